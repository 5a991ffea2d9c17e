for so in paper_1808_10292_b200/librsort.so .exp/librsort_rot.so paper_1808_10292_b200/librsort.so .exp/librsort_rot.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/k1_probe.py 20 24 26 27 28 30
done
timeout 600 ncu --set full --clock-control none -k regex:k_digit_hist -s 3 -c 1 -o gpurun_out/k1_27 python scripts/k1_probe.py 27 > gpurun_out/k1_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_digit_hist -c 20 python scripts/k1_probe.py 20 27 2>&1 | grep -E "gpu__time_duration|k_digit" | head -40
