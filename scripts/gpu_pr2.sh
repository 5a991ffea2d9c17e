python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base g16 g32 g64; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 24:u32:16 27:u32:16 > gpurun_out/qpr2_$v.log 2>&1
  echo "== $v"; grep -h "n=2\|r16_" gpurun_out/qpr2_$v.log
done
RS_LIB_PATH=paper_1808_10292_b200/librsort_g16.so python scripts/quick_bench.py 27:u32:16 > gpurun_out/pr2_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:k16_scatter -s 2 -c 1 -o gpurun_out/pr2_g16 env RS_LIB_PATH=paper_1808_10292_b200/librsort_g16.so python scripts/quick_bench.py 27:u32:16 > gpurun_out/pr2_ncu.log 2>&1; echo ncu rc=$?
