# pairs rank / scatter batch sizes below 8 (RS_AR_GP / RS_AR_GSP), interleaved twice
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_gp4.so .exp/librsort_gp6.so .exp/librsort_gsp4.so .exp/librsort_gsp6.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 26:pairs 28:pairs 30:pairs | grep -E "onesweep"
done; done
