# keys store-phase batch (RS_AR_SGK) A/B, interleaved twice
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_sgk2.so .exp/librsort_sgk8.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 26 27 31 28:u64 | grep -E "onesweep"
done; done
