python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
RS_LIB_PATH=$PWD/.exp/librsort_wc32.so timeout 600 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -2
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_wc32.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 27 31 27:u32:8:gauss | grep -E "onesweep|u32"
done; done
