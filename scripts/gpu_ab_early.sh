# K3 u32: next tile's first load batch issued before [store] (RS_AR_EARLY) A/B + parity with the variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
RS_LIB_PATH=$PWD/.exp/librsort_early.so timeout 900 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -1
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_early.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 26 27 28 31 | grep -E "onesweep"
done; done
