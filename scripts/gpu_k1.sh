# K1 A/B: RS_K1_V 0 (per-pass runtime shifts), 1 (key pre-shifted once), 2 (default: + XOR-swizzled 16-copy slot)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -2
for rep in 1 2; do
for so in .exp/librsort_k1v0.so .exp/librsort_k1v1.so paper_1808_10292_b200/librsort.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/k1_probe.py 26:u64 28:u64 30:u64 26 27 28 30
done
done
for so in .exp/librsort_k1v0.so paper_1808_10292_b200/librsort.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 30:pairs 28:u64 27 31 | grep -E "pairs|u64|u32|hist"
done
