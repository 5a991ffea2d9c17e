# radix-65536: partitions per SM (generic scatter at 2-3 CTAs per SM) A/B + parity with the widest variant
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
RS_LIB_PATH=$PWD/.exp/librsort_r16g4m2.so timeout 900 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -m "gpu and not slow" -k "16 or radix65536" 2>&1 | tail -1
for so in paper_1808_10292_b200/librsort.so .exp/librsort_r16g2m2.so .exp/librsort_r16g3m3.so .exp/librsort_r16g4m2.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 24:u32:16 27:u32:16 24:pairs:16 | grep -E "b=16|r16_scatter|r16_count|r16_offsets"
done
