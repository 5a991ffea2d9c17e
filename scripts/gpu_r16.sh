# radix-65536 scan rewrite: parity tests + A/B (previous commit vs working tree) + the c2b16 bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -1
for rep in 1 2; do for so in .exp/librsort_r16prev.so paper_1808_10292_b200/librsort.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 24:u32:16 27:u32:16 | grep -E "b=16|r16_"
done; done
python bench.py --config c2b16 --no-cpu-baseline --graph > gpurun_out/b_c2b16.json 2> gpurun_out/b_c2b16.err; echo "bench rc=$?"
