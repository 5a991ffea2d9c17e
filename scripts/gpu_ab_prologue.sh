# single-GPU sort launch-sequence A/B (previous commit vs working tree): tests, quick_bench, c1 bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_radix.py tests/test_gpu_gsd.py tests/test_gpu_net.py tests/test_gpu_nccl_p1.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -1
for rep in 1 2; do for so in .exp/librsort_k3prev.so paper_1808_10292_b200/librsort.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 20 24 27 31 | grep -E "^u32"
done; done
for so in .exp/librsort_k3prev.so paper_1808_10292_b200/librsort.so .exp/librsort_k3prev.so paper_1808_10292_b200/librsort.so; do
  RS_LIB_PATH=$PWD/$so python bench.py --config c1 --no-cpu-baseline --graph --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$so c1', d['value'], d['graph_replay']['value'])"
  RS_LIB_PATH=$PWD/$so python bench.py --config c3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$so c3', d['value'])"
done
python bench.py --config c1 --no-cpu-baseline --graph > gpurun_out/b_c1.json 2> gpurun_out/b_c1.err; echo "bench c1 rc=$?"
