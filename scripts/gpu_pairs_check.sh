python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_radix.py tests/test_gpu_gsd.py tests/test_gpu_net.py tests/test_gpu_nccl_p1.py -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_radix.py -q -x -p no:cacheprovider -k "config5 or pairs_above" 2>&1 | tail -2
python bench.py --config c5 --no-cpu-baseline > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; echo "bench c5 rc=$?"
python bench.py --config c4 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "bench c4 rc=$?"
