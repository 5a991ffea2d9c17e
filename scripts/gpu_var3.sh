python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in wst wstlpc; do
  RS_LIB_PATH=paper_1808_10292_b200/librsort_$v.so timeout 900 python -m pytest tests/test_gpu_radix.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/t_$v.log 2>&1
  tail -1 gpurun_out/t_$v.log
done
for v in base lpc wst wstlpc; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 28:u64 28:pairs > gpurun_out/qb3_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb3_$v.log
done
