python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_radix.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/t_def.log 2>&1; echo "default $(tail -1 gpurun_out/t_def.log)"
for v in base gs4 gs11 gs22; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 31 28:u64 > gpurun_out/qb10_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb10_$v.log
done
