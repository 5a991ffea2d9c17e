python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base ovl; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 28:u64 > gpurun_out/qb2_$v.log 2>&1
done
RS_LIB_PATH=paper_1808_10292_b200/librsort_ovl.so timeout 900 python -m pytest tests/test_gpu_radix.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/t_ovl.log 2>&1
tail -2 gpurun_out/t_ovl.log
grep -h "n=2\|pass" gpurun_out/qb2_*.log
