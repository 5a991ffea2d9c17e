python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in krlpc kr72lpc; do
  RS_LIB_PATH=paper_1808_10292_b200/librsort_$v.so timeout 900 python -m pytest tests/test_gpu_radix.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/t_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/t_$v.log)"
done
for v in base lpc krlpc kr80lpc kr72lpc kr64lpc lpc72; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 > gpurun_out/qb4_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb4_$v.log
done
