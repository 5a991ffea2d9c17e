python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in krlpcsc kr80lpcsc f84 fsg8 fg11 fg4 f80g10; do
  L=paper_1808_10292_b200/librsort_$v.so
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 > gpurun_out/qb6_$v.log 2>&1
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 > gpurun_out/qb6b_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb6_$v.log gpurun_out/qb6b_$v.log
done
