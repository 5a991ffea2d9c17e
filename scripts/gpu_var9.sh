python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base gr22 gr44 gr88 lb4 lb16; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 27 31 31 > gpurun_out/qb9_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb9_$v.log
done
