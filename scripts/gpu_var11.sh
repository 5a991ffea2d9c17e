python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base k80 k72 k64; do
  if [ $v = base ]; then L=paper_1808_10292_b200/librsort.so; else L=paper_1808_10292_b200/librsort_$v.so; fi
  RS_LIB_PATH=$L python scripts/quick_bench.py 26 27 27 28 29 31 > gpurun_out/qb11_$v.log 2>&1
  echo "== $v"; grep -h "pass" gpurun_out/qb11_$v.log
done
