# pairs pass re-sweep at look-back window 4 (quick_bench, interleaved twice)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_pk32.so .exp/librsort_pk16.so .exp/librsort_pgp12.so .exp/librsort_pgsp12.so .exp/librsort_plb3k32.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 26:pairs 28:pairs 30:pairs | grep -E "onesweep"
done; done
