# look-back window A/B for the pairs pass (quick_bench, interleaved twice): RS_AR_LB_P builds
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do for so in paper_1808_10292_b200/librsort.so .exp/librsort_lbp1.so .exp/librsort_lbp2.so .exp/librsort_lbp3.so .exp/librsort_lbp4.so .exp/librsort_lbp6.so; do
  echo "== $so"; RS_LIB_PATH=$PWD/$so timeout 300 python scripts/quick_bench.py 26:pairs 28:pairs 30:pairs | grep -E "onesweep"
done; done
