# A/B: programmatic dependent launch along K1 -> K2 -> K3 x P -> K4 (default) vs plain launches (RS_PDL=0)
A=paper_1808_10292_b200/librsort_nopdl.so; B=paper_1808_10292_b200/librsort.so
for rep in 1 2; do for so in $A $B; do
  echo "== $so"; RS_NO_KTIMING=1 RS_LIB_PATH="$PWD/$so" timeout 300 python scripts/quick_bench.py 20 22 24 26 27 31 28:pairs 24:u64 2>&1 | grep -E "b=8"
done; done
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_fast.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for so in $A $B; do for c in c1 c2 c3; do echo "== bench $c $so"; RS_LIB_PATH=$PWD/$so python bench.py --config $c --no-cpu-baseline --graph 2>/dev/null > gpurun_out/pdl_$c.json; python scripts/bench_summary.py < gpurun_out/pdl_$c.json; done; done
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; python scripts/bench_summary.py < gpurun_out/b_c4.json
