# PDL gated to u32 keys <= 2^24: suite, smoke, quick sizes, c1/c2/c4 bench lines
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_fast.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
RS_NO_KTIMING=1 timeout 300 python scripts/quick_bench.py 20 24 27 24:u64 20:pairs 2>&1 | grep -E "b=8"
for c in c1 c2; do python bench.py --config $c --no-cpu-baseline --graph 2>/dev/null > gpurun_out/b_$c.json; python scripts/bench_summary.py < gpurun_out/b_$c.json; done
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; python scripts/bench_summary.py < gpurun_out/b_c4.json
