# bench lines of the small configurations with the final build (c1, c2, c2b16)
for c in c1 c2 c2b16; do python bench.py --config $c --no-cpu-baseline --graph 2> gpurun_out/b_$c.err > gpurun_out/b_$c.json; echo "bench $c rc=$?"; python scripts/bench_summary.py < gpurun_out/b_$c.json; done
