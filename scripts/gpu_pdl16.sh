# PDL along the radix-65536 chain: never (1) / always (2), parity tests of radix 65536, c2b16 bench line
timeout 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for v in 1 2; do
  echo "== pdl $v"; RS_PDL=$v RS_NO_KTIMING=1 timeout 300 python scripts/quick_bench.py 20:u32:16 22:u32:16 24:u32:16 25:u32:16 26:u32:16 27:u32:16 24:pairs:16 24:u64:16 2>&1 | grep -E "b=16"
done; done
python bench.py --config c2b16 --no-cpu-baseline --graph 2> gpurun_out/b_c2b16.err > gpurun_out/b_c2b16.json; python scripts/bench_summary.py < gpurun_out/b_c2b16.json
