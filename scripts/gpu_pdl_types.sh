# PDL forced off (1) / on (2) for every key type at small and mid n; the new parity test
timeout 600 python -m pytest tests/test_gpu_radix.py -q -p no:cacheprovider -k "programmatic or edge_sizes or native" 2>&1 | tail -1
for rep in 1 2; do for v in 1 2; do
  echo "== pdl $v"; RS_PDL=$v RS_NO_KTIMING=1 timeout 300 python scripts/quick_bench.py 20 22 24 25 20:u64 22:u64 24:u64 20:pairs 22:pairs 24:pairs 2>&1 | grep -E "b=8"
done; done
