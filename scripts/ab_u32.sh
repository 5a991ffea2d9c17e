# A/B of u32 pass builds: quick_bench at 2^27 and 2^31 for each .so given (twice, interleaved)
for rep in 1 2; do
for so in "$@"; do
  echo "== $so"; RS_LIB_PATH="$PWD/$so" timeout 300 python scripts/quick_bench.py 27 31 2>&1 | grep -E "onesweep"
done
done
