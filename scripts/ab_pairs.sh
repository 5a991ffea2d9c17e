# A/B of pairs pass builds: quick_bench at 2^28 and 2^30 pairs for each .so given
for so in "$@"; do
  echo "== $so"; RS_LIB_PATH="$PWD/$so" timeout 300 python scripts/quick_bench.py 28:pairs 30:pairs 2>&1 | grep -E "pairs|onesweep"
done
