# A/B of whole-sort builds: quick_bench over a few sizes for each .so given (twice, interleaved)
for rep in 1 2; do
for so in "$@"; do
  echo "== $so"; RS_LIB_PATH="$PWD/$so" timeout 300 python scripts/quick_bench.py ${AB_SIZES:-24 27 31 28:pairs} 2>&1 | grep -E "b=8|onesweep|hist"
done
done
