#!/bin/bash
# per-pass timing of the default pass and its ranking variants (development aid)
cd "$(dirname "$0")/.."
SIZES=${SIZES:-"27 31 27:pairs 27:u64"}
for rv in ${RVS:-3 0}; do
  echo "=== rank_variant=$rv"
  RS_RANK_VARIANT=$rv python scripts/quick_bench.py $SIZES 2>&1 | grep -E "Gkeys|onesweep|hist"
done
