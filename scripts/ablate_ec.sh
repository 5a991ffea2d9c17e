#!/bin/bash
# timing ablations of the default (early-counts) pass, output invalid: 1 look-back, 2 rank, 4 store, 8 count
cd "$(dirname "$0")/.."
for skip in 0 1 2 4 8 3 5 6 7 15; do
  echo "=== debug_skip=$skip"
  RS_DEBUG_SKIP=$skip python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "onesweep"
done
