#!/bin/bash
# timing ablations of design 5 (libraries built with -DRS_AR_ABLATE=k under .exp/abk, output invalid)
cd "$(dirname "$0")/.."
echo "=== full"; RS_ONE_PASS=1 python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "onesweep"
for ab in 1 2 4 3 7; do
  echo "=== ablate=$ab (1 no look-back, 2 no store, 4 no scatter)"
  RS_LIB_PATH=.exp/ab$ab/librsort.so RS_ONE_PASS=1 python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "onesweep"
done
