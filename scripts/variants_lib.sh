#!/bin/bash
# time the default library and each .exp/<variant>/librsort.so (development aid)
cd "$(dirname "$0")/.."
echo "=== default"; python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "Gkeys|onesweep"
for d in ${VARIANTS}; do
  echo "=== $d"; RS_LIB_PATH=.exp/$d/librsort.so python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "Gkeys|onesweep"
done
