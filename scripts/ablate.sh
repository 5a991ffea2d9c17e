#!/bin/bash
# timing ablations of the onesweep pass (output invalid): scripts/ablate.sh "256 24 3"
cd "$(dirname "$0")/.."
set -- $1
tag="$1_$2_$3"
RS_NVCC_DEFINES="-DRS_U32_T=$1 -DRS_U32_KPT=$2 -DRS_U32_MINB=$3" RS_LIB_PATH=/tmp/rs_$tag.so RS_OBJ_DIR=/tmp/obj_$tag \
  python paper_1808_10292_b200/build.py --force > /tmp/build_$tag.log 2>&1 || { tail -5 /tmp/build_$tag.log; exit 1; }
for skip in 0 1 2 4 8 3 5 7 15; do
  echo "=== cfg=$tag debug_skip=$skip"
  RS_LIB_PATH=/tmp/rs_$tag.so RS_DEBUG_SKIP=$skip python scripts/quick_bench.py ${SIZES:-27} 2>&1 | grep -E "onesweep"
done
