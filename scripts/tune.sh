#!/bin/bash
# Build and time tile-config variants on the GPU box (development aid).
# usage: scripts/tune.sh "512 12 2" "512 8 3" ...   (u32 keys-only: threads kpt minblocks)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  set -- $cfg
  tag="$1_$2_$3"
  RS_NVCC_DEFINES="-DRS_U32_T=$1 -DRS_U32_KPT=$2 -DRS_U32_MINB=$3 ${EXTRA_DEFINES}" RS_LIB_PATH=/tmp/rs_$tag.so RS_OBJ_DIR=/tmp/obj_$tag \
    python paper_1808_10292_b200/build.py --force > /tmp/build_$tag.log 2>&1 || { echo "build $cfg failed"; tail -5 /tmp/build_$tag.log; continue; }
  for rv in ${RANK_VARIANTS:-0 1}; do
    echo "=== u32 cfg=$cfg rank_variant=$rv"
    RS_LIB_PATH=/tmp/rs_$tag.so RS_RANK_VARIANT=$rv python scripts/quick_bench.py ${TUNE_SIZES:-27} 2>&1 | grep -E "Gkeys|onesweep|hist"
  done
done
