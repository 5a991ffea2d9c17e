#!/bin/bash
# design-2 pass: sweep tile configs x rank variants (development aid)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  set -- $cfg
  tag="ec_$1_$2_$3"
  RS_NVCC_DEFINES="-DRS_EC_U32_T=$1 -DRS_EC_U32_KPT=$2 -DRS_EC_U32_MINB=$3" RS_LIB_PATH=/tmp/rs_$tag.so RS_OBJ_DIR=/tmp/obj_$tag \
    python paper_1808_10292_b200/build.py --force > /tmp/build_$tag.log 2>&1 || { echo "build $cfg failed"; continue; }
  for rv in ${RANK_VARIANTS:-0 3}; do
    echo "=== ec cfg=$cfg rank_variant=$rv"
    RS_RANK_VARIANT=$rv RS_LIB_PATH=/tmp/rs_$tag.so python scripts/quick_bench.py ${TUNE_SIZES:-27} 2>&1 | grep -E "onesweep"
  done
done
