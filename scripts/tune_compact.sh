#!/bin/bash
# compact design-2 layout: 256 x KPT x MINB sweeps (development aid)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  set -- $cfg
  tag="ecc_$1_$2_$3"
  RS_NVCC_DEFINES="-DRS_EC_U32_T=$1 -DRS_EC_U32_KPT=$2 -DRS_EC_U32_MINB=$3" RS_LIB_PATH=/tmp/rs_$tag.so RS_OBJ_DIR=/tmp/obj_$tag \
    python paper_1808_10292_b200/build.py --force > /tmp/build_$tag.log 2>&1 || { echo "build $cfg failed"; continue; }
  echo "=== compact cfg=$cfg"
  RS_COMPACT=1 RS_LIB_PATH=/tmp/rs_$tag.so python scripts/quick_bench.py ${TUNE_SIZES:-27} 2>&1 | grep -E "onesweep"
done
