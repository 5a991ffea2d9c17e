#!/bin/bash
# Build and time early-counts pass configs: scripts/tune_ec.sh "256 16 4" ... (ranking threads, kpt, minblocks)
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  set -- $cfg
  tag="ec_$1_$2_$3"
  RS_NVCC_DEFINES="-DRS_EC_U32_T=$1 -DRS_EC_U32_KPT=$2 -DRS_EC_U32_MINB=$3 ${EXTRA_DEFINES}" RS_LIB_PATH=/tmp/rs_$tag.so RS_OBJ_DIR=/tmp/obj_$tag \
    python paper_1808_10292_b200/build.py --force > /tmp/build_$tag.log 2>&1 || { echo "build $cfg failed"; grep -E "error|fatal" /tmp/build_$tag.log | head -3; continue; }
  echo "=== ec cfg=$cfg"
  RS_PASS_DESIGN=${PASS_DESIGN:-2} RS_LIB_PATH=/tmp/rs_$tag.so python scripts/quick_bench.py ${TUNE_SIZES:-27} 2>&1 | grep -E "Gkeys|onesweep"
done
