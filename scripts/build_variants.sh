#!/bin/bash
# build .exp/<name>/librsort.so for each "name:-DDEFINE ..." argument, each with its
# own object directory (development aid; run sequentially to keep the builds apart)
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  mkdir -p .exp/$name/obj
  RS_OBJ_DIR=.exp/$name/obj RS_NVCC_DEFINES="$defs" RS_LIB_PATH=.exp/$name/librsort.so \
    python -c "import paper_1808_10292_b200.build as b; b.build(force=True)" > .exp/$name/build.log 2>&1 \
    && echo "built $name" || echo "FAILED $name"
done
