# chained launch (every pass in one kernel) vs one launch per pass; .so variants in .exp/
S="${AB_SIZES:-24 27 31 28:pairs 28:u64}"
for rep in $(seq ${AB_REPS:-2}); do
echo "== per-pass launches (lib_cg, chain=0)"; RS_CHAIN=0 RS_LIB_PATH=$PWD/.exp/lib_cg.so timeout 300 python scripts/quick_bench.py $S 2>&1 | grep -E "b=8|onesweep"
for v in "$@"; do echo "== chained $v"; RS_CHAIN=1 RS_LIB_PATH=$PWD/.exp/lib_$v.so timeout 300 python scripts/quick_bench.py $S 2>&1 | grep -E "b=8|onesweep"; done
done
