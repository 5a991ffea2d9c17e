timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_fast.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
RS_NO_KTIMING=1 timeout 300 python scripts/quick_bench.py 20 25 26 20:u64 22:u64 24:u64 22:pairs 24:pairs 2>&1 | grep -E "b=8"
