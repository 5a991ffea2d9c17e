# the driver's round-end GPU tier: every -m gpu test (slow ones included) and smoke()
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/t_full.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t_full.log
python -c "import __graft_entry__ as g; g.smoke()"
