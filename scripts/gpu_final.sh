# final state: the driver's round-end tier (every -m gpu test, smoke) and the c4 / c5 bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests/ -x -q -m gpu -p no:cacheprovider > gpurun_out/t_full.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_full.log
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; python scripts/bench_summary.py < gpurun_out/b_c4.json
python bench.py --config c5 --no-cpu-baseline > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; python scripts/bench_summary.py < gpurun_out/b_c5.json
python bench.py --config c2b16 --no-cpu-baseline --graph > gpurun_out/b_c2b16.json 2> gpurun_out/b_c2b16.err; python scripts/bench_summary.py < gpurun_out/b_c2b16.json
