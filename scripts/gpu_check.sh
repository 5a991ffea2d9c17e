python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider -x > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_fast.log
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "bench c4 rc=$?"
python bench.py --config c3 --no-cpu-baseline > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo "bench c3 rc=$?"
timeout 300 python scripts/quick_bench.py 26 27 28 31 > gpurun_out/qb.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()"
