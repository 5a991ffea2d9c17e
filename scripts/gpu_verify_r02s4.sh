# re-entry check of the committed state: build, fast GPU suite, smoke, c4 and c3 bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_fast.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "bench c4 rc=$?"; cat gpurun_out/b_c4.json
python bench.py --config c3 --no-cpu-baseline --graph > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err; echo "bench c3 rc=$?"
