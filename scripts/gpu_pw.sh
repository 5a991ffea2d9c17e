python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/gsd_local_bench.py 31 8 > gpurun_out/pw_bench.log 2>&1; cat gpurun_out/pw_bench.log
python scripts/gsd_local_bench.py 28 8 > gpurun_out/pw_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pw_merge -s 8 -c 1 -o gpurun_out/pw28 python scripts/gsd_local_bench.py 28 8 > gpurun_out/pw_ncu.log 2>&1; echo ncu rc=$?
