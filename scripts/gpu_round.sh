# full GPU round: tests, bench lines, launch list and one ncu capture of K3 at c4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/t_fast.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/t_fast.log
python bench.py > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo "bench c4 rc=$?"
for c in c3 c1 c2 c2b16; do python bench.py --config $c --no-cpu-baseline --graph > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo "bench $c rc=$?"; done
python bench.py --config c5 --no-cpu-baseline > gpurun_out/b_c5.json 2> gpurun_out/b_c5.err; echo "bench c5 rc=$?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 12 -c 1 -o gpurun_out/k3_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
