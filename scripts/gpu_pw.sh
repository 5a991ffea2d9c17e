# p-way merge study: parity of the GSD paths, per-phase times of 8 in-process ranks at
# 2^31 total (2^28 per rank), and k_pw_merge's own duration / instructions under ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gsd.py -q -p no:cacheprovider > gpurun_out/t_gsd.log 2>&1; echo "gsd tests rc=$?"; tail -1 gpurun_out/t_gsd.log
timeout 600 python scripts/gsd_local_bench.py 31 8 gsd > gpurun_out/pw_bench.txt 2>&1; echo "pw bench rc=$?"
cat gpurun_out/pw_bench.txt
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_pw_merge -c 8 --csv \
    python scripts/gsd_local_bench.py 31 8 gsd > gpurun_out/ncu_pw.csv 2>&1; echo "ncu pw rc=$?"
python3 -c "import csv; rows=[r for r in csv.reader(open('gpurun_out/ncu_pw.csv')) if len(r)>10]; h=rows[0]; ix={k:i for i,k in enumerate(h)}; [print(r[ix['Metric Name']], r[ix['Metric Value']]) for r in rows[1:]]"
if [ -n "$PW_FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pw_merge -c 1 -o gpurun_out/pw_c4 \
    python scripts/gsd_local_bench.py 31 8 gsd > gpurun_out/ncu_pwf.log 2>&1; echo "ncu pw full rc=$?"
fi
