# small-n breakdown: per-kernel durations (ncu, serialised) of one 2^20 / 2^22 u32 sort
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/quick_bench.py 20 22 > gpurun_out/qb_small.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__warps_launched.sum --clock-control none -s 40 -c 14 \
  python scripts/quick_bench.py 20 > gpurun_out/ncu_small20.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 12 -c 1 -o gpurun_out/k3_small20 \
  python scripts/quick_bench.py 20 > gpurun_out/ncu_small20_full.log 2>&1; echo rc=$?
