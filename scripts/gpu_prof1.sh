# ncu source-level profile of the u32 radix-256 pass (K3) at 2^27 (one pass, both variants)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/plain27.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 3 -c 1 -o gpurun_out/k3_base27 \
    env RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/ncu_base27.log 2>&1
RS_LIB_PATH=paper_1808_10292_b200/librsort_lpc.so RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/plain27l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 3 -c 1 -o gpurun_out/k3_lpc27 \
    env RS_LIB_PATH=paper_1808_10292_b200/librsort_lpc.so RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/ncu_lpc27.log 2>&1
ls -la gpurun_out
