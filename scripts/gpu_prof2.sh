python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
RS_LIB_PATH=paper_1808_10292_b200/librsort_wst.so RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/plain27w.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 3 -c 1 -o gpurun_out/k3_wst27 \
    env RS_LIB_PATH=paper_1808_10292_b200/librsort_wst.so RS_ONE_PASS=1 python scripts/quick_bench.py 27 > gpurun_out/ncu_wst27.log 2>&1
ls gpurun_out
