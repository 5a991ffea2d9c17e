# ncu --set full of one pairs K3 launch at config c5 (bench.py), then the c5 bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > gpurun_out/plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 24 -c 1 -o gpurun_out/k3_pairs_c5 \
    python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-verify > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
