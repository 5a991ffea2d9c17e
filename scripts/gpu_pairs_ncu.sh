# ncu --set full of the (u64, u32) pairs pass at 2^28 pairs (quick_bench), source-level
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/quick_bench.py 28:pairs 30:pairs > gpurun_out/qb_pairs.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep_ar -s 10 -c 1 -o gpurun_out/k3_pairs28 \
   python scripts/quick_bench.py 28:pairs > gpurun_out/ncu_pairs.log 2>&1; echo "ncu rc=$?"
