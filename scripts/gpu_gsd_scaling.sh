# per-rank device times of the collective sort at p = 2, 4, 8 (in-process ranks on one B200):
# event times per phase, then the serialised ncu launch list of each run
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "31 2 gsd u32" "31 4 gsd u32" "31 8 gsd u32" "30 2 gsd pairs" "30 4 gsd pairs" "30 8 gsd pairs"; do
  set -- $cfg; tag=c$([ "$4" = u32 ] && echo 4 || echo 5)_p$2
  timeout 900 python scripts/gsd_local_bench.py $cfg > gpurun_out/gsdl_$tag.txt 2>&1; echo "$tag rc=$?"; head -1 gpurun_out/gsdl_$tag.txt
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gsdl_$tag.csv \
     python scripts/gsd_local_bench.py $cfg > /dev/null 2>&1; echo "ncu $tag rc=$?"
done
