# per-rank device time of every collective mode at config 4, p = 8 (in-process ranks, ncu-serialised)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in gsd ger gvr pr4 btn oet; do
  timeout 900 python scripts/gsd_local_bench.py 31 8 $m > gpurun_out/mode_$m.txt 2>&1; echo "$m rc=$?"; head -1 gpurun_out/mode_$m.txt
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mode_$m.csv \
     python scripts/gsd_local_bench.py 31 8 $m > /dev/null 2>&1; echo "ncu $m rc=$?"
done
