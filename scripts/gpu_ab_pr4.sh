# PR4 pull kernel A/B (previous commit vs working tree) + PR4 parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gsd.py tests/test_gpu_nccl_p1.py -q -x -p no:cacheprovider -k "pr4 or config4" 2>&1 | tail -1
for so in .exp/librsort_prprev.so paper_1808_10292_b200/librsort.so; do
  RS_LIB_PATH=$PWD/$so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_pull_pieces \
     --log-file gpurun_out/pr_$(basename $so).csv python scripts/gsd_local_bench.py 31 8 pr4 > gpurun_out/pr_$(basename $so).txt 2>&1
  head -1 gpurun_out/pr_$(basename $so).txt
  python3 -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/pr_$(basename $so).csv')) if len(r)>10]
ix={k:i for i,k in enumerate(rows[0])}
v=sorted(float(r[ix['Metric Value']].replace(',','')) for r in rows[1:])
print('$so k_pull_pieces us: median %.1f (n=%d)' % (v[len(v)//2]/1e3 if rows[1][ix['Metric Unit']] in ('ns','nsecond') else v[len(v)//2], len(v)))"
done
