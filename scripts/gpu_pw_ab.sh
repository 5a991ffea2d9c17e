# A/B of k_pw_merge builds: serialized per-launch durations (one ncu metric, one pass)
# usage: bash scripts/gpu_pw_ab.sh lib1.so lib2.so ...
for so in "$@"; do
  RS_LIB_PATH=$PWD/$so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pw_merge -c 8 --csv \
      python scripts/gsd_local_bench.py ${PW_LG:-31} ${PW_P:-8} gsd ${PW_KIND:-u32} > gpurun_out/ab_$(basename $so).csv 2>&1
  python3 -c "
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/ab_$(basename $so).csv')) if len(r)>10]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
v=[float(r[ix['Metric Value']].replace(',','')) for r in rows[1:]]
print('$so', 'k_pw_merge us:', ' '.join('%.1f'%(x/1e3) for x in v), ' median %.1f'%(sorted(v)[len(v)//2]/1e3))
"
done
