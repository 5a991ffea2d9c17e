import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
hdr=r[0]; vals=r[2]
d=dict(zip(hdr,vals))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size','sm__inst_executed.sum','smsp__inst_executed.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','dram__cycles_active.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum.pct_of_peak_sustained_elapsed','dram__bytes_write.sum.pct_of_peak_sustained_elapsed','lts__t_sectors_srcunit_tex.sum','lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed']:
    print(k, d.get(k))
items=[]
for h,v in d.items():
    if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
        try: items.append((float(v),h))
        except: pass
tot=sum(v for v,h in items)
for v,h in sorted(items,reverse=True)[:9]: print(f"{100*v/tot:5.1f}% {h.replace('smsp__pcsamp_warps_issue_stalled_','')}")
