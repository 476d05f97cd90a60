import csv, sys, re, subprocess, collections
rep = sys.argv[1]
raw = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines()))
h,u,v=r[0],r[1],r[2]
want = r'gpu__time_duration.sum$|dram__bytes_(read|write)\.sum$|dram__throughput.avg.pct_of_peak_sustained_elapsed$|lts__t_sectors_srcunit_tex_op_read.sum$|l1tex__t_sector_hit_rate.pct$|lts__t_sector_hit_rate.pct$|smsp__pcsamp_warps_issue_stalled_(long_scoreboard|barrier|short_scoreboard|wait|selected|not_selected|lg_throttle|mio_throttle|math_pipe_throttle|dispatch_stall|no_instruction)$|sm__warps_active.avg.pct_of_peak_sustained_active$|launch__registers_per_thread$'
for name,unit,val in zip(h,u,v):
    if re.search(want,name): print(f'{name:70s} {val} {unit}')
src = subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','cuda,sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
for i,row in enumerate(rows[:10]):
    if 'Warp Stall Sampling (All Samples)' in row: hdr=row; st=i+1; break
iS=hdr.index('Warp Stall Sampling (All Samples)')
agg=collections.Counter(); tot=0
for row in rows[st:]:
    if len(row)<=iS or not row[0]: continue
    try: s=int(row[iS])
    except: continue
    agg[(int(row[0]), row[1].strip()[:90])]+=s; tot+=s
print('total samples (cuda lines)', tot)
for k,val in agg.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 30): print(f'{val:7d} {100*val/tot:5.1f}% L{k[0]}: {k[1]}')
