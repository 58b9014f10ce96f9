R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
hdr=r[0]
want=['Duration','Executed Ipc Active','Issue Slots Busy','L2 Cache Throughput','Achieved Occupancy','Registers Per Thread','Warp Cycles Per Issued Instruction','Executed Instructions','L2 Hit Rate','Compute (SM) Throughput','Grid Size','Dynamic Shared Memory Per Block','Theoretical Occupancy']
for row in r[1:]:
    if row[hdr.index('Metric Name')] in want: print(row[hdr.index('Metric Name')].ljust(40), row[hdr.index('Metric Unit')].ljust(10), row[hdr.index('Metric Value')])
"
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]; v=r[2] if len(r)>2 else r[1]
d=dict(zip(h,v))
def f(x):
    try: return float(x.replace(',',''))
    except: return 0.0
items=[(k.replace('smsp__pcsamp_warps_issue_stalled_',''),f(d[k])) for k in h if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
tot=sum(x for k,x in items)
print(' '.join('%s=%.1f%%'%(k,100*x/tot) for k,x in sorted(items,key=lambda kv:-kv[1])[:10]))
for k in ['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum']:
    if k in d: print(k, d[k])
"
