#!/bin/bash
# one-screen summary of an ncu report: time, DRAM bytes, issue/pipe utilisation, stall reasons
rep=$1
ncu -i $rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','sm__cycles_elapsed.avg.per_second','smsp__inst_executed.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
for w in want:
  if w in h: print(f'{w:70s} {v[h.index(w)]}')
st=[(h[i],float(v[i].replace(',',''))) for i in range(len(h)) if h[i].startswith('smsp__pcsamp_warps_issue_stalled_') and not h[i].endswith('not_issued')]
tot=sum(x for _,x in st)
print('stall samples:', ' '.join(f'{k[33:]}={100*x/tot:.1f}%' for k,x in sorted(st,key=lambda t:-t[1]) if x/tot>0.01))
"
