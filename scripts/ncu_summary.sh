#!/bin/bash
# Key metrics of an ncu --set full capture (run here, no GPU needed).
ncu -i "$1" --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; u=rows[1]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__bytes.sum.per_second',
'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed',
'sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','launch__block_size',
'launch__shared_mem_per_block_dynamic','smsp__inst_executed.sum','sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active',
'sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','lts__t_bytes.sum']
for d in rows[2:]:
  for i,k in enumerate(h):
    if k in keys: print(f'{k:75s} {d[i]} {u[i]}')
  print()
"
