#!/bin/bash
# usage: tools/ncu_extract.sh <report.ncu-rep> <out.csv>  -- the counters DESIGN.md / profiles quote
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c '
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr = rows[0]
keep = [i for i, h in enumerate(hdr) if any(k in h for k in (
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct",
    "sm__pipe_tensor_cycles_active", "sm__inst_executed_pipe_tensor", "sm__warps_active.avg.pct", "launch__registers_per_thread",
    "sm__throughput.avg.pct", "l1tex__throughput.avg.pct", "lts__throughput.avg.pct", "sm__inst_executed.sum",
    "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct", "smsp__issue_active.avg.pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct",
    "launch__occupancy_limit", "sm__inst_executed_pipe_lsu", "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
    "sm__pipe_tensor_op", "smsp__pipe_tensor", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed_op_shared"))]
w = csv.writer(sys.stdout)
for r in rows:
    w.writerow([r[i] for i in keep if i < len(r)])
' > "$2"
