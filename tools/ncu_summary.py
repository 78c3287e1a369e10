#!/usr/bin/env python3
"""Key metrics + stall reasons of each kernel in an ncu report. usage: ncu_summary.py report [kernel_regex]"""
import csv, io, re, subprocess, sys

args = ["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", f"regex:{sys.argv[2]}"]
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = rows[0]
pat = re.compile(r"^(Kernel Name|gpu__time_duration.sum|smsp__inst_executed.sum|smsp__issue_active.avg.pct_of_peak_sustained_active|"
                 r"sm__warps_active.avg.pct_of_peak_sustained_active|dram__bytes_read.sum|dram__bytes_write.sum|"
                 r"launch__registers_per_thread|launch__grid_size|launch__block_size|launch__occupancy_limit_.*|"
                 r"lts__t_sector_hit_rate.pct|lts__throughput.avg.pct_of_peak_sustained_elapsed|"
                 r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum|sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio)$")
for r in rows[2:]:
    for i, w in enumerate(h):
        if pat.match(w):
            v = r[i]
            if "stalled" in w:
                try:
                    if float(v) < 0.1:
                        continue
                except ValueError:
                    pass
                w = w.replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", "")
            print(f"{w:60s} {rows[1][i]:10s} {v}")
    print()
