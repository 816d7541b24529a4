#!/usr/bin/env python
"""Key metrics + stall breakdown per kernel from an ncu --page raw --csv export."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.per_cycle_active", "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
for d in data:
    print("---", d[idx["Kernel Name"]][:60])
    for k in KEYS:
        if k in idx:
            print(f"   {k:62s} {d[idx[k]]} {units[idx[k]]}")
    st = [(hdr[i], float(d[i])) for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_")
          and not hdr[i].endswith("not_issued") and d[i] not in ("", "n/a")]
    tot = sum(v for _, v in st) or 1
    print("   stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                                   for h, v in sorted(st, key=lambda x: -x[1])[:6]))
