#!/usr/bin/env python3
"""Summary of an ncu report (raw page): the metrics B200_PROFILING.md lists
plus the warp-stall breakdown.  usage: ncu_summary2.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
for r in rows[2:]:
    for k in WANT:
        if k in h:
            print(f"{k:70s} {r[h.index(k)]}")
    stalls = [(k, r[i]) for i, k in enumerate(h) if k.startswith("smsp__average_warp_latency_issue_stalled_")
              or (k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct"))]
    vals = []
    for k, v in stalls:
        try:
            vals.append((float(v), k))
        except ValueError:
            pass
    for v, k in sorted(vals, reverse=True)[:10]:
        print(f"  stall {k:68s} {v:8.2f}")
    print()
