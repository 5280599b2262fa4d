#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics, pipe utilisation, stall reasons,
and per-instruction-group counts.  Usage: python scripts/ncu_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k][1]:>20s} {d[k][0]}")
stalls = [(h, v) for h, (u, v) in d.items() if h.startswith("smsp__average_warp_latency_issue_stalled") or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
tot = 0.0
items = []
for h, v in stalls:
    if h.endswith("_not_issued"):
        continue
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        continue
    items.append((x, h))
    tot += x
print("-- stall samples (pcsamp) --")
for x, h in sorted(items, reverse=True)[:12]:
    print(f"{h:80s} {x:12.0f} {100 * x / max(tot, 1):5.1f}%")
