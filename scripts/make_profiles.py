#!/usr/bin/env python3
"""Condense ncu reports from gpurun_out/ into committed summaries under profiles/.

    python scripts/make_profiles.py TAG REPORT.ncu-rep [LAUNCHES.csv]

Writes profiles/<TAG>_kpz_ncu.txt (key metrics, stall reasons, instruction
mix) and updates profiles/ncu_summary.json (per-launch DRAM traffic that
bench.py reports as roofline.traffic)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
here = os.path.dirname(os.path.abspath(__file__))
s1 = subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), rep], capture_output=True, text=True).stdout
s2 = subprocess.run([sys.executable, os.path.join(here, "ncu_insts.py"), rep], capture_output=True, text=True).stdout
out = os.path.join(ROOT, "profiles", f"{tag}_kpz_ncu.txt")
with open(out, "w") as f:
    f.write(f"# ncu --set full --clock-control none, one kpz_dtr_phase_kernel launch (L=65536, p=1 q=0, "
            f"default plan 1024x128, sub=4)\n")
    f.write(f"# source report: {os.path.relpath(rep, ROOT)} (not committed; regenerate with scripts/ncu_kpz.sh)\n\n")
    f.write(s1 + "\n# instruction groups by execution count\n" + s2)
vals = {}
for ln in s1.splitlines():
    parts = ln.split()
    if len(parts) >= 2:
        vals[parts[0]] = parts[1]
        if parts[0] == "gpu__time_duration.sum" and len(parts) > 2:  # -> ms
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(parts[2], 1.0)
            vals[parts[0]] = str(float(parts[1]) * scale)
summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
mb = 1e6
try:
    rd = float(vals["dram__bytes_read.sum"]) * mb
    wr = float(vals["dram__bytes_write.sum"]) * mb
    summ["kpz_dtr_phase"] = {"tag": tag, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                             "duration_ms": float(vals["gpu__time_duration.sum"]),
                             "inst_executed": float(vals["smsp__inst_executed.sum"]),
                             "issue_active_pct": float(vals["sm__issue_active.avg.pct_of_peak_sustained_elapsed"]),
                             "alu_pipe_pct": float(vals["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]),
                             "smem_wavefront_pct": float(vals["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]),
                             "sub": int(os.environ.get("LFG_PROFILE_SUB", "4")),
                             "note": "one launch = one DT phase of a sub-sweep = L^2/(4 sub) attempts on average"}
    k = summ["kpz_dtr_phase"]
    dram_pct = 100.0 * (rd + wr) / (k["duration_ms"] * 1e-3) / 7.7e12 if k["duration_ms"] else 0.0
    k["binding"] = (f"SM issue / ALU pipe (profiles/{tag}_kpz_ncu.txt: issue {k['issue_active_pct']:.0f}%, "
                    f"ALU {k['alu_pipe_pct']:.0f}%, DRAM {dram_pct:.0f}% of 7.7 TB/s)")
except KeyError as e:
    print("missing", e)
json.dump(summ, open(summ_path, "w"), indent=1)
if launches:
    import csv
    rows = list(csv.reader(open(launches)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ix = {k: i for i, k in enumerate(h)}
    agg = {}
    for r in rows[hdr + 1:]:
        if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)  # -> usecond
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) -- "
                "bench.py --steps 2 --warmup 1\n# kernel, launches, total_us, share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k}, {n}, {t:.1f}, {t / tot:.3f}\n")
print("wrote", out)
