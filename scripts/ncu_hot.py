#!/usr/bin/env python3
"""Per-instruction stall samples of an ncu report, hottest first, with the
instruction text.  Usage: python scripts/ncu_hot.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
recs = []
tot = 0
for r in rows[2:]:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    tot += s
    recs.append((r[ix["Address"]][-5:], r[ix["Source"]].strip(), s, n))
print("total samples", tot)
if "--seq" in sys.argv:
    for a, src, s, n in recs:
        if n:
            print(f"{a} {s:6d} {n:>10d}  {src}")
else:
    for a, src, s, n in sorted(recs, key=lambda x: -x[2])[:top]:
        print(f"{a} {s:6d} {100*s/tot:5.1f}% {n:>10d}  {src}")
