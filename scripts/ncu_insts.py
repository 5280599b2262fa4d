#!/usr/bin/env python3
"""Group executed SASS instructions of an ncu report by execution count and opcode.
Usage: python scripts/ncu_insts.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot = 0
groups = defaultdict(list)
for r in rows[2:]:
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    tot += n
    src = r[ix["Source"]].strip()
    op = src.split()[1] if src.startswith("@") else src.split()[0]
    groups[n].append(op)
print("total executed", tot)
for n, ops in sorted(groups.items(), key=lambda kv: -kv[0] * len(kv[1]))[:8]:
    c = Counter(o.split(".")[0] for o in ops)
    print(f"count {n:>10d} x {len(ops):4d} instr = {100 * n * len(ops) / tot:5.1f}%  ", dict(c.most_common(14)))
