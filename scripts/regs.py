"""Registers / spills per kernel from the nvcc -Xptxas -v build log.
usage: python scripts/regs.py [pattern] [log]"""
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
log = sys.argv[2] if len(sys.argv) > 2 else "paper_1204_5072_b200/_lib/liblfg.so.build.log"
cur = None
for line in open(log):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        if pat in name:
            print(m.group(1), name.replace("lfg::", "").replace("(lfg::KpzPhaseArgs)", ""))
        cur = None
