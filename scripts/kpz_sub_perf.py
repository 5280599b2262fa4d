#!/usr/bin/env python3
"""KPZ DTr sweep throughput (attempts/ns, device counters) for plan sub = 1, 4, 8 at
L = 2^16 (p = 1) and L = 2^17 (p = 0.95, q = 0.05).  Usage: python scripts/kpz_sub_perf.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402

stream = torch.cuda.Stream()
for L, p, q, steps in ((1 << 16, 1.0, 0.0, 10), (1 << 17, 0.95, 0.05, 3)):
    for sub in (4, 8, 1):
        with lfg.KpzLattice(L, p, q, 7, sub=sub) as k:
            k.set_stream(stream.cuda_stream)
            k.make_flat_slopes()
            k.sweep(2)
            a0 = k.counters().attempts
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            k.sweep_async(steps)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            att = k.counters().attempts - a0
            print(json.dumps({"L": L, "p": p, "q": q, "sub": sub, "att_per_ns": att / (ms * 1e6),
                              "ms_per_mcs": ms / steps}), flush=True)
