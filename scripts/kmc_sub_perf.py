#!/usr/bin/env python3
"""KMC DT sweep throughput (attempts/ns) for plan sub = 1 and sub = 4 at the given sizes
(16^3 blocks, both active, c = 0.5, eps = 1.5).  Usage: python scripts/kmc_sub_perf.py [L ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402

stream = torch.cuda.Stream()
for L in [int(a) for a in sys.argv[1:]] or [256, 1024]:
    steps = 30 if L <= 256 else 8
    for sub in (1, 4):
        k = lfg.KmcLattice(L, 1.5, True, 7, block=16, sub=sub)
        k.set_stream(stream.cuda_stream)
        k.make_random_alloy(0.5, 3)
        k.sweep_async(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        k.sweep_async(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"L": L, "sub": sub, "att_per_ns": (L ** 3 // 2) * steps / (ms * 1e6)}), flush=True)
        k.close()
