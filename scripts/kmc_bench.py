#!/usr/bin/env python3
"""Time the KMC DT sweep (attempts/ns) for each DT block size and active mode.
Usage: python scripts/kmc_bench.py [L] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
stream = torch.cuda.Stream()
for bk in (16, 32):
    for both in (True, False):
        k = lfg.KmcLattice(L, 1.5, both, 7, block=bk)
        k.set_stream(stream.cuda_stream)
        k.make_random_alloy(0.5, 3)
        k.sweep_async(5)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        k.sweep_async(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"L": L, "bk": bk, "both": both, "att_per_ns": (L ** 3 // 2) * steps / (ms * 1e6),
                          "ms_per_mcs": ms / steps, "open_bonds": k.open_bonds_per_particle()}), flush=True)
        k.close()
