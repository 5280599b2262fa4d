#!/usr/bin/env python3
"""BASELINE configs[0] on the GPU: KPZ L = 2^10, p = 1, q = 0, flat start, 1000 MCS, one seed
(and 16 seeds as one replica batch), timed with CUDA events around the sweeps."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402

L, MCS = 1024, 1000
st = torch.cuda.Stream()
for seeds in ([1], list(range(1, 17))):
    k = lfg.KpzLattice(L, 1.0, 0.0, seeds=seeds)
    k.set_stream(st.cuda_stream)
    k.make_flat_slopes()
    k.sweep_async(3)
    torch.cuda.synchronize()
    k.make_flat_slopes()
    k.reset_counters()
    k.sweep_index = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    k.sweep_async(MCS)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"L": L, "mcs": MCS, "seeds": len(seeds), "plan": k.plan, "seconds": ms / 1e3,
                      "attempts_per_ns": len(seeds) * L * L * MCS / (ms * 1e6),
                      "w2_seed1": k.interface_width(0)}), flush=True)
    k.close()
