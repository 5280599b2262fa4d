"""Time the W^2 readout (lfg_kpz_width_sums_async) at L = 2^16 on the device
with CUDA events on the handle's stream; print JSON.  Usage: python scripts/w2_time.py [L] [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_1204_5072_b200 as lfg
from paper_1204_5072_b200 import _native

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
st = torch.cuda.Stream()
out = torch.empty(3, dtype=torch.int64).pin_memory()
with lfg.KpzLattice(L, 1.0, 0.0, 5) as k:
    k.make_flat_slopes()
    k.sweep(3)
    k.set_stream(st.cuda_stream)
    ref = k.width_sums()
    for _ in range(3):
        k.width_sums_async(out.data_ptr())
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        k.width_sums_async(out.data_ptr())
    e1.record(st)
    st.synchronize()
    ms = e0.elapsed_time(e1) / reps
    got = (int(out[0]), int(out[1]))
bytes_read = L * L / 8
print(json.dumps({"L": L, "ms_per_readout": ms, "GBps_of_spin_read": bytes_read / ms / 1e6,
                  "sums_match_sync_call": got == tuple(ref), "sum": got[0], "sum2": got[1]}))
