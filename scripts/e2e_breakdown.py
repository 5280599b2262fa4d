#!/usr/bin/env python3
"""Wall-clock breakdown of one e2e step (bench.py e2e leg) at L = 2^16."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
wpr = L // 64
x0 = np.full(L * wpr, 0x5555555555555555, np.uint64)
y0 = np.zeros((L, wpr), np.uint64)
y0[0::2, :] = np.uint64(0xFFFFFFFFFFFFFFFF)
hx = torch.from_numpy(x0.view(np.int64)).pin_memory()
hy = torch.from_numpy(y0.reshape(-1).view(np.int64)).pin_memory()
k = lfg.KpzLattice(L, 1.0, 0.0, 5)
dev = torch.empty(L * wpr * 2, dtype=torch.int64, device="cuda")
for it in range(3):
    t = [time.perf_counter()]
    k.upload_ptr(hx.data_ptr(), hy.data_ptr()); t.append(time.perf_counter())
    k.sweep(1); t.append(time.perf_counter())
    w2 = k.interface_width(); t.append(time.perf_counter())
    k.download_ptr(hx.data_ptr(), hy.data_ptr()); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"upload {d[0]:.2f} ms  sweep {d[1]:.2f}  width {d[2]:.2f}  download {d[3]:.2f}  total {sum(d):.2f}")
# raw PCIe
torch.cuda.synchronize()
for it in range(3):
    t0 = time.perf_counter()
    dev[:L * wpr].copy_(hx, non_blocking=True); dev[L * wpr:].copy_(hy, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    hx.copy_(dev[:L * wpr], non_blocking=True); hy.copy_(dev[L * wpr:], non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    gb = 2 * L * wpr * 8 / 1e9
    print(f"raw H2D {gb / (t1 - t0):.1f} GB/s  D2H {gb / (t2 - t1):.1f} GB/s")
