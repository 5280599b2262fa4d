#!/usr/bin/env python3
"""Host<->device copy bandwidth of this box (pinned, 1 GiB): H2D alone, D2H alone, both at
once on two streams -- the ceiling of bench.py's e2e leg (1 GiB in + 1 GiB out per lattice-step)."""
import json
import time

import torch

n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return reps * n / (time.perf_counter() - t0) / 1e9


run(True, True, 1)
print(json.dumps({"h2d_GBps": run(True, False), "d2h_GBps": run(False, True),
                  "duplex_GBps_per_direction": run(True, True)}))
