#!/usr/bin/env python3
"""Compute side of the slab-sharded KMC sweep (BASELINE configs[4], 1024^3) on one GPU.

Each GPU of an N-GPU run executes one rank's slab phases (lfg_kmc_slab_phase over L/N
planes); timing rank 0's launches alone gives the per-GPU compute time, and
    eff_compute(N) = T_single / (N * T_rank0)
bounds the strong-scaling efficiency from the compute side (plane exchanges excluded).

    python scripts/slab_compute_proxy.py [both]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402
from paper_1204_5072_b200.shard import CudaSlabEngine, SlabPlan  # noqa: E402

L, EPS, BK = 1024, 1.5, 16
both = bool(int(sys.argv[1])) if len(sys.argv) > 1 else True
SWEEPS, WARM = 5, 2


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


st = torch.cuda.Stream()
with lfg.KmcLattice(L, EPS, both, 7, block=BK) as k:
    k.set_stream(st.cuda_stream)
    k.make_random_alloy(0.5, 3)
    k.sweep_async(WARM)
    t_single = timed(st, lambda: k.sweep_async(SWEEPS)) / SWEEPS
out = {"L": L, "both": both, "block": BK, "single_ms_per_mcs": t_single,
       "single_attempts_per_ns": L ** 3 // 2 / (t_single * 1e6), "ranks": {}}
for world in (2, 4, 8):
    pl = SlabPlan(L, world, BK)
    e = CudaSlabEngine(pl, EPS, both, 7, 0)
    try:
        e.init_random_alloy(0, pl.cap, 0.5, 3)

        def run(n, s0):
            for s in range(s0, s0 + n):
                for kk in range(8):
                    b0, nb = pl.block_rows(0)
                    e.phase(s, kk, b0, nb)

        run(WARM, 0)
        t_rank = timed(e.stream, lambda: run(SWEEPS, WARM)) / SWEEPS
        out["ranks"][world] = {"rank0_ms_per_mcs": t_rank, "eff_compute": t_single / (world * t_rank),
                               "projected_attempts_per_ns": L ** 3 // 2 / (t_rank * 1e6)}
    finally:
        e.close()
print(json.dumps(out))
