#!/usr/bin/env python3
"""Compute side of the strip-sharded KPZ sweep (BASELINE configs[2], L = 2^17) on one GPU.

One rank's share of an MCS on N GPUs is its strip: 4 phase launches per sub-sweep over L/N rows
(lfg_kpz_strip_phase).  Timing rank 0's launches alone on one B200 gives the per-GPU
compute time of an N-GPU run (each GPU runs exactly this workload); against the
single-lattice sweep it bounds the strong-scaling efficiency from the compute side:
    eff_compute(N) = T_single / (N * T_rank0).
Exchanges (one ghost row per phase, the per-sweep roll, the step barriers) are not
included; this is a proxy for the part of the N-GPU run that one GPU can measure.

    python scripts/shard_compute_proxy.py [p q]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1204_5072_b200 as lfg  # noqa: E402
from paper_1204_5072_b200.shard import CudaStripEngine, StripPlan  # noqa: E402

L = 1 << 17
p = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
q = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
SWEEPS, WARM = 6, 2


def timed(stream, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


st = torch.cuda.Stream()
with lfg.KpzLattice(L, p, q, 1) as k:
    k.set_stream(st.cuda_stream)
    k.make_flat_slopes()
    k.sweep_async(WARM)
    t_single = timed(st, lambda: k.sweep_async(SWEEPS)) / SWEEPS
    bx, by = k.plan
out = {"L": L, "p": p, "q": q, "plan": [bx, by], "single_ms_per_sweep": t_single,
       "single_attempts_per_ns": L * L / (t_single * 1e6), "ranks": {}}
for world in (2, 4, 8):
    pl = StripPlan(L, world, bx, by)
    e = CudaStripEngine(pl, p, q, 1, 0)
    try:
        # the ring buffer starts all-zero (a valid spin field); its content does not change the cost

        def run(n, s0):  # n MCS from MCS s0: pl.sub sub-sweeps of 4 phases each
            for s in range(s0 * pl.sub, (s0 + n) * pl.sub):
                for kk in range(4):
                    b0, nb = pl.block_rows(0)
                    e.phase(s, kk, b0, nb)

        run(WARM, 0)
        t_rank = timed(e.stream, lambda: run(SWEEPS, WARM)) / SWEEPS
        out["ranks"][world] = {"rank0_ms_per_sweep": t_rank,
                               "eff_compute": t_single / (world * t_rank),
                               "projected_attempts_per_ns": L * L / (t_rank * 1e6)}
    finally:
        e.close()
print(json.dumps(out))
