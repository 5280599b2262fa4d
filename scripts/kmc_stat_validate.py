#!/usr/bin/env python3
"""Statistical tier for the KMC path: GPU two-layer DT vs the reference's
sequential Metropolis sweep (kmc_mcs_sequential, kmc.cpp:5-18).

    python scripts/kmc_stat_validate.py --L 64 --t 200 --seeds 256 --both 0 --out gpurun_out/kmc_stats.json

Observable: open bonds per particle (open_bonds_per_particle, kmc.cpp:20-40)
at t = 1, 2, 5, 10, 20, 50, 100, 200 MCS from a random 50/50 alloy
(make_random_alloy, lattice.cpp:117-132; eps = 1.5).  GPU: KmcLattice (default
plan, 16^3 blocks), Philox alloy init; reference: the unmodified sources
(oracle/_ref, lcg64 streams, one seed per realization) on all host cores.
Reports ensemble means, standard errors and z = (gpu - ref) / combined SE.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def ref_run(args):
    L, c, eps, both, seed, ts = args
    import pyoracle

    ref = pyoracle.RefLib()
    w, st = ref.make_random_alloy(L, c, "lcg64", seed)
    out, t = [], 0
    for tt in ts:
        _, st = ref.kmc_sweep_sequential(L, w, eps, both, "lcg64", st, tt - t)
        t = tt
        out.append(ref.open_bonds_per_particle(L, w))
    return out


def gpu_runs(L, c, eps, both, seeds, ts, block, sub=0):
    import paper_1204_5072_b200 as lfg

    ob = np.zeros((len(seeds), len(ts)))
    for i, s in enumerate(seeds):
        with lfg.KmcLattice(L, eps, bool(both), s, block=block, sub=sub) as k:
            k.make_random_alloy(c, s ^ 0x5DEECE66D)
            t = 0
            for j, tt in enumerate(ts):
                k.sweep_async(tt - t)
                t = tt
                ob[i, j] = k.open_bonds_per_particle()
    return ob


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--t", type=int, default=200)
    ap.add_argument("--seeds", type=int, default=256)
    ap.add_argument("--ref-seeds", type=int, default=None)
    ap.add_argument("--both", type=int, default=0)
    ap.add_argument("--eps", type=float, default=1.5)
    ap.add_argument("--c", type=float, default=0.5)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--sub", type=int, default=0, help="sub-sweeps per MCS (0: plan default 1; 4)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ts = [t for t in (1, 2, 5, 10, 20, 50, 100, 200, 500, 1000) if t <= a.t]
    if ts[-1] != a.t:
        ts.append(a.t)
    seeds = [7919 * (i + 1) for i in range(a.seeds)]
    t0 = time.time()
    g = gpu_runs(a.L, a.c, a.eps, a.both, seeds, ts, a.block, a.sub)
    tg = time.time() - t0
    nref = a.ref_seeds or a.seeds
    t0 = time.time()
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        r = np.array(list(ex.map(ref_run, [(a.L, a.c, a.eps, a.both, 13 * i + 1, ts) for i in range(nref)])))
    tr = time.time() - t0
    gm, gs = g.mean(0), g.std(0, ddof=1) / math.sqrt(len(seeds))
    rm, rs = r.mean(0), r.std(0, ddof=1) / math.sqrt(nref)
    z = (gm - rm) / np.sqrt(gs ** 2 + rs ** 2)
    rep = {"L": a.L, "c": a.c, "eps": a.eps, "both": a.both, "sub": a.sub or 1, "t": ts, "gpu_seeds": len(seeds), "ref_seeds": nref,
           "gpu_seconds": tg, "ref_seconds": tr, "gpu": {"mean": gm.tolist(), "se": gs.tolist()},
           "ref": {"mean": rm.tolist(), "se": rs.tolist()}, "z": z.tolist(), "max_abs_z": float(np.max(np.abs(z))),
           "rel_final": float(gm[-1] / rm[-1] - 1.0)}
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(rep, f)
    print(json.dumps({k: rep[k] for k in ("L", "both", "gpu_seeds", "ref_seeds", "max_abs_z", "rel_final")}))
    for j, t in enumerate(ts):
        print(f"t={t:5d}  gpu {gm[j]:.5f} +- {gs[j]:.5f}   ref {rm[j]:.5f} +- {rs[j]:.5f}   z {z[j]:+.2f}")


if __name__ == "__main__":
    main()
