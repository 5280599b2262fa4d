#!/usr/bin/env python3
"""Statistical tier: GPU two-layer DTr vs the reference's sequential sweep.

    python scripts/stat_validate.py --L 256 --t 100 --seeds 200 --out gpurun_out/stats.json

Observables at sample times t (MCS), per realization:
  * W^2(t)   -- interface_width (kpz.cpp:62-81), device scan vs lf::interface_width
  * <h>(t)   -- -1 + 2 (deposits - detaches) / L^2 (the flat
                mean height is -1)
The reference ensemble runs lf::kpz_sweep_sequential (oracle/_ref = the
unmodified sources, lcg64 streams, one seed per realization) on all host
cores.  Reports ensemble means, standard errors, z = (gpu - ref)/combined SE,
and the growth exponent beta from the same estimator on both sides
(least-squares slope of log <W^2> vs log t over [t_lo, t_hi], /2).
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


def sample_times(tmax: int):
    ts = sorted({max(1, int(round(1.1 ** k))) for k in range(0, 200) if round(1.1 ** k) <= tmax} | {tmax})
    return ts


def ref_run(args):
    L, p, q, seed, ts = args
    import pyoracle

    ref = pyoracle.RefLib()
    x, y = ref.make_flat(L)
    st, t, w2, hm = seed, 0, [], []
    dep = 0
    for tt in ts:
        c, st = ref.kpz_sweep_sequential(L, x, y, p, q, "lcg64", st, tt - t)
        t = tt
        w2.append(ref.interface_width(L, x, y))
        if q == 0.0:
            dep += int(c[1])
            hm.append(-1.0 + 2.0 * dep / (L * L))
    return w2, hm


def gpu_runs(L, p, q, seeds, ts, block_x, block_y, sub=0):
    import paper_1204_5072_b200 as lfg

    w2 = np.zeros((len(seeds), len(ts)))
    hm = np.zeros((len(seeds), len(ts)))
    chunk = 64
    for c0 in range(0, len(seeds), chunk):
        ss = seeds[c0:c0 + chunk]
        with lfg.KpzLattice(L, p, q, seeds=ss, block_x=block_x, block_y=block_y, sub=sub) as k:
            k.make_flat_slopes()
            t = 0
            for j, tt in enumerate(ts):
                k.sweep_async(tt - t)
                t = tt
                for r in range(len(ss)):
                    w2[c0 + r, j] = k.interface_width(r)
                    c = k.counters(r)
                    hm[c0 + r, j] = -1.0 + 2.0 * (c.deposits - c.detaches) / (L * L)
    return w2, hm


def beta_fit(ts, w2mean, lo, hi):
    t = np.array(ts, float)
    m = (t >= lo) & (t <= hi)
    if m.sum() < 2:
        return None
    slope = np.polyfit(np.log(t[m]), np.log(np.asarray(w2mean)[m]), 1)[0]
    return slope / 2.0


def per_seed_beta(ts, w2, lo, hi):
    out = [beta_fit(ts, row, lo, hi) for row in w2]
    return np.array([b for b in out if b is not None])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--t", type=int, default=100)
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--ref-seeds", type=int, default=None)
    ap.add_argument("--p", type=float, default=1.0)
    ap.add_argument("--q", type=float, default=0.0)
    ap.add_argument("--block-x", type=int, default=0)
    ap.add_argument("--block-y", type=int, default=0)
    ap.add_argument("--beta-lo", type=int, default=32)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--seed-base", type=int, default=0, help="offset of the GPU and reference seed sets")
    ap.add_argument("--sub", type=int, default=0, help="DTr sub-sweeps per MCS (0: plan default 4; 1: paper)")
    ap.add_argument("--ref-json", default=None,
                    help="reuse the reference ensemble (t, ref means / SEs, ref_seeds) of an earlier report")
    ap.add_argument("--save-samples", action="store_true", help="store per-seed W^2(t) and <h>(t)")
    a = ap.parse_args()
    ts = sample_times(a.t)
    seeds = [1000003 * (i + 1) + a.seed_base for i in range(a.seeds)]
    t0 = time.time()
    gw, gh = gpu_runs(a.L, a.p, a.q, seeds, ts, a.block_x, a.block_y, a.sub)
    tg = time.time() - t0
    rep = {"L": a.L, "p": a.p, "q": a.q, "t": ts, "gpu_seeds": a.seeds, "gpu_seconds": tg, "sub": a.sub or 4,
           "gpu": {"w2_mean": gw.mean(0).tolist(), "w2_se": (gw.std(0, ddof=1) / math.sqrt(len(seeds))).tolist(),
                   "h_mean": gh.mean(0).tolist(), "h_se": (gh.std(0, ddof=1) / math.sqrt(len(seeds))).tolist()}}
    if a.save_samples:
        rep["gpu"]["w2"] = gw.tolist()
        rep["gpu"]["h"] = gh.tolist()
    if a.no_ref:
        lo, hi = a.beta_lo, a.t
        sg = per_seed_beta(ts, gw, lo, hi)
        rep["beta"] = {"window": [lo, hi], "estimator": "slope of log <W^2> vs log t, /2",
                       "gpu": beta_fit(ts, gw.mean(0), lo, hi),
                       "gpu_per_seed_mean": float(sg.mean()) if len(sg) else None,
                       "gpu_per_seed_se": float(sg.std(ddof=1) / math.sqrt(len(sg))) if len(sg) > 1 else None}
    if a.ref_json:
        with open(a.ref_json) as f:
            old = json.load(f)
        assert old["t"] == ts and old["L"] == a.L and old["p"] == a.p and old["q"] == a.q, "incompatible reference"
        R = old["ref"]
        rep["ref_seeds"] = old["ref_seeds"]
        rep["ref_source"] = a.ref_json
        rep["ref"] = R
        g = rep["gpu"]
        zw = (np.array(g["w2_mean"]) - np.array(R["w2_mean"])) / np.hypot(g["w2_se"], R["w2_se"])
        rep["z_w2"] = zw.tolist()
        rep["max_abs_z_w2"] = float(np.max(np.abs(zw)))
        if "h_mean" in R:
            zh = (np.array(g["h_mean"]) - np.array(R["h_mean"])) / np.hypot(g["h_se"], R["h_se"])
            rep["z_h"] = zh.tolist()
            rep["max_abs_z_h"] = float(np.max(np.abs(zh)))
        lo, hi = a.beta_lo, a.t
        rep["beta"] = {"window": [lo, hi], "estimator": "slope of log <W^2> vs log t, /2",
                       "gpu": beta_fit(ts, gw.mean(0), lo, hi), "ref": beta_fit(ts, R["w2_mean"], lo, hi)}
        rep["beta"]["diff"] = rep["beta"]["gpu"] - rep["beta"]["ref"]
    elif not a.no_ref:
        nref = a.ref_seeds or a.seeds
        t0 = time.time()
        with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
            res = list(ex.map(ref_run, [(a.L, a.p, a.q, 7 * i + 1 + a.seed_base, ts) for i in range(nref)]))
        tr = time.time() - t0
        rw = np.array([r[0] for r in res])
        rh = np.array([r[1] for r in res]) if a.q == 0.0 else None
        rep["ref_seeds"] = nref
        rep["ref_seconds"] = tr
        rep["ref"] = {"w2_mean": rw.mean(0).tolist(), "w2_se": (rw.std(0, ddof=1) / math.sqrt(nref)).tolist()}
        zw = (gw.mean(0) - rw.mean(0)) / np.sqrt(gw.var(0, ddof=1) / len(seeds) + rw.var(0, ddof=1) / nref)
        rep["z_w2"] = zw.tolist()
        if rh is not None:
            rep["ref"]["h_mean"] = rh.mean(0).tolist()
            rep["ref"]["h_se"] = (rh.std(0, ddof=1) / math.sqrt(nref)).tolist()
            zh = (gh.mean(0) - rh.mean(0)) / np.sqrt(gh.var(0, ddof=1) / len(seeds) + rh.var(0, ddof=1) / nref)
            rep["z_h"] = zh.tolist()
        lo, hi = a.beta_lo, a.t
        bg, br = beta_fit(ts, gw.mean(0), lo, hi), beta_fit(ts, rw.mean(0), lo, hi)
        sg, sr = per_seed_beta(ts, gw, lo, hi), per_seed_beta(ts, rw, lo, hi)
        rep["beta"] = {"window": [lo, hi], "estimator": "slope of log <W^2> vs log t, /2",
                       "gpu": bg, "ref": br, "diff": None if bg is None or br is None else bg - br,
                       "gpu_per_seed_mean": float(sg.mean()) if len(sg) else None,
                       "gpu_per_seed_se": float(sg.std(ddof=1) / math.sqrt(len(sg))) if len(sg) > 1 else None,
                       "ref_per_seed_mean": float(sr.mean()) if len(sr) else None,
                       "ref_per_seed_se": float(sr.std(ddof=1) / math.sqrt(len(sr))) if len(sr) > 1 else None}
        rep["max_abs_z_w2"] = float(np.max(np.abs(zw)))
        if rh is not None:
            rep["max_abs_z_h"] = float(np.max(np.abs(zh)))
    txt = json.dumps(rep)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            f.write(txt)
    summary = {k: rep.get(k) for k in ("L", "gpu_seeds", "ref_seeds", "max_abs_z_w2", "max_abs_z_h", "beta")}
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
