#!/usr/bin/env python3
"""Generate tests/golden/golden.json by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every value below is produced by oracle/_ref/liblfref.so, i.e. by the
reference sources under /root/reference/proj/src compiled as they lie plus
oracle/ref_shim.cpp.  The DTr cases drive lf::detail::kpz_attempt_impl<false>
(kpz.hpp:71-107) through the schedule in oracle/oracle_core.hpp; the KMC DT
cases use lf::exchange_probability (kmc.hpp:70-76).  Philox KATs are the
published Random123 vectors (the reference has no counter-based RNG).

Lattices are recorded by SHA-256 of their little-endian words (plus the full
words for the smallest cases) so the fixtures stay small.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import pyoracle as po  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# (L, bx, by, p, q, seed, sweep0, nsweeps, sub): sub = 4 is the default plan
# (sub-sweeps + Poisson tile counts), sub = 1 the paper's single-origin scheme,
# sub = 8 eight sub-sweeps per MCS.
KPZ_DTR_CASES = [
    (64, 32, 32, 1.0, 0.0, 1, 0, 1, 4),
    (64, 32, 32, 1.0, 0.0, 1, 0, 4, 4),
    (64, 32, 16, 0.95, 0.05, 7, 3, 3, 4),
    (128, 64, 32, 1.0, 0.0, 2, 0, 3, 4),
    (128, 32, 64, 0.5, 0.5, 3, 10, 2, 4),
    (256, 128, 64, 1.0, 0.0, 11, 0, 2, 4),
    (256, 64, 128, 0.95, 0.05, 12, 5, 2, 4),
    (512, 256, 128, 1.0, 0.0, 1, 0, 2, 4),
    (1024, 512, 128, 1.0, 0.0, 1, 0, 1, 4),
    (1024, 512, 64, 0.95, 0.05, 5, 100, 1, 4),
    (2048, 1024, 128, 1.0, 0.0, 1, 0, 1, 4),
    (2048, 1024, 128, 0.25, 0.75, 9, 0, 1, 4),
    (64, 32, 32, 1.0, 0.0, 1, 0, 2, 1),
    (256, 128, 64, 0.95, 0.05, 12, 5, 2, 1),
    (1024, 512, 128, 1.0, 0.0, 1, 0, 1, 1),
    (2048, 1024, 128, 0.25, 0.75, 9, 0, 1, 1),
    (64, 32, 16, 1.0, 0.0, 4, 0, 3, 8),
    (256, 128, 64, 0.95, 0.05, 12, 5, 2, 8),
    (1024, 512, 128, 1.0, 0.0, 1, 0, 1, 8),
    (2048, 1024, 128, 0.95, 0.05, 9, 3, 1, 8),
]

# (L, bk, eps, both, c, alloy_seed, seed, sweep0, nsweeps)
KMC_DT_CASES = [  # (..., sub): sub = 4 is the four-sub-sweep plan option
    (32, 16, 1.5, 0, 0.5, 5, 3, 0, 2, 1),
    (32, 16, 1.5, 1, 0.5, 5, 3, 0, 2, 1),
    (64, 16, 1.5, 1, 0.325, 1, 9, 7, 1, 1),
    (64, 32, 0.5, 0, 0.5, 2, 4, 0, 1, 1),
    (64, 16, 0.0, 1, 0.5, 3, 4, 0, 1, 1),
    (32, 16, 1.5, 1, 0.5, 5, 3, 0, 2, 4),
    (64, 16, 1.5, 0, 0.325, 1, 9, 7, 1, 4),
    (64, 32, 1.5, 1, 0.5, 2, 4, 0, 1, 4),
]


def main() -> None:
    ref = po.RefLib()
    out: dict = {"generated_by": "tests/golden/make_golden.py (reference sources via oracle/_ref)"}

    out["philox_kat"] = [  # Random123 published KATs for philox4x32_10
        {"ctr": [0, 0, 0, 0], "key": [0, 0], "out": [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]},
        {"ctr": [0xFFFFFFFF] * 4, "key": [0xFFFFFFFF] * 2, "out": [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]},
        {"ctr": [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], "key": [0xA4093822, 0x299F31D0],
         "out": [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]},
    ]

    rng = []
    for kind in ("lcg32", "lcg64", "tinymt"):
        for seed, sid in ((12345, 0), (1, 0), (0, 0), (7, 3)):
            rng.append({"kind": kind, "seed": seed, "stream_id": sid,
                        "draws": ref.rng_draws(kind, seed, 8, sid).tolist()})
    rng.append({"kind": "lcg64", "seed": 12345, "stream_id": 0, "skip": 1000,
                "draws": ref.rng_draws("lcg64", 12345, 4, 0, 1000).tolist()})
    out["rng"] = rng
    out["split_streams"] = [
        {"kind": k, "seed": 7, "count": 3, "stride": 1 << 40,
         "states": [int(v) for v in ref.split_streams_state(k, 7, 3)]} for k in ("lcg32", "lcg64")]

    flat = []
    for L in (4, 8, 64, 256):
        x, y = ref.make_flat(L)
        h = ref.reconstruct_heights(L, x, y)
        flat.append({"L": L, "w2": ref.interface_width(L, x, y), "sx": sha(x), "sy": sha(y),
                     "sum": int(h.astype(np.int64).sum()), "sum2": int((h.astype(np.int64) ** 2).sum())})
    out["kpz_flat"] = flat

    # Single attempts on flat L=8.
    att = []
    for (i, j) in ((1, 1), (0, 0), (3, 5), (2, 2)):
        x, y = ref.make_flat(8)
        o = ref.kpz_attempt(8, x, y, i, j, 1.0, 0.0, 0.5)
        att.append({"i": i, "j": j, "outcome": o, "x": [int(v) for v in x], "y": [int(v) for v in y]})
    out["kpz_attempt_flat8"] = att

    # Sequential reference sweeps (the statistical oracle), lcg64.
    seq = []
    for (L, p, q, seed, sweeps) in ((64, 1.0, 0.0, 99, 1), (64, 0.95, 0.05, 3, 2), (256, 1.0, 0.0, 1, 2)):
        x, y = ref.make_flat(L)
        c, st = ref.kpz_sweep_sequential(L, x, y, p, q, "lcg64", seed, sweeps)
        seq.append({"L": L, "p": p, "q": q, "seed": seed, "sweeps": sweeps, "attempts": int(c[0]),
                    "successes": int(c[1]), "state": int(st), "sx": sha(x), "sy": sha(y),
                    "w2": ref.interface_width(L, x, y)})
    out["kpz_sequential"] = seq

    # C1 trajectory head (L=1024, p=1, q=0, lcg64 seed 1): W2 at t = 1, 2, 4, 8.
    L = 1024
    x, y = ref.make_flat(L)
    st, t, traj = 1, 0, []
    for target in (1, 2, 4, 8):
        _, st = ref.kpz_sweep_sequential(L, x, y, 1.0, 0.0, "lcg64", st, target - t)
        t = target
        traj.append({"t": t, "w2": ref.interface_width(L, x, y)})
    out["kpz_c1_head"] = traj

    dtr = []
    for (L, bx, by, p, q, seed, sweep0, ns, sub) in KPZ_DTR_CASES:
        x, y = ref.make_flat(L)
        c = ref.kpz_sweep_dtr(L, x, y, p, q, seed, sweep0, ns, bx, by, sub)
        h = ref.reconstruct_heights(L, x, y).astype(np.int64)
        rec = {"L": L, "bx": bx, "by": by, "p": p, "q": q, "seed": seed, "sweep0": sweep0,
               "nsweeps": ns, "sub": sub, "counters": [int(v) for v in c], "sx": sha(x), "sy": sha(y),
               "w2": ref.interface_width(L, x, y), "sum": int(h.sum()), "sum2": int((h ** 2).sum())}
        if L == 64:
            rec["x"] = [int(v) for v in x]
            rec["y"] = [int(v) for v in y]
        dtr.append(rec)
    out["kpz_dtr"] = dtr

    alloys = []
    for (L, c, seed) in ((16, 0.5, 5), (64, 0.325, 1), (32, 0.5, 5), (64, 0.5, 2)):
        w, st = ref.make_random_alloy(L, c, "lcg64", seed)
        alloys.append({"L": L, "c": c, "seed": seed, "count_b": ref.count_b(L, w), "sha": sha(w),
                       "open_bonds": ref.open_bonds_per_particle(L, w), "state": int(st)})
    out["kmc_alloy"] = alloys

    kseq = []
    for both in (0, 1):
        w, st = ref.make_random_alloy(16, 0.5, "lcg64", 5)
        c, st2 = ref.kmc_sweep_sequential(16, w, 1.5, both, "lcg64", st, 1)
        kseq.append({"L": 16, "both": both, "eps": 1.5, "attempts": int(c[0]), "successes": int(c[1]),
                     "sha": sha(w), "open_bonds": ref.open_bonds_per_particle(16, w)})
    out["kmc_sequential"] = kseq

    kdt = []
    for (L, bk, eps, both, c, aseed, seed, sweep0, ns, sub) in KMC_DT_CASES:
        w, _ = ref.make_random_alloy(L, c, "lcg64", aseed)
        cnt = ref.kmc_sweep_dt(L, w, eps, both, seed, sweep0, ns, bk, sub)
        kdt.append({"L": L, "bk": bk, "eps": eps, "both": both, "c": c, "alloy_seed": aseed, "seed": seed, "sub": sub,
                    "sweep0": sweep0, "nsweeps": ns, "counters": [int(v) for v in cnt], "sha": sha(w),
                    "count_b": ref.count_b(L, w), "open_bonds": ref.open_bonds_per_particle(L, w)})
    out["kmc_dt"] = kdt

    out["metropolis_eps1.5"] = [ref.metropolis_prob(12, 12 - d, 1.5) for d in range(13)]

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
