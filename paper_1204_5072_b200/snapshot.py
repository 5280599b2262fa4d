"""Snapshot / exact-resume format (the reference has none).

One ``.npz`` file per lattice: the state in the reference's own word layout (KPZ: the two
slope planes of every replica, lattice.hpp:56-97; KMC: the occupancy words,
lattice.hpp:107-135) plus a JSON header with everything the counter-based RNG needs to
continue the trajectory bit for bit: model parameters, seeds, DT plan, the next sweep index
and the cumulative counters.  Loading re-uploads the words (KPZ: with the closure check of
lfg_kpz_upload) and restores the sweep index, so ``load(path).sweep(n)`` equals the
uninterrupted run.
"""
from __future__ import annotations

import json

import numpy as np

FORMAT = "lfg-snapshot"
VERSION = 1


def _header(model: str, **kw) -> np.ndarray:
    return np.frombuffer(json.dumps({"format": FORMAT, "version": VERSION, "model": model, **kw}).encode(),
                         dtype=np.uint8)


def _read(path: str, model: str):
    with np.load(path) as z:
        hdr = json.loads(bytes(z["header"]).decode())
        arrays = {k: z[k] for k in z.files if k != "header"}
    if hdr.get("format") != FORMAT or hdr.get("model") != model:
        raise ValueError(f"{path}: not an {FORMAT} file for model {model!r}")
    if int(hdr.get("version", 0)) > VERSION:
        raise ValueError(f"{path}: snapshot version {hdr['version']} is newer than {VERSION}")
    return hdr, arrays


def save_kpz(k, path: str) -> None:
    xs, ys, cnt = [], [], []
    for r in range(k.replicas):
        x, y = k.download(r)
        xs.append(x)
        ys.append(y)
        c = k.counters(r)
        cnt.append([int(c.attempts), int(c.deposits), int(c.detaches)])
    hdr = _header("kpz", L=k.L, p=k.p, q=k.q, seeds=[int(s) for s in k.seeds], plan=list(k.plan) + [int(k.sub)],
                  sweep_index=k.sweep_index, counters=cnt)
    np.savez(path, header=hdr, x=np.stack(xs), y=np.stack(ys))


def load_kpz(path: str, device: int = 0):
    from . import KpzLattice

    hdr, a = _read(path, "kpz")
    k = KpzLattice(int(hdr["L"]), float(hdr["p"]), float(hdr["q"]), seeds=hdr["seeds"],
                   block_x=int(hdr["plan"][0]), block_y=int(hdr["plan"][1]),
                   sub=int(hdr["plan"][2]) if len(hdr["plan"]) > 2 else 1, device=device)
    try:
        for r in range(k.replicas):
            k.upload(a["x"][r], a["y"][r], r)
        k.sweep_index = int(hdr["sweep_index"])
        k._cnt_base = [tuple(int(v) for v in c) for c in hdr["counters"]]
    except Exception:
        k.close()
        raise
    return k


def save_kmc(k, path: str) -> None:
    c = k.counters()
    hdr = _header("kmc", L=k.L, eps=k.eps, both_active=k.both_active, seed=k.seed, plan=k.plan, sub=k.sub,
                  sweep_index=k.sweep_index, counters=[int(c.attempts), int(c.successes)])
    np.savez(path, header=hdr, words=k.download())


def load_kmc(path: str, device: int = 0):
    from . import KmcLattice

    hdr, a = _read(path, "kmc")
    k = KmcLattice(int(hdr["L"]), float(hdr["eps"]), bool(hdr["both_active"]), int(hdr["seed"]),
                   block=int(hdr["plan"]), sub=int(hdr.get("sub", 1)), device=device)
    try:
        k.upload(a["words"])
        k.sweep_index = int(hdr["sweep_index"])
        k._cnt_base = tuple(int(v) for v in hdr["counters"])
    except Exception:
        k.close()
        raise
    return k
