#!/usr/bin/env python3
"""C1 statistical tier over many independent 64 + 64 seed sets (default plan): the
distribution of max|z| over the 59 sample times for reference vs reference (the null)
and GPU vs reference, and the pooled bias.  Usage: python scripts/c1_null.py OUT.json"""
import glob
import itertools
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
files = [os.path.join(ROOT, "profiles/stats/r02", f) for f in ("C1_64.json", "C1_64_b5000.json", "C1_64_b9000.json")]
files += sorted(glob.glob(os.path.join(ROOT, "profiles/stats/r02/c1sets/C1_64_b*.json")))
sets = [json.load(open(f)) for f in files]
t = np.array(sets[0]["t"])


def arr(d, side, key):
    return np.array(d[side][key], dtype=float)


def maxz(a, b, key):
    m = arr(a[0], a[1], key + "_mean") - arr(b[0], b[1], key + "_mean")
    se = np.sqrt(arr(a[0], a[1], key + "_se") ** 2 + arr(b[0], b[1], key + "_se") ** 2)
    z = m / se
    return float(np.abs(z).max()), float(z.mean())


out = {"sets": [os.path.relpath(f, ROOT) for f in files], "n_sets": len(sets), "seeds_per_set": 64}
for key in ("w2", "h"):
    null = [maxz((a, "ref"), (b, "ref"), key)[0] for a, b in itertools.combinations(sets, 2)]
    gvr = [maxz((g, "gpu"), (r, "ref"), key) for g in sets for r in sets]
    out[key] = {
        "null_ref_vs_ref": {"pairs": len(null), "max_abs_z_median": float(np.median(null)),
                            "frac_above_3": float(np.mean(np.array(null) > 3)), "max": float(max(null))},
        "gpu_vs_ref": {"pairs": len(gvr), "max_abs_z_median": float(np.median([m for m, _ in gvr])),
                       "frac_above_3": float(np.mean(np.array([m for m, _ in gvr]) > 3)),
                       "mean_z_median": float(np.median([z for _, z in gvr]))},
    }
    # pooled over all sets: GPU vs reference at every t
    n = len(sets)
    gm = np.mean([arr(d, "gpu", key + "_mean") for d in sets], axis=0)
    rm = np.mean([arr(d, "ref", key + "_mean") for d in sets], axis=0)
    gse = np.sqrt(np.sum([arr(d, "gpu", key + "_se") ** 2 for d in sets], axis=0)) / n
    rse = np.sqrt(np.sum([arr(d, "ref", key + "_se") ** 2 for d in sets], axis=0)) / n
    z = (gm - rm) / np.sqrt(gse ** 2 + rse ** 2)
    rel = (gm / rm - 1) * 100
    out[key]["pooled"] = {"seeds_each_side": 64 * n, "max_abs_z": float(np.abs(z).max()), "mean_z": float(z.mean()),
                          "rel_diff_pct_mean_t_ge_10": float(rel[t >= 10].mean()),
                          "rel_diff_pct_at": {str(int(tt)): float(rel[i]) for i, tt in enumerate(t)
                                              if int(tt) in (1, 10, 100, 1000)}}
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "/dev/stdout", "w"), indent=1)
