#!/usr/bin/env python3
"""Compare dt_explore ensembles against a reference ensemble (rs): relative W^2 / <h>
difference and z-score per sample time.  Usage: compare.py REF.json A.json [B.json ...]"""
import json
import sys


def load(p):
    with open(p) as f:
        return json.load(f)


ref = load(sys.argv[1])
for p in sys.argv[2:]:
    d = load(p)
    print(f"== {p}  (mini={d.get('mini')} counts={d.get('counts')} thin={d.get('thin')} "
          f"skip={d.get('skip')} tc={d.get('tc')} td={d.get('td')} tlog={d.get('tlog')} "
          f"{d['bx']}x{d['by']} reps={d['replicas']} {d['seconds']:.1f}s)")
    for i, t in enumerate(d["t"]):
        if t not in ref["t"]:
            continue
        j = ref["t"].index(t)
        a, sa, b, sb = d["w2_mean"][i], d["w2_se"][i], ref["w2_mean"][j], ref["w2_se"][j]
        z = (a - b) / (sa * sa + sb * sb) ** 0.5
        ha, hsa, hb, hsb = d["h_mean"][i], d["h_se"][i], ref["h_mean"][j], ref["h_se"][j]
        zh = (ha - hb) / max(1e-300, (hsa * hsa + hsb * hsb) ** 0.5)
        print(f"  t={t:5d} W2 {a:9.5f} vs {b:9.5f} rel {100*(a/b-1):+7.3f}% z {z:+6.1f} | "
              f"dh {100*(ha/hb-1):+8.4f}% z {zh:+6.1f}")
