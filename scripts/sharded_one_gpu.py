#!/usr/bin/env python3
"""Overhead of the one-process sharded KPZ handle (lfg_kpz_create_sharded) with all
strips on ONE GPU: configs[2]'s lattice (L = 2^17, p = 0.95, q = 0.05) as 1, 2, 4, 8
strips.  The strips share the GPU's SMs, so the ideal is the single-lattice rate; the gap
is the cost of the per-sub-sweep peer copies and per-phase event ordering (host API calls
and the smaller per-strip grids), i.e. an upper bound on the exchange overhead of the
N-GPU path apart from NVLink transfer time.  Prints one JSON line per strip count."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1204_5072_b200 as lfg  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
for n in (1, 2, 4, 8):
    if n == 1:
        lat = lfg.KpzLattice(L, 0.95, 0.05, 1)
    else:
        lat = lfg.ShardedKpzLattice(L, 0.95, 0.05, 1, devices=[0] * n)
    lat.make_flat_slopes()
    lat.sweep(2)
    c0 = lat.counters().attempts
    t0 = time.perf_counter()
    lat.sweep(steps)
    att = lat.counters().attempts - c0  # counters synchronise
    dt = time.perf_counter() - t0
    print(json.dumps({"L": L, "strips": n, "attempts_per_ns": att / (dt * 1e9), "ms_per_mcs": dt * 1e3 / steps}),
          flush=True)
    lat.close()
