#!/usr/bin/env python3
"""Small runs of every sweep-kernel path, for compute-sanitizer (scripts/sanitize.sh).

    python scripts/sanitize_cases.py [case ...]   (cases: see CASES below)

Each case runs a few sweeps through the C ABI and compares the lattice and
counters with the CPU oracle (test infrastructure, oracle/), so a sanitizer
pass is also a parity pass.  Kernel selection knobs (LFG_KMC_WIDE) are set by
sanitize.sh per case."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_1204_5072_b200 as lfg  # noqa: E402
import pyoracle  # noqa: E402

orc = pyoracle.Oracle()


def kpz(L, p, q, bx, by, sweeps=1, seed=11, sub=4, strips=0):
    x, y = orc.kpz_flat(L)
    c_ref = orc.kpz_sweep_dtr(L, x, y, p, q, seed, 0, sweeps, bx, by, sub)
    if strips:  # one-process sharded handle, all strips on device 0
        with lfg.ShardedKpzLattice(L, p, q, seed, devices=[0] * strips, block_x=bx, block_y=by, sub=sub) as k:
            k.make_flat_slopes()
            c = k.sweep(sweeps)
            gx, gy = k.download()
            w2 = k.interface_width()
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist(), (c, c_ref)
        assert np.array_equal(gx, x) and np.array_equal(gy, y)
        assert w2 == orc.interface_width(L, x, y)
        return
    with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by, sub=sub) as k:
        k.make_flat_slopes()
        c = k.sweep(sweeps)
        gx, gy = k.download()
        w2 = k.interface_width()
    assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist(), (c, c_ref)
    assert np.array_equal(gx, x) and np.array_equal(gy, y)
    assert w2 == orc.interface_width(L, x, y)


def kmc(L, both, bk, sweeps=1, seed=3, share=1):
    w, _ = orc.kmc_random_alloy(L, 0.5, "lcg64", 5)
    w_ref = w.copy()
    c_ref = orc.kmc_sweep_dt(L, w_ref, 1.5, int(both), seed, 0, sweeps, bk)
    with lfg.KmcLattice(L, 1.5, both, seed, block=bk) as k:
        if share > 1:
            k.set_concurrency(share)  # launcher sizes its kernel choice as if `share` lattices ran together
        k.upload(w)
        c = k.sweep(sweeps)
        g = k.download()
        ob = k.open_bond_sums()
    assert [c.attempts, c.successes] == c_ref.tolist(), (c, c_ref)
    assert np.array_equal(g, w_ref)
    assert tuple(ob) == tuple(orc.kmc_open_bond_sums(L, w_ref))


CASES = {
    "kpz_full": lambda: kpz(2048, 1.0, 0.0, 1024, 128),          # 1024-wide path (bulk copies at the wrap), chained phases
    "kpz_general": lambda: kpz(2048, 0.95, 0.05, 1024, 128),     # p < 1 acceptance draws
    "kpz_tensor": lambda: kpz(4096, 1.0, 0.0, 1024, 128),        # TMA tensor-map staging / write-back away from the wrap
    "kpz_small": lambda: kpz(256, 0.95, 0.05, 128, 64),          # generic staging (block narrower than 1024)
    "kpz_sub1": lambda: kpz(2048, 0.95, 0.05, 1024, 128, sub=1),  # the paper's scheme (512 rounds, no skips)
    "kpz_sub8": lambda: kpz(2048, 0.95, 0.05, 1024, 128, sub=8),  # eight sub-sweeps (68 rounds, Poisson(1/4) skips)
    "kpz_sharded": lambda: kpz(2048, 0.95, 0.05, 1024, 128, strips=4),  # one-process sharded handle
    "kmc_wide": lambda: kmc(64, True, 16),                       # producer/consumer 16^3 kernel (LFG_KMC_PC=0: full warp)
    "kmc_wide1": lambda: kmc(64, True, 16),                      # (run with LFG_KMC_PC=0: single full-warp kernel)
    "kmc_narrow": lambda: kmc(64, False, 16),                    # 8-lane 16^3 kernel (env LFG_KMC_WIDE=0)
    "kmc_quad": lambda: kmc(64, True, 16, share=512),            # 4-blocks-per-warp 16^3 kernel (512^3+ regime)
    "kmc_32": lambda: kmc(64, True, 32),                         # 32^3 blocks
}

if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        CASES[name]()
        print(f"{name}: OK (bit-exact vs oracle)", flush=True)
