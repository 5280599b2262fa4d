"""Bit-exact parity at the BASELINE sizes (run with -m gpu on a B200).

The CUDA path (through the C ABI, liblfg.so) against the oracle restatement
(oracle/_build/liboracle.so, itself pinned to the unmodified reference in
tests/test_oracle.py) on the lattices the benchmark and the scaling runs use:

  * KPZ configs[1]  L = 2^16, p = 1,                 1 sweep, default plan (1024 x 128)
  * KPZ configs[2]  L = 2^17, p = 0.95, q = 0.05,    1 sweep, single lattice, and
                    the strip-sharded path with k = 2, 4, 8 shards on one B200
  * KMC configs[3]  256^3, both active modes,        2 sweeps (the full-warp kernel)
  * KMC 512^3 / 1024^3 (configs[4]'s lattice)        1 sweep  (the 4-blocks-per-warp kernel)

The oracle runs the same two-layer DT schedule on all host cores (block rows
of a phase are independent, oracle_core.hpp parallel_rows).  Tolerance: none --
lattice words and counters must be identical.  Reference semantics:
kpz.hpp:71-107 (attempt), kmc.hpp:80-112 (exchange).
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lfg():
    import paper_1204_5072_b200 as m

    if m.device_count() < 1:
        pytest.fail("no CUDA device visible to liblfg.so")
    return m


def _device_spins_to_host(k):
    """The lattice's spin words ([L][L/32] uint32) copied device -> host."""
    import ctypes as C

    import torch

    from paper_1204_5072_b200 import _native

    ptr, nbytes = k.device_spins()
    t = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda:0")
    k.synchronize()
    _native.check(_native.lib().lfg_copy_async(C.c_void_p(t.data_ptr()), C.c_void_p(ptr), nbytes, None, 0))
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def _kpz_oracle_after(oracle, L, p, q, seed, nsweeps, bx, by):
    x, y = oracle.kpz_flat(L)
    c = oracle.kpz_sweep_dtr(L, x, y, p, q, seed, 0, nsweeps, bx, by)
    return x, y, c


def test_kpz_c2_bench_lattice_one_sweep(lfg, oracle):
    """configs[1]: L = 2^16, p = 1, flat start, the production plan (TMA-staged FULL kernel)."""
    L, seed = 1 << 16, 20260
    with lfg.KpzLattice(L, 1.0, 0.0, seed) as k:
        bx, by = k.plan
        assert (bx, by) == (1024, 128)
        k.make_flat_slopes()
        c = k.sweep(1)
        gx, gy = k.download()
        sums = k.width_sums()
    x, y, cref = _kpz_oracle_after(oracle, L, 1.0, 0.0, seed, 1, bx, by)
    assert [c.attempts, c.successes, c.deposits, c.detaches] == cref.tolist()
    assert np.array_equal(gx, x)
    assert np.array_equal(gy, y)
    assert sums == oracle.kpz_width_sums(L, x, y)


@pytest.fixture(scope="module")
def c3(lfg, oracle):
    """configs[2]'s lattice after one sweep: oracle planes + the single-GPU spins."""
    L, p, q, seed = 1 << 17, 0.95, 0.05, 1
    with lfg.KpzLattice(L, p, q, seed) as k:
        bx, by = k.plan
        k.make_flat_slopes()
        c = k.sweep(1)
        gx, gy = k.download()
        spins = _device_spins_to_host(k)
        sums = k.width_sums()
    x, y, cref = _kpz_oracle_after(oracle, L, p, q, seed, 1, bx, by)
    same = bool(np.array_equal(gx, x) and np.array_equal(gy, y))
    del gx, gy
    return dict(L=L, p=p, q=q, seed=seed, bx=bx, by=by, c=c, cref=cref, same=same, spins=spins, sums=sums,
                osums=oracle.kpz_width_sums(L, x, y))


def test_kpz_c3_lattice_one_sweep(c3):
    """configs[2] on one GPU: L = 2^17, p = 0.95, q = 0.05 (acceptance draws, GENERAL kernel)."""
    c = c3["c"]
    assert [c.attempts, c.successes, c.deposits, c.detaches] == c3["cref"].tolist()
    assert c3["same"], "L=2^17 lattice differs from the oracle"
    assert c3["sums"] == c3["osums"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_kpz_c3_strip_shards_one_sweep(lfg, c3, world):
    """configs[2] strip-sharded into k shards on one B200 (LocalComm row exchange):
    the gathered spin rows equal the single lattice's, which equal the oracle's."""
    from paper_1204_5072_b200.shard import CudaStripEngine, LocalComm, ShardedKpz, StripPlan

    L, p, q, seed = c3["L"], c3["p"], c3["q"], c3["seed"]
    pl = StripPlan(L, world, c3["bx"], c3["by"])
    engines = [CudaStripEngine(pl, p, q, seed, 0) for _ in range(world)]
    try:
        sk = ShardedKpz(pl, seed, engines, list(range(world)), LocalComm(engines))
        sk.make_flat_slopes()
        sk.sweep(1)
        dep, det = sk.counters_local()
        assert (dep, det) == (c3["c"].deposits, c3["c"].detaches)
        rows = sk.gather_rows().cpu().numpy()
        assert np.array_equal(rows.reshape(-1).view(np.uint32), c3["spins"].reshape(-1).view(np.uint32))
        assert sk.width_sums() == c3["sums"]
    finally:
        for e in engines:
            e.close()


@pytest.mark.parametrize("both,sub", [(1, 1), (0, 1), (1, 4)])
def test_kmc_c4_two_sweeps(lfg, oracle, both, sub):
    """configs[3]: 256^3, c = 0.5, eps = 1.5, 2 sweeps, both active modes (the
    producer/consumer kernel), and the four-sub-sweep plan option."""
    L, eps, seed = 256, 1.5, 31 + both
    w0, _ = oracle.kmc_random_alloy(L, 0.5, "lcg64", 7)
    w = w0.copy()
    cref = oracle.kmc_sweep_dt(L, w, eps, both, seed, 0, 2, 16, sub=sub)
    with lfg.KmcLattice(L, eps, bool(both), seed, block=16, sub=sub) as k:
        k.upload(w0)
        c = k.sweep(2)
        g = k.download()
        ob = k.open_bond_sums()
    assert [c.attempts, c.successes] == cref.tolist()
    assert np.array_equal(g, w)
    assert tuple(ob) == tuple(oracle.kmc_open_bond_sums(L, w))


@pytest.mark.parametrize("L,both,sub", [(512, 1, 1), (1024, 1, 1), (1024, 0, 1), (512, 1, 4)])
def test_kmc_four_blocks_per_warp_kernel(lfg, oracle, L, both, sub):
    """The 4-blocks-per-warp kernel (>= 2368 active 16^3 blocks per phase: 512^3,
    and configs[4]'s 1024^3 lattice) against the oracle, not against its siblings."""
    eps, seed = 1.5, 900 + L + both
    with lfg.KmcLattice(L, eps, bool(both), seed, block=16, sub=sub) as k:
        k.make_random_alloy(0.5, 11)
        w = k.download()
        c = k.sweep(1)
        g = k.download()
    cref = oracle.kmc_sweep_dt(L, w, eps, both, seed, 0, 1, 16, sub=sub)
    assert [c.attempts, c.successes] == cref.tolist()
    assert np.array_equal(g, w)
