"""Strip-sharded KPZ on one B200 (run with -m gpu).

k shards live on cuda:0 and exchange rows in-process (LocalComm); the result
must be bit-identical to the single-lattice run, because the RNG is keyed on
global tile/block ids of the shifted frame.  The exact
W² of the sharded lattice (segments combined across shards) must equal the
single-lattice scan.
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


@pytest.mark.parametrize("L,world,p,q,nsweeps", [(2048, 2, 1.0, 0.0, 3), (2048, 4, 0.95, 0.05, 2),
                                                 (4096, 8, 1.0, 0.0, 2), (4096, 2, 0.5, 0.5, 2)])
def test_sharded_equals_single(lfg, L, world, p, q, nsweeps):
    from strip_cpu_engine import spins_to_slopes

    from paper_1204_5072_b200.shard import CudaStripEngine, LocalComm, ShardedKpz, StripPlan

    seed = 4242 + world
    with lfg.KpzLattice(L, p, q, seed) as k:
        bx, by = k.plan
        k.make_flat_slopes()
        c = k.sweep(nsweeps)
        x, y = k.download()
        ref_sums = k.width_sums()
    pl = StripPlan(L, world, bx, by)
    engines = [CudaStripEngine(pl, p, q, seed, 0) for _ in range(world)]
    try:
        sk = ShardedKpz(pl, seed, engines, list(range(world)), LocalComm(engines))
        sk.make_flat_slopes()
        sk.sweep(nsweeps)
        dep, det = sk.counters_local()
        assert (dep, det) == (c.deposits, c.detaches)
        rows = sk.gather_rows().numpy().view(np.uint32)
        px, py = spins_to_slopes(rows, L)
        assert np.array_equal(px, x) and np.array_equal(py, y)
        assert sk.width_sums() == ref_sums
    finally:
        for e in engines:
            e.close()


# ----------------------------------------------------------------- KMC z-slabs
@pytest.mark.parametrize("L,world,bk,both,nsweeps", [(128, 2, 16, 1, 2), (128, 4, 16, 0, 2),
                                                     (256, 8, 16, 1, 1), (128, 2, 32, 1, 2)])
def test_sharded_kmc_equals_single(lfg, L, world, bk, both, nsweeps):
    """k z-slabs on cuda:0 (LocalComm plane exchanges) == the single lattice,
    bit for bit: words, exchange count and open-bond sums."""
    from paper_1204_5072_b200.shard import CudaSlabEngine, LocalComm, ShardedKmc, SlabPlan

    seed, eps = 77 + world, 1.5
    with lfg.KmcLattice(L, eps, bool(both), seed, block=bk) as k:
        k.make_random_alloy(0.5, 5)
        w0 = k.download()
        c = k.sweep(nsweeps)
        ref = k.download()
        ref_ob = k.open_bond_sums()
    pl = SlabPlan(L, world, bk)
    engines = [CudaSlabEngine(pl, eps, bool(both), seed, 0) for _ in range(world)]
    try:
        sk = ShardedKmc(pl, seed, engines, list(range(world)), LocalComm(engines))
        sk.make_random_alloy(0.5, 5)  # position-keyed Philox init: same sites as the single lattice
        assert np.array_equal(sk.gather_planes().numpy().reshape(-1).view(np.uint64), w0)
        sk.sweep(nsweeps)
        assert sk.successes() == c.successes
        assert np.array_equal(sk.gather_planes().numpy().reshape(-1).view(np.uint64), ref)
        assert sk.open_bond_sums() == tuple(ref_ob)
    finally:
        for e in engines:
            e.close()
