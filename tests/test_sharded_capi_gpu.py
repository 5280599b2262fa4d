"""The one-process, N-GPU sharded KPZ handle of the C ABI (lfg_kpz_create_sharded,
include/lfg.h): strips on several devices -- here several strips on the one GPU of the
test box -- driven by one host thread give the single-lattice trajectory bit for bit
(counters, the reference-layout slope planes, W^2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lfg():
    import paper_1204_5072_b200 as m

    if m.device_count() < 1:
        pytest.fail("no CUDA device visible to liblfg.so")
    return m


@pytest.mark.parametrize("n,p,q,sub", [(2, 1.0, 0.0, 4), (4, 0.95, 0.05, 4), (8, 1.0, 0.0, 4), (2, 0.7, 0.3, 1)])
def test_sharded_equals_single(lfg, n, p, q, sub):
    L, seed = 2048, 99
    with lfg.KpzLattice(L, p, q, seed, sub=sub) as k, \
            lfg.ShardedKpzLattice(L, p, q, seed, devices=[0] * n, sub=sub) as s:
        k.make_flat_slopes()
        s.make_flat_slopes()
        c1 = k.sweep(3)
        c2 = s.sweep(3)
        assert [c1.attempts, c1.successes, c1.deposits, c1.detaches] == \
               [c2.attempts, c2.successes, c2.deposits, c2.detaches]
        x1, y1 = k.download()
        x2, y2 = s.download()
        assert np.array_equal(x1, x2) and np.array_equal(y1, y2)
        assert s.width_sums() == k.width_sums()
        assert s.interface_width() == k.interface_width()
        assert s.sweep_index == 3


def test_sharded_upload_resume(lfg, oracle):
    """Upload a rough closed field at MCS index 5, sweep, compare with the oracle."""
    L, seed = 2048, 7
    x, y = oracle.kpz_flat(L)
    oracle.kpz_sweep_dtr(L, x, y, 0.95, 0.05, seed, 0, 2, 1024, 128)
    xr, yr = x.copy(), y.copy()
    c_ref = oracle.kpz_sweep_dtr(L, xr, yr, 0.95, 0.05, seed, 5, 1, 1024, 128)
    with lfg.ShardedKpzLattice(L, 0.95, 0.05, seed, devices=[0, 0, 0, 0]) as s:
        s.sweep_index = 5
        s.upload(x, y)
        c = s.sweep(1)
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist()
        gx, gy = s.download()
        assert np.array_equal(gx, xr) and np.array_equal(gy, yr)


def test_sharded_rejects_bad_geometry(lfg):
    with pytest.raises(lfg.InvalidArgument):
        lfg.ShardedKpzLattice(1024, devices=[0] * 8)  # strip height 128 < 2 * block_y


@pytest.mark.parametrize("n,both,L", [(2, True, 128), (4, False, 128), (8, True, 256)])
def test_sharded_kmc_equals_single(lfg, n, both, L):
    """KMC z-slabs (lfg_kmc_create_sharded) == one lattice, bit for bit."""
    with lfg.KmcLattice(L, 1.5, both, 21) as k, lfg.ShardedKmcLattice(L, 1.5, both, 21, devices=[0] * n) as s:
        k.make_random_alloy(0.5, 4)
        s.make_random_alloy(0.5, 4)
        assert np.array_equal(k.download(), s.download())
        c1 = k.sweep(3)
        c2 = s.sweep(3)
        assert (c1.attempts, c1.successes) == (c2.attempts, c2.successes)
        assert np.array_equal(k.download(), s.download())
        assert k.open_bond_sums() == s.open_bond_sums()
        assert s.open_bonds_per_particle() == k.open_bonds_per_particle()


def test_sharded_kmc_upload_vs_oracle(lfg, oracle):
    L = 128
    w, _ = oracle.kmc_random_alloy(L, 0.5, "lcg64", 8)
    w_ref = w.copy()
    c_ref = oracle.kmc_sweep_dt(L, w_ref, 1.5, 1, 17, 4, 2, 16)
    with lfg.ShardedKmcLattice(L, 1.5, True, 17, devices=[0, 0]) as s:
        s.sweep_index = 4
        s.upload(w)
        c = s.sweep(2)
        assert [c.attempts, c.successes] == c_ref.tolist()
        assert np.array_equal(s.download(), w_ref)


def test_sharded_kmc_sub4_equals_single(lfg):
    """KMC plan option sub = 4 (four sub-sweeps per MCS): slabs == one lattice."""
    L = 128
    with lfg.KmcLattice(L, 1.5, True, 5, sub=4) as k, lfg.ShardedKmcLattice(L, 1.5, True, 5, devices=[0] * 4,
                                                                            sub=4) as s:
        k.make_random_alloy(0.5, 6)
        s.make_random_alloy(0.5, 6)
        c1, c2 = k.sweep(2), s.sweep(2)
        assert (c1.attempts, c1.successes) == (c2.attempts, c2.successes)
        assert np.array_equal(k.download(), s.download())
