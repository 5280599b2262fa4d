"""Snapshot / exact resume (paper_1204_5072_b200/snapshot.py): a lattice
saved after n sweeps and reloaded continues bit for bit like the uninterrupted run (the RNG
is counter-based: (seed, sweep index) -> draws).  Run with -m gpu."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lfg():
    import paper_1204_5072_b200 as m

    if m.device_count() < 1:
        pytest.fail("no CUDA device visible to liblfg.so")
    return m


def test_kpz_snapshot_resume(lfg, tmp_path):
    path = str(tmp_path / "kpz.npz")
    with lfg.KpzLattice(512, 0.95, 0.05, seeds=[11, 12], block_x=128, block_y=64) as a:
        a.make_flat_slopes()
        a.sweep(3)
        a.save(path)
        a.sweep(4)
        ref = [(a.download(r), a.counters(r), a.width_sums(r)) for r in range(2)]
    with lfg.KpzLattice.load(path) as b:
        assert b.sweep_index == 3 and b.plan == (128, 64) and b.seeds == [11, 12]
        b.sweep(4)
        for r in range(2):
            (x, y), c, ws = ref[r]
            bx, by = b.download(r)
            assert np.array_equal(bx, x) and np.array_equal(by, y)
            cb = b.counters(r)
            assert (cb.attempts, cb.deposits, cb.detaches) == (c.attempts, c.deposits, c.detaches)
            assert b.width_sums(r) == ws


def test_kmc_snapshot_resume(lfg, tmp_path):
    path = str(tmp_path / "kmc.npz")
    with lfg.KmcLattice(64, 1.5, True, 21) as a:
        a.make_random_alloy(0.4, 5)
        a.sweep(2)
        a.save(path)
        a.sweep(3)
        w, c = a.download(), a.counters()
    with lfg.KmcLattice.load(path) as b:
        assert b.sweep_index == 2 and b.both_active and b.eps == 1.5
        b.sweep(3)
        assert np.array_equal(b.download(), w)
        cb = b.counters()
        assert (cb.attempts, cb.successes) == (c.attempts, c.successes)


def test_snapshot_rejects_wrong_model(lfg, tmp_path):
    path = str(tmp_path / "kmc.npz")
    with lfg.KmcLattice(32) as a:
        a.save(path)
    with pytest.raises(ValueError):
        lfg.KpzLattice.load(path)
