"""CPU tests of the z-slab-sharded KMC driver (paper_1204_5072_b200/shard.py,
SlabPlan / ShardedKmc).

* plan invariants: every roll / ghost / write-back send has its matching
  receive, and after a roll every rank owns exactly its new window;
* a real world_size-2 run over torch.distributed (gloo, 127.0.0.1) with the
  CPU slab engine, compared bit for bit (lattice words, exchange count, open
  bonds) with the oracle's full-lattice DT sweep.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from paper_1204_5072_b200.shard import SlabPlan  # noqa: E402


def test_slab_plan_geometry():
    pl = SlabPlan(1024, 8, 16)
    assert pl.H == 128 and pl.cap >= pl.H + 4 * 16 + 4 and pl.cap & (pl.cap - 1) == 0
    assert pl.wpp == 1024 * 1024 // 32
    with pytest.raises(ValueError):
        SlabPlan(128, 8, 16)  # H = 16 is not a multiple of 2*bk
    assert SlabPlan(64, 1, 16).cap == 64


def _match(ops, L):
    s = sorted((r, p, b % L, n) for r in ops for (k, p, b, n) in ops[r] if k == "send")
    v = sorted((p, r, b % L, n) for r in ops for (k, p, b, n) in ops[r] if k == "recv")
    return s == v


@pytest.mark.parametrize("world", [2, 4, 8])
def test_slab_exchanges_match(world):
    bk = 16
    L = 2 * bk * world * 2
    pl = SlabPlan(L, world, bk)
    rs = np.random.RandomState(world)
    for _ in range(40):
        o1, o2 = int(rs.randint(0, 2 * bk)), int(rs.randint(0, 2 * bk))
        ops = {r: pl.roll(o1, o2, r) for r in range(world)}
        assert _match(ops, L)
        for r in range(world):
            own = {(pl.start(o1, r) + i) % L for i in range(pl.H)}
            for (k, peer, b, n) in ops[r]:
                planes = {(b + i) % L for i in range(n)}
                own = own - planes if k == "send" else own | planes
            assert own == {(pl.start(o2, r) + i) % L for i in range(pl.H)}
        for sz in (0, 1):
            assert _match({r: pl.ghost(o2, r, sz, 2) for r in range(world)}, L)
            assert _match({r: pl.ghost(o2, r, sz, 1) for r in range(world)}, L)
            wb = {r: pl.writeback(o2, r, sz) for r in range(world)}
            assert _match(wb, L)
            for r in range(world):  # the plane sent back is the one just beyond the slab on side sz
                s = pl.start(o2, r)
                (kind, _, b, n), = [op for op in wb[r] if op[0] == "send"]
                assert n == 1 and b % L == ((s + pl.H) % L if sz else (s - 1) % L)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, L, bk, eps, both, seed, nsweeps, out_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import pyoracle
    from slab_cpu_engine import CpuSlabEngine

    from paper_1204_5072_b200.shard import DistComm, ShardedKmc, SlabPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pl = SlabPlan(L, world, bk)
    orc = pyoracle.Oracle()
    eng = CpuSlabEngine(pl, eps, both, seed, orc)
    w0, _ = orc.kmc_random_alloy(L, 0.5, "lcg64", 11)
    sk = ShardedKmc(pl, seed, [eng], [rank], DistComm(eng), origin=eng.origin)
    sk.upload(w0, sweep_index=2)
    sk.sweep(nsweeps)
    full = sk.gather_planes().numpy()
    succ = sk.successes()
    ob = sk.open_bond_sums()
    if rank == 0:
        np.savez(out_path, full=full, succ=succ, ob=np.array(ob, np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("both", [0, 1])
def test_sharded_kmc_gloo_world2_matches_oracle(tmp_path, oracle, both):
    L, bk, eps, seed, nsweeps = 64, 16, 1.5, 9, 3
    out = str(tmp_path / "slab.npz")
    mp.spawn(_worker, args=(2, _free_port(), L, bk, eps, both, seed, nsweeps, out), nprocs=2, join=True)
    w, _ = oracle.kmc_random_alloy(L, 0.5, "lcg64", 11)
    c = oracle.kmc_sweep_dt(L, w, eps, both, seed, 2, nsweeps, bk)
    got = np.load(out)
    assert np.array_equal(got["full"].reshape(-1).view(np.uint64), w)
    assert int(got["succ"]) == int(c[1])
    assert tuple(got["ob"]) == oracle.kmc_open_bond_sums(L, w)
