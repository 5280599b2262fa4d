"""CPU tests of the strip-sharded driver (paper_1204_5072_b200/shard.py).

* plan invariants: every roll/ghost send has its matching receive and after a
  roll every rank owns exactly its new window;
* a real world_size-2 run over torch.distributed (gloo, 127.0.0.1) with the
  pure-Python strip engine, compared bit for bit with the full-lattice oracle.
"""
import os
import socket

import numpy as np
import pytest

import sys as _sys
_sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1204_5072_b200.shard import StripPlan


def test_plan_geometry():
    pl = StripPlan(2048, 4, 1024, 128)
    assert pl.H == 512 and pl.cap >= pl.H + 4 * 128 + 2 and pl.cap & (pl.cap - 1) == 0
    with pytest.raises(ValueError):
        StripPlan(1024, 8, 512, 128)  # H = 128 is not a multiple of 2*by
    assert StripPlan(1024, 1, 512, 128).cap == 1024


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_roll_and_ghost_plans_match(world):
    L, by = 256 * world if world != 3 else 96 * 4, 16
    if L % world:
        pytest.skip("world must divide L")
    pl = StripPlan(L, world, 32, by)
    rs = np.random.RandomState(world)
    for _ in range(50):
        o1, o2 = int(rs.randint(0, 2 * by)), int(rs.randint(0, 2 * by))
        ops = {r: pl.roll(o1, o2, r) for r in range(world)}
        sends = sorted((r, peer, b % L, n) for r in ops for (k, peer, b, n) in ops[r] if k == "send")
        recvs = sorted((peer, r, b % L, n) for r in ops for (k, peer, b, n) in ops[r] if k == "recv")
        assert sends == recvs
        for r in range(world):  # ownership after the roll
            own = {(pl.start(o1, r) + i) % L for i in range(pl.H)}
            for (k, peer, b, n) in ops[r]:
                rows = {(b + i) % L for i in range(n)}
                own = own - rows if k == "send" else own | rows
            assert own == {(pl.start(o2, r) + i) % L for i in range(pl.H)}
        for sy in (0, 1):
            g = {r: pl.ghost(o2, r, sy) for r in range(world)}
            s = sorted((r, p, b % L, n) for r in g for (k, p, b, n) in g[r] if k == "send")
            v = sorted((p, r, b % L, n) for r in g for (k, p, b, n) in g[r] if k == "recv")
            assert s == v


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, L, bx, by, p, q, seed, nsweeps, out_path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import pyoracle
    from strip_cpu_engine import CpuStripEngine

    from paper_1204_5072_b200.shard import DistComm, ShardedKpz, StripPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pl = StripPlan(L, world, bx, by)
    orc = pyoracle.Oracle()
    eng = CpuStripEngine(pl, p, q, seed, orc)
    sk = ShardedKpz(pl, seed, [eng], [rank], DistComm(eng))
    # the first sweep's window comes from the driver; fill it flat
    from paper_1204_5072_b200 import shard as shard_mod

    shard_mod.sweep_origin = lambda plan, sd, s: (lambda d: (int(d[0]), int(d[1]), [int(v) for v in d[2:]]))(
        orc.kpz_sweep_draw(plan.L, plan.bx, plan.by, sd, s))
    sk.make_flat_slopes()
    sk.sweep(nsweeps)
    rows = sk.gather_rows()
    dep, det = sk.counters_local()
    c = torch.tensor([dep, det], dtype=torch.int64)
    dist.all_reduce(c)
    ws = sk.width_sums()
    if rank == 0:
        np.save(out_path, rows.numpy())
        np.save(out_path + ".cnt.npy", c.numpy())
        np.save(out_path + ".w.npy", np.array(ws, dtype=np.int64))
    dist.destroy_process_group()


@pytest.mark.parametrize("p,q", [(1.0, 0.0), (0.7, 0.3)])
def test_gloo_world2_matches_full_lattice_oracle(tmp_path, oracle, p, q):
    from strip_cpu_engine import spins_to_slopes

    L, bx, by, seed, ns = 128, 64, 16, 99, 2
    out = str(tmp_path / "rows.npy")
    mp.spawn(_worker, args=(2, _free_port(), L, bx, by, p, q, seed, ns, out), nprocs=2, join=True)
    rows = np.load(out).view(np.uint32)
    cnt = np.load(out + ".cnt.npy")
    x, y = oracle.kpz_flat(L)
    c = oracle.kpz_sweep_dtr(L, x, y, p, q, seed, 0, ns, bx, by)
    px, py = spins_to_slopes(rows, L)
    assert (px == x).all() and (py == y).all()
    assert [int(cnt[0]), int(cnt[1])] == [int(c[2]), int(c[3])]
    # W^2 sums of the sharded lattice (row pieces chained across ranks) == interface_width's
    assert tuple(int(v) for v in np.load(out + ".w.npy")) == oracle.kpz_width_sums(L, x, y)
