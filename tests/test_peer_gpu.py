"""Peer-memory strip sharding (PeerComm: CUDA IPC + fused write-back push + device-side
step barrier, no NCCL) with two processes on cuda:0 (run with -m gpu).

Both ranks map each other's ring buffers through CUDA IPC exactly as ranks on
different GPUs of a node would over NVLink; the sharded trajectory must equal the
single-lattice one bit for bit (counters, slope planes, W^2).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, L, p, q, seed, nsweeps, out):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    import torch
    import torch.distributed as dist

    from paper_1204_5072_b200.shard import CudaStripEngine, PeerComm, ShardedKpz, StripPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pl = StripPlan(L, world, min(1024, L // 2), min(128, L // 2))
    eng = CudaStripEngine(pl, p, q, seed, 0)
    comm = PeerComm(eng, max_spins=1 << 23)
    sk = ShardedKpz(pl, seed, [eng], [rank], comm)
    sk.make_flat_slopes()
    sk.sweep(nsweeps)
    rows = sk.gather_rows().numpy()
    dep, det = sk.counters_local()
    t = torch.tensor([dep, det], dtype=torch.int64)
    dist.all_reduce(t)
    sums = sk.width_sums()
    if rank == 0:
        np.savez(out, rows=rows, cnt=t.numpy(), sums=np.array(sums, np.int64))
    dist.barrier()
    comm.close()
    eng.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,p,q,nsweeps", [(2, 1.0, 0.0, 3), (4, 0.95, 0.05, 2)])
def test_peer_sharded_equals_single(tmp_path, world, p, q, nsweeps):
    sys.path.insert(0, HERE)
    from strip_cpu_engine import spins_to_slopes

    import paper_1204_5072_b200 as lfg

    L, seed = 2048, 606 + world
    out = str(tmp_path / "peer.npz")
    mp.start_processes(_worker, args=(world, _free_port(), L, p, q, seed, nsweeps, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    with lfg.KpzLattice(L, p, q, seed) as k:
        k.make_flat_slopes()
        c = k.sweep(nsweeps)
        x, y = k.download()
        ref_sums = k.width_sums()
    assert tuple(got["cnt"]) == (c.deposits, c.detaches)
    px, py = spins_to_slopes(got["rows"].view(np.uint32), L)
    assert np.array_equal(px, x) and np.array_equal(py, y)
    assert tuple(got["sums"]) == ref_sums


def _kmc_worker(rank, world, port, L, both, seed, nsweeps, out):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import torch.distributed as dist

    from paper_1204_5072_b200.shard import CudaSlabEngine, PeerComm, ShardedKmc, SlabPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    pl = SlabPlan(L, world, 16)
    eng = CudaSlabEngine(pl, 1.5, both, seed, 0)
    comm = PeerComm(eng, max_spins=1 << 23)
    sk = ShardedKmc(pl, seed, [eng], [rank], comm)
    sk.make_random_alloy(0.5, 5)
    sk.sweep(nsweeps)
    planes = sk.gather_planes().numpy()
    succ = sk.successes()
    ob = sk.open_bond_sums()
    if rank == 0:
        np.savez(out, planes=planes, succ=succ, ob=np.array(ob, np.int64))
    dist.barrier()
    comm.close()
    eng.close()
    dist.destroy_process_group()


def test_peer_sharded_kmc_equals_single(tmp_path):
    import paper_1204_5072_b200 as lfg

    L, both, seed, nsweeps, world = 128, True, 91, 2, 2
    out = str(tmp_path / "kmc.npz")
    mp.start_processes(_kmc_worker, args=(world, _free_port(), L, both, seed, nsweeps, out), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    with lfg.KmcLattice(L, 1.5, both, seed, block=16) as k:
        k.make_random_alloy(0.5, 5)
        c = k.sweep(nsweeps)
        ref = k.download()
        ref_ob = k.open_bond_sums()
    assert int(got["succ"]) == c.successes
    assert np.array_equal(got["planes"].reshape(-1).view(np.uint64), ref)
    assert tuple(got["ob"]) == tuple(ref_ob)
