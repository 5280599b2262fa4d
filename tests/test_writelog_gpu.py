"""Write-disjointness of the GPU DT schedule (SPEC.md:510 acceptance 7),
checked by the reference's own lf::WriteLog (write_log.hpp:10-60) over the write sets the
B200 kernel actually executed (run with -m gpu).

The debug instantiation of the phase kernel (lfg_kpz_debug_record_anchors) records every
attempt: tile, anchor, inner set, accepted.  Each accepted attempt writes the four slope
bits that kpz_attempt_impl records (kpz.hpp:97-105): sigma_x at (i,j), (i+1,j) and sigma_y
at (i,j), (i,j+1).  Two logs are checked per sweep:
  * round level: a barrier interval = one (phase, single-hit round); workers = tiles of all
    blocks active in the phase;
  * block level: a barrier interval = one phase; workers = device blocks (all rounds of all
    active blocks run concurrently).
A third, deliberately wrong model (all rounds of a phase in one interval, workers = tiles)
must report violations -- the checker can see races.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lfg():
    import paper_1204_5072_b200 as m

    if m.device_count() < 1:
        pytest.fail("no CUDA device visible to liblfg.so")
    return m


def _writes(L, ox, oy, rec):
    """Decode records -> (tile id, accepted mask, write sites [n, 4]) in the reference's site
    numbering (x plane: j*L + i, y plane: L*L + j*L + i)."""
    m = L - 1
    tile = (rec & 0xFFFFF).astype(np.int64)
    xd = (rec >> 20) & 15
    yd = (rec >> 24) & 7
    hx = (rec >> 27) & 1
    hy = (rec >> 28) & 1
    acc = ((rec >> 29) & 1).astype(bool)
    gx, gy = tile % (L // 32), tile // (L // 32)
    i = (ox + 32 * gx + 16 * hx + xd) & m
    j = (oy + 16 * gy + 8 * hy + yd) & m
    n = L * L
    sites = np.stack([j * L + i, j * L + ((i + 1) & m), n + j * L + i, n + ((j + 1) & m) * L + i], axis=1)
    return tile, acc, sites.astype(np.int64)


def _np_log(workers, acc, sites):
    """Vectorised _log_arrays: workers / acc [G, T] (interval g, worker slot t),
    sites [G, T, 4]; an accepted attempt writes its four sites."""
    G, T = workers.shape
    nw = np.where(acc, 4, 0).reshape(-1)
    goff = np.arange(G + 1, dtype=np.int64) * T
    woff = np.concatenate([[0], np.cumsum(nw)]).astype(np.int64)
    ws = sites.reshape(-1, 4)[acc.reshape(-1)].reshape(-1).astype(np.int64)
    return goff, workers.reshape(-1).astype(np.int32), woff, (ws if ws.size else np.zeros(1, np.int64))


@pytest.mark.parametrize("L,bx,by,sub,p,q,nsweeps", [
    (256, 64, 32, 4, 1.0, 0.0, 30), (256, 64, 32, 4, 0.95, 0.05, 30), (256, 64, 32, 1, 0.95, 0.05, 30),
    (2048, 1024, 128, 4, 1.0, 0.0, 2), (2048, 1024, 128, 4, 0.95, 0.05, 2), (2048, 1024, 128, 1, 1.0, 0.0, 1),
    (2048, 1024, 128, 8, 0.95, 0.05, 1), (256, 64, 32, 8, 1.0, 0.0, 10)])
def test_dt_write_sets_are_disjoint(lfg, oracle, reflib, L, bx, by, sub, p, q, nsweeps):
    """Every plan incl. the production 1024 x 128 TMA path (L = 2048) and all sub modes."""
    import torch

    seed = 4711
    rounds = {1: 512, 4: 132, 8: 68}[sub]
    ntiles = L * L // 512
    nrec = ntiles * rounds * sub
    buf = torch.zeros(nrec, dtype=torch.int32, device="cuda")
    ntile_x = L // 32
    tpb_x, tpb_y = bx // 32, by // 16
    nblocks = (L // bx) * (L // by)
    total_rw = total_bw = 0
    with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by, sub=sub) as k:
        lfg._native.check(lfg._native.lib().lfg_kpz_debug_record_anchors(k._h, buf.data_ptr(), nrec))
        k.make_flat_slopes()
        for s in range(nsweeps):
            c = k.sweep(1)
            rec = buf.cpu().numpy().view(np.uint32).reshape(sub, 4, rounds, ntiles // 4)
            skipped = ((rec >> 30) & 1).astype(bool)
            assert int((~skipped).sum()) == c.attempts  # every attempt recorded once
            nacc = 0
            for kk in range(sub):
                d = oracle.kpz_sweep_draw(L, bx, by, seed, s * sub + kk)
                tile, acc, sites = _writes(L, int(d[0]), int(d[1]), rec[kk].reshape(-1))
                assert not (acc & skipped[kk].reshape(-1)).any()
                nacc += int(acc.sum())
                T = ntiles // 4
                tile = tile.reshape(4 * rounds, T)
                acc = acc.reshape(4 * rounds, T)
                sites = sites.reshape(4 * rounds, T, 4)
                # round level: one interval per (phase, round), workers = tiles
                nv, nw, first = reflib.writelog_violations(ntiles, *_np_log(tile, acc, sites))
                assert nv == 0, (s, kk, first)
                # block level: one interval per phase, workers = device blocks
                blk = (tile // ntile_x // tpb_y) * (L // bx) + (tile % ntile_x) // tpb_x
                bw = blk.reshape(4, rounds * T)
                nv2, nw2, first2 = reflib.writelog_violations(
                    nblocks, *_np_log(bw, acc.reshape(4, rounds * T), sites.reshape(4, rounds * T, 4)))
                assert nv2 == 0, (s, kk, first2)
                assert nw == nw2
                total_rw += nw
                total_bw += nw2
                if s == 0 and kk == 0:  # negative control: a phase as one interval with tiles as workers must race
                    nvw, _, _ = reflib.writelog_violations(
                        ntiles, *_np_log(tile.reshape(4, rounds * T), acc.reshape(4, rounds * T),
                                         sites.reshape(4, rounds * T, 4)))
                    assert nvw > 0
            assert nacc == c.successes
        lfg._native.check(lfg._native.lib().lfg_kpz_debug_record_anchors(k._h, None, 0))
    assert total_rw > 0 and total_bw > 0


@pytest.mark.parametrize("both,share", [(True, 1), (False, 1), (True, 512)])
def test_kmc_write_sets_are_disjoint(lfg, reflib, both, share):
    """KMC (16^3 plan): the exchanges the GPU kernels make -- the producer/consumer
    kernel of sparse phases and the 4-blocks-per-warp kernel of dense ones (forced by
    a concurrency hint) -- recorded site by site (lfg_kmc_debug_record_writes, the
    write hooks of kmc.hpp:105-110) and checked by the reference's WriteLog: no site
    written by two tiles in one single-hit round, nor by two blocks in one phase."""
    import torch

    L, nsweeps = 64, 12
    nact = (L // 16) ** 3 // 8  # active blocks per phase
    buf = torch.zeros(L ** 3, dtype=torch.int32, device="cuda")
    with lfg.KmcLattice(L, 1.5, both, 31) as k:
        if share > 1:
            k.set_concurrency(share)
        k.make_random_alloy(0.5, 9)
        lfg._native.check(lfg._native.lib().lfg_kmc_debug_record_writes(k._h, buf.data_ptr(), L ** 3))
        tot = 0
        for s in range(nsweeps):
            c = k.sweep(1)
            rec = buf.cpu().numpy().view(np.uint32).reshape(8, 256, nact, 8, 2)
            done = rec[..., 0] != 0xFFFFFFFF
            assert int(done.sum()) == c.successes  # every exchange recorded once
            sites = rec.astype(np.int64)
            tiles = np.broadcast_to(np.arange(nact * 8).reshape(nact, 8), (8, 256, nact, 8))
            blocks = np.broadcast_to(np.arange(nact).reshape(nact, 1), (8, 256, nact, 8))
            G = 8 * 256
            # round level: one interval per (phase, round), workers = tiles
            nv, nw, first = reflib.writelog_violations(
                nact * 8, *_np_log2(tiles.reshape(G, -1), done.reshape(G, -1), sites.reshape(G, -1, 2)))
            assert nv == 0, (s, first)
            # block level: one interval per phase, workers = device blocks
            nv2, nw2, first2 = reflib.writelog_violations(
                nact, *_np_log2(blocks.reshape(8, -1), done.reshape(8, -1), sites.reshape(8, -1, 2)))
            assert nv2 == 0, (s, first2)
            assert nw == nw2 == 2 * c.successes
            tot += nw
            if s == 0:  # negative control: a phase as one interval with tiles as workers must race
                nvw, _, _ = reflib.writelog_violations(
                    nact * 8, *_np_log2(tiles.reshape(8, -1), done.reshape(8, -1), sites.reshape(8, -1, 2)))
                assert nvw > 0
        lfg._native.check(lfg._native.lib().lfg_kmc_debug_record_writes(k._h, None, 0))
    assert tot > 0


def _np_log2(workers, done, sites):
    """_np_log for attempts that write two sites (KMC exchanges)."""
    G, T = workers.shape
    nw = np.where(done, 2, 0).reshape(-1)
    goff = np.arange(G + 1, dtype=np.int64) * T
    woff = np.concatenate([[0], np.cumsum(nw)]).astype(np.int64)
    ws = sites.reshape(-1, 2)[done.reshape(-1)].reshape(-1).astype(np.int64)
    return goff, workers.reshape(-1).astype(np.int32), woff, (ws if ws.size else np.zeros(1, np.int64))
