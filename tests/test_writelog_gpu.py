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


def _log_arrays(groups):
    """groups: list of lists of (worker, sites[k]) -> flat arrays for ref_writelog_violations."""
    goff, tw, woff, ws = [0], [], [0], []
    for g in groups:
        for worker, sites in g:
            tw.append(worker)
            ws.extend(sites)
            woff.append(len(ws))
        goff.append(len(tw))
    return (np.array(goff, np.int64), np.array(tw, np.int32), np.array(woff, np.int64),
            np.array(ws if ws else [0], np.int64))


@pytest.mark.parametrize("p,q", [(1.0, 0.0), (0.95, 0.05)])
def test_dt_write_sets_are_disjoint(lfg, oracle, reflib, p, q):
    import torch

    L, bx, by, seed, nsweeps = 256, 64, 32, 4711, 100
    buf = torch.zeros(L * L, dtype=torch.int32, device="cuda")
    ntile_x = L // 32
    tpb_x, tpb_y = bx // 32, by // 16
    total_rw = total_bw = 0
    with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by) as k:
        lfg._native.check(lfg._native.lib().lfg_kpz_debug_record_anchors(k._h, buf.data_ptr(), L * L))
        k.make_flat_slopes()
        for s in range(nsweeps):
            c = k.sweep(1)
            rec = buf.cpu().numpy().view(np.uint32).reshape(4, 512, -1)
            d = oracle.kpz_sweep_draw(L, bx, by, seed, s)
            ox, oy = int(d[0]), int(d[1])
            tile, acc, sites = _writes(L, ox, oy, rec.reshape(-1))
            assert acc.sum() == c.successes and rec.size == L * L  # every attempt recorded once
            tile = tile.reshape(4, 512, -1)
            acc = acc.reshape(4, 512, -1)
            sites = sites.reshape(4, 512, -1, 4)
            rounds, blocks = [], []
            for ph in range(4):
                per_block = {}
                for r in range(512):
                    g = [(int(tile[ph, r, t]), sites[ph, r, t].tolist() if acc[ph, r, t] else [])
                         for t in range(tile.shape[2])]
                    rounds.append(g)
                    for (w, ss) in g:
                        b = (w // ntile_x // tpb_y) * (L // bx) + (w % ntile_x) // tpb_x
                        per_block.setdefault(b, []).extend(ss)
                blocks.append(list(per_block.items()))
            nv, nw, first = reflib.writelog_violations(L * L // 512, *_log_arrays(rounds))
            assert nv == 0, (s, first)
            nv2, nw2, first2 = reflib.writelog_violations((L // bx) * (L // by), *_log_arrays(blocks))
            assert nv2 == 0, (s, first2)
            assert nw == nw2 == 4 * c.successes
            total_rw += nw
            total_bw += nw2
            if s == 0:  # negative control: a phase as one interval with tiles as workers must race
                wrong = [[w for g in rounds[ph * 512:(ph + 1) * 512] for w in g] for ph in range(4)]
                nvw, _, _ = reflib.writelog_violations(L * L // 512, *_log_arrays(wrong))
                assert nvw > 0
        lfg._native.check(lfg._native.lib().lfg_kpz_debug_record_anchors(k._h, None, 0))
    assert total_rw > 0 and total_bw > 0
