"""GPU parity tests for the KPZ DTr path (run with -m gpu on a B200).

The CUDA path (paper_1204_5072_b200 -> liblfg.so) is compared bit-for-bit with
  * the golden vectors produced by the unmodified reference
    (tests/golden/golden.json: DTr schedule driving lf::detail::kpz_attempt_impl),
  * the live oracle restatement (oracle/_build/liboracle.so) on seeded inputs.
Tolerance: none -- integer/bit state must match exactly; W^2 is compared as
the same double expression over exact int64 sums.
"""
import hashlib
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def lfg():
    import paper_1204_5072_b200 as m

    if m.device_count() < 1:
        pytest.fail("no CUDA device visible to liblfg.so")
    return m


def test_flat_init_matches_reference(lfg, oracle, golden):
    for g in golden["kpz_flat"]:
        L = g["L"]
        if L < 64:
            continue
        with lfg.KpzLattice(L) as k:
            k.make_flat_slopes()
            x, y = k.download()
            assert sha(x) == g["sx"] and sha(y) == g["sy"]
            assert k.interface_width() == g["w2"] == 0.5
            assert k.width_sums() == (g["sum"], g["sum2"])


def test_default_state_is_all_zero_slopes(lfg):
    # SlopeField(L) constructor (lattice.cpp:20-25): all words zero.
    with lfg.KpzLattice(64) as k:
        x, y = k.download()
        assert not x.any() and not y.any()


@pytest.mark.parametrize("case", range(16))
def test_dtr_golden_bit_exact(lfg, golden, case):
    g = golden["kpz_dtr"][case]
    L = g["L"]
    with lfg.KpzLattice(L, g["p"], g["q"], g["seed"], block_x=g["bx"], block_y=g["by"], sub=g["sub"]) as k:
        k.make_flat_slopes()
        k.sweep_index = g["sweep0"]
        c = k.sweep(g["nsweeps"])
        assert [c.attempts, c.successes, c.deposits, c.detaches] == g["counters"]
        x, y = k.download()
        assert sha(x) == g["sx"] and sha(y) == g["sy"]
        assert k.width_sums() == (g["sum"], g["sum2"])
        assert k.interface_width() == g["w2"]


def test_dtr_live_oracle_random(lfg, oracle):
    rs = np.random.RandomState(2024)
    for _ in range(10):
        L = int(rs.choice([64, 128, 256, 512]))
        bx = int(rs.choice([b for b in (32, 64, 128, 256) if 2 * b <= L]))
        by = int(rs.choice([b for b in (16, 32, 64, 128) if 2 * b <= L]))
        p, q = [(1.0, 0.0), (0.95, 0.05), (0.3, 0.7), (0.0, 1.0), (1.0, 0.5)][rs.randint(5)]
        seed = int(rs.randint(0, 2**63))
        s0 = int(rs.randint(0, 1000))
        x, y = oracle.kpz_flat(L)
        c_ref = oracle.kpz_sweep_dtr(L, x, y, p, q, seed, s0, 3, bx, by)
        with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by) as k:
            k.make_flat_slopes()
            k.sweep_index = s0
            c = k.sweep(3)
            gx, gy = k.download()
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist(), (L, bx, by, p, q)
        assert (gx == x).all() and (gy == y).all(), (L, bx, by, p, q)


def test_upload_download_roundtrip_and_continue(lfg, oracle):
    L = 256
    x, y = oracle.kpz_flat(L)
    oracle.kpz_sweep_dtr(L, x, y, 0.7, 0.3, 9, 0, 4, 64, 32)  # a rough, closed field
    with lfg.KpzLattice(L, 0.7, 0.3, 9, block_x=64, block_y=32) as k:
        k.upload(x, y)
        gx, gy = k.download()
        assert (gx == x).all() and (gy == y).all()
        assert k.width_sums() == oracle.kpz_width_sums(L, x, y)
        assert (k.reconstruct_heights() == oracle.reconstruct_heights(L, x, y)).all()
        # continue the trajectory from the uploaded state
        k.sweep_index = 4
        c = k.sweep(2)
        c_ref = oracle.kpz_sweep_dtr(L, x, y, 0.7, 0.3, 9, 4, 2, 64, 32)
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist()
        gx, gy = k.download()
        assert (gx == x).all() and (gy == y).all()


def test_upload_rejects_non_integrable(lfg, oracle):
    L = 64
    x, y = oracle.kpz_flat(L)
    x[3] ^= np.uint64(1 << 5)  # single slope flip -> heights path-dependent
    with lfg.KpzLattice(L) as k:
        k.make_flat_slopes()
        with pytest.raises(lfg.ClosureError, match="closure"):
            k.upload(x, y)
        # state unchanged after the failed upload
        fx, fy = oracle.kpz_flat(L)
        gx, gy = k.download()
        assert (gx == fx).all() and (gy == fy).all()


def test_wrong_word_count_rejected(lfg):
    with lfg.KpzLattice(64) as k:
        with pytest.raises(lfg.InvalidArgument):
            k.upload(np.zeros(10, np.uint64), np.zeros(10, np.uint64))


def test_split_sweeps_equal_one_call(lfg):
    # counter-based RNG: (seed, sweep index) -> exact resume
    L = 256
    with lfg.KpzLattice(L, 1.0, 0.0, 5) as a, lfg.KpzLattice(L, 1.0, 0.0, 5) as b:
        a.make_flat_slopes()
        b.make_flat_slopes()
        ca = a.sweep(5)
        cb1 = b.sweep(2)
        cb2 = b.sweep(3)
        assert ca.successes == cb1.successes + cb2.successes
        assert b.sweep_index == 5
        xa, ya = a.download()
        xb, yb = b.download()
        assert (xa == xb).all() and (ya == yb).all()


def test_phase_api_equals_sweep(lfg):
    L = 512
    with lfg.KpzLattice(L, 1.0, 0.0, 77) as a, lfg.KpzLattice(L, 1.0, 0.0, 77) as b:
        a.make_flat_slopes()
        b.make_flat_slopes()
        a.sweep(2)
        for s in range(2 * a.sub):  # the phase API takes the sub-sweep index s' = MCS * sub + k
            for ph in range(4):
                b.phase(s, ph)
        b.synchronize()
        ca, cb = a.counters(), b.counters()
        assert (ca.attempts, ca.deposits) == (cb.attempts, cb.deposits)
        xa, ya = a.download()
        xb, yb = b.download()
        assert (xa == xb).all() and (ya == yb).all()


def test_replica_batch_equals_single_runs(lfg):
    L = 256
    seeds = [3, 11, 2**40 + 7]
    with lfg.KpzLattice(L, 0.95, 0.05, seeds=seeds) as kb:
        kb.make_flat_slopes()
        cs = kb.sweep(3)
        for r, s in enumerate(seeds):
            with lfg.KpzLattice(L, 0.95, 0.05, s) as k1:
                k1.make_flat_slopes()
                c1 = k1.sweep(3)
                assert (cs[r].deposits, cs[r].detaches) == (c1.deposits, c1.detaches)
                assert all((a == b).all() for a, b in zip(kb.download(r), k1.download()))


def test_large_lattice_properties(lfg, oracle):
    # L=4096 with the production block geometry (1024 x 128): exact accounting,
    # closure, W^2 consistency between the device scan and the oracle scan.
    L = 4096
    with lfg.KpzLattice(L, 1.0, 0.0, 1) as k:
        assert k.plan == (1024, 128)
        k.make_flat_slopes()
        c = k.sweep(3)
        assert abs(c.attempts - 3 * L * L) < 6 * L * 3 ** 0.5  # sub = 4: mean L^2, sd L per MCS
        assert c.successes == c.deposits and c.detaches == 0
        x, y = k.download()
        assert oracle.closure_holds(L, x, y)
        assert k.width_sums() == oracle.kpz_width_sums(L, x, y)
        # mean height identity: sum over successes (p=1): anchored mean moves by 2 per deposit
        # relative to the flat sum -L^2 only through the anchor; check via heights directly
        h = k.reconstruct_heights().astype(np.int64)
        assert (h.sum(), (h * h).sum()) == k.width_sums()


def test_block_height_256_matches_oracle(lfg, oracle):
    # 8-warp CTAs (block_y = 256): the block-boundary part of the DT deficit is 45 % smaller
    # than with the default 128 (profiles/stats_r01.md), at 3 % lower throughput
    for (L, p, q, bx, by, n) in [(2048, 1.0, 0.0, 1024, 256, 2), (2048, 0.95, 0.05, 1024, 256, 2),
                                 (1024, 0.95, 0.05, 256, 256, 2), (4096, 1.0, 0.5, 1024, 256, 1)]:
        x, y = oracle.kpz_flat(L)
        c_ref = oracle.kpz_sweep_dtr(L, x, y, p, q, 17, 0, n, bx, by)
        with lfg.KpzLattice(L, p, q, 17, block_x=bx, block_y=by) as k:
            k.make_flat_slopes()
            c = k.sweep(n)
            gx, gy = k.download()
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist(), (L, bx, by, p, q)
        assert (gx == x).all() and (gy == y).all(), (L, bx, by, p, q)


def test_large_lattice_matches_oracle_one_sweep(lfg, oracle):
    L = 2048
    # (1, 0.5) and (0, 1): thresholds of exactly 2^32 and 0 on the TMA-staged path, where the
    # acceptance compare is 32-bit with the "threshold == 2^32" predicate
    for (p, q) in ((1.0, 0.0), (0.95, 0.05), (1.0, 0.5), (0.0, 1.0)):
        x, y = oracle.kpz_flat(L)
        c_ref = oracle.kpz_sweep_dtr(L, x, y, p, q, 31, 0, 1, 1024, 128)
        with lfg.KpzLattice(L, p, q, 31) as k:
            k.make_flat_slopes()
            c = k.sweep(1)
            gx, gy = k.download()
        assert [c.attempts, c.successes, c.deposits, c.detaches] == c_ref.tolist()
        assert (gx == x).all() and (gy == y).all()


_SWEEP_KERNEL_PROG = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import paper_1204_5072_b200 as lfg
out = []
for (L, p, q, seed, bx, by, n) in json.loads(sys.argv[2]):
    with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by) as k:
        k.make_flat_slopes()
        c = k.sweep(n)
        x, y = k.download()
        out.append([c.deposits, c.detaches, hashlib.sha256(x.tobytes() + y.tobytes()).hexdigest()])
print(json.dumps(out))
"""


def test_sweep_kernel_matches_phase_launches(lfg):
    """The persistent whole-sweep kernel (LFG_KPZ_SWEEP_KERNEL=1, flag-ordered
    phases) reproduces the four-launch sweep bit for bit."""
    import hashlib
    import json
    import subprocess

    cases = [(2048, 1.0, 0.0, 5, 1024, 128, 3), (4096, 0.95, 0.05, 6, 1024, 64, 2), (1024, 1.0, 0.0, 7, 256, 32, 2)]
    ref = []
    for (L, p, q, seed, bx, by, n) in cases:
        with lfg.KpzLattice(L, p, q, seed, block_x=bx, block_y=by) as k:
            k.make_flat_slopes()
            c = k.sweep(n)
            x, y = k.download()
            ref.append([c.deposits, c.detaches, hashlib.sha256(x.tobytes() + y.tobytes()).hexdigest()])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LFG_KPZ_SWEEP_KERNEL="1")
    r = subprocess.run([sys.executable, "-c", _SWEEP_KERNEL_PROG, root, json.dumps(cases)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1]) == ref


_REPLICA_PROG = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import paper_1204_5072_b200 as lfg
out = []
for (L, p, q, seeds, bx, by, n) in json.loads(sys.argv[2]):
    with lfg.KpzLattice(L, p, q, seeds=seeds, block_x=bx, block_y=by) as k:
        k.make_flat_slopes()
        cs = k.sweep(n)
        cs = cs if isinstance(cs, list) else [cs]
        for r in range(len(seeds)):
            x, y = k.download(r)
            out.append([cs[r].deposits, cs[r].detaches, hashlib.sha256(x.tobytes() + y.tobytes()).hexdigest()])
print(json.dumps(out))
"""


def test_chained_phases_match_plain_launches():
    """Chained phase launches (programmatic dependent launch; each block waits for
    the previous phase's blocks around it, with a per-replica set order) give the
    lattices of plain stream-ordered launches (LFG_KPZ_PDL=0) bit for bit --
    several replicas with different seeds in one launch, many blocks per phase."""
    import json
    import subprocess

    cases = [(4096, 0.95, 0.05, [5, 6, 7, 2**33 + 1, 99], 1024, 128, 3),
             (2048, 1.0, 0.0, [11, 12, 13], 256, 32, 4),
             (8192, 1.0, 0.0, [21], 1024, 128, 2)]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for pdl in ("1", "0"):
        env = dict(os.environ, LFG_KPZ_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _REPLICA_PROG, root, json.dumps(cases)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]


def test_async_transfers_match_sync_calls(lfg, oracle):
    """upload_async / sweep_async / width_sums_async / download_async on two
    handles with their own streams == the synchronous calls."""
    import torch

    L = 2048
    x0, y0 = oracle.kpz_flat(L)
    ref = []
    for seed in (31, 32):
        with lfg.KpzLattice(L, 0.95, 0.05, seed) as k:
            k.upload(x0, y0)
            k.sweep(2)
            ref.append((k.width_sums(), *k.download()))
    ks = [lfg.KpzLattice(L, 0.95, 0.05, seed) for seed in (31, 32)]
    sts = [torch.cuda.Stream() for _ in ks]
    hx = [torch.from_numpy(x0.view(np.int64).copy()).pin_memory() for _ in ks]
    hy = [torch.from_numpy(y0.view(np.int64).copy()).pin_memory() for _ in ks]
    o3 = torch.zeros((2, 3), dtype=torch.int64).pin_memory()
    try:
        for i, k in enumerate(ks):
            k.set_stream(sts[i].cuda_stream)
        for _ in range(2):
            for i, k in enumerate(ks):
                k.upload_ptr_async(hx[i].data_ptr(), hy[i].data_ptr())
                k.sweep_async(1)
                k.width_sums_async(o3[i].data_ptr())
                k.download_ptr_async(hx[i].data_ptr(), hy[i].data_ptr())
        for i, k in enumerate(ks):
            k.synchronize()
            k.upload_check()
            s, s2 = int(o3[i, 0]), int(o3[i, 1]) + int(o3[i, 2])
            # each step re-uploads the previous step's download: 2 sweeps from the flat start
            assert (s, s2) == tuple(ref[i][0])
            assert np.array_equal(hx[i].numpy().view(np.uint64), ref[i][1])
            assert np.array_equal(hy[i].numpy().view(np.uint64), ref[i][2])
    finally:
        for k in ks:
            k.close()


def test_upload_async_check_reports_closure(lfg, oracle):
    import torch

    L = 64
    x, y = oracle.kpz_flat(L)
    x[3] ^= np.uint64(1 << 5)
    hx = torch.from_numpy(x.view(np.int64).copy()).pin_memory()
    hy = torch.from_numpy(y.view(np.int64).copy()).pin_memory()
    with lfg.KpzLattice(L) as k:
        k.upload_ptr_async(hx.data_ptr(), hy.data_ptr())
        with pytest.raises(lfg.ClosureError, match="closure"):
            k.upload_check()
        k.upload_check()  # the failure was reported once


def test_bench_size_properties(lfg, oracle):
    """L = 2^16 (the bench lattice, BASELINE configs[1]) with the production plan: two sweeps,
    then the downloaded reference-layout slope field is closed (integrable), the row sums of
    sigma_x and column sums of sigma_y are conserved, and the attempt accounting is exact."""
    L = 1 << 16
    with lfg.KpzLattice(L, 1.0, 0.0, 99) as k:
        assert k.plan == (1024, 128)
        k.make_flat_slopes()
        x0, y0 = k.download()
        c = k.sweep(2)
        assert abs(c.attempts - 2 * L * L) < 6 * L * 2 ** 0.5  # sub = 4: mean L^2, sd L per MCS
        assert c.detaches == 0 and c.deposits > 0.1 * c.attempts
        x, y = k.download()
    wpr = L // 64

    def row_ones(w):  # +1 bits per row
        return np.bitwise_count(w.reshape(L, wpr)).sum(axis=1, dtype=np.int64)

    def col_ones(w):  # +1 bits per column, in row chunks (the unpacked lattice is 4 GiB)
        acc = np.zeros(L, np.int64)
        rows = w.reshape(L, wpr)
        for r0 in range(0, L, 512):
            acc += np.unpackbits(rows[r0:r0 + 512].view(np.uint8), axis=1, bitorder="little").sum(axis=0, dtype=np.int64)
        return acc

    assert np.array_equal(row_ones(x), row_ones(x0))  # sigma_x row sums
    assert np.array_equal(col_ones(y), col_ones(y0))  # sigma_y column sums
    assert oracle.closure_holds(L, x, y)


@pytest.mark.parametrize("L", [4, 8, 16, 32, 64, 256])
def test_host_readouts_any_field(lfg, reflib, L):
    """interface_width / reconstruct_heights of host SlopeFields through the
    handle-free device readouts: every power-of-two L >= 4 and fields that are
    not integrable (random bits), against the unmodified reference."""
    rs = np.random.RandomState(L)
    nw = (L * L + 63) // 64
    for trial in range(3):
        if trial == 0:
            x, y = reflib.make_flat(L)
            for _ in range(2):
                reflib.kpz_sweep_sequential(L, x, y, 0.9, 0.1, "lcg64", 5 + L, 1)
        else:
            x = rs.randint(0, 2**63, size=nw, dtype=np.int64).view(np.uint64)
            y = rs.randint(0, 2**63, size=nw, dtype=np.int64).view(np.uint64)
            if L * L < 64:
                x &= np.uint64((1 << (L * L)) - 1)
                y &= np.uint64((1 << (L * L)) - 1)
        assert lfg.interface_width(L, x, y) == reflib.interface_width(L, x, y)
        try:
            ref_h = reflib.reconstruct_heights(L, x, y)
        except Exception:
            ref_h = None
        if ref_h is None:
            with pytest.raises(lfg.ClosureError):
                lfg.reconstruct_heights(L, x, y)
        else:
            assert np.array_equal(lfg.reconstruct_heights(L, x, y), ref_h)


def test_heights_readout_refuses_unclosed_state(lfg, reflib):
    """The device's default state (all slopes -1, SlopeField(L)) is swept like the
    reference but is not integrable: lfg_kpz_heights raises like
    reconstruct_heights (kpz.cpp:42-44); after make_flat_slopes it succeeds."""
    L = 64
    with lfg.KpzLattice(L) as k:
        with pytest.raises(lfg.ClosureError):
            k.reconstruct_heights()
        x, y = k.download()
        assert k.interface_width() == reflib.interface_width(L, x, y)
        k.make_flat_slopes()
        k.sweep(2)
        x, y = k.download()
        assert np.array_equal(k.reconstruct_heights(), reflib.reconstruct_heights(L, x, y))


def test_upload_rejects_unclosed_plaquettes(lfg, oracle):
    """Negating the four slopes around a site that is not a local extremum is a
    single spin flip -- the spin re-derivation check passes -- but the
    plaquettes around the site no longer close (heights would be
    path-dependent): the upload is rejected and the state is unchanged."""
    L = 64
    x, y = oracle.kpz_flat(L)
    i, j = 10, 21  # flat state: s_x(i) = +1, s_x(i+1) = -1, s_y(j) = -1, s_y(j+1) = +1
    for (plane, ii, jj) in ((x, i, j), (x, i + 1, j), (y, i, j), (y, i, j + 1)):
        idx = jj * L + ii
        plane[idx >> 6] ^= np.uint64(1 << (idx & 63))
    # closure_holds (row/column sums) still passes; reconstruct_heights' full
    # path-independence check (kpz.cpp:35-47) does not
    assert oracle.closure_holds(L, x, y)
    with pytest.raises(RuntimeError):
        oracle.reconstruct_heights(L, x, y)
    with lfg.KpzLattice(L) as k:
        k.make_flat_slopes()
        before = k.download()
        with pytest.raises(lfg.ClosureError):
            k.upload(x, y)
        after = k.download()
        assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1])
