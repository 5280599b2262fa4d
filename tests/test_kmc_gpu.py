"""GPU parity tests for the KMC two-layer DT path (run with -m gpu on a B200).

Bit-exact against the reference-produced golden vectors (tests/golden/golden.json:
the DT schedule with lf::exchange_probability, kmc.hpp:70-76) and against the
live oracle restatement on seeded inputs.
"""
import hashlib

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


@pytest.mark.parametrize("case", range(8))
def test_kmc_dt_golden_bit_exact(lfg, oracle, golden, case):
    g = golden["kmc_dt"][case]
    L = g["L"]
    w, _ = oracle.kmc_random_alloy(L, g["c"], "lcg64", g["alloy_seed"])
    with lfg.KmcLattice(L, g["eps"], bool(g["both"]), g["seed"], block=g["bk"], sub=g["sub"]) as k:
        k.upload(w)
        k.sweep_index = g["sweep0"]
        c = k.sweep(g["nsweeps"])
        assert [c.attempts, c.successes] == g["counters"]
        gw = k.download()
        assert sha(gw) == g["sha"]
        assert k.count_b() == g["count_b"]
        assert k.open_bonds_per_particle() == g["open_bonds"]


def test_kmc_live_oracle_random(lfg, oracle):
    rs = np.random.RandomState(7)
    for _ in range(8):
        L = int(rs.choice([32, 64]))
        bk = int(rs.choice([b for b in (16, 32) if 2 * b <= L]))
        eps = float(rs.choice([0.0, 0.5, 1.5, 3.0]))
        both = bool(rs.randint(2))
        c = float(rs.choice([0.1, 0.325, 0.5, 0.8]))
        seed = int(rs.randint(0, 2**62))
        sub = int(rs.choice([1, 4]))
        w, _ = oracle.kmc_random_alloy(L, c, "lcg64", int(rs.randint(1, 1000)))
        w_ref = w.copy()
        c_ref = oracle.kmc_sweep_dt(L, w_ref, eps, both, seed, 3, 2, bk, sub)
        with lfg.KmcLattice(L, eps, both, seed, block=bk, sub=sub) as k:
            k.upload(w)
            k.sweep_index = 3
            cc = k.sweep(2)
            gw = k.download()
        assert [cc.attempts, cc.successes] == c_ref.tolist(), (L, bk, eps, both, c)
        assert np.array_equal(gw, w_ref), (L, bk, eps, both, c)


def test_open_bonds_and_count_b(lfg, oracle, golden):
    for a in golden["kmc_alloy"]:
        L = a["L"]
        if L < 32:
            continue
        w, _ = oracle.kmc_random_alloy(L, a["c"], "lcg64", a["seed"])
        with lfg.KmcLattice(L) as k:
            k.upload(w)
            assert k.count_b() == a["count_b"]
            np_, no = k.open_bond_sums()
            assert (np_, no) == oracle.kmc_open_bond_sums(L, w)
            assert k.open_bonds_per_particle() == a["open_bonds"]


def test_open_bonds_no_particles_is_domain_error(lfg):
    with lfg.KmcLattice(32) as k:  # all A (OccupancyLattice ctor)
        with pytest.raises(lfg.DomainError, match="no B particles"):
            k.open_bonds_per_particle()


def test_init_random_alloy_statistics(lfg, oracle):
    L = 64
    n_valid = L ** 3 // 2
    with lfg.KmcLattice(L) as k:
        k.make_random_alloy(0.325, 11)
        w = k.download()
        nb = k.count_b()
        # odd-parity sites stay empty (lattice.hpp:104-106)
        bits = np.unpackbits(w.view(np.uint8), bitorder="little").reshape(L, L, L)
        z, y, x = np.indices((L, L, L))
        assert bits[((x ^ y ^ z) & 1) == 1].sum() == 0
        mu, sd = 0.325 * n_valid, np.sqrt(n_valid * 0.325 * 0.675)
        assert abs(nb - mu) < 5 * sd
        # determinism and seed dependence
        k.make_random_alloy(0.325, 11)
        assert np.array_equal(k.download(), w)
        k.make_random_alloy(0.325, 12)
        assert not np.array_equal(k.download(), w)
        k.make_random_alloy(0.0, 3)
        assert k.count_b() == 0
        k.make_random_alloy(1.0, 3)
        assert k.count_b() == n_valid
        with pytest.raises(lfg.InvalidArgument):
            k.make_random_alloy(1.5, 3)


def test_conservation_accounting_and_quench(lfg):
    # SPEC acceptance 6 (species conservation) and the quench observable trend.
    L = 128
    with lfg.KmcLattice(L, 1.5, True, 5) as k:
        k.make_random_alloy(0.5, 2)
        n0 = k.count_b()
        ob0 = k.open_bonds_per_particle()
        c = k.sweep(20)
        assert c.attempts == 20 * L ** 3 // 2
        assert k.count_b() == n0
        ob1 = k.open_bonds_per_particle()
        assert ob1 < ob0 - 0.1


def test_kmc_phase_api_and_resume(lfg, oracle):
    L = 64
    w, _ = oracle.kmc_random_alloy(L, 0.5, "lcg64", 4)
    with lfg.KmcLattice(L, 1.5, False, 9) as a, lfg.KmcLattice(L, 1.5, False, 9) as b:
        a.upload(w)
        b.upload(w)
        a.sweep(3)
        b.sweep(1)
        for s in (1, 2):
            for ph in range(8):
                b.phase(s, ph)
        b.synchronize()
        assert np.array_equal(a.download(), b.download())
        assert a.counters().successes == b.counters().successes


@pytest.mark.parametrize("both", [False, True])
def test_kmc_large_d_thresholds(lfg, oracle, both):
    """Small eps makes every Metropolis threshold d = 1..12 matter (exp(-d eps) ~ 0.5..0.95):
    the 16^3 kernel's 8-thread CTAs must still see the whole 13-entry table."""
    L, eps, seed = 64, 0.05, 321
    w, _ = oracle.kmc_random_alloy(L, 0.5, "lcg64", 8)
    w_ref = w.copy()
    c_ref = oracle.kmc_sweep_dt(L, w_ref, eps, both, seed, 0, 3, 16)
    with lfg.KmcLattice(L, eps, both, seed, block=16) as k:
        k.upload(w)
        c = k.sweep(3)
        assert [c.attempts, c.successes] == c_ref.tolist()
        assert np.array_equal(k.download(), w_ref)


_KMC_PROG = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1204_5072_b200 as lfg
out = []
for (L, eps, both, seed, n) in json.loads(sys.argv[2]):
    with lfg.KmcLattice(L, eps, both, seed, block=16) as k:
        k.make_random_alloy(0.5, seed + 1)
        c = k.sweep(n)
        out.append([c.attempts, c.successes, hashlib.sha256(np.ascontiguousarray(k.download()).tobytes()).hexdigest()])
print(json.dumps(out))
"""


def test_kmc_16_kernels_agree():
    """The four 16^3 paths -- the producer/consumer warp pair and the single
    full-warp kernel (latency-bound phases; LFG_KMC_PC=1/0), the 8-lane kernel
    with one block per warp, and with four blocks per warp (>= 2368 active
    blocks, L = 512) -- give the same lattice (LFG_KMC_WIDE=0/1/2)."""
    import json
    import os
    import subprocess
    import sys

    cases = [(64, 1.5, True, 3, 3), (128, 0.3, False, 4, 2), (512, 1.5, True, 5, 1)]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mode, pc in (("0", "1"), ("1", "1"), ("2", "1"), ("1", "0"), ("2", "0")):
        env = dict(os.environ, LFG_KMC_WIDE=mode, LFG_KMC_PC=pc)
        r = subprocess.run([sys.executable, "-c", _KMC_PROG, root, json.dumps(cases)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert all(o == outs[0] for o in outs[1:])
