"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
(``paper_1204_5072_b200``) never does.

Two libraries:
  * ``Oracle``  -> oracle/_build/liboracle.so, the plain C++ restatement
    (oracle/oracle.cpp); always buildable (``make -C oracle``).
  * ``RefLib``  -> oracle/_ref/liblfref.so, the UNMODIFIED reference sources
    (/root/reference/proj/src) plus oracle/ref_shim.cpp; built only where the
    reference is present, travels to the GPU box as a prebuilt file.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblfref.so")

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

KIND = {"lcg32": 0, "lcg64": 1, "tinymt": 2}


def words2(L: int) -> int:
    return (L * L + 63) // 64


def words3(L: int) -> int:
    return (L * L * L + 63) // 64


def _sig(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


class Oracle:
    """The restatement (oracle/oracle.cpp)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        self.lib = lib
        I32, I64, U32, U64, D, I = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_int
        _sig(lib, "orc_philox4x32_10", None, u32p, u32p, u32p)
        _sig(lib, "orc_rng_draws", None, I, U64, U32, U64, u32p, I64)
        _sig(lib, "orc_lcg64_skip", U64, U64, U64)
        _sig(lib, "orc_split_streams_lcg", I, I, U64, I, U64, u64p)
        _sig(lib, "orc_kpz_flat", I, I32, u64p, u64p)
        _sig(lib, "orc_kpz_width_sums", None, I32, u64p, u64p, C.POINTER(I64), C.POINTER(I64))
        _sig(lib, "orc_width_from_sums", D, I32, I64, I64)
        _sig(lib, "orc_kpz_reconstruct_heights", I, I32, u64p, u64p, i32p)
        _sig(lib, "orc_kpz_closure_holds", I, I32, u64p, u64p)
        _sig(lib, "orc_kpz_sweep_sequential", I, I32, u64p, u64p, D, D, I, C.POINTER(U64), I, i64p)
        _sig(lib, "orc_kpz_sweep_dtr", I, I32, u64p, u64p, D, D, U64, U64, I32, I32, I32, I32, i64p)
        _sig(lib, "orc_kpz_sweep_draw", None, I32, I32, I32, U64, U64, i32p)
        _sig(lib, "orc_kmc_random_alloy", I, I32, D, I, U64, U32, u64p, C.POINTER(U64))
        _sig(lib, "orc_kmc_sweep_sequential", I, I32, u64p, D, I, I, C.POINTER(U64), I, i64p)
        _sig(lib, "orc_kmc_sweep_dt", I, I32, u64p, D, I, U64, U64, I32, I32, I32, i64p)
        _sig(lib, "orc_kmc_dt_phase_rows", I, I32, u64p, D, I, U64, U64, I32, I32, I32, I32, I32, i64p)
        _sig(lib, "orc_kmc_sweep_draw", None, I32, I32, U64, U64, i32p)
        _sig(lib, "orc_kmc_open_bond_sums_planes", None, I32, u64p, I32, I32, C.POINTER(I64), C.POINTER(I64))
        _sig(lib, "orc_kmc_open_bond_sums", None, I32, u64p, C.POINTER(I64), C.POINTER(I64))
        _sig(lib, "orc_kmc_count_b", I64, I32, u64p)

    # -- RNG ------------------------------------------------------------
    def philox(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.lib.orc_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def rng_draws(self, kind: str, seed: int, n: int, stream_id: int = 0, skip: int = 0):
        out = np.zeros(n, np.uint32)
        self.lib.orc_rng_draws(KIND[kind], seed, stream_id, skip, out, n)
        return out

    def lcg64_skip(self, state: int, n: int) -> int:
        return int(self.lib.orc_lcg64_skip(state, n))

    def split_streams_lcg(self, kind: str, seed: int, count: int, stride: int = 1 << 40):
        out = np.zeros(count, np.uint64)
        assert self.lib.orc_split_streams_lcg(KIND[kind], seed, count, stride, out) == 0
        return out

    # -- KPZ ------------------------------------------------------------
    def kpz_flat(self, L: int):
        x = np.zeros(words2(L), np.uint64)
        y = np.zeros(words2(L), np.uint64)
        if self.lib.orc_kpz_flat(L, x, y) != 0:
            raise ValueError("SlopeField: size must be a power of two >= 4")
        return x, y

    def kpz_width_sums(self, L, x, y):
        s, s2 = C.c_int64(), C.c_int64()
        self.lib.orc_kpz_width_sums(L, x, y, C.byref(s), C.byref(s2))
        return s.value, s2.value

    def width_from_sums(self, L, s, s2) -> float:
        return float(self.lib.orc_width_from_sums(L, s, s2))

    def interface_width(self, L, x, y) -> float:
        return self.width_from_sums(L, *self.kpz_width_sums(L, x, y))

    def reconstruct_heights(self, L, x, y):
        h = np.zeros(L * L, np.int32)
        if self.lib.orc_kpz_reconstruct_heights(L, x, y, h) != 0:
            raise RuntimeError("reconstruct_heights: slope field violates closure")
        return h.reshape(L, L)

    def closure_holds(self, L, x, y) -> bool:
        return bool(self.lib.orc_kpz_closure_holds(L, x, y))

    def kpz_sweep_sequential(self, L, x, y, p, q, kind, state, sweeps):
        c = np.zeros(4, np.int64)
        st = C.c_uint64(state)
        assert self.lib.orc_kpz_sweep_sequential(L, x, y, p, q, KIND[kind], C.byref(st), sweeps, c) == 0
        return c, st.value

    def kpz_sweep_dtr(self, L, x, y, p, q, seed, sweep0, nsweeps, bx, by, sub=4):
        """MCS sweep0 .. sweep0+nsweeps-1 of the DTr schedule (sub sub-sweeps each);
        counters [attempts, successes, deposits, detaches]."""
        c = np.zeros(4, np.int64)
        rc = self.lib.orc_kpz_sweep_dtr(L, x, y, p, q, seed, sweep0, nsweeps, bx, by, sub, c)
        if rc != 0:
            raise ValueError("KpzParams: invalid p/q")
        return c

    def kpz_sweep_draw(self, L, bx, by, seed, sweep):
        out = np.zeros(6, np.int32)
        self.lib.orc_kpz_sweep_draw(L, bx, by, seed, sweep, out)
        return out

    # -- KMC ------------------------------------------------------------
    def kmc_random_alloy(self, L, c, kind, seed, stream_id=0):
        w = np.zeros(words3(L), np.uint64)
        st = C.c_uint64()
        assert self.lib.orc_kmc_random_alloy(L, c, KIND[kind], seed, stream_id, w, C.byref(st)) == 0
        return w, st.value

    def kmc_sweep_sequential(self, L, w, eps, both, kind, state, steps):
        c = np.zeros(2, np.int64)
        st = C.c_uint64(state)
        assert self.lib.orc_kmc_sweep_sequential(L, w, eps, int(both), KIND[kind], C.byref(st), steps, c) == 0
        return c, st.value

    def kmc_sweep_dt(self, L, w, eps, both, seed, sweep0, nsweeps, bk, sub=1):
        """MCS sweep0 .. sweep0+nsweeps-1 of the KMC DT schedule (sub sub-sweeps each)."""
        c = np.zeros(2, np.int64)
        assert self.lib.orc_kmc_sweep_dt(L, w, eps, int(both), seed, sweep0, nsweeps, bk, sub, c) == 0
        return c

    def kmc_dt_phase_rows(self, L, w, eps, both, seed, sweep, phase, bk, bz0, nbz, sub=1):
        """One DT phase of sub-sweep `sweep` on block z-rows [bz0, bz0 + nbz); returns [attempts, successes]."""
        c = np.zeros(2, np.int64)
        assert self.lib.orc_kmc_dt_phase_rows(L, w, eps, int(both), seed, sweep, phase, bk, sub, bz0, nbz, c) == 0
        return c

    def kmc_sweep_draw(self, L, bk, seed, sweep):
        """(ox, oy, oz, order[8]) of a KMC DT sweep."""
        out = np.zeros(11, np.int32)
        self.lib.orc_kmc_sweep_draw(L, bk, seed, sweep, out)
        return int(out[0]), int(out[1]), int(out[2]), [int(v) for v in out[3:]]

    def kmc_open_bond_sums_planes(self, L, w, z0, nz):
        a, b = C.c_int64(), C.c_int64()
        self.lib.orc_kmc_open_bond_sums_planes(L, w, z0, nz, C.byref(a), C.byref(b))
        return a.value, b.value

    def kmc_open_bond_sums(self, L, w):
        a, b = C.c_int64(), C.c_int64()
        self.lib.orc_kmc_open_bond_sums(L, w, C.byref(a), C.byref(b))
        return a.value, b.value

    def kmc_count_b(self, L, w) -> int:
        return int(self.lib.orc_kmc_count_b(L, w))


class RefError(Exception):
    pass


class RefLib:
    """The unmodified reference sources + oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (built only where /root/reference exists)")
        lib = C.CDLL(path)
        self.lib = lib
        I32, I64, U32, U64, D, I = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_int
        _sig(lib, "ref_last_error", C.c_char_p)
        _sig(lib, "ref_rng_draws", I, I, U64, U32, U64, u32p, I64)
        _sig(lib, "ref_split_streams_state", I, I, U64, I, U64, u64p)
        _sig(lib, "ref_rng_kind_from_string", I, C.c_char_p, C.POINTER(I))
        _sig(lib, "ref_make_flat", I, I32, u64p, u64p)
        _sig(lib, "ref_interface_width", I, I32, u64p, u64p, C.POINTER(D))
        _sig(lib, "ref_reconstruct_heights", I, I32, u64p, u64p, i32p)
        _sig(lib, "ref_closure_holds", I, I32, u64p, u64p, C.POINTER(I))
        _sig(lib, "ref_kpz_params_validate", I, D, D)
        _sig(lib, "ref_kpz_sweep_sequential", I, I32, u64p, u64p, D, D, I, C.POINTER(U64), I, i64p)
        _sig(lib, "ref_kpz_attempt", I, I32, u64p, u64p, I32, I32, D, D, D, C.POINTER(I))
        _sig(lib, "ref_kpz_attempts_sequential", I, I32, u64p, u64p, D, D, I, C.POINTER(U64), I64, i64p)
        _sig(lib, "ref_kmc_attempts_sequential", I, I32, u64p, D, I, I, C.POINTER(U64), I64, i64p)
        _sig(lib, "ref_kpz_field_create", C.c_void_p, I32, u64p, u64p)
        _sig(lib, "ref_kpz_field_destroy", None, C.c_void_p)
        _sig(lib, "ref_kpz_field_attempts", I, C.c_void_p, D, D, I, C.POINTER(U64), I64, i64p)
        _sig(lib, "ref_kpz_sweep_dtr", I, I32, u64p, u64p, D, D, U64, U64, I32, I32, I32, I32, i64p)
        _sig(lib, "ref_make_random_alloy", I, I32, D, I, U64, u64p, C.POINTER(U64))
        _sig(lib, "ref_kmc_sweep_sequential", I, I32, u64p, D, I, I, C.POINTER(U64), I, i64p)
        _sig(lib, "ref_kmc_sweep_dt", I, I32, u64p, D, I, U64, U64, I32, I32, I32, i64p)
        _sig(lib, "ref_open_bonds_per_particle", I, I32, u64p, C.POINTER(D))
        _sig(lib, "ref_count_b", I, I32, u64p, C.POINTER(I64))
        _sig(lib, "ref_metropolis_prob", I, I, I, D, C.POINTER(D))
        _sig(lib, "ref_fcc_neighbors", I, I32, I32, I32, I32, i32p)
        _sig(lib, "ref_schedule_ahead_of_time_steps", I, I32, I32, I32, i32p, I32, C.POINTER(I32))
        _sig(lib, "ref_writelog_violations", I, I32, I64, i64p, i32p, i64p, i64p, C.POINTER(I64),
             C.POINTER(I64), i64p)

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def rng_draws(self, kind, seed, n, stream_id=0, skip=0):
        out = np.zeros(n, np.uint32)
        self._check(self.lib.ref_rng_draws(KIND[kind], seed, stream_id, skip, out, n))
        return out

    def split_streams_state(self, kind, seed, count, stride=1 << 40):
        out = np.zeros(count, np.uint64)
        self._check(self.lib.ref_split_streams_state(KIND[kind], seed, count, stride, out))
        return out

    def make_flat(self, L):
        x = np.zeros(words2(L), np.uint64)
        y = np.zeros(words2(L), np.uint64)
        self._check(self.lib.ref_make_flat(L, x, y))
        return x, y

    def interface_width(self, L, x, y):
        w = C.c_double()
        self._check(self.lib.ref_interface_width(L, x, y, C.byref(w)))
        return w.value

    def reconstruct_heights(self, L, x, y):
        h = np.zeros(L * L, np.int32)
        self._check(self.lib.ref_reconstruct_heights(L, x, y, h))
        return h.reshape(L, L)

    def closure_holds(self, L, x, y):
        ok = C.c_int()
        self._check(self.lib.ref_closure_holds(L, x, y, C.byref(ok)))
        return bool(ok.value)

    def kpz_sweep_sequential(self, L, x, y, p, q, kind, state, sweeps):
        c = np.zeros(2, np.int64)
        st = C.c_uint64(state)
        self._check(self.lib.ref_kpz_sweep_sequential(L, x, y, p, q, KIND[kind], C.byref(st), sweeps, c))
        return c, st.value

    def kpz_attempts_sequential(self, L, x, y, p, q, kind, state, n):
        """Bounded sample of kpz_sweep_sequential's loop (n attempts)."""
        c = np.zeros(2, np.int64)
        st = C.c_uint64(state)
        self._check(self.lib.ref_kpz_attempts_sequential(L, x, y, p, q, KIND[kind], C.byref(st), n, c))
        return c, st.value

    def kpz_field(self, L, x, y):
        """A reference lf::SlopeField held across calls (timed loops exclude copies)."""
        ptr = self.lib.ref_kpz_field_create(L, x, y)
        if not ptr:
            raise RefError(1, self.lib.ref_last_error().decode())
        ref = self

        class _Field:
            def attempts(self, p, q, kind, state, n):
                c = np.zeros(2, np.int64)
                st = C.c_uint64(state)
                ref._check(ref.lib.ref_kpz_field_attempts(ptr, p, q, KIND[kind], C.byref(st), n, c))
                return c, st.value

            def close(self):
                ref.lib.ref_kpz_field_destroy(ptr)

        return _Field()

    def kmc_attempts_sequential(self, L, w, eps, both, kind, state, n):
        c = np.zeros(2, np.int64)
        st = C.c_uint64(state)
        self._check(self.lib.ref_kmc_attempts_sequential(L, w, eps, int(both), KIND[kind], C.byref(st), n, c))
        return c, st.value

    def kpz_attempt(self, L, x, y, i, j, p, q, r):
        o = C.c_int()
        self._check(self.lib.ref_kpz_attempt(L, x, y, i, j, p, q, r, C.byref(o)))
        return o.value

    def kpz_sweep_dtr(self, L, x, y, p, q, seed, sweep0, nsweeps, bx, by, sub=4):
        c = np.zeros(4, np.int64)
        self._check(self.lib.ref_kpz_sweep_dtr(L, x, y, p, q, seed, sweep0, nsweeps, bx, by, sub, c))
        return c

    def make_random_alloy(self, L, c, kind, seed):
        w = np.zeros(words3(L), np.uint64)
        st = C.c_uint64()
        self._check(self.lib.ref_make_random_alloy(L, c, KIND[kind], seed, w, C.byref(st)))
        return w, st.value

    def kmc_sweep_sequential(self, L, w, eps, both, kind, state, steps):
        c = np.zeros(2, np.int64)
        st = C.c_uint64(state)
        self._check(self.lib.ref_kmc_sweep_sequential(L, w, eps, int(both), KIND[kind], C.byref(st), steps, c))
        return c, st.value

    def kmc_sweep_dt(self, L, w, eps, both, seed, sweep0, nsweeps, bk, sub=1):
        c = np.zeros(2, np.int64)
        self._check(self.lib.ref_kmc_sweep_dt(L, w, eps, int(both), seed, sweep0, nsweeps, bk, sub, c))
        return c

    def open_bonds_per_particle(self, L, w):
        o = C.c_double()
        self._check(self.lib.ref_open_bonds_per_particle(L, w, C.byref(o)))
        return o.value

    def count_b(self, L, w):
        o = C.c_int64()
        self._check(self.lib.ref_count_b(L, w, C.byref(o)))
        return o.value

    def writelog_violations(self, workers, group_off, task_worker, task_woff, write_site):
        """lf::WriteLog over a recorded schedule (groups = barrier intervals); returns
        (violations, writes, first violation (site, worker_a, worker_b) or None)."""
        nv, nw = C.c_int64(), C.c_int64()
        first = np.zeros(3, np.int64)
        self._check(self.lib.ref_writelog_violations(
            int(workers), len(group_off) - 1, np.ascontiguousarray(group_off, np.int64),
            np.ascontiguousarray(task_worker, np.int32), np.ascontiguousarray(task_woff, np.int64),
            np.ascontiguousarray(write_site, np.int64), C.byref(nv), C.byref(nw), first))
        return nv.value, nw.value, (tuple(int(v) for v in first) if nv.value else None)

    def metropolis_prob(self, ni, nf, eps):
        o = C.c_double()
        self._check(self.lib.ref_metropolis_prob(ni, nf, eps, C.byref(o)))
        return o.value


def try_ref() -> "RefLib | None":
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None
