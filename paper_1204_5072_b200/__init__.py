"""B200-native KPZ octahedron DT/DTr sweep and binary-alloy KMC (arXiv 1204.5072).

Host-side mirror of the reference's simulation API (namespace ``lf``,
/root/reference/proj/include/lf) over the C ABI in include/lfg.h.  The
compute path is the sm_100a library ``_lib/liblfg.so``; there is no CPU
fallback.  Names follow the reference:

    lf::SlopeField + make_flat_slopes + kpz_sweep_sequential + interface_width
        -> KpzLattice(L, p, q, seed).make_flat_slopes() / .sweep(n) / .interface_width()
    lf::OccupancyLattice + make_random_alloy + kmc_mcs_sequential + open_bonds_per_particle
        -> KmcLattice(L, eps, both_active, seed).make_random_alloy(c) / .sweep(n) / ...
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from ._native import (ClosureError, Counters, CudaError, DeviceOutOfMemory, DomainError,  # noqa: F401
                      InvalidArgument, KmcPlan, KpzPlan, LfgError, TransportError, check, device_count)

__all__ = ["KpzLattice", "ShardedKpzLattice", "KmcLattice", "ShardedKmcLattice", "Counters", "LfgError", "InvalidArgument", "ClosureError",
           "DomainError", "CudaError", "device_count", "words2", "words3", "interface_width",
           "width_sums", "reconstruct_heights", "open_bond_sums", "open_bonds_per_particle"]


def words2(L: int) -> int:
    return (L * L + 63) // 64


def words3(L: int) -> int:
    return (L * L * L + 63) // 64


def _u64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a


# ---------------------------------------------------------------- host-lattice readouts
# The reference's free functions on host words (any power-of-two L >= 4,
# integrable or not), computed on the device (include/lfg.h "readouts of host
# lattices"; kpz.cpp:21-81, kmc.cpp:20-40).
def width_sums(L: int, x, y, device: int = 0):
    """interface_width's exact int64 (sum h, sum h^2) of a host SlopeField."""
    x, y = _u64(x), _u64(y)
    s, s2 = C.c_int64(), C.c_int64()
    check(_native.lib().lfg_kpz_width_sums_host(device, L, x.ctypes.data, y.ctypes.data, x.size, C.byref(s),
                                                C.byref(s2)))
    return int(s.value), int(s2.value)


def interface_width(L: int, x, y, device: int = 0) -> float:
    s, s2 = width_sums(L, x, y, device)
    n = float(L * L)  # kpz.cpp:78-80
    mean = s / n
    return s2 / n - mean * mean


def reconstruct_heights(L: int, x, y, device: int = 0) -> np.ndarray:
    """reconstruct_heights (kpz.cpp:21-49) -> int32 [L, L] indexed [j, i];
    ClosureError when path-dependent."""
    x, y = _u64(x), _u64(y)
    h = np.empty(L * L, np.int32)
    check(_native.lib().lfg_kpz_heights_host(device, L, x.ctypes.data, y.ctypes.data, x.size, h.ctypes.data, h.size))
    return h.reshape(L, L)


def open_bond_sums(L: int, words, device: int = 0):
    w = _u64(words)
    a, b = C.c_int64(), C.c_int64()
    check(_native.lib().lfg_kmc_open_bond_sums_host(device, L, w.ctypes.data, w.size, C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


def open_bonds_per_particle(L: int, words, device: int = 0) -> float:
    npart, nopen = open_bond_sums(L, words, device)
    if npart == 0:
        raise DomainError("open_bonds_per_particle: no B particles in lattice")
    return nopen / npart


class KpzLattice:
    """Device-resident slope field(s) advanced by the two-layer DTr sweep.

    ``replicas > 1`` (or ``seeds=[...]``) holds independent lattices that one
    launch advances together (ensembles, e.g. W(t) over 16 seeds).
    ``sub``: sub-sweeps per MCS (0 = 4, the statistically matched scheme; 8 =
    eight sub-sweeps, half the residual <h> bias; 1 = the paper's single-origin
    scheme), include/lfg.h ``lfg_kpz_plan``.
    """

    def __init__(self, L: int, p: float = 1.0, q: float = 0.0, seed: int = 1, *, seeds=None,
                 block_x: int = 0, block_y: int = 0, sub: int = 0, device: int = 0):
        self._h = None
        L_ = _native.lib()
        seeds = [int(seed)] if seeds is None else [int(s) for s in seeds]
        arr = (C.c_uint64 * len(seeds))(*seeds)
        plan = KpzPlan(block_x, block_y, sub)
        h = C.c_void_p()
        check(L_.lfg_kpz_create_batch(C.byref(h), L, float(p), float(q), arr, len(seeds), C.byref(plan), device))
        self._h = h
        self.L = int(L)
        self.replicas = len(seeds)
        self.device = device
        self.p, self.q, self.seeds = float(p), float(q), list(seeds)
        self._cnt_base = [(0, 0, 0)] * len(seeds)  # (attempts, deposits, detaches) restored by load()
        got = KpzPlan()
        check(L_.lfg_kpz_get_plan(h, C.byref(got)))
        self.plan = (int(got.block_x), int(got.block_y))
        self.sub = int(got.sub)

    # -- lifetime ---------------------------------------------------------
    def close(self) -> None:
        if self._h is not None:
            _native.lib().lfg_kpz_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- lattice state ----------------------------------------------------
    def make_flat_slopes(self) -> "KpzLattice":
        """make_flat_slopes (lattice.cpp:71-82) on every replica."""
        check(_native.lib().lfg_kpz_init_flat(self._h))
        return self

    init_flat = make_flat_slopes

    def upload(self, x, y, replica: int = 0) -> None:
        x, y = _u64(x), _u64(y)
        n = words2(self.L)
        if x.size != n or y.size != n:
            raise InvalidArgument(f"upload: expected {n} words per plane")
        check(_native.lib().lfg_kpz_upload(self._h, replica, x.ctypes.data, y.ctypes.data, n))

    def upload_ptr(self, x_ptr: int, y_ptr: int, replica: int = 0) -> None:
        """Upload from raw host pointers (e.g. pinned torch tensors)."""
        check(_native.lib().lfg_kpz_upload(self._h, replica, x_ptr, y_ptr, words2(self.L)))

    def download(self, replica: int = 0):
        n = words2(self.L)
        x = np.empty(n, np.uint64)
        y = np.empty(n, np.uint64)
        check(_native.lib().lfg_kpz_download(self._h, replica, x.ctypes.data, y.ctypes.data, n))
        return x, y

    def download_ptr(self, x_ptr: int, y_ptr: int, replica: int = 0) -> None:
        check(_native.lib().lfg_kpz_download(self._h, replica, x_ptr, y_ptr, words2(self.L)))

    # stream-ordered host transfers (pinned pointers; complete at synchronize())
    def upload_ptr_async(self, x_ptr: int, y_ptr: int, replica: int = 0) -> None:
        check(_native.lib().lfg_kpz_upload_async(self._h, replica, x_ptr, y_ptr, words2(self.L)))

    def upload_check(self) -> None:
        """Raise ClosureError if an upload_ptr_async since the last check was not integrable."""
        check(_native.lib().lfg_kpz_upload_check(self._h))

    def download_ptr_async(self, x_ptr: int, y_ptr: int, replica: int = 0) -> None:
        check(_native.lib().lfg_kpz_download_async(self._h, replica, x_ptr, y_ptr, words2(self.L)))

    def width_sums_async(self, out3_ptr: int, replica: int = 0) -> None:
        """Enqueue the W^2 scan; pinned int64[3] at out3_ptr holds (sum h, s2a, s2b) after synchronize()."""
        check(_native.lib().lfg_kpz_width_sums_async(self._h, replica, out3_ptr))

    # -- dynamics ---------------------------------------------------------
    def sweep(self, sweeps: int = 1):
        """kpz_sweep_sequential(f, params, rng, sweeps) (kpz.cpp:5-19) -> Counters
        (a list of Counters when replicas > 1)."""
        out = (Counters * self.replicas)()
        check(_native.lib().lfg_kpz_sweep(self._h, int(sweeps), out))
        return out[0] if self.replicas == 1 else list(out)

    def sweep_async(self, sweeps: int = 1) -> None:
        check(_native.lib().lfg_kpz_sweep_async(self._h, int(sweeps)))

    def phase(self, sweep: int, phase: int) -> None:
        check(_native.lib().lfg_kpz_phase(self._h, int(sweep), int(phase)))

    def counters(self, replica: int = 0) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kpz_counters(self._h, replica, C.byref(c)))
        a0, d0, e0 = self._cnt_base[replica]
        if a0 or d0 or e0:
            c.attempts += a0
            c.deposits += d0
            c.detaches += e0
            c.successes += d0 + e0
        return c

    def reset_counters(self) -> None:
        check(_native.lib().lfg_kpz_reset_counters(self._h))
        self._cnt_base = [(0, 0, 0)] * self.replicas

    # -- snapshot / exact resume ------------------
    def save(self, path: str) -> None:
        """Snapshot: the reference's slope planes of every replica + (p, q, seeds, plan,
        next sweep index, counters).  The counter-based RNG makes load() + sweep(n) continue
        the trajectory bit for bit."""
        from .snapshot import save_kpz

        save_kpz(self, path)

    @classmethod
    def load(cls, path: str, device: int = 0) -> "KpzLattice":
        from .snapshot import load_kpz

        return load_kpz(path, device)

    # -- observables ------------------------------------------------------
    def width_sums(self, replica: int = 0):
        s, s2 = C.c_int64(), C.c_int64()
        check(_native.lib().lfg_kpz_width_sums(self._h, replica, C.byref(s), C.byref(s2)))
        return int(s.value), int(s2.value)

    def interface_width(self, replica: int = 0) -> float:
        """interface_width(const SlopeField&) (kpz.cpp:62-81)."""
        w = C.c_double()
        check(_native.lib().lfg_kpz_interface_width(self._h, replica, C.byref(w)))
        return float(w.value)

    def reconstruct_heights(self, replica: int = 0) -> np.ndarray:
        """reconstruct_heights (kpz.cpp:21-49) -> int32 [L, L] indexed [j, i]."""
        h = np.empty(self.L * self.L, np.int32)
        check(_native.lib().lfg_kpz_heights(self._h, replica, h.ctypes.data, h.size))
        return h.reshape(self.L, self.L)

    # -- state / plumbing -------------------------------------------------
    def set_params(self, p: float, q: float) -> None:
        check(_native.lib().lfg_kpz_set_params(self._h, float(p), float(q)))
        self.p, self.q = float(p), float(q)

    @property
    def sweep_index(self) -> int:
        v = C.c_uint64()
        check(_native.lib().lfg_kpz_get_sweep_index(self._h, C.byref(v)))
        return int(v.value)

    @sweep_index.setter
    def sweep_index(self, v: int) -> None:
        check(_native.lib().lfg_kpz_set_sweep_index(self._h, int(v)))

    def set_seed(self, seed: int, replica: int = 0) -> None:
        check(_native.lib().lfg_kpz_set_seed(self._h, replica, int(seed)))
        self.seeds[replica] = int(seed)

    def set_stream(self, stream_ptr: int) -> None:
        check(_native.lib().lfg_kpz_set_stream(self._h, C.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        check(_native.lib().lfg_kpz_synchronize(self._h))

    def device_spins(self, replica: int = 0):
        p, n = C.c_void_p(), C.c_size_t()
        check(_native.lib().lfg_kpz_device_spins(self._h, replica, C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)


class ShardedKpzLattice:
    """BASELINE configs[2]: one lattice split into y-strips over several GPUs, driven by
    this one process through the C ABI (lfg_kpz_create_sharded).  Same trajectory, bit
    for bit, as KpzLattice with the same L, p, q, seed and plan.  ``devices``: one CUDA
    device per strip (may repeat, e.g. [0, 0] for two strips on one GPU)."""

    def __init__(self, L: int, p: float = 1.0, q: float = 0.0, seed: int = 1, *, devices=(0, 1),
                 block_x: int = 0, block_y: int = 0, sub: int = 0):
        self._h = None
        devs = [int(d) for d in devices]
        arr = (C.c_int32 * len(devs))(*devs)
        plan = KpzPlan(block_x, block_y, sub)
        h = C.c_void_p()
        check(_native.lib().lfg_kpz_create_sharded(C.byref(h), L, float(p), float(q), int(seed), C.byref(plan),
                                                   len(devs), arr))
        self._h, self.L, self.devices = h, int(L), devs

    def close(self) -> None:
        if self._h is not None:
            _native.lib().lfg_kpz_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def make_flat_slopes(self) -> "ShardedKpzLattice":
        check(_native.lib().lfg_kpz_sharded_init_flat(self._h))
        return self

    def upload(self, x, y) -> None:
        x, y = _u64(x), _u64(y)
        check(_native.lib().lfg_kpz_sharded_upload(self._h, x.ctypes.data, y.ctypes.data, x.size))

    def download(self):
        n = words2(self.L)
        x = np.empty(n, np.uint64)
        y = np.empty(n, np.uint64)
        check(_native.lib().lfg_kpz_sharded_download(self._h, x.ctypes.data, y.ctypes.data, n))
        return x, y

    def sweep(self, sweeps: int = 1) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kpz_sharded_sweep(self._h, int(sweeps), C.byref(c)))
        return c

    def counters(self) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kpz_sharded_counters(self._h, C.byref(c)))
        return c

    def width_sums(self):
        s, s2 = C.c_int64(), C.c_int64()
        check(_native.lib().lfg_kpz_sharded_width_sums(self._h, C.byref(s), C.byref(s2)))
        return int(s.value), int(s2.value)

    def interface_width(self) -> float:
        w = C.c_double()
        check(_native.lib().lfg_kpz_sharded_interface_width(self._h, C.byref(w)))
        return float(w.value)

    @property
    def sweep_index(self) -> int:
        v = C.c_uint64()
        check(_native.lib().lfg_kpz_sharded_get_sweep_index(self._h, C.byref(v)))
        return int(v.value)

    @sweep_index.setter
    def sweep_index(self, v: int) -> None:
        check(_native.lib().lfg_kpz_sharded_set_sweep_index(self._h, int(v)))


class KmcLattice:
    """Device-resident fcc binary-alloy occupancy advanced by the two-layer DT sweep."""

    def __init__(self, L: int, eps: float = 1.5, both_active: bool = False, seed: int = 1, *,
                 block: int = 0, sub: int = 0, device: int = 0):
        self._h = None
        L_ = _native.lib()
        if not hasattr(L_, "lfg_kmc_create"):
            raise ImportError("liblfg.so was built without the KMC path")
        plan = KmcPlan(block, sub)
        h = C.c_void_p()
        check(L_.lfg_kmc_create(C.byref(h), L, float(eps), int(bool(both_active)), int(seed), C.byref(plan),
                                device))
        self._h = h
        self.L = int(L)
        self.device = device
        self.eps, self.both_active, self.seed = float(eps), bool(both_active), int(seed)
        self._cnt_base = (0, 0)  # (attempts, exchanges) restored by load()
        got = KmcPlan()
        check(L_.lfg_kmc_get_plan(h, C.byref(got)))
        self.plan = int(got.block)
        self.sub = int(got.sub)

    def close(self) -> None:
        if self._h is not None:
            _native.lib().lfg_kmc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def upload(self, words) -> None:
        w = _u64(words)
        n = words3(self.L)
        if w.size != n:
            raise InvalidArgument(f"upload: expected {n} words")
        check(_native.lib().lfg_kmc_upload(self._h, w.ctypes.data, n))

    def download(self) -> np.ndarray:
        n = words3(self.L)
        w = np.empty(n, np.uint64)
        check(_native.lib().lfg_kmc_download(self._h, w.ctypes.data, n))
        return w

    def make_random_alloy(self, c: float, seed: int) -> "KmcLattice":
        """make_random_alloy (lattice.cpp:117-132) with the device counter RNG."""
        check(_native.lib().lfg_kmc_init_random_alloy(self._h, float(c), int(seed)))
        return self

    def sweep(self, steps: int = 1) -> Counters:
        """kmc_mcs_sequential (kmc.cpp:5-18) -> Counters."""
        c = Counters()
        check(_native.lib().lfg_kmc_sweep(self._h, int(steps), C.byref(c)))
        return c

    def sweep_async(self, steps: int = 1) -> None:
        check(_native.lib().lfg_kmc_sweep_async(self._h, int(steps)))

    def phase(self, sweep: int, phase: int) -> None:
        check(_native.lib().lfg_kmc_phase(self._h, int(sweep), int(phase)))

    def counters(self) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kmc_counters(self._h, C.byref(c)))
        a0, s0 = self._cnt_base
        if a0 or s0:
            c.attempts += a0
            c.successes += s0
            c.deposits += s0
        return c

    def reset_counters(self) -> None:
        check(_native.lib().lfg_kmc_reset_counters(self._h))
        self._cnt_base = (0, 0)

    def save(self, path: str) -> None:
        """Snapshot: occupancy words (reference layout) + (eps, mode, seed, plan, next sweep
        index, counters); load() + sweep(n) continues bit for bit."""
        from .snapshot import save_kmc

        save_kmc(self, path)

    @classmethod
    def load(cls, path: str, device: int = 0) -> "KmcLattice":
        from .snapshot import load_kmc

        return load_kmc(path, device)

    def open_bond_sums(self):
        a, b = C.c_int64(), C.c_int64()
        check(_native.lib().lfg_kmc_open_bond_sums(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def open_bonds_per_particle(self) -> float:
        """open_bonds_per_particle (kmc.cpp:20-40)."""
        v = C.c_double()
        check(_native.lib().lfg_kmc_open_bonds_per_particle(self._h, C.byref(v)))
        return float(v.value)

    def count_b(self) -> int:
        v = C.c_int64()
        check(_native.lib().lfg_kmc_count_b(self._h, C.byref(v)))
        return int(v.value)

    def set_params(self, eps: float, both_active: bool) -> None:
        check(_native.lib().lfg_kmc_set_params(self._h, float(eps), int(bool(both_active))))
        self.eps, self.both_active = float(eps), bool(both_active)

    @property
    def sweep_index(self) -> int:
        v = C.c_uint64()
        check(_native.lib().lfg_kmc_get_sweep_index(self._h, C.byref(v)))
        return int(v.value)

    @sweep_index.setter
    def sweep_index(self, v: int) -> None:
        check(_native.lib().lfg_kmc_set_sweep_index(self._h, int(v)))

    def set_seed(self, seed: int) -> None:
        check(_native.lib().lfg_kmc_set_seed(self._h, int(seed)))
        self.seed = int(seed)

    def set_stream(self, stream_ptr: int) -> None:
        check(_native.lib().lfg_kmc_set_stream(self._h, C.c_void_p(stream_ptr)))

    def set_concurrency(self, lattices: int) -> None:
        """Hint: `lattices` handles sweep side by side (kernel choice only)."""
        check(_native.lib().lfg_kmc_set_concurrency(self._h, int(lattices)))

    def synchronize(self) -> None:
        check(_native.lib().lfg_kmc_synchronize(self._h))

    def device_words(self):
        p, n = C.c_void_p(), C.c_size_t()
        check(_native.lib().lfg_kmc_device_words(self._h, C.byref(p), C.byref(n)))
        return int(p.value or 0), int(n.value)
class ShardedKmcLattice:
    """BASELINE configs[4]: one KMC lattice cut into z-slabs over several GPUs, driven by
    this one process through the C ABI (lfg_kmc_create_sharded).  Same trajectory, bit for
    bit, as KmcLattice with the same L, eps, mode, seed and plan."""

    def __init__(self, L: int, eps: float = 1.5, both_active: bool = True, seed: int = 1, *, devices=(0, 1),
                 block: int = 0, sub: int = 0):
        self._h = None
        devs = [int(d) for d in devices]
        arr = (C.c_int32 * len(devs))(*devs)
        plan = KmcPlan(block, sub)
        h = C.c_void_p()
        check(_native.lib().lfg_kmc_create_sharded(C.byref(h), L, float(eps), int(bool(both_active)), int(seed),
                                                   C.byref(plan), len(devs), arr))
        self._h, self.L, self.devices = h, int(L), devs

    def close(self) -> None:
        if self._h is not None:
            _native.lib().lfg_kmc_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def make_random_alloy(self, c: float, alloy_seed: int) -> "ShardedKmcLattice":
        check(_native.lib().lfg_kmc_sharded_init_random_alloy(self._h, float(c), int(alloy_seed)))
        return self

    def upload(self, words) -> None:
        w = _u64(words)
        check(_native.lib().lfg_kmc_sharded_upload(self._h, w.ctypes.data, w.size))

    def download(self):
        w = np.empty(self.L ** 3 // 64, np.uint64)
        check(_native.lib().lfg_kmc_sharded_download(self._h, w.ctypes.data, w.size))
        return w

    def sweep(self, sweeps: int = 1) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kmc_sharded_sweep(self._h, int(sweeps), C.byref(c)))
        return c

    def counters(self) -> Counters:
        c = Counters()
        check(_native.lib().lfg_kmc_sharded_counters(self._h, C.byref(c)))
        return c

    def open_bond_sums(self):
        a, b = C.c_int64(), C.c_int64()
        check(_native.lib().lfg_kmc_sharded_open_bond_sums(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def open_bonds_per_particle(self) -> float:
        v = C.c_double()
        check(_native.lib().lfg_kmc_sharded_open_bonds_per_particle(self._h, C.byref(v)))
        return float(v.value)

    @property
    def sweep_index(self) -> int:
        v = C.c_uint64()
        check(_native.lib().lfg_kmc_sharded_get_sweep_index(self._h, C.byref(v)))
        return int(v.value)

    @sweep_index.setter
    def sweep_index(self, v: int) -> None:
        check(_native.lib().lfg_kmc_sharded_set_sweep_index(self._h, int(v)))


