"""ctypes binding of the C ABI (include/lfg.h) -> paper_1204_5072_b200/_lib/liblfg.so.

There is no fallback: if the sm_100a library is missing, importing the
device classes raises immediately (build it with ``python -m
paper_1204_5072_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFG_LIB") or os.path.join(PKG, "_lib", "liblfg.so")
HEADERS = [os.path.join(os.path.dirname(PKG), "include", h) for h in ("lfg.h", "lfg_kmc.h")]

LFG_OK, LFG_EINVAL, LFG_ECLOSURE, LFG_EDOMAIN, LFG_ECUDA, LFG_ENCCL, LFG_ENOMEM = range(7)


class LfgError(Exception):
    status = -1


class InvalidArgument(LfgError, ValueError):
    """std::invalid_argument in the reference."""
    status = LFG_EINVAL


class ClosureError(LfgError, RuntimeError):
    """std::runtime_error (closure violation, kpz.cpp:42-44)."""
    status = LFG_ECLOSURE


class DomainError(LfgError, ArithmeticError):
    """std::domain_error (no B particles, kmc.cpp:36-38)."""
    status = LFG_EDOMAIN


class CudaError(LfgError, RuntimeError):
    status = LFG_ECUDA


class TransportError(LfgError, RuntimeError):
    status = LFG_ENCCL


class DeviceOutOfMemory(LfgError, MemoryError):
    status = LFG_ENOMEM


_EXC = {LFG_EINVAL: InvalidArgument, LFG_ECLOSURE: ClosureError, LFG_EDOMAIN: DomainError,
        LFG_ECUDA: CudaError, LFG_ENCCL: TransportError, LFG_ENOMEM: DeviceOutOfMemory}


class Counters(C.Structure):
    """lf::Counters (counters.hpp:10-19) + deposit/detach split."""
    _fields_ = [("attempts", C.c_int64), ("successes", C.c_int64),
                ("deposits", C.c_int64), ("detaches", C.c_int64)]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}

    def __repr__(self) -> str:
        return f"Counters({self.as_dict()})"


class KpzPlan(C.Structure):
    """lfg_kpz_plan (include/lfg.h): block_x, block_y, sub (0 = defaults)."""
    _fields_ = [("block_x", C.c_int32), ("block_y", C.c_int32), ("sub", C.c_int32)]


class KmcPlan(C.Structure):
    """lfg_kmc_plan (include/lfg_kmc.h): block, sub (0 = defaults)."""
    _fields_ = [("block", C.c_int32), ("sub", C.c_int32)]


_lib = None


def _sig(lib, name, *args):
    f = getattr(lib, name)
    f.restype = C.c_int
    f.argtypes = list(args)


def lib() -> C.CDLL:
    """Load liblfg.so once (RTLD_GLOBAL so the CUDA runtime state is shared)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: the CUDA library must be built "
                          "(python -m paper_1204_5072_b200.build); there is no CPU fallback")
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I32, I64, U64, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
    L.lfg_last_error.restype = C.c_char_p
    L.lfg_last_error.argtypes = []
    _sig(L, "lfg_abi_version")
    _sig(L, "lfg_device_count", C.POINTER(C.c_int))
    # KPZ
    _sig(L, "lfg_kpz_create", C.POINTER(P), I32, D, D, U64, C.POINTER(KpzPlan), I32)
    _sig(L, "lfg_kpz_create_batch", C.POINTER(P), I32, D, D, C.POINTER(U64), I32, C.POINTER(KpzPlan), I32)
    _sig(L, "lfg_kpz_destroy", P)
    _sig(L, "lfg_kpz_get_plan", P, C.POINTER(KpzPlan))
    _sig(L, "lfg_kpz_init_flat", P)
    _sig(L, "lfg_kpz_upload", P, I32, P, P, SZ)
    _sig(L, "lfg_kpz_download", P, I32, P, P, SZ)
    _sig(L, "lfg_kpz_upload_async", P, I32, P, P, SZ)
    _sig(L, "lfg_kpz_upload_check", P)
    _sig(L, "lfg_kpz_download_async", P, I32, P, P, SZ)
    _sig(L, "lfg_kpz_width_sums_async", P, I32, P)
    _sig(L, "lfg_kpz_debug_record_anchors", P, P, SZ)
    _sig(L, "lfg_kpz_sweep", P, I64, C.POINTER(Counters))
    _sig(L, "lfg_kpz_sweep_async", P, I64)
    _sig(L, "lfg_kpz_phase", P, U64, I32)
    _sig(L, "lfg_kpz_counters", P, I32, C.POINTER(Counters))
    _sig(L, "lfg_kpz_reset_counters", P)
    _sig(L, "lfg_kpz_width_sums", P, I32, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kpz_interface_width", P, I32, C.POINTER(D))
    _sig(L, "lfg_kpz_heights", P, I32, P, SZ)
    _sig(L, "lfg_kpz_set_params", P, D, D)
    _sig(L, "lfg_kpz_set_sweep_index", P, U64)
    _sig(L, "lfg_kpz_get_sweep_index", P, C.POINTER(U64))
    _sig(L, "lfg_kpz_set_seed", P, I32, U64)
    _sig(L, "lfg_kpz_set_stream", P, P)
    _sig(L, "lfg_kpz_synchronize", P)
    _sig(L, "lfg_kpz_device_spins", P, I32, C.POINTER(P), C.POINTER(SZ))
    # strip-sharded path
    _sig(L, "lfg_kpz_create_strip", C.POINTER(P), I32, D, D, U64, C.POINTER(KpzPlan), I32)
    _sig(L, "lfg_kpz_sweep_origin", I32, C.POINTER(KpzPlan), U64, U64, C.POINTER(I32))
    _sig(L, "lfg_kpz_strip_phase", P, P, I32, I32, I32, U64, I32)
    _sig(L, "lfg_kpz_strip_phase_push", P, P, I32, I32, I32, U64, I32, P, I32, P, I32)
    _sig(L, "lfg_ipc_get_handle", P, P, C.POINTER(U64))
    _sig(L, "lfg_ipc_open_handle", P, I32, C.POINTER(P))
    _sig(L, "lfg_ipc_close", P, I32)
    _sig(L, "lfg_peer_signal", P, P, P, C.c_uint32, I32)
    _sig(L, "lfg_peer_wait", P, P, P, C.c_uint32, U64, P, I32)
    _sig(L, "lfg_copy_async", P, P, SZ, P, I32)
    _sig(L, "lfg_kpz_strip_fill", P, P, I32, I32, I32, I32)
    _sig(L, "lfg_kpz_strip_row0_heights", P, P, I32, P)
    _sig(L, "lfg_kpz_strip_width_partials", P, P, I32, I32, I32, I32, P, P, P)
    _sig(L, "lfg_kpz_width_combine", P, P, P, P, P, I32, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kpz_strip_width_rows", P, P, I32, I32, I32, C.POINTER(I64))
    # sharded lattice: one process, N GPUs (include/lfg.h)
    _sig(L, "lfg_kpz_create_sharded", C.POINTER(P), I32, D, D, U64, C.POINTER(KpzPlan), I32, C.POINTER(I32))
    _sig(L, "lfg_kpz_sharded_destroy", P)
    _sig(L, "lfg_kpz_sharded_init_flat", P)
    _sig(L, "lfg_kpz_sharded_upload", P, P, P, C.c_size_t)
    _sig(L, "lfg_kpz_sharded_download", P, P, P, C.c_size_t)
    _sig(L, "lfg_kpz_sharded_sweep", P, C.c_int64, C.POINTER(Counters))
    _sig(L, "lfg_kpz_sharded_counters", P, C.POINTER(Counters))
    _sig(L, "lfg_kpz_sharded_width_sums", P, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kpz_sharded_interface_width", P, C.POINTER(D))
    _sig(L, "lfg_kpz_sharded_set_sweep_index", P, U64)
    _sig(L, "lfg_kpz_sharded_get_sweep_index", P, C.POINTER(U64))
    _sig(L, "lfg_kmc_create_sharded", C.POINTER(P), I32, D, I32, U64, C.POINTER(KmcPlan), I32, C.POINTER(I32))
    _sig(L, "lfg_kmc_sharded_destroy", P)
    _sig(L, "lfg_kmc_sharded_init_random_alloy", P, D, U64)
    _sig(L, "lfg_kmc_sharded_upload", P, P, C.c_size_t)
    _sig(L, "lfg_kmc_sharded_download", P, P, C.c_size_t)
    _sig(L, "lfg_kmc_sharded_sweep", P, C.c_int64, C.POINTER(Counters))
    _sig(L, "lfg_kmc_sharded_counters", P, C.POINTER(Counters))
    _sig(L, "lfg_kmc_sharded_open_bond_sums", P, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kmc_sharded_open_bonds_per_particle", P, C.POINTER(D))
    _sig(L, "lfg_kmc_sharded_set_sweep_index", P, U64)
    _sig(L, "lfg_kmc_sharded_get_sweep_index", P, C.POINTER(U64))
    _sig(L, "lfg_kpz_set_abort_flag", P, P)
    # readouts of host lattices (no handle)
    _sig(L, "lfg_kpz_width_sums_host", I32, I32, P, P, SZ, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kpz_heights_host", I32, I32, P, P, SZ, P, SZ)
    _sig(L, "lfg_heights_width_sums_host", I32, P, SZ, C.POINTER(I64), C.POINTER(I64))
    _bind_kmc(L)
    _lib = L
    return L


def _bind_kmc(L) -> None:
    if not hasattr(L, "lfg_kmc_create"):
        return
    P, I32, I64, U64, D, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t
    _sig(L, "lfg_kmc_create", C.POINTER(P), I32, D, I32, U64, C.POINTER(KmcPlan), I32)
    _sig(L, "lfg_kmc_destroy", P)
    _sig(L, "lfg_kmc_get_plan", P, C.POINTER(KmcPlan))
    _sig(L, "lfg_kmc_upload", P, P, SZ)
    _sig(L, "lfg_kmc_download", P, P, SZ)
    _sig(L, "lfg_kmc_init_random_alloy", P, D, U64)
    _sig(L, "lfg_kmc_sweep", P, I64, C.POINTER(Counters))
    _sig(L, "lfg_kmc_sweep_async", P, I64)
    _sig(L, "lfg_kmc_phase", P, U64, I32)
    _sig(L, "lfg_kmc_counters", P, C.POINTER(Counters))
    _sig(L, "lfg_kmc_reset_counters", P)
    _sig(L, "lfg_kmc_open_bond_sums", P, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kmc_open_bonds_per_particle", P, C.POINTER(D))
    _sig(L, "lfg_kmc_open_bond_sums_host", I32, I32, P, SZ, C.POINTER(I64), C.POINTER(I64))
    _sig(L, "lfg_kmc_count_b", P, C.POINTER(I64))
    _sig(L, "lfg_kmc_set_params", P, D, I32)
    _sig(L, "lfg_kmc_set_sweep_index", P, U64)
    _sig(L, "lfg_kmc_get_sweep_index", P, C.POINTER(U64))
    _sig(L, "lfg_kmc_set_seed", P, U64)
    _sig(L, "lfg_kmc_set_stream", P, P)
    _sig(L, "lfg_kmc_set_concurrency", P, I32)
    _sig(L, "lfg_kmc_debug_record_writes", P, P, C.c_size_t)
    _sig(L, "lfg_kmc_set_abort_flag", P, P)
    _sig(L, "lfg_kmc_synchronize", P)
    _sig(L, "lfg_kmc_device_words", P, C.POINTER(P), C.POINTER(SZ))
    # z-slab sharded path
    _sig(L, "lfg_kmc_create_slab", C.POINTER(P), I32, D, I32, U64, C.POINTER(KmcPlan), I32)
    _sig(L, "lfg_kmc_sweep_origin", I32, C.POINTER(KmcPlan), U64, U64, C.POINTER(I32))
    _sig(L, "lfg_kmc_slab_phase", P, P, I32, I32, I32, U64, I32)
    _sig(L, "lfg_kmc_slab_init_random_alloy", P, P, I32, I32, I32, D, U64)
    _sig(L, "lfg_kmc_slab_open_bond_sums", P, P, I32, I32, I32, C.POINTER(I64), C.POINTER(I64))


def check(rc: int) -> None:
    if rc != LFG_OK:
        msg = lib().lfg_last_error().decode(errors="replace")
        raise _EXC.get(rc, LfgError)(msg)


def declared_symbols() -> list[str]:
    """Every function declared in include/*.h (for the export test)."""
    names: list[str] = []
    for h in HEADERS:
        if os.path.exists(h):
            names += re.findall(r"LFG_API\s+[\w\s\*]+?\b(lfg_\w+)\s*\(", open(h).read())
    return names


def device_count() -> int:
    n = C.c_int(0)
    check(lib().lfg_device_count(C.byref(n)))
    return int(n.value)
