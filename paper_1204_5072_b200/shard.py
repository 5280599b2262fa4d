"""Strip-sharded KPZ DTr sweep across GPUs.

Partition.  With `world` ranks, H = L/world rows per rank, H a multiple of
2*block_y.  In sweep s (origin oy_s), rank g owns the rows
[oy_s + g H, oy_s + (g+1) H) (mod L) of the lattice -- exactly the block rows
[g H/by, (g+1) H/by) of the sweep's shifted frame -- so every device block of
every phase lives on one rank and the per-rank kernel is the single-GPU
kernel restricted to those block rows (lfg_kpz_strip_phase).

Storage.  Each rank holds a device ring buffer of C rows (power of two
>= H + 4 by + 2; C = L when world == 1): global row y sits at slot y & (C-1),
so the strip, its two ghost rows and the rows in flight during an ownership
roll never collide and nothing is ever shifted in memory.

Exchanges (the only collective traffic; all NCCL send/recv between ring
neighbours, one L/32-word row = 16 KiB at L = 2^17):
  * per sweep, the ownership roll: the origin moves by d = oy_s - oy_{s-1}
    in (-2 by, 2 by); |d| rows move to the neighbour on one side and |d|
    arrive from the other;
  * per phase, one ghost row: a phase of block-row parity sy reads exactly
    one row outside the strip -- the first row of rank g+1 (sy = 1) or the
    last row of rank g-1 (sy = 0) -- and no phase writes outside the strip.
The RNG is keyed on global tile/block ids of the shifted frame, so the
sharded trajectory is bit-identical to the single-GPU one for any world size
(tests/test_shard_gpu.py, tests/test_shard_cpu.py).

Execution back-ends (`comm`):
  * DistComm: torch.distributed point-to-point (NCCL over NVLink on B200,
    gloo on CPU for the world_size-2 tests);
  * LocalComm: all shards in one process (e.g. k shards on one GPU), rows
    copied directly -- used to prove bit-identity with a single device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native


def next_pow2(v: int) -> int:
    p = 1
    while p < v:
        p <<= 1
    return p


# ----------------------------------------------------------------------------- plan
@dataclass(frozen=True)
class StripPlan:
    L: int
    world: int
    bx: int
    by: int
    sub: int = 4  # sub-sweeps per MCS (include/lfg.h lfg_kpz_plan.sub); ownership rolls per sub-sweep

    def __post_init__(self):
        if self.L % self.world:
            raise ValueError("world must divide L")
        if self.world > 1 and self.H % (2 * self.by):
            raise ValueError(f"strip height L/world = {self.H} must be a multiple of 2*block_y = {2 * self.by}")

    @property
    def H(self) -> int:
        return self.L // self.world

    @property
    def cap(self) -> int:
        return self.L if self.world == 1 else min(self.L, next_pow2(self.H + 4 * self.by + 2))

    @property
    def wpr(self) -> int:
        return self.L // 32

    def start(self, oy: int, rank: int) -> int:
        return (oy + rank * self.H) % self.L

    def block_rows(self, rank: int):
        return rank * self.H // self.by, self.H // self.by

    def roll(self, oy_old: int, oy_new: int, rank: int):
        """Row moves when the origin goes from oy_old to oy_new:
        list of (kind, peer, row_begin, count)."""
        if self.world == 1 or oy_old == oy_new:
            return []
        d = oy_new - oy_old
        s = self.start(oy_old, rank)
        up, dn = (rank + 1) % self.world, (rank - 1) % self.world
        if d > 0:
            return [("send", dn, s, d), ("recv", up, s + self.H, d)]
        return [("send", up, s + self.H + d, -d), ("recv", dn, s + d, -d)]

    def ghost(self, oy: int, rank: int, sy: int):
        """The one ghost row a phase of block-row parity sy reads, refreshed."""
        if self.world == 1:
            return []
        s = self.start(oy, rank)
        up, dn = (rank + 1) % self.world, (rank - 1) % self.world
        if sy == 1:  # top block row active: needs row s+H (first row of rank+1)
            return [("send", dn, s, 1), ("recv", up, s + self.H, 1)]
        return [("send", up, s + self.H - 1, 1), ("recv", dn, s - 1, 1)]  # bottom: last row of rank-1

    def pieces(self, row_begin: int, count: int):
        """Split global rows [row_begin, +count) mod L into contiguous slot ranges
        of the ring buffer: list of (slot_begin, n)."""
        out = []
        y = row_begin % self.L
        left = count
        while left > 0:
            slot = y % self.cap
            n = min(left, self.cap - slot, self.L - y)
            out.append((slot, n))
            y = (y + n) % self.L
            left -= n
        return out

    def row_pieces_global(self, row_begin: int, count: int):
        """Split global rows into pieces that do not wrap past row L-1: (start, n)."""
        out = []
        y = row_begin % self.L
        left = count
        while left > 0:
            n = min(left, self.L - y)
            out.append((y, n))
            y = (y + n) % self.L
            left -= n
        return out


# ----------------------------------------------------------------------------- engines
class CudaStripEngine:
    """One rank's strip on a CUDA device: ring buffer (torch uint32 rows) +
    a strip handle of liblfg.so (lfg_kpz_create_strip)."""

    def __init__(self, plan: StripPlan, p: float, q: float, seed: int, device: int = 0):
        import torch

        self.plan = plan
        self.device = device
        self.torch = torch
        self.buf = torch.zeros((plan.cap, plan.wpr), dtype=torch.int32, device=f"cuda:{device}")
        lib = _native.lib()
        h = C.c_void_p()
        kp = _native.KpzPlan(plan.bx, plan.by, plan.sub)
        _native.check(lib.lfg_kpz_create_strip(C.byref(h), plan.L, float(p), float(q), int(seed), C.byref(kp),
                                               device))
        self.h = h
        self.stream = torch.cuda.Stream(device=device)
        # the zero fill above ran on torch's current stream; the library works on self.stream
        self.stream.wait_stream(torch.cuda.current_stream(device))
        _native.check(lib.lfg_kpz_set_stream(h, C.c_void_p(self.stream.cuda_stream)))

    def close(self):
        if self.h is not None:
            _native.lib().lfg_kpz_destroy(self.h)
            self.h = None

    def rows(self, slot: int, n: int):
        return self.buf[slot:slot + n]

    def sync(self):
        self.stream.synchronize()

    def set_abort_flag(self, ptr: int):
        _native.check(_native.lib().lfg_kpz_set_abort_flag(self.h, C.c_void_p(ptr) if ptr else None))

    def fill(self, row_begin: int, count: int, pattern: int):
        _native.check(_native.lib().lfg_kpz_strip_fill(self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap,
                                                       row_begin, count, pattern))

    def phase(self, sweep: int, phase: int, brow0: int, nbrow: int):
        _native.check(_native.lib().lfg_kpz_strip_phase(self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap,
                                                        brow0, nbrow, int(sweep), phase))

    def phase_push(self, sweep: int, phase: int, brow0: int, nbrow: int, peer_dn, row_dn: int, peer_up,
                   row_up: int):
        _native.check(_native.lib().lfg_kpz_strip_phase_push(
            self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap, brow0, nbrow, int(sweep), phase,
            C.c_void_p(peer_dn) if peer_dn else None, int(row_dn), C.c_void_p(peer_up) if peer_up else None,
            int(row_up)))

    def counters(self):
        c = _native.Counters()
        _native.check(_native.lib().lfg_kpz_counters(self.h, 0, C.byref(c)))
        return c

    def width_rows(self, row_begin: int, count: int):
        """(sum h_rel, sum h_rel^2, net column-0 step) of global rows
        [row_begin, +count) (no wrap), heights relative to the row below."""
        out = (C.c_int64 * 3)()
        _native.check(_native.lib().lfg_kpz_strip_width_rows(self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap,
                                                             row_begin, count, out))
        return int(out[0]), int(out[1]), int(out[2])


def sweep_origin(plan: StripPlan, seed: int, sweep: int):
    """(ox, oy, [set of phase 0..3]) of global sub-sweep `sweep` (= MCS * plan.sub + k)."""
    out = (C.c_int32 * 6)()
    kp = _native.KpzPlan(plan.bx, plan.by, plan.sub)
    _native.check(_native.lib().lfg_kpz_sweep_origin(plan.L, C.byref(kp), int(seed), int(sweep),
                                                     C.cast(out, C.POINTER(C.c_int32))))
    return int(out[0]), int(out[1]), [int(out[2 + k]) for k in range(4)]


# ----------------------------------------------------------------------------- comms
class LocalComm:
    """All shards in one process: ops are executed as direct row copies."""

    def __init__(self, engines):
        self.engines = engines
        self.world = len(engines)

    def exchange(self, ops_per_rank):
        # a send of rows [b, b+n) from rank r lands in the same global rows of `peer`
        for r, ops in enumerate(ops_per_rank):
            for kind, peer, b, n in ops:
                if kind != "send":
                    continue
                src, dst = self.engines[r], self.engines[peer]
                torch = dst.torch
                # on the destination engine's stream, after everything already
                # queued on both engines' streams
                with torch.cuda.stream(dst.stream):
                    dst.stream.wait_stream(src.stream)
                    for (slot, m) in src.plan.pieces(b, n):
                        dst.rows(slot, m).copy_(src.rows(slot, m))
                    src.stream.wait_stream(dst.stream)  # src rows not overwritten before the copy reads them
                dst.sync()


class DistComm:
    """torch.distributed point-to-point between ring neighbours (one shard per process)."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves CPU tensors only: device rows are staged through host
        # memory (used to exercise the distributed path with several ranks on
        # one GPU); NCCL sends device rows directly over NVLink.
        self.stage = dist.get_backend(group) == "gloo" and getattr(engine.buf, "is_cuda", False)

    def exchange(self, ops):
        """Post the matched sends/receives of this rank.  Device buffers over NCCL:
        the P2P ops are ordered after the work already on the engine's stream and
        the stream waits for them on the device (no host synchronisation), so the
        next phase kernel on that stream consumes the received rows in order.
        gloo with device buffers stages through host memory (synchronous)."""
        dist = self.dist
        e = self.engine
        if not ops:
            return
        on_device = getattr(e.buf, "is_cuda", False)
        if on_device and not self.stage:
            torch = e.torch
            with torch.cuda.stream(e.stream):
                p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, e.rows(slot, m), peer, self.group)
                       for kind, peer, b, n in ops for (slot, m) in e.plan.pieces(b, n)]
                for w in dist.batch_isend_irecv(p2p):
                    w.wait()  # stream-ordered wait on the engine's stream
            return
        e.sync()
        p2p, unstage = [], []
        for kind, peer, b, n in ops:
            for (slot, m) in e.plan.pieces(b, n):
                t = e.rows(slot, m)
                if self.stage:
                    h = t.cpu() if kind == "send" else t.new_empty(t.shape, device="cpu")
                    if kind == "recv":
                        unstage.append((t, h))
                    t = h
                p2p.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, t, peer, self.group))
        if p2p:
            for w in dist.batch_isend_irecv(p2p):
                w.wait()
        for t, h in unstage:
            t.copy_(h)
        if on_device:
            e.torch.cuda.current_stream(e.buf.device).synchronize()


class PeerComm(DistComm):
    """Single-node shard exchange over NVLink peer memory, without a collective
    library and without host synchronisation (one process per GPU).

    Each rank exports its ring buffer and a two-word step-flag array through CUDA
    IPC; neighbours open them once.  Rows move by peer copies on the engine's
    stream (rolls, readout ghosts) or -- in the sweep -- are stored straight into
    the neighbour's ring by the phase kernel's write-back
    (lfg_kpz_strip_phase_push), and a device-side step barrier
    (lfg_peer_signal / lfg_peer_wait: release/acquire flags in peer memory)
    orders each phase after both neighbours' previous phase.  torch.distributed
    (any backend) is used only at setup to swap the IPC handles and by the
    readouts' reductions.  A wait that never completes sets an error flag
    (checked after every sweep) instead of hanging."""

    fused_push = True

    def __init__(self, engine, group=None, max_spins: int = 1 << 24):
        super().__init__(engine, group)
        e = engine
        torch = e.torch
        lib = _native.lib()
        self.lib = lib
        self.device = e.buf.device.index or 0
        self.flags = torch.zeros(2, dtype=torch.int32, device=e.buf.device)  # [from lower, from upper]
        self.err = torch.zeros(1, dtype=torch.int32, device=e.buf.device)
        self.max_spins = int(max_spins)
        torch.cuda.current_stream(e.buf.device).synchronize()  # zero fills done before peers see the flags
        e.sync()
        # a neighbour that never arrives sets err (peer_wait); the engine's phase
        # kernels then skip instead of updating against stale ghost rows
        e.set_abort_flag(self.err.data_ptr())
        mine = []
        for t in (e.buf, self.flags):
            hd, off = (C.c_char * 64)(), C.c_uint64()
            _native.check(lib.lfg_ipc_get_handle(C.c_void_p(t.data_ptr()), hd, C.byref(off)))
            mine.append((bytes(hd), int(off.value)))
        allh = [None] * self.world
        self.dist.all_gather_object(allh, mine, group=self.group)
        self.up, self.dn = (self.rank + 1) % self.world, (self.rank - 1) % self.world
        self._opened, self._bases = {}, []
        for peer in {self.up, self.dn}:
            ptrs = []
            for hbytes, off in allh[peer]:
                p = C.c_void_p()
                _native.check(lib.lfg_ipc_open_handle(C.create_string_buffer(hbytes, 64), self.device, C.byref(p)))
                self._bases.append(int(p.value))
                ptrs.append(int(p.value) + off)
            self._opened[peer] = ptrs  # (ring buffer, flags)
        self.epoch = 0

    def close(self):
        if getattr(self.engine, "h", None) is not None:
            self.engine.set_abort_flag(0)  # self.err goes away with this object
        for p in self._bases:
            self.lib.lfg_ipc_close(C.c_void_p(p), self.device)
        self._opened, self._bases = {}, []

    def peer_ring(self, peer: int) -> int:
        return self._opened[peer][0]

    def step(self):
        """Device-side barrier with both neighbours (stream-ordered)."""
        self.epoch += 1
        st = C.c_void_p(self.engine.stream.cuda_stream)
        f_up = self._opened[self.up][1] + 0   # I am the upper neighbour's lower neighbour: its slot 0
        f_dn = self._opened[self.dn][1] + 4   # ... and the lower neighbour's upper neighbour: its slot 1
        _native.check(self.lib.lfg_peer_signal(st, C.c_void_p(f_up), C.c_void_p(f_dn), self.epoch, self.device))
        fl = self.flags.data_ptr()
        _native.check(self.lib.lfg_peer_wait(st, C.c_void_p(fl), C.c_void_p(fl + 4), self.epoch, self.max_spins,
                                             C.c_void_p(self.err.data_ptr()), self.device))

    def check(self):
        if int(self.err.item()) != 0:
            raise _native.TransportError("peer step barrier timed out (a neighbour did not arrive)")

    def exchange(self, ops):
        """Generic row exchange: barrier, my sends as peer copies into the
        receivers' rings (same slots), barrier."""
        if not ops:
            return
        e = self.engine
        st = C.c_void_p(e.stream.cuda_stream)
        row_bytes = e.buf.shape[1] * 4
        self.step()
        for kind, peer, b, n in ops:
            if kind != "send":
                continue
            base = self.peer_ring(peer)
            for (slot, m) in e.plan.pieces(b, n):
                _native.check(self.lib.lfg_copy_async(C.c_void_p(base + slot * row_bytes),
                                                      C.c_void_p(e.rows(slot, m).data_ptr()), m * row_bytes, st,
                                                      self.device))
        self.step()


# ----------------------------------------------------------------------------- driver
class ShardedKpz:
    """Strip-sharded lattice.  `engines` are this process's shards (all of them
    for LocalComm, exactly one for DistComm); `ranks` their global ranks."""

    def __init__(self, plan: StripPlan, seed: int, engines, ranks, comm):
        self.plan = plan
        self.seed = seed
        self.engines = list(engines)
        self.ranks = list(ranks)
        self.comm = comm
        self.sweep_index = 0
        self.oy = None  # origin the current row ownership refers to

    # ---- initial state -------------------------------------------------------
    def make_flat_slopes(self, sweep_index: int = 0):
        """Each rank fills its window for the first sweep's origin plus both ghosts
        (no communication)."""
        self.sweep_index = sweep_index
        _, oy, _ = sweep_origin(self.plan, self.seed, sweep_index * self.plan.sub)
        for e, r in zip(self.engines, self.ranks):
            e.fill(self.plan.start(oy, r) - 1, self.plan.H + 2, 0)
        for e in self.engines:
            e.sync()
        self.oy = oy

    # ---- sweeps --------------------------------------------------------------
    def _exchange(self, fn):
        if isinstance(self.comm, LocalComm):
            self.comm.exchange([fn(r) for r in self.ranks])
        else:
            self.comm.exchange(fn(self.ranks[0]))

    def sweep(self, n: int = 1):
        pl = self.plan
        if getattr(self.comm, "fused_push", False):
            return self._sweep_fused(n)
        for _ in range(n):
            for s in range(self.sweep_index * pl.sub, (self.sweep_index + 1) * pl.sub):  # sub-sweeps
                _, oy, sets = sweep_origin(pl, self.seed, s)
                if oy != self.oy:
                    old = self.oy
                    self._exchange(lambda r: pl.roll(old, oy, r))
                    self.oy = oy
                for k in range(4):
                    sy = sets[k] >> 1
                    self._exchange(lambda r: pl.ghost(oy, r, sy))
                    for e, r in zip(self.engines, self.ranks):
                        b0, nb = pl.block_rows(r)
                        e.phase(s, k, b0, nb)
            self.sweep_index += 1
        for e in self.engines:
            e.sync()

    def _sweep_fused(self, n: int):
        """Peer-memory sweep: per sweep the roll and a full refresh of both ghost
        rows (peer copies), then per phase one device-side step barrier and the
        phase kernel, whose write-back also stores the strip's first row into the
        lower neighbour's ring (sy = 0 phases, when that row changes) or its last
        row into the upper neighbour's ring (sy = 1)."""
        pl, comm = self.plan, self.comm
        e, r = self.engines[0], self.ranks[0]
        for _ in range(n):
            for s in range(self.sweep_index * pl.sub, (self.sweep_index + 1) * pl.sub):  # sub-sweeps
                _, oy, sets = sweep_origin(pl, self.seed, s)
                ops = []
                if oy != self.oy:
                    ops += pl.roll(self.oy, oy, r)
                    self.oy = oy
                comm.exchange(ops)
                comm.exchange(pl.ghost(oy, r, 0) + pl.ghost(oy, r, 1))
                first = pl.start(oy, r)
                last = (first + pl.H - 1) % pl.L
                b0, nb = pl.block_rows(r)
                for k in range(4):
                    sy = sets[k] >> 1
                    comm.step()
                    if sy == 0:
                        e.phase_push(s, k, b0, nb, comm.peer_ring(comm.dn), first, None, -1)
                    else:
                        e.phase_push(s, k, b0, nb, None, -1, comm.peer_ring(comm.up), last)
            self.sweep_index += 1
        comm.step()
        e.sync()
        comm.check()

    def counters_local(self):
        tot = [0, 0]
        for e in self.engines:
            c = e.counters()
            tot[0] += c.deposits
            tot[1] += c.detaches
        return tot

    # ---- readout -------------------------------------------------------------
    def owned_pieces(self, rank: int):
        return self.plan.row_pieces_global(self.plan.start(self.oy, rank), self.plan.H)

    def gather_rows(self):
        """Full lattice of spin rows as one CPU int32 tensor [L, L/32].  With
        DistComm every rank contributes its owned rows (all_reduce of disjoint
        row sets); with LocalComm the shards are read directly."""
        import torch

        L, wpr = self.plan.L, self.plan.wpr
        out = torch.zeros((L, wpr), dtype=torch.int32)
        for e, r in zip(self.engines, self.ranks):
            e.sync()
            for (a, n) in self.owned_pieces(r):
                y = a
                for (slot, m) in self.plan.pieces(a, n):
                    out[y:y + m] = e.rows(slot, m).cpu()
                    y += m
        if isinstance(self.comm, DistComm):
            dist = self.comm.dist
            dev = "cpu" if self.comm.stage else self.engines[0].buf.device
            t = out.to(dev)
            # rows are disjoint across ranks: XOR-free sum of int32 words is exact
            # only without overflow, so reduce as int64 halves
            lo = (t & 0xFFFF).to(torch.int64)
            hi = ((t >> 16) & 0xFFFF).to(torch.int64)
            dist.all_reduce(lo, group=self.comm.group)
            dist.all_reduce(hi, group=self.comm.group)
            out = ((hi << 16) | lo).to(torch.int32).cpu()
        return out

    def width_sums(self):
        """interface_width sums (kpz.cpp:62-81) of the sharded lattice: exact
        (sum h, sum h^2) with h(0,0) = 0.  Every rank scans its owned rows in row
        order (lfg_kpz_strip_width_rows: heights relative to the column-0 height
        of the row below each piece) and the pieces are chained in global row
        order from row 0:  sum h += s1 + n L B,  sum h^2 += s2 + 2 B s1 + n L B^2,
        B += D.  Only (start, rows, s1, s2, D) per piece crosses ranks."""
        pl = self.plan
        # each piece reads the row below it (s_y of its first column-0 site)
        for sy in (0, 1):
            self._exchange(lambda r: pl.ghost(self.oy, r, sy))
        pieces = []
        for e, r in zip(self.engines, self.ranks):
            for (a, n) in self.owned_pieces(r):
                s1, s2, d = e.width_rows(a, n)
                pieces.append((a, n, s1, s2, d))
        if isinstance(self.comm, DistComm):
            allp = [None] * self.comm.world
            self.comm.dist.all_gather_object(allp, pieces, group=self.comm.group)
            pieces = [t for lst in allp for t in lst]
        pieces.sort(key=lambda t: t[0])
        assert pieces and pieces[0][0] == 0 and sum(t[1] for t in pieces) == pl.L
        S1 = S2 = B = 0
        for (_, n, s1, s2, d) in pieces:
            m = n * pl.L
            S1 += s1 + m * B
            S2 += s2 + 2 * B * s1 + m * B * B
            B += d
        return S1, S2

    def interface_width(self) -> float:
        s, s2 = self.width_sums()
        n = float(self.plan.L * self.plan.L)  # kpz.cpp:78-80
        mean = s / n
        return s2 / n - mean * mean


# ============================================================================= KMC z-slabs
# the 3-D lattice is cut into z-slabs of H = L/world
# planes, H a multiple of 2*bk, so the block z-rows on either side of a slab
# boundary are never active in the same phase.  In sweep s (origin oz_s) rank g
# owns planes [oz_s + g H, oz_s + (g+1) H) (mod L) = block z-rows
# [g H/bk, (g+1) H/bk) of the shifted frame.  Reach (kmc.hpp:140-141): a phase
# reads two planes beyond the slab and writes one beyond it, so around each
# phase of z-parity sz:
#   * before: the two ghost planes on the active side are refreshed from the
#     neighbour that owns them;
#   * after: the one ghost plane the phase may have modified goes back to its
#     owner (whose own blocks next to it were inactive in that phase).
# Per sweep the ownership rolls with oz exactly as for the KPZ strips.  Plane
# traffic per boundary: 2 planes in + 1 plane back per phase (128 KiB each at
# L = 1024), plus < 2 bk planes per sweep for the roll.
@dataclass(frozen=True)
class SlabPlan:
    L: int
    world: int
    bk: int
    sub: int = 1  # sub-sweeps per MCS (include/lfg_kmc.h lfg_kmc_plan.sub); ownership rolls per sub-sweep

    def __post_init__(self):
        if self.L % self.world:
            raise ValueError("world must divide L")
        if self.world > 1 and self.H % (2 * self.bk):
            raise ValueError(f"slab height L/world = {self.H} must be a multiple of 2*block = {2 * self.bk}")

    @property
    def H(self) -> int:
        return self.L // self.world

    @property
    def cap(self) -> int:
        return self.L if self.world == 1 else min(self.L, next_pow2(self.H + 4 * self.bk + 4))

    @property
    def wpp(self) -> int:  # uint32 words per plane
        return self.L * self.L // 32

    def start(self, oz: int, rank: int) -> int:
        return (oz + rank * self.H) % self.L

    def block_rows(self, rank: int):
        return rank * self.H // self.bk, self.H // self.bk

    def roll(self, oz_old: int, oz_new: int, rank: int):
        if self.world == 1 or oz_old == oz_new:
            return []
        d = oz_new - oz_old
        s = self.start(oz_old, rank)
        up, dn = (rank + 1) % self.world, (rank - 1) % self.world
        if d > 0:
            return [("send", dn, s, d), ("recv", up, s + self.H, d)]
        return [("send", up, s + self.H + d, -d), ("recv", dn, s + d, -d)]

    def ghost(self, oz: int, rank: int, sz: int, depth: int = 2):
        """Refresh the `depth` planes beyond the slab on side sz (1: above, 0: below)."""
        if self.world == 1:
            return []
        s = self.start(oz, rank)
        up, dn = (rank + 1) % self.world, (rank - 1) % self.world
        if sz == 1:
            return [("send", dn, s, depth), ("recv", up, s + self.H, depth)]
        return [("send", up, s + self.H - depth, depth), ("recv", dn, s - depth, depth)]

    def writeback(self, oz: int, rank: int, sz: int):
        """Return the ghost plane a phase of z-parity sz may have written to its owner."""
        if self.world == 1:
            return []
        s = self.start(oz, rank)
        up, dn = (rank + 1) % self.world, (rank - 1) % self.world
        if sz == 1:
            return [("send", up, s + self.H, 1), ("recv", dn, s, 1)]
        return [("send", dn, s - 1, 1), ("recv", up, s + self.H - 1, 1)]

    def pieces(self, z_begin: int, count: int):
        """Split global planes [z_begin, +count) mod L into ring-slot ranges (slot, n)."""
        out = []
        z = z_begin % self.L
        left = count
        while left > 0:
            slot = z % self.cap
            n = min(left, self.cap - slot, self.L - z)
            out.append((slot, n))
            z = (z + n) % self.L
            left -= n
        return out

    def plane_pieces_global(self, z_begin: int, count: int):
        out = []
        z = z_begin % self.L
        left = count
        while left > 0:
            n = min(left, self.L - z)
            out.append((z, n))
            z = (z + n) % self.L
            left -= n
        return out


class CudaSlabEngine:
    """One rank's z-slab on a CUDA device: a ring buffer of planes (torch int32
    [cap, L*L/32]) + a slab handle of liblfg.so (lfg_kmc_create_slab)."""

    def __init__(self, plan: SlabPlan, eps: float, both: bool, seed: int, device: int = 0):
        import torch

        self.plan = plan
        self.torch = torch
        self.buf = torch.zeros((plan.cap, plan.wpp), dtype=torch.int32, device=f"cuda:{device}")
        lib = _native.lib()
        h = C.c_void_p()
        kp = _native.KmcPlan(plan.bk, plan.sub)
        _native.check(lib.lfg_kmc_create_slab(C.byref(h), plan.L, float(eps), int(bool(both)), int(seed),
                                              C.byref(kp), device))
        self.h = h
        self.stream = torch.cuda.Stream(device=device)
        self.stream.wait_stream(torch.cuda.current_stream(device))  # after the zero fill of buf
        _native.check(lib.lfg_kmc_set_stream(h, C.c_void_p(self.stream.cuda_stream)))

    def close(self):
        if self.h is not None:
            _native.lib().lfg_kmc_destroy(self.h)
            self.h = None

    def rows(self, slot: int, n: int):
        return self.buf[slot:slot + n]

    def sync(self):
        self.stream.synchronize()

    def set_abort_flag(self, ptr: int):
        _native.check(_native.lib().lfg_kmc_set_abort_flag(self.h, C.c_void_p(ptr) if ptr else None))

    def init_random_alloy(self, z_begin: int, count: int, c: float, seed: int):
        _native.check(_native.lib().lfg_kmc_slab_init_random_alloy(
            self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap, z_begin, count, float(c), int(seed)))

    def load_planes(self, words_u64, z_begin: int, count: int):
        """Copy global planes [z_begin, +count) of a host lattice (uint64 words) into the ring."""
        import numpy as np

        full = np.asarray(words_u64).view(np.uint32).view(np.int32).reshape(self.plan.L, self.plan.wpp)
        with self.torch.cuda.stream(self.stream):  # ordered with the library's kernels
            for (z, n) in self.plan.plane_pieces_global(z_begin, count):
                for (slot, m) in self.plan.pieces(z, n):
                    self.buf[slot:slot + m].copy_(self.torch.from_numpy(full[z:z + m].copy()))
                    z += m

    def phase(self, sweep: int, phase: int, bz0: int, nbz: int):
        _native.check(_native.lib().lfg_kmc_slab_phase(self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap,
                                                       bz0, nbz, int(sweep), phase))

    def successes(self) -> int:
        c = _native.Counters()
        _native.check(_native.lib().lfg_kmc_counters(self.h, C.byref(c)))
        return int(c.successes)

    def open_bond_sums(self, z_begin: int, count: int):
        a, b = C.c_int64(), C.c_int64()
        _native.check(_native.lib().lfg_kmc_slab_open_bond_sums(
            self.h, C.c_void_p(self.buf.data_ptr()), self.plan.cap, z_begin, count, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)


def kmc_sweep_origin(plan: SlabPlan, seed: int, sweep: int):
    """(ox, oy, oz, [set of phase 0..7]) of global sub-sweep `sweep` (= MCS * plan.sub + k)."""
    out = (C.c_int32 * 11)()
    kp = _native.KmcPlan(plan.bk, plan.sub)
    _native.check(_native.lib().lfg_kmc_sweep_origin(plan.L, C.byref(kp), int(seed), int(sweep),
                                                     C.cast(out, C.POINTER(C.c_int32))))
    return int(out[0]), int(out[1]), int(out[2]), [int(out[3 + k]) for k in range(8)]


class ShardedKmc:
    """z-slab-sharded KMC lattice (SlabPlan); `engines`/`ranks`/`comm` as for
    ShardedKpz.  `origin` maps (plan, seed, sweep) to (ox, oy, oz, order); it
    defaults to the library's draw (tests may pass the oracle's)."""

    def __init__(self, plan: SlabPlan, seed: int, engines, ranks, comm, origin=None):
        self.plan = plan
        self.seed = seed
        self.engines = list(engines)
        self.ranks = list(ranks)
        self.comm = comm
        self.origin = origin or kmc_sweep_origin
        self.sweep_index = 0
        self.oz = None

    def _exchange(self, fn):
        if isinstance(self.comm, LocalComm):
            self.comm.exchange([fn(r) for r in self.ranks])
        else:
            self.comm.exchange(fn(self.ranks[0]))

    def _window(self, rank):
        return self.plan.start(self.oz, rank) - 2, self.plan.H + 4  # owned planes + two ghosts per side

    # ---- initial state (no communication: the init is position-keyed) ------
    def make_random_alloy(self, c: float, alloy_seed: int, sweep_index: int = 0):
        self.sweep_index = sweep_index
        self.oz = self.origin(self.plan, self.seed, sweep_index * self.plan.sub)[2]
        for e, r in zip(self.engines, self.ranks):
            z, n = self._window(r)
            e.init_random_alloy(z, n, c, alloy_seed)
        for e in self.engines:
            e.sync()

    def upload(self, words_u64, sweep_index: int = 0):
        """Every rank takes its window of a full host lattice (reference word layout)."""
        self.sweep_index = sweep_index
        self.oz = self.origin(self.plan, self.seed, sweep_index * self.plan.sub)[2]
        for e, r in zip(self.engines, self.ranks):
            z, n = self._window(r)
            e.load_planes(words_u64, z, n)
        for e in self.engines:
            e.sync()

    # ---- sweeps ------------------------------------------------------------
    def sweep(self, n: int = 1):
        pl = self.plan
        for _ in range(n):
            for s in range(self.sweep_index * pl.sub, (self.sweep_index + 1) * pl.sub):  # sub-sweeps
                _, _, oz, order = self.origin(pl, self.seed, s)
                if oz != self.oz:
                    old = self.oz
                    self._exchange(lambda r: pl.roll(old, oz, r))
                    self.oz = oz
                for k in range(8):
                    sz = order[k] >> 2
                    self._exchange(lambda r: pl.ghost(oz, r, sz, 2))
                    for e, r in zip(self.engines, self.ranks):
                        b0, nb = pl.block_rows(r)
                        e.phase(s, k, b0, nb)
                    self._exchange(lambda r: pl.writeback(oz, r, sz))
            self.sweep_index += 1
        for e in self.engines:
            e.sync()

    def _allreduce(self, vals):
        if isinstance(self.comm, DistComm):
            import torch

            t = torch.tensor(vals, dtype=torch.int64)
            if not self.comm.stage and self.engines[0].buf.is_cuda:
                t = t.to(self.engines[0].buf.device)
            self.comm.dist.all_reduce(t, group=self.comm.group)
            return [int(v) for v in t.cpu().tolist()]
        return vals

    def successes(self) -> int:
        return self._allreduce([sum(e.successes() for e in self.engines)])[0]

    # ---- readout -----------------------------------------------------------
    def owned_pieces(self, rank: int):
        return self.plan.plane_pieces_global(self.plan.start(self.oz, rank), self.plan.H)

    def open_bond_sums(self):
        """open_bonds_per_particle (kmc.cpp:20-40) sums over the whole lattice."""
        pl = self.plan
        for sz in (0, 1):
            self._exchange(lambda r: pl.ghost(self.oz, r, sz, 1))
        np_, no = 0, 0
        for e, r in zip(self.engines, self.ranks):
            for (z, n) in self.owned_pieces(r):
                a, b = e.open_bond_sums(z, n)
                np_ += a
                no += b
        return tuple(self._allreduce([np_, no]))

    def gather_planes(self):
        """Full lattice as a CPU int32 tensor [L, L*L/32] (owned planes of every rank)."""
        import torch

        L, wpp = self.plan.L, self.plan.wpp
        out = torch.zeros((L, wpp), dtype=torch.int32)
        for e, r in zip(self.engines, self.ranks):
            e.sync()
            for (a, n) in self.owned_pieces(r):
                z = a
                for (slot, m) in self.plan.pieces(a, n):
                    out[z:z + m] = e.rows(slot, m).cpu()
                    z += m
        if isinstance(self.comm, DistComm):
            dist = self.comm.dist
            dev = "cpu" if self.comm.stage else self.engines[0].buf.device
            t = out.to(dev)
            lo = (t & 0xFFFF).to(torch.int64)
            hi = ((t >> 16) & 0xFFFF).to(torch.int64)
            dist.all_reduce(lo, group=self.comm.group)
            dist.all_reduce(hi, group=self.comm.group)
            out = ((hi << 16) | lo).to(torch.int32).cpu()
        return out
