"""CPU strip engine for the sharded-driver tests -- TEST INFRASTRUCTURE ONLY.

A pure-Python restatement of one DT phase of the KPZ kernel
on a ring buffer of spin rows, with the interface of
paper_1204_5072_b200.shard.CudaStripEngine, so the multi-process driver
(roll + ghost exchange over torch.distributed/gloo) can run without a GPU.
Philox comes from the oracle restatement (oracle/_build/liboracle.so).
"""
from __future__ import annotations

import numpy as np
import torch

import pyoracle

TAG_SWEEP, TAG_SET, TAG_ANCHOR, TAG_ACCEPT = 1, 2, 3, 4


class CpuStripEngine:
    def __init__(self, plan, p, q, seed, oracle: pyoracle.Oracle):
        self.plan, self.p, self.q, self.seed, self.orc = plan, p, q, seed, oracle
        self.buf = torch.zeros((plan.cap, plan.wpr), dtype=torch.int32)
        self.dep = 0
        self.det = 0
        self.thrP = self._thr(p)
        self.thrQ = self._thr(q)

    @staticmethod
    def _thr(x):
        import math

        return 0 if x <= 0 else (1 << 32 if x >= 1 else math.ceil(x * 4294967296.0))

    def draw(self, sweep, tag, c0, c1):
        ctr = [c0 & 0xFFFFFFFF, c1 & 0xFFFFFFFF, sweep & 0xFFFFFFFF, (tag << 24) | ((sweep >> 32) & 0xFFFFFF)]
        key = [self.seed & 0xFFFFFFFF, (self.seed >> 32) & 0xFFFFFFFF]
        return [int(v) for v in self.orc.philox(ctr, key)]

    def rows(self, slot, n):
        return self.buf[slot:slot + n]

    def sync(self):
        pass

    def close(self):
        pass

    def fill(self, row_begin, count, pattern):
        pats = [0x66666666, 0x99999999, 0x99999999, 0x66666666] if pattern == 0 else \
               [0xAAAAAAAA, 0x55555555, 0xAAAAAAAA, 0x55555555]
        L, cap = self.plan.L, self.plan.cap
        for k in range(count):
            y = (row_begin + k) % L
            self.buf[y & (cap - 1)] = torch.tensor(np.full(self.plan.wpr, pats[y & 3], np.uint32).view(np.int32))

    def counters(self):
        class C:
            pass

        c = C()
        c.deposits, c.detaches = self.dep, self.det
        return c

    def width_rows(self, row_begin, count):
        """Row-order W^2 piece (the contract of lfg_kpz_strip_width_rows):
        (sum h_rel, sum h_rel^2, D) over global rows [row_begin, +count), heights
        relative to the column-0 height of the row below (0 at global row 0)."""
        L, cap = self.plan.L, self.plan.cap
        w = self.buf.numpy().view(np.uint32)
        s1 = s2 = 0
        V = 0
        for k in range(count):
            g = (row_begin + k) % L
            bits = np.unpackbits(w[g & (cap - 1)].view(np.uint8), bitorder="little").astype(np.int64)
            if g != 0:
                below = int(w[((g - 1) % L) & (cap - 1), 0]) & 1
                V += 1 if int(bits[0]) == below else -1
            steps = np.where(bits[1:] == bits[:-1], 1, -1)
            h = V + np.concatenate([[0], np.cumsum(steps)])
            s1 += int(h.sum())
            s2 += int((h * h).sum())
        return s1, s2, V

    # ---- one phase -------------------------------------------------------------
    def phase(self, sweep, k, brow0, nbrow):
        pl = self.plan
        L, cap, bx, by = pl.L, pl.cap, pl.bx, pl.by
        w = self.buf.numpy().view(np.uint32)
        W = self.draw(sweep, TAG_SWEEP, 0, 0)
        qx = 128 if bx >= 64 else 32  # x-origin quantum (lfg_common.cuh kpz_ox_quantum)
        ox = qx * ((W[0] * (2 * bx // qx)) >> 32)
        oy = (W[1] * 2 * by) >> 32
        sub = getattr(pl, "sub", 4)
        rounds = {1: 512, 4: 132, 8: 68}[sub]
        perm = self.orc.kpz_sweep_draw(L, bx, by, self.seed, sweep)[2:]
        st = int(perm[k])
        sx, sy = st & 1, st >> 1
        twx, thy = bx // 32, by // 16

        def get(i, j):
            i %= L
            j %= L
            return (int(w[j & (cap - 1), i >> 5]) >> (i & 31)) & 1

        for byi in range(brow0 + sy, brow0 + nbrow, 2):
            for bxi in range(sx, L // bx, 2):
                block_id = byi * (L // bx) + bxi
                anc = {}
                smask = {}
                sw = None
                for r in range(rounds):
                    if r % 64 == 0:
                        sw = self.draw(sweep, TAG_SET, block_id, r >> 6)
                    inner = (sw[(r >> 4) & 3] >> (2 * (r & 15))) & 3
                    hx, hy = inner & 1, inner >> 1
                    for ty in range(thy):
                        for tx in range(twx):
                            gx, gy = bxi * twx + tx, byi * thy + ty
                            tid = gy * (L // 32) + gx
                            if r % 16 == 0:
                                anc[tid] = self.draw(sweep, TAG_ANCHOR, tid, r >> 4)
                            a4 = anc[tid]
                            if r == 0:  # sub = 4 / 8: Poisson attempt count via skipped 4-round groups
                                v = (a4[2] & 0xFF) | ((a4[3] & 0xFF) << 8)
                                tails = (7701, 471, 19, 1) if sub == 4 else (14497, 1735, 143, 9)
                                K = sum(v >= 65536 - t for t in tails)
                                rep_ = 0x11111111 if sub == 4 else 0x1111
                                smask[tid] = [0x0, 0x8, 0xA, 0xE, 0xF][K] * rep_ if sub != 1 else 0
                            if r < 128 and (smask[tid] >> (r >> 2)) & 1:
                                continue
                            kk, h = r & 15, (r >> 3) & 1
                            xd = (a4[h] >> (28 - 4 * (kk & 7))) & 15
                            yd = (a4[2 + h] >> (29 - 3 * (kk & 7))) & 7
                            i = (ox + 32 * gx + 16 * hx + xd) % L
                            j = (oy + 16 * gy + 8 * hy + yd) % L
                            S = get(i, j)
                            R, U, Lf, D = get(i + 1, j), get(i, j + 1), get(i - 1, j), get(i, j - 1)
                            dep = R == S and U == S and Lf != S and D != S
                            det = R != S and U != S and Lf == S and D == S
                            if not (dep or det):
                                continue
                            thr = self.thrP if dep else self.thrQ
                            if thr == 0:
                                continue
                            if thr < (1 << 32) and not self.draw(sweep, TAG_ACCEPT, tid, r >> 2)[r & 3] < thr:
                                continue
                            w[j & (cap - 1), i >> 5] ^= np.uint32(1 << (i & 31))
                            self.dep += dep
                            self.det += det


def spins_to_slopes(f: np.ndarray, L: int):
    """[L, L/32] uint32 spin rows -> reference SlopeField planes (uint64 words)."""
    bits = np.unpackbits(f.view(np.uint8), bitorder="little").reshape(L, L).astype(np.uint8)
    left = np.roll(bits, 1, axis=1)
    down = np.roll(bits, 1, axis=0)
    sx = (1 - (bits ^ left)).astype(np.uint8)
    sy = (1 - (bits ^ down)).astype(np.uint8)
    px = np.packbits(sx.reshape(-1), bitorder="little").view(np.uint64)
    py = np.packbits(sy.reshape(-1), bitorder="little").view(np.uint64)
    return px, py
