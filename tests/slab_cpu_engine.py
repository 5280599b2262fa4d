"""CPU z-slab engine for the KMC sharded-driver tests -- TEST INFRASTRUCTURE ONLY.

Implements the interface of paper_1204_5072_b200.shard.CudaSlabEngine on a
CPU ring buffer of planes.  A phase expands the slab's planes (+-2 ghosts) of
the ring into a full-size scratch lattice and runs the oracle's DT phase
restricted to the rank's block z-rows (oracle/oracle.cpp,
orc_kmc_dt_phase_rows), so the multi-process driver (roll, ghost and
write-back plane exchanges over torch.distributed/gloo) runs without a GPU.
"""
from __future__ import annotations

import numpy as np
import torch

import pyoracle


class CpuSlabEngine:
    def __init__(self, plan, eps, both, seed, oracle: pyoracle.Oracle):
        self.plan, self.eps, self.both, self.seed, self.orc = plan, eps, both, seed, oracle
        self.buf = torch.zeros((plan.cap, plan.wpp), dtype=torch.int32)
        self.succ = 0

    def origin(self, plan, seed, sweep):
        return self.orc.kmc_sweep_draw(plan.L, plan.bk, seed, sweep)

    def rows(self, slot, n):
        return self.buf[slot:slot + n]

    def sync(self):
        pass

    def close(self):
        pass

    def _planes(self, z0, n):
        L, cap = self.plan.L, self.plan.cap
        return [((z0 + k) % L, ((z0 + k) % L) & (cap - 1)) for k in range(n)]

    def load_planes(self, words_u64, z0, n):
        full = np.asarray(words_u64).view(np.uint32).view(np.int32).reshape(self.plan.L, self.plan.wpp)
        for z, slot in self._planes(z0, n):
            self.buf[slot] = torch.from_numpy(full[z].copy())

    def _expand(self, z0, n):
        full = np.zeros((self.plan.L, self.plan.wpp), np.uint32)
        for z, slot in self._planes(z0, n):
            full[z] = self.buf[slot].numpy().view(np.uint32)
        return full

    def phase(self, sweep, phase, bz0, nbz):
        pl = self.plan
        oz = self.origin(pl, self.seed, sweep)[2]
        z0, n = oz + bz0 * pl.bk - 2, nbz * pl.bk + 4
        full = self._expand(z0, n)
        w = full.reshape(-1).view(np.uint64)
        c = self.orc.kmc_dt_phase_rows(pl.L, w, self.eps, self.both, self.seed, sweep, phase, pl.bk, bz0, nbz,
                                       getattr(pl, "sub", 1))
        self.succ += int(c[1])
        for z, slot in self._planes(z0, n):
            self.buf[slot] = torch.from_numpy(full[z].view(np.int32).copy())

    def successes(self):
        return self.succ

    def open_bond_sums(self, z0, n):
        full = self._expand(z0 - 1, n + 2)
        return self.orc.kmc_open_bond_sums_planes(self.plan.L, full.reshape(-1).view(np.uint64), z0, n)
