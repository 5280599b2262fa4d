"""Experiment runner and time-series CSV ("harness").

The reference specifies (but does not implement) a harness that runs a model for a duration,
samples observables on a schedule and writes CSV rows
``t, observable_name, value, attempts, successes, wall_ms, realization_id`` preceded by
``#``-prefixed config-echo lines.  This module is that harness over the
B200 path: KPZ two-layer DTr (observable W², plus ⟨h⟩ = -1 + 2 (dep - det) / L²) and KMC
two-layer DT (observable open bonds per particle).  Realizations run as independent
lattices with seeds ``seed + r``, several at once on their own CUDA streams
(``concurrency``, CLI ``--concurrency``); wall time is measured around the update calls
only.  There is no CPU scheduler here: the CLI's ``--scheduler`` accepts the
two-layer DT schedule the device implements.
"""
from __future__ import annotations

import csv
import io
import time
from dataclasses import asdict, dataclass, field
from typing import List, Optional

from . import InvalidArgument, KmcLattice, KpzLattice

CSV_COLUMNS = ("t", "observable_name", "value", "attempts", "successes", "wall_ms", "realization_id")


@dataclass
class ExperimentConfig:
    """ExperimentConfig."""
    model: str                      # "kpz" | "kmc"
    size: int
    mcs: int
    seed: int = 1
    realizations: int = 1
    samples: Optional[List[int]] = None  # sample times (MCS); default: 0, round(1.1^k), mcs
    # KPZ
    p: float = 1.0
    q: float = 0.0
    block_x: int = 0
    block_y: int = 0
    sub: int = 0          # KPZ sub-sweeps per MCS (0: plan default 4; 1: the paper's scheme)
    # KMC
    conc: float = 0.5
    eps: float = 1.5
    both_active: bool = False
    block: int = 0
    alloy_seed: Optional[int] = None
    device: int = 0
    concurrency: int = 8            # realizations in flight at once (own streams)
    extra: dict = field(default_factory=dict)

    def validate(self) -> None:
        if self.model not in ("kpz", "kmc"):
            raise InvalidArgument(f"model must be kpz or kmc, got {self.model!r}")
        if self.size < 4 or self.size & (self.size - 1):
            raise InvalidArgument(f"size must be a power of two >= 4, got {self.size}")
        if self.mcs < 0:
            raise InvalidArgument("mcs must be >= 0")
        if self.realizations < 1:
            raise InvalidArgument("realizations must be >= 1")
        if self.concurrency < 1:
            raise InvalidArgument("concurrency must be >= 1")
        if self.model == "kmc" and not (0.0 <= self.conc <= 1.0):
            raise InvalidArgument("conc must lie in [0, 1]")

    def sample_times(self) -> List[int]:
        if self.samples is not None:
            ts = sorted({int(t) for t in self.samples if 0 <= int(t) <= self.mcs} | {self.mcs})
        else:
            ts = sorted({0, self.mcs} | {int(round(1.1 ** k)) for k in range(400) if round(1.1 ** k) <= self.mcs})
        return ts


@dataclass
class Row:
    t: int
    observable_name: str
    value: float
    attempts: int
    successes: int
    wall_ms: float
    realization_id: int


def _kpz_open(cfg: ExperimentConfig, r: int) -> KpzLattice:
    k = KpzLattice(cfg.size, cfg.p, cfg.q, cfg.seed + r, block_x=cfg.block_x, block_y=cfg.block_y,
                   sub=cfg.sub, device=cfg.device)
    k.make_flat_slopes()
    return k


def _kpz_observe(cfg: ExperimentConfig, k: KpzLattice):
    L = cfg.size
    c = k.counters()
    succ = c.deposits + c.detaches
    return succ, int(c.attempts), [("W2", k.interface_width()),
                                   ("mean_height", -1.0 + 2.0 * (c.deposits - c.detaches) / (L * L))]


def _kmc_open(cfg: ExperimentConfig, r: int) -> KmcLattice:
    k = KmcLattice(cfg.size, cfg.eps, cfg.both_active, cfg.seed + r, block=cfg.block, device=cfg.device)
    k.make_random_alloy(cfg.conc, (cfg.alloy_seed if cfg.alloy_seed is not None else cfg.seed) + 7919 * r)
    return k


def _kmc_observe(cfg: ExperimentConfig, k: KmcLattice):
    c = k.counters()
    return c.successes, int(c.attempts), [("open_bonds_per_particle", k.open_bonds_per_particle())]


def _run_batch(cfg: ExperimentConfig, rids: List[int]) -> List[Row]:
    """Realizations `rids` side by side: every lattice has its own CUDA stream, so one
    interval's sweeps of all of them are in flight together (a 256^3 KMC phase fills a
    ninth of the GPU; several realizations fill it).  Wall time: from issuing the
    interval's sweeps to the last one finishing, attributed equally to the realizations."""
    kpz = cfg.model == "kpz"
    opener, observe = (_kpz_open, _kpz_observe) if kpz else (_kmc_open, _kmc_observe)
    lats = []
    try:
        for r in rids:
            lats.append(opener(cfg, r))
            if not kpz and len(rids) > 1:
                lats[-1].set_concurrency(len(rids))
        out = {r: [] for r in rids}
        t, wall = 0, 0.0
        for ts in cfg.sample_times():
            if ts > t:
                t0 = time.perf_counter()
                if len(lats) == 1:
                    lats[0].sweep_async(ts - t)
                else:  # round-robin, one MCS at a time, so all streams stay fed
                    for _ in range(ts - t):
                        for k in lats:
                            k.sweep_async(1)
                for k in lats:
                    k.synchronize()
                wall += (time.perf_counter() - t0) * 1e3 / len(lats)
                t = ts
            for r, k in zip(rids, lats):
                succ, att, obs = observe(cfg, k)  # device counters: attempts actually made
                out[r].extend(Row(t, name, v, att, succ, wall, r) for name, v in obs)
        return [row for r in rids for row in out[r]]
    finally:
        for k in lats:
            k.close()


def run_experiment(cfg: ExperimentConfig) -> List[Row]:
    """run_experiment: every realization's time series, in order.
    Realizations run in concurrent batches of ``cfg.concurrency`` lattices (1: one after
    another); the lattices and their series do not depend on the batching."""
    cfg.validate()
    rows: List[Row] = []
    step = max(1, int(cfg.concurrency))
    for r0 in range(0, cfg.realizations, step):
        rows.extend(_run_batch(cfg, list(range(r0, min(cfg.realizations, r0 + step)))))
    return rows


def throughput(rows: List[Row]) -> dict:
    """ThroughputReport: attempts per wall-second of the update calls."""
    last = {}
    for row in rows:
        last[row.realization_id] = row
    att = sum(r.attempts for r in last.values())
    wall = sum(r.wall_ms for r in last.values()) / 1e3
    return {"attempts": att, "update_seconds": wall, "updates_per_second": att / wall if wall > 0 else None}


def write_csv(cfg: ExperimentConfig, rows: List[Row], out) -> None:
    """CSV with a '#'-prefixed config echo and the fixed header."""
    for k, v in asdict(cfg).items():
        if k != "extra":
            out.write(f"# {k}: {v}\n")
    w = csv.writer(out, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for r in rows:
        w.writerow([r.t, r.observable_name, repr(float(r.value)), r.attempts, r.successes, f"{r.wall_ms:.3f}",
                    r.realization_id])


def read_csv(text: str):
    """Parse a harness CSV back into (config dict, rows) -- the round-trip property of SPEC.md:484."""
    meta, body = {}, []
    for ln in text.splitlines():
        if ln.startswith("# "):
            k, _, v = ln[2:].partition(": ")
            meta[k] = v
        elif ln.strip():
            body.append(ln)
    rd = csv.reader(io.StringIO("\n".join(body)))
    header = next(rd)
    if tuple(header) != CSV_COLUMNS:
        raise ValueError(f"unexpected CSV header {header}")
    rows = [Row(int(a), b, float(c), int(d), int(e), float(f), int(g)) for a, b, c, d, e, f, g in rd]
    return meta, rows
