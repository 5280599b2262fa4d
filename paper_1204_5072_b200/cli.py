"""Command-line front end ("cli").

    python -m paper_1204_5072_b200.cli kpz --size 256 --mcs 100 --p 1 --q 0 --out w2.csv
    python -m paper_1204_5072_b200.cli kmc --size 64 --conc 0.325 --eps 1.5 --mcs 1000 --out ob.csv
    python -m paper_1204_5072_b200.cli bench --size 65536 --mcs 20
    python -m paper_1204_5072_b200.cli verify [-m gpu]

Flags follow the SPEC: --size --mcs --seed --realizations --out, --p --q (kpz), --conc --eps
--both-active (kmc), --scheduler.  The device implements the two-layer double tiling with
single-hit inner rounds; ``--scheduler`` accepts ``twolayer``
(alias ``doubletile``) and rejects the CPU-only schedulers (seq, cache, deadborder) with a
one-line diagnostic, as it does for a non-power-of-two size.  --block-edge
sets the device block (KMC edge, KPZ height), --tile-edge the KPZ block width.  Exit codes:
0 ok, 2 usage / invalid value, 1 runtime failure.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

SCHEDULERS = {"twolayer": "twolayer", "doubletile": "twolayer"}
CPU_ONLY = ("seq", "cache", "deadborder")


class UsageError(Exception):
    pass


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1204_5072_b200.cli",
                                 description="B200 KPZ / KMC lattice Monte Carlo (arXiv 1204.5072 hot path)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--size", type=int, default=256)
        p.add_argument("--mcs", type=int, default=100)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--realizations", type=int, default=1)
        p.add_argument("--scheduler", default="twolayer")
        p.add_argument("--single-hit", action="store_true", default=True,
                       help="single-hit inner rounds (always on: the device schedule)")
        p.add_argument("--block-edge", type=int, default=0)
        p.add_argument("--tile-edge", type=int, default=0)
        p.add_argument("--samples", default=None, help="comma-separated sample times (default: 1.1^k)")
        p.add_argument("--device", type=int, default=0)
        p.add_argument("--concurrency", type=int, default=8,
                       help="realizations in flight at once, each on its own stream (1: sequential)")
        p.add_argument("--out", default=None, help="CSV file (default: stdout)")

    k = sub.add_parser("kpz", help="KPZ octahedron model, W^2(t) and <h>(t)")
    common(k)
    k.add_argument("--p", type=float, default=1.0)
    k.add_argument("--q", type=float, default=0.0)
    k.add_argument("--sub", type=int, default=0, choices=[0, 1, 4, 8],
                   help="DTr sub-sweeps per MCS: 4 (default) statistically matched, 8 with half the residual "
                        "<h> bias, 1 the paper's scheme with exact L^2 attempts per MCS")
    m = sub.add_parser("kmc", help="fcc binary-alloy KMC, open bonds per particle (t)")
    common(m)
    m.add_argument("--conc", type=float, default=0.5)
    m.add_argument("--eps", type=float, default=1.5)
    m.add_argument("--both-active", action="store_true")
    b = sub.add_parser("bench", help="KPZ throughput (attempts/ns) of the device sweep")
    common(b)
    b.add_argument("--p", type=float, default=1.0)
    b.add_argument("--q", type=float, default=0.0)
    v = sub.add_parser("verify", help="run the invariant / oracle suites (pytest)")
    v.add_argument("-m", "--marker", default="not gpu", help="pytest marker expression")
    return ap


def _config(a):
    from .harness import ExperimentConfig

    sched = SCHEDULERS.get(a.scheduler)
    if sched is None:
        if a.scheduler in CPU_ONLY:
            raise UsageError(f"scheduler {a.scheduler!r} is a CPU scheduler; the device runs 'twolayer' "
                             f"(two-layer double tiling, single-hit)")
        raise UsageError(f"unknown scheduler {a.scheduler!r} (choices: twolayer, doubletile)")
    if a.size < 4 or a.size & (a.size - 1):
        raise UsageError(f"size must be a power of two, got {a.size}")
    if a.mcs < 0 or a.realizations < 1 or a.concurrency < 1:
        raise UsageError("mcs must be >= 0, realizations >= 1 and concurrency >= 1")
    samples = [int(x) for x in a.samples.split(",")] if a.samples else None
    if a.cmd in ("kpz", "bench"):
        if not (0.0 <= a.p <= 1.0 and 0.0 <= a.q <= 1.0) or a.p + a.q <= 0.0:
            raise UsageError("p and q must lie in [0,1] with p + q > 0")
        return ExperimentConfig("kpz", a.size, a.mcs, a.seed, a.realizations, samples, p=a.p, q=a.q,
                                block_x=a.tile_edge, block_y=a.block_edge, sub=getattr(a, "sub", 0),
                                device=a.device, concurrency=a.concurrency)
    if not 0.0 <= a.conc <= 1.0 or a.eps < 0.0:
        raise UsageError("conc must lie in [0,1] and eps >= 0")
    return ExperimentConfig("kmc", a.size, a.mcs, a.seed, a.realizations, samples, conc=a.conc, eps=a.eps,
                            both_active=a.both_active, block=a.block_edge, device=a.device,
                            concurrency=a.concurrency)


def parse_and_run(argv=None) -> int:
    """parse_and_run."""
    ap = _parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse already printed usage
        return 2 if e.code else 0
    if a.cmd == "verify":
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        return subprocess.call([sys.executable, "-m", "pytest", os.path.join(root, "tests"), "-q", "-m", a.marker])
    try:
        cfg = _config(a)
    except UsageError as e:
        sys.stderr.write(f"error: {e}\n")
        ap.print_usage(sys.stderr)
        return 2
    from . import LfgError
    from .harness import run_experiment, throughput, write_csv

    try:
        if a.cmd == "bench":
            cfg.samples = [cfg.mcs]
            rows = run_experiment(cfg)
            rep = throughput(rows)
            print(json.dumps({"size": cfg.size, "mcs": cfg.mcs, "attempts": rep["attempts"],
                              "attempts_per_ns": rep["updates_per_second"] / 1e9,
                              "note": "host wall clock around lfg_kpz_sweep (SPEC.md:454); bench.py has the "
                                      "device-timed figure"}))
            return 0
        rows = run_experiment(cfg)
    except LfgError as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
    if a.out:
        with open(a.out, "w", encoding="utf-8") as f:
            write_csv(cfg, rows, f)
    else:
        write_csv(cfg, rows, sys.stdout)
    return 0


def main() -> None:
    sys.exit(parse_and_run())


if __name__ == "__main__":
    main()
