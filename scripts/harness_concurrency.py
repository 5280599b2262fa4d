#!/usr/bin/env python3
"""Ensemble throughput of the harness with realizations run one after another vs several
in flight (own streams): KMC 256^3 (BASELINE C4 size) and KPZ 4096^2.
Usage: python scripts/harness_concurrency.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1204_5072_b200.harness import ExperimentConfig, run_experiment, throughput  # noqa: E402

for model, size, mcs, kw in (("kmc", 256, 40, dict(conc=0.5, eps=1.5, both_active=True)),
                             ("kpz", 4096, 200, dict(p=1.0, q=0.0))):
    for conc in (1, 8):
        cfg = ExperimentConfig(model, size, mcs, seed=3, realizations=8, samples=[mcs // 2], concurrency=conc, **kw)
        rep = throughput(run_experiment(cfg))
        print(json.dumps({"model": model, "size": size, "realizations": 8, "concurrency": conc,
                          "attempts_per_ns": rep["updates_per_second"] / 1e9}), flush=True)
