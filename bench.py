#!/usr/bin/env python3
"""Benchmark: KPZ 2+1-d DTr sweep, site-update attempts/ns (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one Monte Carlo step (L^2 attempts) of the two-layer DTr sweep on
the synthetic flat start (make_flat_slopes, lattice.cpp:71-82) at L = 2^16,
p = 1, q = 0 -- BASELINE.json configs[1], the configuration the metric is
quoted on.  The 512 MiB spin lattice (1 GiB in the reference's two-plane
layout) is 4x the 126 MB L2, so every timed sweep streams from HBM (no flush
needed).

Rank 0 prints ONE JSON line.  Multi-GPU (torchrun, one rank per GPU): see
--mode; the device-timed value is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "site-update attempts/ns (KPZ 2+1d, L=2^16²) at 1/2/4/8 B200; % HBM roofline"
ALG_BYTES_PER_ATTEMPT = 0.5  # sigma_x + sigma_y, 1 bit each, read + written once per MCS


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--L", type=int, default=1 << 16)
    ap.add_argument("--p", type=float, default=1.0)
    ap.add_argument("--q", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for ln in open(self.path):
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def host_info():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return os.cpu_count() or 1, model


def flat_words(L):
    """make_flat_slopes (lattice.cpp:71-82) as uint64 words, built vectorised."""
    import numpy as np

    wpr = L // 64
    x = np.full(L * wpr, 0x5555555555555555, np.uint64)  # sigma_x = +1 iff i even
    y = np.zeros((L, wpr), np.uint64)
    y[0::2, :] = np.uint64(0xFFFFFFFFFFFFFFFF)            # sigma_y = +1 iff j even
    return x, y.reshape(-1)


# ----------------------------------------------------------------------------- CPU legs
def reference_sample(L, p, q, seconds, threads):
    """Time the reference's own kpz_sweep_sequential loop body (oracle/_ref =
    the unmodified reference sources) on `threads` host threads, one
    independent replica each (the reference has no parallel sweep)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle

    ref = pyoracle.try_ref()
    kind = "reference"
    if ref is None:
        raise RuntimeError("oracle/_ref/liblfref.so missing: build it where /root/reference exists")
    x0, y0 = flat_words(L)
    fields = [ref.kpz_field(L, x0, y0) for _ in range(threads)]
    del x0, y0
    # calibrate on one thread (warms the replica's pages and caches)
    n_cal = 1 << 22
    t = time.perf_counter()
    fields[0].attempts(p, q, "lcg64", 1, n_cal)
    rate1 = n_cal / (time.perf_counter() - t)
    n = max(n_cal, int(rate1 * seconds))
    results = [None] * threads

    def work(r):
        t0 = time.perf_counter()
        fields[r].attempts(p, q, "lcg64", 1 + r, n)
        results[r] = time.perf_counter() - t0

    ths = [threading.Thread(target=work, args=(r,)) for r in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    wall = time.perf_counter() - t0
    for fl in fields:
        fl.close()
    agg = threads * n / (wall * 1e9)
    return {"value": agg, "unit": "attempts/ns", "cores": threads, "kind": kind,
            "sample": f"{n} attempts of kpz_sweep_sequential's loop (kpz.cpp:12-16) per thread on a flat "
                      f"L={L} lattice (1 GiB/replica), {threads} independent replicas, wall {wall:.1f}s"}


def cpu_threads_for(L):
    ncpu, _ = host_info()
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    per = 2 * (L * L // 8) + (256 << 20)
    return max(1, min(ncpu, int(avail * 0.6 // per)))


# ----------------------------------------------------------------------------- main legs
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = cpu_threads_for(args.L)
    per_step = []
    cb = None
    for s in range(args.warmup + args.steps):
        r = reference_sample(args.L, args.p, args.q, max(2.0, args.cpu_seconds / 4), threads)
        if s >= args.warmup:
            per_step.append(r["value"])
            cb = r
    v = statistics.median(per_step)
    ncpu, model = host_info()
    line = {"metric": METRIC, "value": v, "unit": "attempts/ns", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (flat start)",
            "config": {"workload": f"KPZ octahedron, L={args.L}, p={args.p}, q={args.q}, flat start",
                       "cpu_model": model, "nproc": ncpu},
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": "attempts/ns", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch

    import paper_1204_5072_b200 as lfg

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = args.L
    stream = torch.cuda.current_stream()
    k = lfg.KpzLattice(L, args.p, args.q, args.seed + rank, device=local)
    k.set_stream(stream.cuda_stream)
    k.make_flat_slopes()
    attempts_per_step = L * L

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up
    k.sweep_async(args.warmup)
    barrier()
    # timed region
    clocks = ClockSampler(local)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    k.sweep_async(args.steps)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * attempts_per_step * args.steps / (ms * 1e6)  # attempts/ns, whole job
    c = k.counters()

    # dominant kernel: per-launch event timing of the phase kernel on the same stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
    s0 = k.sweep_index
    for i, (a, b) in enumerate(ev):
        a.record(stream)
        k.phase(s0 + i // 4, i % 4)
        b.record(stream)
    k.sweep_index = s0 + 2
    torch.cuda.synchronize()
    launch_ms = [a.elapsed_time(b) for a, b in ev]
    avg_launch_ms = statistics.mean(launch_ms)
    peak, peak_kind = measured_peaks()
    bytes_per_launch = ALG_BYTES_PER_ATTEMPT * attempts_per_step / 4
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get("kpz_dtr_phase", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_kind,
                "kernel": "kpz_dtr_phase_kernel", "avg_launch_ms": avg_launch_ms,
                "alg_bytes_per_launch": bytes_per_launch,
                "note": "algorithmic bytes = 0.5 B/attempt (two 1-bit slope planes read+written once per "
                        "MCS, SURVEY.md §8(d)); the device stores 1 spin bit per site, so actual HBM "
                        "traffic is about half of that; the kernel is issue/SMEM bound, not HBM bound"}

    # end-to-end through the public API with host buffers (rank-local)
    e2e = None
    if not args.no_e2e:
        import numpy as np

        x0, y0 = flat_words(L)
        hx = torch.from_numpy(x0.view(np.int64)).pin_memory()
        hy = torch.from_numpy(y0.view(np.int64)).pin_memory()
        ke = lfg.KpzLattice(L, args.p, args.q, args.seed + 1000 + rank, device=local)
        ke.upload_ptr(hx.data_ptr(), hy.data_ptr())
        ke.sweep(1)
        ke.download_ptr(hx.data_ptr(), hy.data_ptr())
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ke.upload_ptr(hx.data_ptr(), hy.data_ptr())       # host SlopeField -> device
            ke.sweep(1)                                       # kpz_sweep_sequential(f, params, rng, 1)
            w2 = ke.interface_width()                         # W^2 readout (d2h)
            ke.download_ptr(hx.data_ptr(), hy.data_ptr())     # device -> host SlopeField
        barrier()
        dt = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": world * attempts_per_step * args.e2e_steps / (dt * 1e9), "unit": "attempts/ns",
               "h2d_bytes_per_step": 2 * L * L // 8, "d2h_bytes_per_step": 2 * L * L // 8 + 24 + 32,
               "steps": args.e2e_steps,
               "step": "lfg_kpz_upload(host SlopeField planes, pinned) + lfg_kpz_sweep(1 MCS) + "
                       "lfg_kpz_interface_width + lfg_kpz_download", "w2_last": w2}
        ke.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_sample(L, args.p, args.q, args.cpu_seconds, 1)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "attempts/ns", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "attempts/ns", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (flat start)",
                "config": {"workload": f"KPZ octahedron DTr, L={L}x{L}, p={args.p}, q={args.q}, flat start, "
                                       f"1 MCS per step (BASELINE.json configs[1])",
                           "plan": {"block_x": k.plan[0], "block_y": k.plan[1], "domain": "16x8"},
                           "parallelism": f"replica-per-GPU x{world}" if world > 1 else "1 GPU",
                           "l2": "lattice 512 MiB >> 126 MB L2: no flush needed",
                           "successes_per_step": c.successes / max(1, c.attempts // attempts_per_step)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": 4 * args.steps}
        print(json.dumps(line), flush=True)
    k.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
