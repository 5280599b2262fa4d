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
    ap.add_argument("--L", type=int, default=0,
                    help="lattice edge (0: 2^16, the metric's configs[1] lattice, at every N)")
    ap.add_argument("--p", type=float, default=1.0)
    ap.add_argument("--q", type=float, default=0.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--block-x", type=int, default=0, help="DT device block width (0: library default)")
    ap.add_argument("--block-y", type=int, default=0, help="DT device block height (0: library default)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--e2e-lattices", type=int, default=3, help="lattices (seeds) pipelined in the e2e leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kmc", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the configs[2] (L=2^17, p=0.95, q=0.05) sub-measurement")
    a = ap.parse_args()
    a.L = a.L or (1 << 16)
    return a


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
class ReferenceReplicas:
    """`threads` independent reference lattices (oracle/_ref = the unmodified
    reference sources; the reference has no parallel sweep), each a persistent
    lf::SlopeField so timed samples exclude host copies."""

    def __init__(self, L, p, q, threads):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle

        self.ref = pyoracle.try_ref()
        if self.ref is None:
            raise RuntimeError("oracle/_ref/liblfref.so missing: build it where /root/reference exists")
        self.L, self.p, self.q, self.threads = L, p, q, threads
        x0, y0 = flat_words(L)
        self.fields = [self.ref.kpz_field(L, x0, y0) for _ in range(threads)]
        self.state = [1 + r for r in range(threads)]
        self.rate1 = None

    def calibrate(self, n=1 << 21):
        t = time.perf_counter()
        _, self.state[0] = self.fields[0].attempts(self.p, self.q, "lcg64", self.state[0], n)
        self.rate1 = n / (time.perf_counter() - t)
        return self.rate1

    def sample(self, seconds):
        if self.rate1 is None:
            self.calibrate()
        n = max(1 << 20, int(self.rate1 * seconds))

        def work(r):
            _, self.state[r] = self.fields[r].attempts(self.p, self.q, "lcg64", self.state[r], n)

        ths = [threading.Thread(target=work, args=(r,)) for r in range(self.threads)]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        wall = time.perf_counter() - t0
        return self.threads * n / (wall * 1e9), n, wall

    def close(self):
        for f in self.fields:
            f.close()

    def describe(self, n, wall):
        return (f"{n} attempts of kpz_sweep_sequential's loop (kpz.cpp:12-16) per thread on a flat L={self.L} "
                f"lattice (1 GiB/replica), {self.threads} independent replicas, wall {wall:.1f}s")


def reference_sample(L, p, q, seconds, threads):
    rr = ReferenceReplicas(L, p, q, threads)
    try:
        v, n, wall = rr.sample(seconds)
        return {"value": v, "unit": "attempts/ns", "cores": threads, "kind": "reference", "sample": rr.describe(n, wall)}
    finally:
        rr.close()


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
    rr = ReferenceReplicas(args.L, args.p, args.q, threads)
    rr.calibrate()
    step_s = max(1.0, min(4.0, 150.0 / max(1, args.warmup + args.steps)))
    vals = []
    n = wall = 0
    for s in range(args.warmup + args.steps):
        v, n, wall = rr.sample(step_s)
        if s >= args.warmup:
            vals.append(v)
    rr.close()
    v = statistics.median(vals)
    ncpu, model = host_info()
    line = {"metric": METRIC, "value": v, "unit": "attempts/ns", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (flat start)",
            "config": {"workload": f"KPZ octahedron, L={args.L}, p={args.p}, q={args.q}, flat start; reference "
                                   f"random-sequential sweep (lf::kpz_sweep_sequential), bounded sample per step",
                       "cpu_model": model, "nproc": ncpu},
            "cpu_baseline": {"value": v, "unit": "attempts/ns", "cores": threads, "kind": "reference",
                             "sample": rr.describe(n, wall)},
            "e2e": {"value": v, "unit": "attempts/ns", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def duplex_copy_gbps(torch, ha, hb, device, reps=3):
    """GB/s per direction with one pinned H2D and one D2H copy in flight at once."""
    da = torch.empty_like(ha, device=f"cuda:{device}")
    db = torch.empty_like(hb, device=f"cuda:{device}")
    s1, s2 = torch.cuda.Stream(device=device), torch.cuda.Stream(device=device)
    for i in range(reps + 1):  # the first round is untimed (first touch of the device buffers)
        if i == 1:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            da.copy_(ha, non_blocking=True)
        with torch.cuda.stream(s2):
            hb.copy_(db, non_blocking=True)
        if i == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    del da, db
    return reps * ha.numel() * ha.element_size() / dt / 1e9


def kmc_measure(lfg, torch, stream, steps, warmup, L=256):
    """BASELINE configs[3]: 3-D fcc binary alloy, 256^3 sc, c = 0.5, eps = 1.5,
    both species active; one step = one MCS (L^3/2 attempts)."""
    out = {}
    for both in (True, False):
        k = lfg.KmcLattice(L, 1.5, both, 7)
        k.set_stream(stream.cuda_stream)
        k.make_random_alloy(0.5, 3)
        k.sweep_async(warmup)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        k.sweep_async(steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out["both" if both else "b_only"] = {"value": (L ** 3 // 2) * steps / (ms * 1e6), "unit": "attempts/ns",
                                             "ms_per_mcs": ms / steps, "open_bonds": k.open_bonds_per_particle()}
        k.close()
    # ensemble: 8 seeds side by side, each lattice on its own stream (sweeps issued
    # round-robin), launches sized for the combined load (lfg_kmc_set_concurrency)
    n = 8
    ks = []
    for i in range(n):
        k = lfg.KmcLattice(L, 1.5, True, 100 + i)
        k.set_concurrency(n)
        k.make_random_alloy(0.5, 200 + i)
        ks.append(k)
    for k in ks:
        k.sweep_async(warmup)
    for k in ks:
        k.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        for k in ks:
            k.sweep_async(1)
    for k in ks:
        k.synchronize()
    dt = time.perf_counter() - t0
    out["ensemble8_both"] = {"value": n * (L ** 3 // 2) * steps / (dt * 1e9), "unit": "attempts/ns",
                             "note": "8 lattices (seeds) on 8 streams, wall clock incl. the final synchronize"}
    for k in ks:
        k.close()
    out["config"] = f"KMC fcc binary alloy {L}^3 sc, c=0.5, eps=1.5, DT blocks 16^3 (BASELINE.json configs[3])"
    out["note"] = ("L2-resident (2 MiB); only L^3/4096 tiles are active per single-hit round, so the 256^3 "
                   "case is latency-bound by construction")
    # BASELINE configs[4] on one GPU: 1024^3, both active (the 4-blocks-per-warp kernel)
    L5, s5 = 1024, 5
    k = lfg.KmcLattice(L5, 1.5, True, 7)
    k.set_stream(stream.cuda_stream)
    k.make_random_alloy(0.5, 3)
    k.sweep_async(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k.sweep_async(s5)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["c5_single_gpu"] = {"value": (L5 ** 3 // 2) * s5 / (ms * 1e6), "unit": "attempts/ns", "ms_per_mcs": ms / s5,
                            "steps": s5, "open_bonds": k.open_bonds_per_particle(),
                            "config": "KMC fcc binary alloy 1024^3 sc, c=0.5, eps=1.5, both active, DT blocks 16^3 "
                                      "(BASELINE.json configs[4] on 1 GPU; 128 MiB lattice > L2)"}
    k.close()
    return out


class KpzRun:
    """One KPZ lattice of the bench with the same interface at every N: the resident
    lattice on this GPU (N = 1) or the strip-sharded lattice across the ranks (N > 1,
    one strip per GPU; peer memory over NVLink, torch.distributed as the fallback)."""

    def __init__(self, lfg, torch, dist, L, p, q, seed, rank, world, local, stream, block_x=0, block_y=0):
        self.torch, self.dist, self.world, self.L = torch, dist, world, L
        if world == 1:
            self.k = k = lfg.KpzLattice(L, p, q, seed, block_x=block_x, block_y=block_y, device=local)
            k.set_stream(stream.cuda_stream)
            k.make_flat_slopes()
            self.stream, self.plan, self.sub = stream, k.plan, k.sub
            self.mode = "1 GPU"
            return
        from paper_1204_5072_b200.shard import CudaStripEngine, DistComm, PeerComm, ShardedKpz, StripPlan

        bx, by = block_x or min(1024, L // 2), block_y or min(128, L // 2)
        self.plan = (bx, by)
        pl = StripPlan(L, world, bx, by)
        self.sub = pl.sub
        eng = CudaStripEngine(pl, p, q, seed, local)
        # Default: peer memory (CUDA IPC over NVLink; ghost rows pushed by the phase
        # kernel's write-back, device-side step barriers).  LFG_COMM=nccl selects
        # torch.distributed P2P; a peer setup failure falls back to it.
        comm, how = None, "torch.distributed " + dist.get_backend()
        if os.environ.get("LFG_COMM", "peer") == "peer":
            try:
                comm, how = PeerComm(eng), "peer memory (CUDA IPC / NVLink), fused write-back push"
            except Exception as ex:  # reported in the JSON line
                how = f"torch.distributed {dist.get_backend()} (peer setup failed: {ex})"
        if comm is None:
            comm = DistComm(eng)
        sk = ShardedKpz(pl, seed, [eng], [rank], comm)
        sk.make_flat_slopes()
        if isinstance(comm, PeerComm):  # a peer barrier that times out anywhere -> everyone falls back
            try:
                sk.sweep(1)
                bad = 0
            except Exception:
                bad = 1
            t = torch.tensor([bad], device="cuda" if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(t)
            if int(t.item()):
                comm.close()
                comm, how = DistComm(eng), f"torch.distributed {dist.get_backend()} (peer barrier timed out)"
                sk = ShardedKpz(pl, seed, [eng], [rank], comm)
                sk.make_flat_slopes()
        self.eng, self.sk, self.rank = eng, sk, rank
        self.stream = eng.stream
        self.mode = (f"strip-sharded x{world} (rows rolled per sub-sweep, one ghost row per phase; {how})")

    def run(self, n):
        if self.world == 1:
            self.k.sweep_async(n)
        else:
            self.sk.sweep(n)

    def done(self):
        """Attempts made so far by the whole job (device counters; sub = 4: Poisson tiles)."""
        if self.world == 1:
            return self.k.counters().attempts
        t = self.torch.tensor([float(self.eng.counters().attempts)], dtype=self.torch.float64,
                              device="cuda" if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t)
        return int(t.item())

    def launch_ms(self, n=8):
        """Mean duration of this rank's dominant-kernel launch (one DT phase), CUDA events on
        the launching stream; the phases are timed after the timed region (no trajectory)."""
        torch = self.torch
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        if self.world == 1:
            s0 = self.k.sweep_index
        else:
            s0 = self.sk.sweep_index
            b0, nb = self.sk.plan.block_rows(self.rank)
        for i, (a, b) in enumerate(ev):
            a.record(self.stream)
            if self.world == 1:
                self.k.phase(s0 * self.sub + i // 4, i % 4)
            else:
                self.eng.phase(s0 * self.sub + i // 4, i % 4, b0, nb)
            b.record(self.stream)
        torch.cuda.synchronize()
        if self.world == 1:
            self.k.sweep_index = s0 + 1
        return statistics.mean(a.elapsed_time(b) for a, b in ev)

    def close(self):
        if self.world == 1:
            self.k.close()


def timed(torch, dist, lat, steps, warmup, barrier, clocks=None):
    """W warm-up MCS, then K MCS between CUDA events on the launching stream with a
    barrier + synchronize on both sides; max over ranks.  -> (attempts/ns, ms, clocks)."""
    lat.run(warmup)
    barrier()
    att0 = lat.done()
    if clocks is not None:
        clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(lat.stream)
    lat.run(steps)
    e1.record(lat.stream)
    barrier()
    clk = clocks.stop() if clocks is not None else None
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    att = lat.done() - att0
    return att / (ms * 1e6), ms, clk


def run_b200(args):
    import torch

    import paper_1204_5072_b200 as lfg

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())  # several ranks may share one GPU (gloo tests)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("LFG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    L = args.L
    stream = torch.cuda.current_stream()
    attempts_per_step = L * L

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    peak, peak_kind = measured_peaks()
    lat = KpzRun(lfg, torch, dist, L, args.p, args.q, args.seed, rank, world, local, stream, args.block_x,
                 args.block_y)
    plan, sub, mode = lat.plan, lat.sub, lat.mode
    stream = lat.stream
    if world == 1:
        k = lat.k
    else:
        eng, sk = lat.eng, lat.sk
    value, ms, clk = timed(torch, dist, lat, args.steps, args.warmup, barrier, ClockSampler(local))

    # dominant kernel: event-timed phase launches on the launching stream (this rank's
    # strip phases at N > 1: per-GPU bytes / per-GPU launch time)
    roofline = None
    if True:
        avg_launch_ms = lat.launch_ms()
        if dist is not None:
            t = torch.tensor([avg_launch_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            avg_launch_ms = float(t.item())
        bytes_per_launch = ALG_BYTES_PER_ATTEMPT * attempts_per_step / world / (4 * sub)  # mean, per GPU
        achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
        traffic, ncu = None, {}
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
                ncu = json.load(f).get("kpz_dtr_phase", {})
            traffic = ncu.get("dram_bytes_per_launch")
        except Exception:
            pass
        # The roofline that binds: SM issue.  Ceiling = warp-instruction issue rate of all
        # SMSPs at the clock sampled during the timed region / warp-instructions per attempt
        # (ncu count of one launch of this kernel at L = 2^16, p = 1).
        issue = None
        if ncu.get("inst_executed") and world == 1 and L == 1 << 16 and args.p == 1.0 and args.q == 0.0:
            wi_per_att = ncu["inst_executed"] / (attempts_per_step / (4 * ncu.get("sub", 1)))
            f_ghz = (clk.get("sm_mhz") or 1965.0) / 1000.0
            ceil_att = 148 * 4 * f_ghz / wi_per_att
            issue = {"achieved_attempts_per_ns": bytes_per_launch / ALG_BYTES_PER_ATTEMPT / (avg_launch_ms * 1e6),
                     "ceiling_attempts_per_ns": ceil_att, "warp_inst_per_attempt": wi_per_att,
                     "frac": bytes_per_launch / ALG_BYTES_PER_ATTEMPT / (avg_launch_ms * 1e6) / ceil_att,
                     "source": f"ncu inst_executed of one launch ({ncu.get('tag')}), 148 SMs x 4 issue slots/clk"}
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "peak_source": peak_kind, "kernel": "kpz_dtr_phase_kernel",
                    "avg_launch_ms": avg_launch_ms, "alg_bytes_per_launch": bytes_per_launch,
                    "binding_unit": ncu.get("binding", "SM issue (profiles/ncu_summary.json)"),
                    "issue_roofline": issue,
                    "note": "algorithmic bytes = 0.5 B/attempt (two 1-bit slope planes read+written once per MCS, "
                            "SURVEY.md §8(d)); the device keeps 1 spin bit per site; the faithful single-hit "
                            "DTr kernel is issue-bound, not HBM-bound (DESIGN.md §4.1)"}

    e2e = None
    if not args.no_e2e and world == 1:
        import numpy as np

        x0, y0 = flat_words(L)
        # (a) one lattice, synchronous reference-style calls: upload, sweep, W^2, download
        hx = torch.from_numpy(x0.view(np.int64)).pin_memory()
        hy = torch.from_numpy(y0.view(np.int64)).pin_memory()
        ke = lfg.KpzLattice(L, args.p, args.q, args.seed + 1000, device=local)
        ke.upload_ptr(hx.data_ptr(), hy.data_ptr())
        ke.sweep(1)
        ke.download_ptr(hx.data_ptr(), hy.data_ptr())
        a_single = ke.counters().attempts
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ke.upload_ptr(hx.data_ptr(), hy.data_ptr())       # host SlopeField -> device
            ke.sweep(1)                                       # kpz_sweep_sequential(f, params, rng, 1)
            w2 = ke.interface_width()                         # W^2 readout (d2h)
            ke.download_ptr(hx.data_ptr(), hy.data_ptr())     # device -> host SlopeField
        barrier()
        dt_single = time.perf_counter() - t0
        single = (ke.counters().attempts - a_single) / (dt_single * 1e9)
        ke.close()
        # (b) headline: two lattices of the same configuration (an ensemble, as in
        # BASELINE configs[1]'s 16 seeds), each on its own stream with the
        # stream-ordered C-ABI calls, so one lattice's device->host copy runs
        # beside the other's host->device copy (full-duplex PCIe).  Every
        # lattice-step still moves its whole SlopeField in and out.
        nl = max(1, args.e2e_lattices)
        hxs = [torch.from_numpy(x0.view(np.int64)).pin_memory() for _ in range(nl)]
        hys = [torch.from_numpy(y0.view(np.int64)).pin_memory() for _ in range(nl)]
        o3 = torch.zeros((nl, 3), dtype=torch.int64).pin_memory()
        sts = [torch.cuda.Stream(device=local) for _ in range(nl)]
        kes = []
        for i in range(nl):
            k2 = lfg.KpzLattice(L, args.p, args.q, args.seed + 2000 + i, device=local)
            k2.set_stream(sts[i].cuda_stream)
            kes.append(k2)

        def lattice_step(i):
            kes[i].upload_ptr_async(hxs[i].data_ptr(), hys[i].data_ptr())
            kes[i].sweep_async(1)
            kes[i].width_sums_async(o3[i].data_ptr())
            kes[i].download_ptr_async(hxs[i].data_ptr(), hys[i].data_ptr())

        for i in range(nl):
            lattice_step(i)
        for k2 in kes:
            k2.synchronize()
            k2.upload_check()
        a_multi = sum(k2.counters().attempts for k2 in kes)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for i in range(nl):
                lattice_step(i)
        for k2 in kes:
            k2.synchronize()
            k2.upload_check()
        barrier()
        dt = time.perf_counter() - t0
        s_, s2_ = int(o3[0, 0]), int(o3[0, 1]) + int(o3[0, 2])
        w2 = s2_ / (L * L) - (s_ / (L * L)) ** 2
        a_multi = sum(k2.counters().attempts for k2 in kes) - a_multi
        e2e = {"value": a_multi / (dt * 1e9), "unit": "attempts/ns",
               "h2d_bytes_per_step": 2 * L * L // 8, "d2h_bytes_per_step": 2 * L * L // 8 + 24,
               "steps": nl * args.e2e_steps,
               "step": f"one lattice-step = lfg_kpz_upload_async(host SlopeField planes, pinned) + 1 MCS + "
                       f"W^2 sums + lfg_kpz_download_async; {nl} lattices (seeds) on {nl} streams, issued "
                       f"round-robin, wall clock incl. the final synchronize and closure checks",
               "single_lattice_sync_calls": single, "w2_last": w2}
        for k2 in kes:
            k2.close()
        # the ceiling of this leg: concurrent H2D + D2H of pinned buffers (scripts/pcie_bw.py)
        try:
            bw = duplex_copy_gbps(torch, hxs[0].view(torch.uint8), hys[0].view(torch.uint8), local)
            e2e["pcie_duplex_GBps_per_direction"] = bw
            e2e["pcie_ceiling_attempts_per_ns"] = attempts_per_step / (2 * L * L // 8 / (bw * 1e9)) / 1e9
        except Exception as ex:  # informational only
            e2e["pcie_duplex_note"] = f"not measured: {ex}"

    elif not args.no_e2e:
        # sharded: each rank moves its strip (spin rows) host<->device around one MCS + distributed W^2
        hbuf = torch.empty_like(eng.buf, device="cpu").pin_memory()
        hbuf.copy_(eng.buf)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            with torch.cuda.stream(eng.stream):       # ordered before the phase kernels / exchanges
                eng.buf.copy_(hbuf, non_blocking=True)
            sk.sweep(1)
            w2 = sk.interface_width()
            with torch.cuda.stream(eng.stream):
                hbuf.copy_(eng.buf, non_blocking=True)
            eng.sync()
        barrier()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        nbytes = eng.buf.numel() * 4 * world
        e2e = {"value": attempts_per_step * args.e2e_steps / (dt * 1e9), "unit": "attempts/ns",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes + 16, "steps": args.e2e_steps,
               "step": "per rank: strip ring buffer host->device, 1 MCS, distributed W^2, device->host",
               "w2_last": w2}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = reference_sample(L, args.p, args.q, args.cpu_seconds, 1)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": "attempts/ns", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    kmc = None
    if rank == 0 and world == 1 and not args.no_kmc:
        kmc = kmc_measure(lfg, torch, stream, steps=20, warmup=3)
    c3 = None
    if not args.no_c3:  # BASELINE configs[2]: L = 2^17, p = 0.95, q = 0.05, at every N (strips at N > 1)
        l3 = KpzRun(lfg, torch, dist, 1 << 17, 0.95, 0.05, 1, rank, world, local, torch.cuda.current_stream())
        v3, ms3, _ = timed(torch, dist, l3, 10, 3, barrier)
        c3 = {"value": v3, "unit": "attempts/ns", "ms_per_mcs": ms3 / 10, "steps": 10, "n_gpus": world,
              "config": f"KPZ DTr L=131072, p=0.95, q=0.05, flat start, plan {l3.plan} sub={l3.sub} "
                        f"(BASELINE.json configs[2]; {l3.mode})"}
        l3.close()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "attempts/ns", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (flat start)",
                "config": {"workload": f"KPZ octahedron DTr, L={L}x{L}, p={args.p}, q={args.q}, flat start, "
                                       f"1 MCS per step (BASELINE.json configs[1]; the same lattice at every N: "
                                       f"strong scaling)",
                           "plan": {"block_x": plan[0], "block_y": plan[1], "domain": "16x8", "sub_sweeps_per_mcs": sub},
                           "parallelism": mode,
                           "l2": f"lattice {L * L // 8 >> 20} MiB ({L * L // 8 // world >> 20} MiB per GPU) >> 126 MB L2: "
                                 f"no flush needed"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": 4 * sub * args.steps, "kmc": kmc, "c3": c3}
        if world == 1:
            line["c3_single_gpu"] = c3
        print(json.dumps(line), flush=True)
    if world == 1:
        k.close()
    else:
        eng.close()
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
