#!/usr/bin/env python3
"""Benchmark of the B200 randomized k-SVD on BASELINE.json's headline configuration.

Workload (config C2, the metric's 1-GPU case): a CelebA-shaped synthetic FP64 matrix
A (202599 x 4096) with a controlled, exponentially decaying spectrum, rank k=64,
oversampling p=10, q=2 power iterations, seed 42. One step = one full
`randomized_ksvd` (Algorithm 1) with A resident in HBM. A (6.6 GB) is much larger than
the 126 MB L2, so every step streams it from HBM (no explicit flush needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0). value = whole-job TFLOP/s with the algorithmic flop
count F = (2q+2)*2*m*n*s + 2*m*s*k (s = k+p), i.e. the reference's arithmetic, not
padded tiles; ms_per_step is the wall time of one solve (max over ranks).
--impl reference times the reference's own CPU implementation (oracle/_ref, compiled
from the unmodified reference sources) on the host cores, on a bounded row sample.
N > 1 runs independent replicas (one per GPU, no data-path collective), weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M, N, K_RANK, P_OVER, Q_POW, SEED = 202599, 4096, 64, 10, 2, 42
METRIC = "rSVD wall ms & TFLOP/s (frac of FP64 TC roofline), 1/2/4/8 B200 vs host CPU"


def flops(m, n, k, p, q):
    s = min(k + p, m, n)
    return (2 * q + 2) * 2.0 * m * n * s + 2.0 * m * s * k


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ----------------------------------------------------------------- CPU reference
def cpu_reference_run(rows: int, threads: int, reps: int = 1):
    """Time randsvd::randomized_ksvd (the unmodified reference library) on the first
    `rows` rows of the synthetic C2 matrix (same n, k, p, q, seed), all host threads."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    a = synth_host(rows, N, SEED)
    if kind == "reference":
        orc.set_max_threads(threads)
        times, _ = orc.timed_solve(a, K_RANK, P_OVER, Q_POW, SEED, reps=reps)
        cores = threads
    else:
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            orc.randomized_ksvd(a, K_RANK, P_OVER, Q_POW, SEED, values_only=False)
            times.append(time.perf_counter() - t0)
        cores = 1
    t = min(times)
    f = flops(rows, N, K_RANK, P_OVER, Q_POW)
    return {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
            "sample": f"{rows}x{N} row block of the C2 synthetic matrix, k={K_RANK} p={P_OVER} "
                      f"q={Q_POW}; {t:.2f} s per solve ({reps} run)",
            "seconds": t}


def synth_host(rows, cols, seed):
    """Host copy of the first rows of the synthetic matrix (same law as synth_device)."""
    rng = np.random.default_rng(seed)
    tau = (K_RANK + P_OVER - 1) / np.log(1e4)
    sig = np.exp(-np.arange(cols) / tau) + 1e-6
    v, _ = np.linalg.qr(rng.standard_normal((cols, cols)))
    g = rng.standard_normal((rows, cols)) / np.sqrt(M)
    return np.ascontiguousarray((g * sig) @ v.T)


# ----------------------------------------------------------------- GPU helpers
def synth_device(torch, m, n, seed, device):
    """A = G diag(sigma) V^T: G Gaussian / sqrt(m) (near-isometric columns), V a random
    orthogonal n x n, sigma_i = exp(-i/tau) + 1e-6 with sigma_1/sigma_s = 1e4 over the
    sketch width (a controlled, decaying spectrum)."""
    gen = torch.Generator(device=device).manual_seed(seed)
    tau = (K_RANK + P_OVER - 1) / np.log(1e4)
    sig = torch.exp(-torch.arange(n, dtype=torch.float64, device=device) / tau) + 1e-6
    v = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=device, generator=gen))[0]
    a = torch.empty(m, n, dtype=torch.float64, device=device)
    step = 16384
    for r0 in range(0, m, step):
        r1 = min(m, r0 + step)
        g = torch.randn(r1 - r0, n, dtype=torch.float64, device=device, generator=gen)
        a[r0:r1] = (g * (sig / np.sqrt(m))) @ v.T
    return a


def fp64_peak(torch, device):
    """Measured FP64 tensor-core peak for the roofline: cuBLAS DGEMM 8192^3, best of 3."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device=device)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=device)
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    return 2 * 8192**3 / (best * 1e-3) / 1e12


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


# ----------------------------------------------------------------- main arms
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rows = args.cpu_rows
    for _ in range(args.warmup):  # untimed warm-up on a quarter-size sample (bounded time)
        cpu_reference_run(max(1024, rows // 4), threads)
    samples = []
    for _ in range(args.steps):
        r = cpu_reference_run(rows, threads)
        samples.append(r)
    secs = [r["seconds"] for r in samples]
    value = statistics.median([r["value"] for r in samples])
    base = samples[0]
    out = {
        "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.median(secs), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (G diag(sigma) V^T, exponential decay, seed 42)",
        "config": {"workload": f"C2 rSVD {M}x{N} k={K_RANK} p={P_OVER} q={Q_POW} FP64, "
                               f"CPU sample {rows}x{N}", "m": M, "n": N, "k": K_RANK,
                   "p": P_OVER, "q": Q_POW, "parallelism": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": base["cores"],
                         "kind": base["kind"], "sample": base["sample"]},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import paper_2110_03423_b200 as P

    rank, world, local_rank = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    m, n, k, p, q = args.m, args.n, K_RANK, P_OVER, Q_POW
    cfg = P.RsvdConfig(k=k, oversample=p, power_q=q, seed=SEED)
    F = flops(m, n, k, p, q)
    solver = P.Solver(local_rank)
    a = synth_device(torch, m, n, SEED + rank, dev)
    peak = fp64_peak(torch, dev)
    torch.cuda.synchronize()

    lib_stream = torch.cuda.ExternalStream(solver.stream, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (also allocates the workspace)
    for _ in range(args.warmup):
        u, s, v, sw = solver.randomized_ksvd_device(a, cfg)
    launches_per_step = solver.last_launch_count()

    # ---- timed region: K device-resident solves
    solver.set_profiling(2)
    solver.reset_stats()
    barrier()
    with ClockSampler(local_rank) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(lib_stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            u, s, v, sw = solver.randomized_ksvd_device(a, cfg)
        e1.record(lib_stream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        barrier()
    dev_ms = e0.elapsed_time(e1)
    stats = solver.kernel_stats("gemm_A")
    solver.set_profiling(0)
    step_ms = dev_ms / args.steps
    if world > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())
    value = world * F / (step_ms * 1e-3) / 1e12

    # ---- e2e: the public host-buffer API (pinned A in, U, sigma, V out), same config
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    a_host_t = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
    a_host_t.copy_(a)
    a_host = a_host_t.numpy()
    del a
    torch.cuda.empty_cache()
    res = solver.randomized_ksvd(a_host, cfg)  # warm the host path
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = solver.randomized_ksvd(a_host, cfg)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * F / e2e_s / 1e12
    sigma_check = float(res.factors.sigma[0])

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded row sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference_run(args.cpu_rows, os.cpu_count() or 1)
        cpu.pop("seconds", None)

    if rank == 0:
        per_launch_ms = stats["ms"] / max(1, stats["count"])
        per_launch_flops = stats["flops"] / max(1, stats["count"])
        achieved = per_launch_flops / (per_launch_ms * 1e-3) / 1e12 if stats["count"] else None
        traffic = load_traffic()
        roof = {"bound": "tensor", "kernel": "gemm_A (FP64 DMMA passes over A: ax + atx)",
                "achieved": round(achieved, 3) if achieved else None, "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": traffic.get("gemm_A_bytes_per_launch") if traffic else None,
                "peak_source": "cuBLAS DGEMM 8192^3 best-of-3 measured in this run "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "launches_timed": stats["count"], "ms_per_launch": round(per_launch_ms, 4),
                "share_of_step": round(stats["ms"] / dev_ms, 4) if dev_ms else None,
                "algorithmic_flops_per_launch": per_launch_flops}
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (G diag(sigma) V^T, exponential decay sigma_1/sigma_s=1e4, seed 42)",
            "config": {"workload": f"C2 rSVD {m}x{n} k={k} p={p} q={q} FP64 (CelebA-shaped)",
                       "m": m, "n": n, "k": k, "p": p, "q": q, "sketch_width": sw,
                       "parallelism": "replicas" if world > 1 else "single GPU",
                       "l2": "A (6.6 GB) >> L2 (126 MB): every pass streams HBM, no flush"},
            "clocks": clocks.summary(),
            "e2e": {"value": round(e2e_value, 4), "unit": "TFLOP/s", "ms_per_step": round(1e3 * e2e_s, 2),
                    "h2d_bytes_per_step": m * n * 8,
                    "d2h_bytes_per_step": (m * k + n * k + k) * 8,
                    "api": "rsvd_b200_randomized_ksvd (host buffers, pinned A)"},
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roof,
            "cpu_baseline": cpu,
            "wall_s_timed": round(wall, 3),
            "sigma1": sigma_check,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--m", type=int, default=M)
    ap.add_argument("--n", type=int, default=N)
    ap.add_argument("--cpu-rows", type=int, default=16384)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
