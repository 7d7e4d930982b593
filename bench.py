#!/usr/bin/env python3
"""Benchmark of the B200 randomized k-SVD on BASELINE.json's configurations.

Default workload (config C2, the metric's 1-GPU case): a CelebA-shaped synthetic FP64
matrix A (202599 x 4096) with a controlled, exponentially decaying spectrum, rank k=64,
oversampling p=10, q=2 power iterations, seed 42. One step = one full `randomized_ksvd`
(Algorithm 1) with A resident in HBM. A (6.6 GB) is much larger than the 126 MB L2, so
every pass streams it from HBM (no explicit flush needed). A is generated on the host by
`synth_host` (numpy, fixed seed) so that both arms, the CPU baseline and the full-size parity
tests (tests/test_gpu_fullsize_parity.py) solve the same bits.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c1|c2|c3|c4|c5|c5ill]

Prints ONE JSON line (rank 0). value = whole-job TFLOP/s with the algorithmic flop count
F = (2q+2)*2*m*n*s + 2*m*s*k (s = k+p), i.e. the reference's arithmetic, not padded
tiles; ms_per_step is the device time of one solve (CUDA events, max over ranks). Repeated
device-resident solves replay the pipeline's cached CUDA graph (one launch per solve).
N > 1 (torchrun): A is row-sharded, each rank holding the config's m rows (weak scaling:
m_total = N*m), and the solve runs collectively with NCCL all-reduces of the Gram and
n x s partial sums (rsvd_b200_randomized_ksvd_sharded_device).
--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from
the unmodified reference sources; else the C restatement) on all host cores, on the same
full-size matrix and config (C1, C2; the larger configs time a stated row sample).
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

METRIC = "rSVD wall ms & TFLOP/s (frac of FP64 TC roofline), 1/2/4/8 B200 vs host CPU"
SEED = 42
# BASELINE.json configs (FP64 ones; C4 is the FP32 weak-scaling case)
CONFIGS = {
    "c1": dict(m=4096, n=4096, k=64, p=10, q=2, spectrum="exp", cpu_rows=4096,
               name="C1 rSVD 4096x4096 k=64 p=10 q=2 FP64 (exponential decay)"),
    "c2": dict(m=202599, n=4096, k=64, p=10, q=2, spectrum="exp", cpu_rows=202599,
               name="C2 rSVD 202599x4096 k=64 p=10 q=2 FP64 (CelebA-shaped)"),
    "c3": dict(m=202599, n=16384, k=128, p=20, q=2, spectrum="exp", cpu_rows=2048,
               name="C3 rSVD 202599x16384 k=128 p=20 q=2 FP64 (CelebA 128x128-shaped)"),
    "c5": dict(m=65536, n=65536, k=32, p=10, q=6, spectrum="slow", cpu_rows=1024,
               name="C5 rSVD 65536x65536 k=32 p=10 q=6 FP64 (slow decay 1/i^0.1)"),
    # C5's shape with sigma_1/sigma_s = 1e10: every CholeskyQR2 breaks down (cond(Y) >> 1e6),
    # so the solve is the optimistic attempt (aborted at the first Cholesky) + the robust
    # rerun with the blocked Householder fallback in every tall QR
    "c5ill": dict(m=65536, n=65536, k=32, p=10, q=6, spectrum="ill", ratio=1e10, cpu_rows=1024,
                  name="C5-ill rSVD 65536x65536 k=32 p=10 q=6 FP64 (sigma_1/sigma_s = 1e10, "
                       "CholeskyQR2 -> Householder fallback)"),
    # FP32 A, 3xTF32 tensor cores; m is per GPU (weak scaling up to 1.6M x 4096 at 8 GPUs).
    # sigma_1/sigma_s = 1e2 keeps the FP32 bar (1e-4 on sigma) meaningful.
    "c4": dict(m=200000, n=4096, k=256, p=16, q=4, spectrum="exp", ratio=1e2, cpu_rows=2048,
               f32=True, name="C4 rSVD 200000x4096 per GPU k=256 p=16 q=4 FP32 (3xTF32)"),
}


def flops(m, n, k, p, q):
    s = min(k + p, m, n)
    return (2 * q + 2) * 2.0 * m * n * s + 2.0 * m * s * k


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def spectrum(cfg, n, xp):
    """Controlled decaying spectra: "exp" sigma_i = exp(-i/tau) + 1e-6 with
    sigma_1/sigma_s = 1e4 over the sketch width; "slow" sigma_i = 1/(i+1)^0.1
    (synth.cpp:37's slow decay); "ill" sigma_i = ratio^(-i/(s-1)) floored at 1e-14
    (sigma_1/sigma_s = ratio over the sketch width)."""
    i = xp.arange(n, dtype=xp.float64)
    if cfg["spectrum"] == "slow":
        return 1.0 / (i + 1.0) ** 0.1
    if cfg["spectrum"] == "ill":
        s = cfg["k"] + cfg["p"]
        return xp.maximum(cfg["ratio"] ** (-i / (s - 1)), 1e-14)
    tau = (cfg["k"] + cfg["p"] - 1) / np.log(cfg.get("ratio", 1e4))
    return xp.exp(-i / tau) + 1e-6


# ----------------------------------------------------------------- synthetic inputs
def synth_host(cfg, rows=None, rank=0, out=None, threads=None):
    """The config's synthetic matrix on the host, identical bits for every arm and test
    (both bench arms, the CPU baseline and the full-size parity tests solve THIS matrix).

    Tall configs: A = G diag(sigma) V^T / sqrt(m) with G Gaussian (numpy PCG64, one
    SeedSequence child per 4096-row chunk, so the chunks are generated in parallel and the
    result does not depend on the thread count; rank r of a weak-scaled run draws its own
    children) and V Haar (QR of a Gaussian, shared by all ranks); n > 8192 uses V = (H D)^T
    instead (a Haar QR of n x n is too slow on the host). Columns of G/sqrt(m) are
    near-isometric, so the singular values are sigma up to (1 +- sqrt(n/m)).
    Square power-of-two configs: the exact Hadamard-conjugated construction of
    _hadamard_rows. `rows` (default m) takes the first rows of the rank's block; `out`
    (rows x n, float64 or float32, e.g. a pinned buffer) receives the matrix."""
    from concurrent.futures import ThreadPoolExecutor
    n, m = cfg["n"], cfg["m"]
    rows = m if rows is None else rows
    if out is None:
        out = np.empty((rows, n), dtype=np.float32 if cfg.get("f32") else np.float64)
    threads = threads or os.cpu_count() or 1
    if m == n and (n & (n - 1)) == 0:
        step = max(1, (1 << 24) // n)

        def had(r0):
            out[r0:min(rows, r0 + step)] = _hadamard_rows(cfg, r0, min(rows, r0 + step), np)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(had, range(0, rows, step)))
        return out
    sig = spectrum(cfg, n, np)
    rng = np.random.default_rng(SEED)
    signs = None
    if n > 8192:
        signs = rng.choice([-1.0, 1.0], size=n)
    else:
        vt = np.ascontiguousarray(np.linalg.qr(rng.standard_normal((n, n)))[0].T)
    chunk = 4096
    nchunks = (rows + chunk - 1) // chunk
    kids = np.random.SeedSequence([SEED, 1 + rank]).spawn(nchunks)
    scale = sig / np.sqrt(m)
    batch = max(1, min(threads, nchunks))
    buf = np.empty((batch * chunk, n))

    def gen(j, slot):
        r = min(chunk, rows - j * chunk)
        g = buf[slot * chunk: slot * chunk + r]
        np.random.default_rng(kids[j]).standard_normal(out=g)
        g *= scale
        return r

    with ThreadPoolExecutor(threads) as ex:
        for j0 in range(0, nchunks, batch):
            js = range(j0, min(nchunks, j0 + batch))
            got = sum(ex.map(lambda t: gen(t[1], t[0]), enumerate(js)))
            r0 = j0 * chunk
            if signs is not None:
                out[r0:r0 + got] = _fwht(buf[:got] * signs, np)
            else:
                out[r0:r0 + got] = buf[:got] @ vt
    return out


def _fwht(x, xp):
    """Normalised fast Walsh-Hadamard transform along the last axis (length 2^j)."""
    n = x.shape[-1]
    h = 1
    y = x.copy()
    while h < n:
        y = y.reshape(*y.shape[:-1], n // (2 * h), 2, h)
        a, b = y[..., 0, :].copy(), y[..., 1, :].copy()
        y[..., 0, :] = a + b
        y[..., 1, :] = a - b
        y = y.reshape(*y.shape[:-3], n)
        h *= 2
    return y / np.sqrt(n)


def _hadamard_rows(cfg, r0, r1, xp, device=None):
    """Rows [r0, r1) of A = D1 H diag(sigma) H D2 P (n = 2^j square): H the normalised
    Walsh-Hadamard matrix, D1/D2 random signs, P a random column permutation. H diag(s) H
    is the dyadic convolution A0[i, j] = f(i xor j), f = H (sigma / sqrt(n)) ... so
    A[i, j] = d1_i d2_j f(i xor pi(j)) is generated elementwise with singular values
    exactly sigma (to rounding)."""
    n = cfg["n"]
    d1, d2, perm, f = _hadamard_parts(cfg)
    i = np.arange(r0, r1)[:, None]
    return d1[r0:r1, None] * d2[None, :] * f[np.bitwise_xor(i, perm[None, :])]


_HAD_CACHE = {}


def _hadamard_parts(cfg):
    key = (cfg["n"], cfg["spectrum"], cfg["k"], cfg["p"], cfg.get("ratio"))
    if key not in _HAD_CACHE:
        n = cfg["n"]
        rng = np.random.default_rng(SEED + 7)
        d1 = rng.choice([-1.0, 1.0], size=n)
        d2 = rng.choice([-1.0, 1.0], size=n)
        perm = rng.permutation(n)
        f = _fwht(spectrum(cfg, n, np)[None, :], np)[0] / np.sqrt(n)
        _HAD_CACHE[key] = (d1, d2, perm, f)
    return _HAD_CACHE[key]


def synth_device(torch, cfg, m, rank, device):
    """synth_host's matrix (rank `rank`'s m rows) copied to `device` (tools/ scripts)."""
    out = synth_host(cfg, m, rank=rank)
    return torch.from_numpy(out).to(device)


def workload_config(cfgd, world):
    """The `config` object of BOTH arms' JSON lines (identical dicts: same workload)."""
    m, n = cfgd["m"], cfgd["n"]
    w = 4 if cfgd.get("f32") else 8
    return {"workload": cfgd["name"], "m": m * world, "m_per_gpu": m, "n": n, "k": cfgd["k"],
            "p": cfgd["p"], "q": cfgd["q"], "seed": SEED,
            "sketch_width": min(cfgd["k"] + cfgd["p"], m * world, n),
            "input": "bench.synth_host (same bits in both arms)",
            "l2": f"A ({m * n * w / 1e9:.1f} GB per GPU) >> L2 (126 MB): every pass streams "
                  "HBM, no flush"}


DATA = "synthetic (controlled decaying spectrum, seed 42; numpy host generator, same A in both arms)"


# ----------------------------------------------------------------- CPU reference
def cpu_reference_run(cfg, a, threads, reps=1, budget_s=None):
    """Time randsvd::randomized_ksvd (the unmodified reference library, all host threads) on
    the host matrix `a` with the config's k, p, q and seed. Returns per-solve seconds (at
    most `reps`; stops early once the next solve would overrun `budget_s`)."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    note = ""
    if a.dtype != np.float64:  # the reference is FP64-only: it runs on the FP32-rounded input
        a = a.astype(np.float64)
        note = " (FP64 reference on the FP32-rounded matrix; it has no FP32 path)"
    k, p, q = cfg["k"], cfg["p"], cfg["q"]
    times = []
    t_start = time.perf_counter()
    if kind == "reference":
        orc.set_max_threads(threads)
        cores = threads
        for _ in range(reps):
            if budget_s and times and (time.perf_counter() - t_start) + max(times) > budget_s:
                break
            t, _ = orc.timed_solve(a, k, p, q, SEED, reps=1)
            times += t
    else:
        cores = 1
        for _ in range(reps):
            if budget_s and times and (time.perf_counter() - t_start) + max(times) > budget_s:
                break
            t0 = time.perf_counter()
            orc.randomized_ksvd(a, k, p, q, SEED, values_only=False)
            times.append(time.perf_counter() - t0)
    rows = a.shape[0]
    f = flops(rows, cfg["n"], k, p, q)
    full = rows == cfg["m"]
    what = (f"the full {rows}x{cfg['n']} matrix" if full else
            f"a {rows}x{cfg['n']} row block (bounded sample) of the {cfg['name'].split()[0]} matrix")
    t = statistics.median(times)
    return {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
            "sample": f"{what}, k={k} p={p} q={q} seed={SEED}; median {t:.2f} s per solve over "
                      f"{len(times)} solve(s){note}",
            "seconds": t, "times": times, "same_config": full}


# ----------------------------------------------------------------- GPU helpers
def tf32x3_peak(torch, device):
    """TF32 dense tensor peak / 3 (three TF32 products per FP32 product). The TF32 rate is
    half the bf16 rate on Blackwell; the bf16 rate is MEASURED_PEAKS.json's (driver-measured
    cuBLAS bf16), falling back to a bf16 8192^3 matmul measured here."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    bf16 = None
    if os.path.exists(path):
        with open(path) as f:
            bf16 = json.load(f).get("bf16_tflops")
    src = "MEASURED_PEAKS.json bf16_tflops"
    if not bf16:
        a = torch.randn(8192, 8192, dtype=torch.bfloat16, device=device)
        c = a @ a
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ a
        e1.record()
        torch.cuda.synchronize()
        bf16 = 2 * 8192**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12
        src = "bf16 8192^3 matmul measured here"
        del a, c
    return bf16 / 2 / 3, f"bf16 {bf16:.0f} TF ({src}) / 2 (TF32) / 3 (3xTF32 products)"


def cublas_dgemm_peak(torch, device):
    """cuBLAS DGEMM 8192^3, best of 3 (library reference point for the FP64 roofline)."""
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
    """SM clock and clock-event (throttle) reasons sampled during the timed region: NVML every
    5 ms from a thread (the first sample lands right at the start, so even a 0.1 s region is
    covered), nvidia-smi -lms 200 as the fallback when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self.lines = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def sample():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), {k for k, v in bits.items() if r & v}))

            sample()  # validate the calls before relying on the thread
            self.nvml = nv

            def loop():
                while not self.stop.wait(0.005):
                    try:
                        sample()
                    except Exception:  # noqa: BLE001 - sampling must never break the bench
                        return
            self.samples.clear()
            self.t = threading.Thread(target=loop, daemon=True)
            sample()
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
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
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self.nvml.nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            mx.append(m_)
            reasons |= r_
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def load_traffic(config):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            t = json.load(f)
        return t.get(config)  # per-config entries: {"c2": {...}, "c4": {...}}
    return None


# ----------------------------------------------------------------- main arms
def run_reference(args):
    """The reference arm: randsvd::randomized_ksvd (oracle/_ref, the unmodified reference
    library) on the host cores, on the SAME matrix and config as our arm (bench.synth_host,
    seed 42; at N > 1 the concatenation of every rank's shard, i.e. the whole weak-scaled
    matrix). Rank 0 alone runs; the others exit. Warm-up solves run on a 4096-row block
    (bounded time); the K timed solves are full-size. If K full solves would overrun
    --ref-budget-s, the line reports how many ran ("steps") next to "steps_requested"."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    rows = args.cpu_rows or cfg["cpu_rows"]
    t0 = time.perf_counter()
    if world == 1:
        a = synth_host(cfg, rows)
    else:
        a = np.concatenate([synth_host(cfg, rows, rank=r) for r in range(world)])
    synth_s = time.perf_counter() - t0
    af = a.astype(np.float64) if a.dtype != np.float64 else a
    if args.warmup:
        cpu_reference_run(cfg, np.ascontiguousarray(af[:4096]), threads, reps=args.warmup)
    run = cpu_reference_run(cfg, af, threads, reps=args.steps, budget_s=args.ref_budget_s)
    f = flops(af.shape[0], cfg["n"], cfg["k"], cfg["p"], cfg["q"])
    value = f / run["seconds"] / 1e12
    conf = workload_config(cfg, world)
    if rows != cfg["m"]:
        conf["workload"] += f" (CPU row sample {rows})"
    out = {
        "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": len(run["times"]), "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * run["seconds"], 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": DATA, "config": conf,
        "parallelism": f"host threads ({threads})",
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": run["cores"],
                         "kind": run["kind"], "sample": run["sample"]},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "seconds_per_solve": [round(t, 3) for t in run["times"]],
        "synth_s": round(synth_s, 1),
        "host": {"cores": threads, "ram_gb": round(os.sysconf("SC_PAGE_SIZE")
                                                   * os.sysconf("SC_PHYS_PAGES") / 2**30, 1)},
    }
    print(json.dumps(out), flush=True)


def run_ours(args):
    import torch
    import paper_2110_03423_b200 as P

    rank, world, local_rank = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # sharded: the row-sharded NCCL solve (always for N > 1; --sharded forces it at N = 1, a
    # one-rank NCCL communicator, to exercise the multi-GPU path on a single GPU)
    sharded = world > 1 or args.sharded
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfgd = CONFIGS[args.config]
    m, n, k, p, q = cfgd["m"], cfgd["n"], cfgd["k"], cfgd["p"], cfgd["q"]
    f32 = cfgd.get("f32", False)
    m_total = m * world
    cfg = P.RsvdConfig(k=k, oversample=p, power_q=q, seed=SEED)
    F = flops(m_total, n, k, p, q)
    solver = P.Solver(local_rank)
    if sharded:
        P.attach_process_group(solver)

    def solve_dev(a):
        if f32:
            if sharded:
                return solver.randomized_ksvd_sharded_f32_device(a, m_total, cfg)
            return solver.randomized_ksvd_f32_device(a, cfg)
        if sharded:
            return solver.randomized_ksvd_sharded_device(a, m_total, cfg)
        return solver.randomized_ksvd_device(a, cfg)

    # e2e outputs: pinned host arrays allocated once and reused (the API's out= buffers)
    e2e_out = tuple(torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
                    for shape in ((m, cfgd["k"]), (cfgd["k"],), (n, cfgd["k"])))

    def solve_host(a_host):
        if f32:
            if sharded:
                return solver.randomized_ksvd_sharded_f32(a_host, m_total, cfg, out=e2e_out)
            return solver.randomized_ksvd_f32(a_host, cfg, out=e2e_out)
        if sharded:
            return solver.randomized_ksvd_sharded(a_host, m_total, cfg, out=e2e_out)
        return solver.randomized_ksvd(a_host, cfg, out=e2e_out)

    # A: bench.synth_host (the same bits the reference arm and the CPU baseline solve),
    # generated straight into pinned host memory (the e2e leg's input), then copied to HBM
    a_host_t = torch.empty((m, n), dtype=torch.float32 if f32 else torch.float64,
                           pin_memory=True)
    a_host = a_host_t.numpy()
    synth_host(cfgd, m, rank=rank, out=a_host)
    a = a_host_t.to(dev)
    peak_cublas = cublas_dgemm_peak(torch, dev) if not f32 else None
    torch.cuda.synchronize()
    lib_stream = torch.cuda.ExternalStream(solver.stream, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if sharded:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (also allocates the workspace and captures the solve's CUDA graph: from the
    # second solve of a shape/buffer set on, a solve is one graph launch of the pipeline)
    for _ in range(args.warmup):
        u, s, v, sw = solve_dev(a)
    launches_per_step = solver.last_launch_count()
    graphs0 = solver.last_info("graph_launches")

    # ---- timed region: K device-resident solves
    barrier()
    with ClockSampler(local_rank) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(lib_stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            u, s, v, sw = solve_dev(a)
        e1.record(lib_stream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        barrier()
    dev_ms = e0.elapsed_time(e1)
    graph_steps = solver.last_info("graph_launches") - graphs0
    robust = {"robust_reruns": solver.last_info("robust_reruns"),
              "householder_fallbacks": solver.last_info("householder_fallbacks")}

    # ---- the same K solves once more with per-launch CUDA events around every pass over A
    # (profiling level 2 runs the pipeline eagerly: events recorded by graph nodes cannot be
    # timed). The kernels are the same; the roofline numbers come from this pass.
    solver.set_profiling(2)
    solver.reset_stats()
    barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(lib_stream)
    for _ in range(args.steps):
        u, s, v, sw = solve_dev(a)
    p1.record(lib_stream)
    p1.synchronize()
    prof_ms = p0.elapsed_time(p1)
    stats = solver.kernel_stats("gemm_A")
    conv_stats = solver.kernel_stats("oz_convert")
    solver.set_profiling(0)
    barrier()
    step_ms = dev_ms / args.steps
    if world > 1:
        t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())
    value = F / (step_ms * 1e-3) / 1e12
    sigma1 = float(s[0].item())

    # ---- e2e: the public host-buffer API (pinned A in, U, sigma, V out), same config
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    del a, u, v
    torch.cuda.empty_cache()
    res = solve_host(a_host)  # warm the host path
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        res = solve_host(a_host)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = F / e2e_s / 1e12

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded row sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rows = min(m, args.cpu_rows or cfgd["cpu_rows"])
        cpu = cpu_reference_run(cfgd, a_host[:rows], os.cpu_count() or 1)
        for key in ("seconds", "times"):
            cpu.pop(key, None)

    if rank == 0:
        if f32:
            peak, peak_src = tf32x3_peak(torch, dev)
            kernel = "gemm_A (3xTF32 tcgen05 passes over A: ax + atx)"
        else:
            peak_dmma = solver.dmma_peak_tflops()
            peak = max(peak_dmma, peak_cublas)
            peak_src = ("max of the DMMA m16n8k16 issue-rate probe (rsvd_b200_dmma_peak, "
                        f"{peak_dmma:.2f}) and cuBLAS DGEMM 8192^3 ({peak_cublas:.2f}), both "
                        "measured in this run; MEASURED_PEAKS.json has no FP64 entry")
            kernel = "gemm_A (FP64 DMMA passes over A: ax + atx)"
        per_launch_ms = stats["ms"] / max(1, stats["count"])
        per_launch_flops = stats["flops"] / max(1, stats["count"])
        achieved = per_launch_flops / (per_launch_ms * 1e-3) / 1e12 if stats["count"] else None
        traffic = load_traffic(args.config)
        # FP64 passes over A on the INT8 tensor cores (Ozaki scheme): the dominant kernel's
        # roofline is the INT8 tensor peak; it executes 28 digit products over the padded width
        oz = (not f32) and solver.last_info("oz_passes") > 0
        fp64_equiv = None
        if oz and achieved:
            sw_ = int(sw)
            np_pad = -(-sw_ // 16) * 16 if sw_ <= 96 else -(-sw_ // 32) * 32
            ops_per_launch = per_launch_flops / sw_ * np_pad * 28
            peak_i8 = solver.imma_peak_tops()
            fp64_equiv = {"achieved_tflops": round(achieved, 3), "dmma_peak_tflops": round(peak, 3),
                          "frac_of_fp64_tc_peak": round(achieved / peak, 4),
                          "note": "algorithmic FP64 flop rate of the emulated passes; can exceed "
                                  "the FP64 tensor peak"}
            achieved = ops_per_launch / (per_launch_ms * 1e-3) / 1e12
            peak_fp64 = peak
            peak = peak_i8
            peak_src = ("tcgen05 kind::i8 M128 N256 K32 issue-rate probe (rsvd_b200_imma_peak), "
                        "measured in this run; MEASURED_PEAKS.json has no INT8 entry")
            stored = solver.last_info("oz_stored_passes") > 0
            kernel = ("gemm_A (FP64 passes over A emulated on the INT8 tensor cores: Ozaki "
                      "scheme, 7 balanced base-256 digits, 28 digit products; ax + atx"
                      + (", from A's digit planes stored once per solve)" if stored else ")"))
            if stored and conv_stats["count"]:
                fp64_equiv["digit_conversion"] = {
                    "kernel": "oz_scan_convert (row scales, NaN/Inf check and both stored "
                              "digit layouts in one pass over A; HBM-bound)",
                    "ms_per_solve": round(conv_stats["ms"] / args.steps, 4),
                    "bytes_per_solve": m * n * 8 + 2 * m * n * 7,
                    "GBps": round((m * n * 8 + 2 * m * n * 7) / (conv_stats["ms"] / args.steps * 1e-3)
                                  / 1e9, 1)}
        roof = {"bound": "tensor", "kernel": kernel,
                "achieved": round(achieved, 3) if achieved else None, "peak": round(peak, 3),
                "unit": "TOPS (INT8)" if oz else "TFLOP/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": traffic.get("gemm_A_bytes_per_launch") if traffic else None,
                "traffic_algorithmic": m * n * (4 if f32 else 7 if (oz and solver.last_info(
                    "oz_stored_passes") > 0) else 8),
                "peak_source": peak_src,
                "launches_timed": stats["count"], "ms_per_launch": round(per_launch_ms, 4),
                "share_of_step": round(stats["ms"] / prof_ms, 4) if prof_ms else None,
                "measured_on": ("a second run of the same K solves with CUDA events around "
                                "every pass over A (eager launches, "
                                f"{prof_ms / args.steps:.3f} ms per solve)"),
                "algorithmic_flops_per_launch": per_launch_flops,
                "step_frac": round(value / world / (peak_fp64 if oz else peak), 4)}
        if fp64_equiv:
            roof["fp64_equivalent"] = fp64_equiv
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": ("f32 (A; 3xTF32 tensor cores, f64 small side)" if f32 else
                      "f64 (passes over A: INT8-emulated FP64, Ozaki scheme)"
                      if solver.last_info("oz_passes") > 0 else "f64"),
            "data": DATA, "config": workload_config(cfgd, world),
            "parallelism": f"row-sharded x{world} (NCCL)" if sharded else "single GPU",
            "sketch_width": sw,
            "clocks": clocks.summary(),
            "e2e": {"value": round(e2e_value, 4), "unit": "TFLOP/s",
                    "ms_per_step": round(1e3 * e2e_s, 2),
                    "h2d_bytes_per_step": m * n * (4 if f32 else 8),
                    "d2h_bytes_per_step": (m * k + n * k + k) * 8,
                    "api": ("rsvd_b200_randomized_ksvd" + ("_sharded" if sharded else "")
                            + ("_f32" if f32 else "")
                            + " (host buffers: pinned A in, pinned reused out= U, sigma, V)")},
            "gpu_launches": launches_per_step * args.steps,
            "cuda_graph": {"timed_steps_as_graph_launch": graph_steps,
                           "kernels_per_solve": launches_per_step},
            "roofline": roof,
            "cpu_baseline": cpu,
            "robust_path": robust,
            "wall_s_timed": round(wall, 3),
            "sigma1": sigma1,
        }
        print(json.dumps(out), flush=True)
    if sharded:
        solver.detach()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-sharded NCCL solve even at one GPU (tests the N > 1 path)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--cpu-rows", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=1500.0,
                    help="reference arm: stop timing full-size solves past this many seconds")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
