"""The paper's §4 evaluation protocol on the B200 (reference:
include/randsvd/bench.hpp:11-123, src/bench.cpp:50-265, src/synth.cpp:28-71).

For each (n, k fraction) cell of a preset grid: build a synthetic m x n matrix with the
preset's spectrum (fast 1/i^2, sharp 1e-4 + 1/(1 + e^{i+1-beta}), slow 1/i^0.1), time the
full-SVD competitor and the B200 ``singular_values_only`` (1 warm-up + `repetitions` runs,
mean / sample std), and record the speed-up ratio, its band and the worst relative error of
the top-k singular values against the full SVD — one CSV row per cell in the reference's
format (``CSV_HEADER``, 17 significant digits).

On the GPU the competitor is the paper's "GESVD-GPU": the vendor full SVD
(``torch.linalg.svdvals`` -> cuSOLVER). Matrices come from the library's own device
``synth_matrix`` (rsvd_b200_synth_matrix: the reference's construction, synth.cpp:58-71,
with the bit-identical sampler stream, the blocked Householder QR and the DMMA GEMM), so
a cell's matrix is the reference's cell matrix to rounding and the rows can be checked
against the reference's own run_grid CSV (tests/test_gpu_grid_parity.py).

  python -m paper_2110_03423_b200.grid --preset fast-2000 [--out grid.csv] [--reps 10]
"""
from __future__ import annotations

import argparse
import math
import statistics
import sys
from dataclasses import dataclass, field

CSV_HEADER = ("spectrum,m,n,k_fraction,k,competitor,mean_competitor_s,std_competitor_s,"
              "mean_ours_s,std_ours_s,ratio,band_lo,band_hi,max_rel_err")


@dataclass
class BenchStats:
    """randsvd::bench::BenchStats (bench.hpp:17-23)."""
    solver_name: str
    n_runs: int = 0
    mean_seconds: float = 0.0
    std_seconds: float = 0.0  # sample std (n - 1); 0 for a single run


@dataclass
class SpeedupRow:
    """randsvd::bench::SpeedupRow (bench.hpp:26-42)."""
    spectrum: str = ""
    m: int = 0
    n: int = 0
    k_fraction: float = 0.0
    k: int = 0
    competitor_name: str = ""
    mean_competitor_s: float = 0.0
    std_competitor_s: float = 0.0
    mean_ours_s: float = 0.0
    std_ours_s: float = 0.0
    ratio: float = 0.0
    band_lo: float = 0.0
    band_hi: float | None = None
    max_rel_err: float = 0.0


@dataclass
class GridConfig:
    """randsvd::bench::GridConfig (bench.hpp:68-79)."""
    spectrum: str = "fast"
    m: int = 500
    n_grid: list = field(default_factory=list)
    k_fractions: list = field(default_factory=lambda: [0.01, 0.03, 0.05, 0.10])
    oversample: int = 10
    power_q: int = 2
    seed: int = 0
    repetitions: int = 10
    tolerance: float = 1e-8
    beta: float | None = None


def summarize(name: str, seconds: list[float]) -> BenchStats:
    """bench.cpp:69-86: mean and sample standard deviation."""
    if not seconds:
        raise ValueError("summarize needs at least one sample")
    mean = sum(seconds) / len(seconds)
    std = statistics.stdev(seconds) if len(seconds) > 1 else 0.0
    return BenchStats(name, len(seconds), mean, std)


def speedup_ratio(competitor: BenchStats, ours: BenchStats) -> SpeedupRow:
    """bench.cpp:94-110: ratio = mean*/mean_ours with the +-std band."""
    if not ours.mean_seconds > 0.0:
        raise ValueError("speedup_ratio needs mean(ours) > 0")
    row = SpeedupRow(competitor_name=competitor.solver_name,
                     mean_competitor_s=competitor.mean_seconds,
                     std_competitor_s=competitor.std_seconds, mean_ours_s=ours.mean_seconds,
                     std_ours_s=ours.std_seconds)
    row.ratio = competitor.mean_seconds / ours.mean_seconds
    row.band_lo = ((competitor.mean_seconds - competitor.std_seconds) /
                   (ours.mean_seconds + ours.std_seconds))
    if ours.mean_seconds > ours.std_seconds:
        row.band_hi = ((competitor.mean_seconds + competitor.std_seconds) /
                       (ours.mean_seconds - ours.std_seconds))
    return row


def fmt17(v: float) -> str:
    return "%.17g" % v


def write_csv(rows: list[SpeedupRow], out) -> None:
    """bench.cpp:174-187."""
    out.write(CSV_HEADER + "\n")
    for r in rows:
        out.write(",".join([r.spectrum, str(r.m), str(r.n), fmt17(r.k_fraction), str(r.k),
                            r.competitor_name, fmt17(r.mean_competitor_s),
                            fmt17(r.std_competitor_s), fmt17(r.mean_ours_s),
                            fmt17(r.std_ours_s), fmt17(r.ratio), fmt17(r.band_lo),
                            fmt17(r.band_hi) if r.band_hi is not None else "",
                            fmt17(r.max_rel_err)]) + "\n")


def preset(name: str) -> GridConfig:
    """bench.cpp:239-260 (the code's q per spectrum: fast 12, sharp 4, slow 6)."""
    small, large = [100, 200, 400], [250, 500, 1000, 2000]
    table = {"fast-small": ("fast", 500, small, 12, 2.0), "sharp-small": ("sharp", 500, small, 4, 2.0),
             "slow-small": ("slow", 500, small, 6, 2.0), "fast-2000": ("fast", 2000, large, 12, 2.0),
             "sharp-2000": ("sharp", 2000, large, 4, 2.0), "slow-2000": ("slow", 2000, large, 6, 2.0),
             "perf-2000": ("fast", 2000, [2000], 12, 2.0)}
    if name not in table:
        raise ValueError(f"unknown bench preset '{name}'")
    spec, m, ns, q, beta = table[name]
    g = GridConfig(spectrum=spec, m=m, n_grid=list(ns), power_q=q)
    if name == "perf-2000":
        g.k_fractions = [0.01]
    return g


def spectrum(kind: str, r: int, beta: float, xp):
    """synth.cpp:28-40 (1-based index i)."""
    i = xp.arange(1, r + 1, dtype=xp.float64)
    if kind == "fast":
        return 1.0 / (i * i)
    if kind == "sharp":
        return 1e-4 + 1.0 / (1.0 + xp.exp(i + 1.0 - beta))
    if kind == "slow":
        return 1.0 / i ** 0.1
    raise ValueError(kind)


def synth_device(solver, m: int, n: int, kind: str, beta: float, seed: int, device):
    """synth::synth_matrix({m, n, kind, seed}) generated by the library on the device."""
    return solver.synth_matrix_device(m, n, kind, beta, seed, device=device)


def run_grid(cfg: GridConfig, solver=None, device: int = 0):
    """bench.cpp:112-172 with the GPU competitor. Returns (rows, errors)."""
    import torch
    from .rsvd import RsvdConfig, default_solver
    s = solver or default_solver()
    dev = torch.device("cuda", device)
    rows, errors = [], []

    def timed(fn, reps):
        fn()  # untimed warm-up
        torch.cuda.synchronize()
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1) * 1e-3)
        return out

    for n in cfg.n_grid:
        for frac in cfg.k_fractions:
            if not (0.0 < frac <= 1.0):
                raise ValueError(f"k fraction must lie in (0, 1], got {fmt17(frac)}")
            k = int(math.ceil(frac * n))
            try:
                beta = cfg.beta if cfg.beta is not None else float(k + 1)
                cell_seed = (cfg.seed + n * 1315423911 + k * 2654435761) % 2**64
                a = synth_device(s, cfg.m, n, cfg.spectrum, beta, cell_seed, dev)
                rc = RsvdConfig(k=k, oversample=cfg.oversample, power_q=cfg.power_q,
                                seed=cell_seed)
                ref = {}
                ours = {}

                def comp():
                    ref["s"] = torch.linalg.svdvals(a)

                def mine():
                    ours["s"] = s.randomized_ksvd_device(a, rc, values_only=True)[1]

                tc = timed(comp, cfg.repetitions)
                to = timed(mine, cfg.repetitions)
                row = speedup_ratio(summarize("full_svd_gpu", tc), summarize("rsvd_b200", to))
                row.spectrum, row.m, row.n, row.k_fraction, row.k = (cfg.spectrum, cfg.m, n,
                                                                     frac, k)
                so, sr = ours["s"].double(), ref["s"][:k].double()
                row.max_rel_err = float(((so - sr).abs() / sr).max())
                rows.append(row)
            except Exception as e:  # noqa: BLE001 — a failing cell is recorded, not fatal
                errors.append((n, frac, str(e)))
    return rows, errors


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--preset", default="perf-2000")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="-")
    args = ap.parse_args(argv)
    cfg = preset(args.preset)
    cfg.repetitions = args.reps
    rows, errors = run_grid(cfg)
    out = sys.stdout if args.out == "-" else open(args.out, "w")
    write_csv(rows, out)
    if out is not sys.stdout:
        out.close()
    flagged = sum(r.max_rel_err > cfg.tolerance for r in rows)
    for n, frac, msg in errors:
        print(f"bench: cell n={n} frac={fmt17(frac)} failed: {msg}", file=sys.stderr)
    print(f"bench: preset={args.preset} rows={len(rows)} flagged={flagged} errors={len(errors)} "
          f"q={cfg.power_q}", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
