"""Whole solves with the passes over A forced onto the INT8-emulated FP64 GEMMs
(RSVD_B200_GEMM=oz, csrc/gemm_oz.cu) at sizes the CPU oracle handles: the same FP64 parity bar
as every other solve (singular values 1e-10 relative, principal angles 1e-8 against the
reference restatement), on sketch widths that take one, two and four column chunks, power
iterations, wide inputs, the row-sharded pipeline, chunked host uploads, the Householder
fallback and the NaN check. Large inputs take this path by default (A >= 2^26 elements); the
full-size C2 parity against the reference library is tests/test_gpu_fullsize_parity.py."""
import numpy as np
import pytest

from test_gpu_parity import check_against
from test_gpu_sharded import check as check_sharded, run_group

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_oz(monkeypatch):
    monkeypatch.setenv("RSVD_B200_GEMM", "oz")


def planted(m, n, k, decay, seed):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    uu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    sig = np.exp(-np.arange(r) * (np.log(decay) / (k + 10)))
    return (uu * sig) @ vv.T


@pytest.mark.parametrize("m,n,k,p,q", [(3000, 700, 32, 10, 2), (4000, 900, 64, 10, 2),
                                       (2500, 1200, 138, 10, 1), (5000, 600, 20, 6, 0),
                                       (900, 3100, 40, 8, 2)])
def test_oz_solve_vs_oracle(solver, port, m, n, k, p, q):
    import paper_2110_03423_b200 as P
    a = planted(m, n, k, 1e4, m + n + k)
    res = solver.randomized_ksvd(a, P.RsvdConfig(k=k, oversample=p, power_q=q, seed=42))
    assert solver.last_info("oz_passes") == 2 * q + 2
    ref = port.randomized_ksvd(a, k, oversample=p, power_q=q, seed=42)
    check_against(res, ref.sigma, ref.u, ref.v, f"oz {m}x{n} k={k}")


@pytest.mark.parametrize("stored", ["1", "0"])
def test_oz_stored_digit_atx_passes(solver, port, monkeypatch, stored):
    """Every pass reads A's stored digits (both layouts written by the fused scan / convert
    pass) on the optimistic path, or forms them in-kernel (RSVD_B200_OZ_STORED=0): both meet
    the oracle bar, and the pass counts say which ran."""
    import paper_2110_03423_b200 as P
    monkeypatch.setenv("RSVD_B200_OZ_STORED", stored)
    a = planted(3000, 640, 40, 1e5, 77)
    q = 2
    res = solver.randomized_ksvd(a, P.RsvdConfig(k=40, power_q=q, seed=11))
    assert solver.last_info("robust_reruns") == 0
    assert solver.last_info("oz_passes") == 2 * q + 2
    assert solver.last_info("oz_stored_passes") == (2 * q + 2 if stored == "1" else 0)
    ref = port.randomized_ksvd(a, 40, power_q=q, seed=11)
    check_against(res, ref.sigma, ref.u, ref.v, f"stored={stored}")


def test_oz_wide_rows_scan_then_tile_conversion(solver, port):
    """Rows wider than 4608 columns are converted by the scan + the streaming tile kernel (the
    fused pass's L2 re-read would not fit); same oracle bar."""
    import paper_2110_03423_b200 as P
    rng = np.random.default_rng(31)
    r = 120
    a = (rng.standard_normal((6000, r)) * np.exp(-np.arange(r) / 12.0)) @ rng.standard_normal(
        (r, 4736)) + 1e-9 * rng.standard_normal((6000, 4736))
    res = solver.randomized_ksvd(a, P.RsvdConfig(k=24, power_q=1, seed=5))
    assert solver.last_info("oz_stored_passes") == 4
    ref = port.randomized_ksvd(a, 24, power_q=1, seed=5)
    check_against(res, ref.sigma, ref.u, ref.v, "wide rows")


def test_oz_robust_rerun_keeps_in_kernel_digits(solver):
    """A CholeskyQR breakdown reruns robustly with the column-scaled in-kernel digits (better
    relative accuracy of the small singular values than the stored, row-scaled ones)."""
    import paper_2110_03423_b200 as P
    a = planted(3000, 400, 20, 1e12, 13)
    solver.randomized_ksvd(a, P.RsvdConfig(k=20, oversample=10, power_q=3, seed=1))
    assert solver.last_info("robust_reruns") == 1
    assert solver.last_info("oz_stored_passes") == 0


def test_oz_badly_scaled_rows_and_columns(solver, port):
    """Rows and columns spanning 12 orders of magnitude: the per-row / per-column fixed-point
    scales keep every pass FP64-accurate in the normwise sense the SVD depends on."""
    import paper_2110_03423_b200 as P
    rng = np.random.default_rng(5)
    a = planted(2000, 500, 24, 1e3, 9)
    a *= np.exp(rng.uniform(-13, 13, 2000))[:, None]
    a *= np.exp(rng.uniform(-13, 13, 500))[None, :]
    res = solver.randomized_ksvd(a, P.RsvdConfig(k=24, power_q=2, seed=3))
    ref = port.randomized_ksvd(a, 24, power_q=2, seed=3)
    check_against(res, ref.sigma, ref.u, ref.v, "badly scaled")


def test_oz_sharded_matches_oracle(port):
    import paper_2110_03423_b200 as P
    a = planted(4000, 600, 30, 1e4, 21)
    cfg = P.RsvdConfig(k=30, power_q=2, seed=7)
    out, err, info = run_group(a, 3, cfg)
    assert not any(err), err
    ref = port.randomized_ksvd(a, 30, power_q=2, seed=7)
    check_sharded(out, 3, ref, 4000)


@pytest.mark.parametrize("m", [37888, 37000])
def test_oz_chunked_upload_bit_identical(solver, monkeypatch, m):
    """Host-buffer solves convert and sketch A chunk by chunk as it lands; the row scales are
    chunk-local and the chunks are whole tiles (the last one partial when m % 128 != 0, its
    pad rows zero digits), so the result equals the device solve's."""
    import torch
    import paper_2110_03423_b200 as P
    a = planted(m, 512, 64, 1e4, 4)
    cfg = P.RsvdConfig(k=64, oversample=10, power_q=2, seed=5)
    monkeypatch.setenv("RSVD_B200_UPLOAD_CHUNK_MB", "4")
    res = solver.randomized_ksvd(a, cfg)
    u_d, s_d, v_d, _ = solver.randomized_ksvd_device(torch.from_numpy(a).cuda(), cfg)
    assert np.array_equal(res.factors.sigma, s_d.cpu().numpy())
    assert np.array_equal(res.factors.u, u_d.cpu().numpy())
    assert np.array_equal(res.factors.v, v_d.cpu().numpy())


def test_oz_householder_fallback(solver, port):
    """An input that breaks CholeskyQR (sigma ratio 1e12): the robust rerun's Householder QRs
    run on the emulated passes too."""
    import paper_2110_03423_b200 as P
    a = planted(3000, 400, 20, 1e12, 13)
    res = solver.randomized_ksvd(a, P.RsvdConfig(k=20, oversample=10, power_q=3, seed=1))
    assert solver.last_info("householder_fallbacks") >= 1
    ref = port.randomized_ksvd(a, 20, oversample=10, power_q=3, seed=1)
    rel = np.abs(res.factors.sigma - ref.sigma) / ref.sigma
    live = ref.sigma > 1e-12 * ref.sigma[0]
    assert rel[live].max() <= 1e-10


def test_oz_nan_is_detected(solver):
    import paper_2110_03423_b200 as P
    a = planted(1000, 300, 10, 100, 2)
    a[517, 201] = np.nan
    with pytest.raises(P.ArgumentError):
        solver.randomized_ksvd(a, P.RsvdConfig(k=10, seed=1))
