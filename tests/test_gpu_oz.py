"""The INT8-emulated FP64 GEMM (csrc/gemm_oz.cu, Ozaki scheme: 7 balanced base-256 digits per
operand, exact int32 products on the tensor cores) against the exact product (long double,
64-bit significand) and against the FP64 DMMA-class bound. The emulation must be an FP64-grade
GEMM: elementwise |err| <= K * max|a_row| * max|b_col| * 2^-50 (operand rounding 2^-54 of the
row / column maximum plus the dropped digit products, analysis in gemm_oz.cu), and a
Frobenius-relative error within a small factor of an FP64 BLAS product's."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


HOOKS = ["rsvd_b200_debug_gemm_oz", "rsvd_b200_debug_gemm_ozd"]


@pytest.fixture(params=HOOKS, ids=["in-kernel digits", "stored digits"])
def hook(request):
    return request.param


def run(solver, mn, a, b, NP, cols, out_t=False, splits=1, hook=HOOKS[0]):
    import torch
    M = a.shape[1] if mn else a.shape[0]
    K = a.shape[0] if mn else a.shape[1]
    out = torch.full((NP, M) if out_t else (M, NP), float("nan"), dtype=torch.float64,
                     device="cuda")
    solver.wait_for_torch()
    st = getattr(solver.lib, hook)(
        solver.h, int(mn), C.c_void_p(a.data_ptr()), M, K, a.stride(0), C.c_void_p(b.data_ptr()),
        b.stride(0), NP, cols, C.c_void_p(out.data_ptr()), out.stride(0), int(out_t), splits)
    assert st == 0, solver.lib.rsvd_b200_last_error().decode()
    return (out.T if out_t else out).cpu().numpy()


def exact(a, b):
    return (a.astype(np.longdouble) @ b.astype(np.longdouble))


def check(got, a, b, label, row_scaled_k=False):
    """a: M x K, b: K x N (numpy float64). row_scaled_k: a = A^T with A's digits scaled per row
    of A, i.e. per contraction index k (the stored-digit atx pass): the fixed point of a_jk is
    relative to max_j |a_jk|, so the bound is K * max_k (max_j |a_jk|) |b_kc| * 2^-50 — the
    normwise FP64 bound — instead of the per-output-row one."""
    ex = exact(a, b)
    err = np.abs(got.astype(np.longdouble) - ex).astype(np.float64)
    K = a.shape[1]
    if row_scaled_k:
        bound = K * (np.abs(a).max(0)[:, None] * np.abs(b)).max(0, keepdims=True) * 2.0 ** -50
    else:
        bound = K * np.abs(a).max(1, keepdims=True) * np.abs(b).max(0, keepdims=True) * 2.0 ** -50
    assert np.all(err <= bound + 1e-300), (label, float((err / np.maximum(bound, 1e-300)).max()))
    if row_scaled_k:
        return
    f64 = a @ b
    e64 = np.linalg.norm((f64.astype(np.longdouble) - ex).astype(np.float64))
    eoz = np.linalg.norm(err)
    nrm = np.linalg.norm(ex.astype(np.float64))
    assert eoz <= max(8 * e64, 1e-15 * nrm), (label, eoz / nrm, e64 / nrm)


def lowrank_decay(rng, m, n, decay):
    r = min(m, n, 300)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (u * np.exp(-np.arange(r) / decay)) @ v.T


@pytest.mark.parametrize("M,K,NP,cols", [(600, 4096, 80, 74), (333, 1000, 16, 16),
                                         (700, 777, 48, 42), (128, 64, 64, 64),
                                         (2000, 96, 128, 120), (257, 4100, 96, 90)])
def test_ax_oz(solver, hook, M, K, NP, cols):
    import torch
    rng = np.random.default_rng(M + K + NP)
    a = lowrank_decay(rng, M, K, 60.0)
    a[3] *= 1e-9  # rows at very different scales
    kp = (K + 1) // 2 * 2 + 2  # TMA rows are 16-byte multiples; ld > K
    ap = np.zeros((M, kp))
    ap[:, :K] = a
    bt = np.zeros((NP, K + 4))
    bt[:cols, :K] = rng.standard_normal((cols, K))
    got = run(solver, False, torch.from_numpy(ap).cuda()[:, :K], torch.from_numpy(bt).cuda()[:, :K],
              NP, cols, hook=hook)
    check(got, a, bt[:, :K].T, f"ax {M}x{K} NP={NP}")
    assert np.all(got[:, cols:] == 0)


@pytest.mark.parametrize("K,M,NP,cols,splits", [(5000, 1024, 80, 74, 1), (5000, 1024, 80, 74, 7),
                                                (3000, 272, 48, 42, 9), (1000, 200, 16, 10, 1),
                                                (20000, 256, 128, 128, 3)])
@pytest.mark.parametrize("out_t", [False, True])
def test_atx_oz(solver, hook, K, M, NP, cols, splits, out_t):
    import torch
    rng = np.random.default_rng(K + M + NP)
    a = lowrank_decay(rng, K, M, 40.0)
    a[:, 5] *= 1e7  # columns at very different scales
    w = np.zeros((K, NP))
    w[:, :cols] = rng.standard_normal((K, cols))
    got = run(solver, True, torch.from_numpy(a).cuda(), torch.from_numpy(w).cuda(), NP, cols,
              out_t, splits, hook=hook)
    check(got, a.T, w, f"atx {K}x{M} NP={NP} splits={splits}", row_scaled_k=hook.endswith("ozd"))


def test_oz_zero_and_tiny(solver, hook):
    import torch
    rng = np.random.default_rng(3)
    a = rng.standard_normal((300, 512))
    a[7] = 0.0                      # an all-zero row
    a[11, :] = 1e-300 * rng.standard_normal(512)
    bt = rng.standard_normal((16, 512))
    got = run(solver, False, torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda(), 16, 16,
              hook=hook)
    assert np.all(got[7] == 0)
    check(got, a, bt.T, "zero/tiny rows")
