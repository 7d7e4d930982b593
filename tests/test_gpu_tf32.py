"""The 3xTF32 tcgen05 GEMM (csrc/gemm_tf32.cu) against an FP64 torch reference of the same
product. Tolerance: |err_ij| <= 1e-5 * (|op(A)| |B|)_ij — FP32-class accuracy (three TF32
products, each operand split as rna_tf32(x) + rna_tf32(x - hi), ~2^-21 per product plus
FP32 accumulation)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def run(solver, mn, a, b, NP, out64, out_t, splits=1):
    import torch
    M = a.shape[1] if mn else a.shape[0]
    dt = torch.float64 if out64 else torch.float32
    out = torch.full((NP, M) if out_t else (M, NP), float("nan"), dtype=dt, device="cuda")
    solver.wait_for_torch()  # inputs come from torch's stream; the solver's is non-blocking
    st = solver.lib.rsvd_b200_debug_gemm_tf32(
        solver.h, int(mn), C.c_void_p(a.data_ptr()), M, a.shape[0] if mn else a.shape[1],
        a.stride(0), C.c_void_p(b.data_ptr()), b.stride(0), NP, C.c_void_p(out.data_ptr()),
        out.stride(0), int(out64), int(out_t), splits)
    assert st == 0, solver.lib.rsvd_b200_last_error().decode()
    return out.T if out_t else out


def check(got, a64, b64, tol=TOL):
    ref = a64 @ b64
    bound = a64.abs() @ b64.abs()
    err = (got.double() - ref).abs()
    ratio = (err / bound.clamp_min(1e-300)).max().item()
    assert ratio <= tol, ratio


@pytest.mark.parametrize("M,K,NP", [(1000, 4096, 80), (333, 1000, 16), (700, 777, 272),
                                    (128, 64, 48), (2000, 96, 288)])
@pytest.mark.parametrize("out64,out_t", [(True, False), (False, False), (True, True)])
def test_ax_tf32(solver, M, K, NP, out64, out_t):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + K + NP)
    kp = (K + 3) // 4 * 4  # TMA rows are 16-byte multiples
    a = torch.randn(M, kp, device="cuda", generator=g)[:, :K]
    bt = torch.randn(NP, kp + 4, device="cuda", generator=g)[:, :K]  # ld > K
    got = run(solver, False, a, bt, NP, out64, out_t)
    check(got, a.double(), bt.double().T)


@pytest.mark.parametrize("K,M,NP,splits", [(5000, 4096, 80, 1), (5000, 4096, 80, 7),
                                           (3000, 272, 272, 9), (1000, 200, 16, 1),
                                           (20000, 1024, 272, 13)])
@pytest.mark.parametrize("out_t", [False, True])
def test_atx_tf32(solver, K, M, NP, splits, out_t):
    import torch
    g = torch.Generator(device="cuda").manual_seed(K + M + NP)
    a = torch.randn(K, M, device="cuda", generator=g)
    w = torch.randn(K, NP, device="cuda", generator=g)
    got = run(solver, True, a, w, NP, True, out_t, splits)
    check(got, a.double().T, w.double())


def test_gram_tf32(solver):
    """Y^T Y through the MN-major kernel with A = W = Y (the tall Gram of CholeskyQR). The
    diagonal sums ~1350 positive terms per split in the tensor core's FP32 accumulator, whose
    rounding is not unbiased: measured 1.4e-5 of the bound (~1e-5 relative on the diagonal),
    the figure DESIGN.md's CholeskyQR tolerance for the FP32 path is based on."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(3)
    y = torch.randn(50000, 272, device="cuda", generator=g)
    got = run(solver, True, y, y, 272, True, False, 37)
    check(got, y.double().T, y.double(), tol=3e-5)


def test_nan_flag_tf32(solver):
    import torch
    a = torch.randn(300, 256, device="cuda")
    a[17, 200] = float("inf")
    bt = torch.randn(16, 256, device="cuda")
    # the flag path is exercised through the solver; here only the product must not hang
    run(solver, False, a, bt, 16, True, False)


def test_cta_pair_variant_subprocess():
    """The opt-in cta_group::2 variant of the K-major kernel (RSVD_B200_TF32_2SM=1, read once
    per process) on the same shapes, in a child process."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, RSVD_B200_TF32_2SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(os.path.dirname(__file__), "test_gpu_tf32.py"),
                        "-k", "test_ax_tf32"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
