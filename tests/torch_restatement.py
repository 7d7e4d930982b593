"""TEST INFRASTRUCTURE ONLY — a full-size checker for configurations the CPU reference cannot
solve inside a test run (C3, C4, C5: minutes to tens of minutes of host time each).

A literal FP64 restatement of the reference's Algorithm 1 in torch on the GPU, using the
vendor libraries (cuBLAS DGEMM, cuSOLVER geqrf/gesvd) — i.e. an implementation that shares
no code with the product's kernels:

    Y0 = A Omega                                       rsvd.cpp:51-59
    W  = QR(Y0).q ; q x { Z = QR(A^T W).q ; W = QR(A Z).q }   rsvd.cpp:61-73
    Q  = W (range_basis keeps every column: full-rank inputs only, asserted)  rsvd.cpp:75-87
    B  = Q^T A ; (U_B, sigma, V_B) = svd(B) ; U = Q U_B[:, :k] ; V = V_B[:, :k]  rsvd.cpp:89-109
    sign: the largest-|entry| of each V column positive, first index on ties, U
          flipped with it                               svd.cpp:237-254

Householder QR gives each Q up to column signs; the signs cancel in every product that
follows (QR(A^T W) depends on W only through W W^T up to signs), and the final factors are
pinned by the sign convention, so the outputs are comparable with the reference's to
rounding. Omega is the reference's own (the oracle port's gaussian_matrix is bit-exact with
the reference's sampler, tests/test_oracle.py). tests/test_gpu_fullsize_parity.py checks
this restatement against the reference library itself at C1 and C2 before trusting it at
C3-C5.
"""
from __future__ import annotations


def rsvd_fp64(a, omega, k: int, q: int):
    """(u, sigma, v) of the reference algorithm on the CUDA tensor `a` (m x n, m >= n,
    float64 or float32 — computed in float64) with the host Omega `omega` (n x s)."""
    import torch

    dev = a.device
    om = torch.from_numpy(omega).to(dev)

    def qr_q(y):
        qf, r = torch.linalg.qr(y)
        d = torch.diagonal(r).abs()
        assert d.min().item() > 1e-13 * torch.linalg.norm(y).item(), "rank-deficient sketch"
        return qf

    def a_mul(x):  # A @ x in float64, A possibly float32 (rounded to float64 exactly)
        if a.dtype == torch.float64:
            return a @ x
        out = torch.empty(a.shape[0], x.shape[1], dtype=torch.float64, device=dev)
        step = 1 << 15
        for r0 in range(0, a.shape[0], step):
            out[r0:r0 + step] = a[r0:r0 + step].double() @ x
        return out

    def at_mul(w):  # A^T @ w
        if a.dtype == torch.float64:
            return a.T @ w
        acc = torch.zeros(a.shape[1], w.shape[1], dtype=torch.float64, device=dev)
        step = 1 << 15
        for r0 in range(0, a.shape[0], step):
            acc += a[r0:r0 + step].double().T @ w[r0:r0 + step]
        return acc

    w = qr_q(a_mul(om))
    for _ in range(q):
        z = qr_q(at_mul(w))
        w = qr_q(a_mul(z))
    bt = at_mul(w)  # B^T = A^T Q  (n x s)
    ub_t, sig, vh_t = torch.linalg.svd(bt, full_matrices=False)  # B^T = V_B diag U_B^T
    vb = ub_t[:, :k]
    ub = vh_t.T[:, :k]
    idx = vb.abs().argmax(dim=0)
    sgn = torch.sign(vb[idx, torch.arange(k, device=dev)])
    sgn[sgn == 0] = 1.0
    vb = vb * sgn
    u = w @ (ub * sgn)
    return u, sig[:k], vb


def principal_angle(x, y) -> float:
    """test_helpers.hpp:66-73 on CUDA tensors: atan2(sigma_max(y - x x^T y), sigma_min(x^T y))."""
    import math

    import torch
    xty = x.T @ y
    res = y - x @ xty
    sine = torch.linalg.svdvals(res)[0].item()
    cosine = min(max(torch.linalg.svdvals(xty)[-1].item(), 0.0), 1.0)
    return math.atan2(sine, cosine)
