"""The single-CTA Cholesky kernel (csrc/linalg_small.cu: 16-wide panels, warp-0 diagonal
factor with lookahead, in-place blocked inversion) through its test hook, against torch's FP64
Cholesky: R^T R = G and R Rinv = I to a few ulps of cond-scaled size, R upper with a positive
diagonal, zero padding, and the breakdown flag (pivot below tol * max diag)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def chol(solver, g, NP, tol=1e-12):
    import torch
    s = g.shape[0]
    G = torch.zeros(NP, NP, dtype=torch.float64, device="cuda")
    G[:s, :s] = g
    R = torch.full((NP, NP), float("nan"), dtype=torch.float64, device="cuda")
    Ri = torch.full((NP, NP), float("nan"), dtype=torch.float64, device="cuda")
    st = C.c_int(-1)
    solver.wait_for_torch()
    rc = solver.lib.rsvd_b200_debug_cholesky(solver.h, C.c_void_p(G.data_ptr()), s, NP,
                                             C.c_void_p(R.data_ptr()), C.c_void_p(Ri.data_ptr()),
                                             tol, C.byref(st))
    from paper_2110_03423_b200.rsvd import _check
    _check(solver.lib, rc)
    return R, Ri, st.value


@pytest.mark.parametrize("s", [1, 2, 3, 7, 15, 16, 17, 31, 33, 48, 64, 74, 100, 128, 136, 148,
                               157])
def test_cholesky_sizes(solver, s):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(s)
    m = torch.randn(2 * s + 3, s, dtype=torch.float64, device="cuda", generator=gen)
    m = m * torch.logspace(0, -3, s, dtype=torch.float64, device="cuda")  # cond(G) ~ 1e6
    g = m.T @ m
    NP = (s + 15) // 16 * 16
    R, Ri, st = chol(solver, g, NP)
    assert st == 0
    Rs, Ris = R[:s, :s], Ri[:s, :s].T  # Ri holds Rinv^T
    assert torch.all(torch.triu(Rs) == Rs) and torch.all(torch.diagonal(Rs) > 0)
    assert torch.all(R[s:, :] == 0) and torch.all(R[:, s:] == 0)
    assert torch.all(Ri[s:, :] == 0) and torch.all(Ri[:, s:] == 0)
    ref = torch.linalg.cholesky(g, upper=True)
    # backward error of the factorisation and of the inverse
    err = ((Rs.T @ Rs - g).abs() / (torch.diagonal(g).sqrt()[:, None] *
                                     torch.diagonal(g).sqrt()[None, :])).max().item()
    assert err < 1e-13, err
    inv_err = (Rs @ Ris - torch.eye(s, dtype=torch.float64, device="cuda")).abs().max().item()
    assert inv_err < 1e-9, inv_err
    rel = ((Rs - ref).abs().max() / ref.abs().max()).item()
    assert rel < 1e-10, rel


def test_cholesky_breakdown(solver):
    import torch
    s = 40
    m = torch.randn(s, s - 5, dtype=torch.float64, device="cuda")
    g = m @ m.T  # rank s - 5: a pivot collapses
    R, Ri, st = chol(solver, g, 48)
    assert st == 1
    g2 = torch.eye(s, dtype=torch.float64, device="cuda")
    g2[7, 7] = float("nan")
    assert chol(solver, g2, 48)[2] == 1


def test_cholesky_rejects_too_wide(solver):
    import torch
    import paper_2110_03423_b200 as P
    g = torch.eye(300, dtype=torch.float64, device="cuda")
    with pytest.raises(P.ArgumentError):
        chol(solver, g, 304)


def jacobi(solver, r, NP):
    import torch
    from paper_2110_03423_b200.rsvd import _check
    s = r.shape[0]
    Rb = torch.zeros(NP, NP, dtype=torch.float64, device="cuda")
    Rb[:s, :s] = r
    sig = torch.full((NP,), float("nan"), dtype=torch.float64, device="cuda")
    U = torch.full((NP, NP), float("nan"), dtype=torch.float64, device="cuda")
    W = torch.full((NP, NP), float("nan"), dtype=torch.float64, device="cuda")
    sw = C.c_int(-2)
    solver.wait_for_torch()
    _check(solver.lib, solver.lib.rsvd_b200_debug_jacobi(
        solver.h, C.c_void_p(Rb.data_ptr()), s, NP, C.c_void_p(sig.data_ptr()),
        C.c_void_p(U.data_ptr()), C.c_void_p(W.data_ptr()), C.byref(sw)))
    return sig, U, W, sw.value


@pytest.mark.parametrize("s,NP", [(s, (s + 15) // 16 * 16) for s in
                                  [1, 2, 5, 8, 9, 42, 64, 65, 74, 80, 81, 96, 97, 112, 113, 148,
                                   200, 272, 320]] + [(70, 112), (100, 128)])
def test_jacobi_sizes(solver, s, NP):
    """All three Jacobi kernels (single CTA s <= 64, the cluster of ceil(s / 16) CTAs for
    64 < s <= 112 — every cluster size from 5 to 7, and NP beyond 16 ceil(s / 16) so the last
    CTA zero-fills the extra rows — and the block Jacobi beyond) on a graded triangular R (the
    shape the pipeline hands over: R_B of B^T = Q_B R_B): sigma against torch's SVD,
    R W = U diag(sigma), orthonormal U and W, descending order, zero padding."""
    import torch
    gen = torch.Generator(device="cuda").manual_seed(1000 + s)
    a = torch.randn(s, s, dtype=torch.float64, device="cuda", generator=gen)
    a = a * torch.logspace(0, -4, s, dtype=torch.float64, device="cuda")
    r = torch.linalg.qr(a.T).R.T.contiguous().T.contiguous()  # upper triangular, graded
    r = torch.triu(r)
    sig, U, W, sweeps = jacobi(solver, r, NP)
    assert 1 <= sweeps <= 30
    ref = torch.linalg.svdvals(r)
    got = sig[:s]
    assert torch.all(got[:-1] >= got[1:])
    assert torch.all(sig[s:] == 0)
    assert torch.all(U[s:] == 0) and torch.all(U[:, s:] == 0)
    assert torch.all(W[s:] == 0) and torch.all(W[:, s:] == 0)
    rel = ((got - ref).abs() / ref).max().item()
    assert rel < 1e-12, rel
    Us, Ws = U[:s, :s], W[:s, :s]
    eye = torch.eye(s, dtype=torch.float64, device="cuda")
    assert (Ws.T @ Ws - eye).abs().max().item() < 1e-12
    assert (Us.T @ Us - eye).abs().max().item() < 1e-10
    recon = (r @ Ws - Us * got[None, :]).abs().max().item() / ref[0].item()
    assert recon < 1e-13, recon


@pytest.mark.parametrize("s,zero_from", [(20, 15), (90, 70)])
def test_jacobi_rank_deficient(solver, s, zero_from):
    """Zero columns: sigma exactly 0 there, U column 0 (completed later by the pipeline);
    s = 90 runs on the cluster kernel."""
    import torch
    r = torch.triu(torch.randn(s, s, dtype=torch.float64, device="cuda"))
    r[:, zero_from:] = 0
    sig, U, W, sweeps = jacobi(solver, r, (s + 15) // 16 * 16)
    assert sweeps >= 1
    assert torch.all(sig[zero_from:s] == 0)
    assert torch.all(U[:s, zero_from:s] == 0)
