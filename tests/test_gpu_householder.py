"""The blocked Householder QR (csrc/householder.cu; the CholeskyQR2 fallback and the
drop-in randsvd::householder_qr) against the reference's unblocked Householder QR
(/root/reference/proj/src/qr.cpp:27-102, through oracle/_ref).

The thin QR with diag(R) >= 0 is unique for a full-rank input, so Q and R are compared
elementwise with a cond-scaled tolerance; rank-deficient inputs (zero / repeated columns,
where the null directions are rounding-determined on both sides) are checked for the
reference's contract: Q^T Q = I, QR = A, R upper triangular with exact zeros below the
diagonal and a non-negative diagonal, and |r_kk| ~ 0 exactly where the reference's is.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _contract(q, r, a, tol=1e-12):
    n = a.shape[1]
    assert np.abs(q.T @ q - np.eye(n)).max() <= tol * max(1, n / 32)
    assert np.abs(q @ r - a).max() <= tol * max(1.0, np.abs(a).max()) * max(1, n / 32)
    assert np.all(np.tril(r, -1) == 0.0)
    assert np.all(np.diag(r) >= 0.0)


@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (300, 1), (64, 64), (65, 64), (1000, 32),
                                 (1000, 33), (2000, 74), (4096, 100), (3000, 288), (288, 288),
                                 (10000, 42), (20000, 150), (700, 300), (1200, 600),
                                 (1500, 800)])
def test_vs_reference(solver, reference, m, n):
    rng = np.random.default_rng(m * 1000 + n)
    a = rng.standard_normal((m, n))
    q, r = solver.householder_qr(a)
    rq, rr = reference.householder_qr(a)
    _contract(q, r, a)
    cond = np.linalg.cond(a)
    assert np.abs(r - rr).max() <= 1e-13 * cond * np.abs(rr).max() * max(1, n / 32)
    assert np.abs(q - rq).max() <= 1e-13 * cond * max(1, n / 32)


def test_graded_columns_vs_reference(solver, reference):
    """Columns scaled over 12 decades (the ill-conditioned sketches the fallback exists
    for): still the reference's factors to a cond-independent relative accuracy per column
    of R (Householder QR is column-scaling invariant in exact arithmetic)."""
    rng = np.random.default_rng(3)
    m, n = 5000, 74
    a = rng.standard_normal((m, n)) * 10.0 ** (-12.0 * np.arange(n) / (n - 1))
    q, r = solver.householder_qr(a)
    rq, rr = reference.householder_qr(a)
    _contract(q, r, a)
    colscale = np.abs(rr).max(axis=0)
    assert (np.abs(r - rr).max(axis=0) / colscale).max() <= 1e-11
    assert np.abs(q - rq).max() <= 1e-10


@pytest.mark.parametrize("kind", ["zero", "repeat", "lowrank"])
def test_rank_deficient(solver, reference, kind):
    rng = np.random.default_rng(11)
    m, n = 3000, 80
    a = rng.standard_normal((m, n))
    if kind == "zero":
        a[:, [0, 5, 40, 79]] = 0.0
    elif kind == "repeat":
        a[:, 33] = a[:, 2]
        a[:, 70] = a[:, 69]
    else:
        a = rng.standard_normal((m, 20)) @ rng.standard_normal((20, n))
    q, r = solver.householder_qr(a)
    rq, rr = reference.householder_qr(a)
    _contract(q, r, a, tol=1e-11)
    tiny = np.abs(np.diag(rr)) <= 1e-10 * np.abs(rr).max()
    assert np.array_equal(np.abs(np.diag(r)) <= 1e-10 * np.abs(r).max(), tiny)
    if kind == "zero":  # exact zero columns: H_k = I and r_kk = 0 on both sides
        assert np.all(np.diag(r)[[0, 5, 40, 79]] == 0.0)


def test_deterministic_and_device_api(solver):
    import torch
    rng = np.random.default_rng(5)
    a = rng.standard_normal((50000, 74))
    q1, r1 = solver.householder_qr(a)
    q2, r2 = solver.householder_qr(a)
    assert np.array_equal(q1, q2) and np.array_equal(r1, r2)
    # device variant with a row stride: the same bits
    big = torch.zeros((50000, 80), dtype=torch.float64, device="cuda")
    big[:, :74] = torch.from_numpy(a).cuda()
    qd, rd = solver.householder_qr_device(big[:, :74])
    torch.cuda.synchronize()
    assert np.array_equal(qd.cpu().numpy(), q1) and np.array_equal(rd.cpu().numpy(), r1)


@pytest.mark.parametrize("m,n", [(202599, 74), (65536, 42), (200000, 272), (4096, 148)])
def test_full_size_vs_cusolver(solver, m, n):
    """BASELINE shapes of the fallback (C2 / C5 sketches, the C4 and C3 widths): both panel
    storage modes (shared memory up to 800 rows per CTA, HBM beyond), against cuSOLVER's
    QR with the same diag(R) >= 0 normalisation; times printed."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(m + n)
    a = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    a *= 10.0 ** (-6.0 * torch.arange(n, device="cuda", dtype=torch.float64) / n)
    q, r = solver.householder_qr_device(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(solver.stream)
    e0.record(st)
    for _ in range(5):
        solver.householder_qr_device(a)
    e1.record(st)
    e1.synchronize()
    print(f"householder_qr {m}x{n}: {e0.elapsed_time(e1) / 5:.3f} ms")
    tq, tr = torch.linalg.qr(a)
    sgn = torch.sign(torch.diagonal(tr))
    sgn[sgn == 0] = 1
    tq, tr = tq * sgn, tr * sgn[:, None]
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    assert (q.T @ q - eye).abs().max().item() <= 1e-13 * n
    assert (q @ r - a).abs().max().item() <= 1e-13 * n * a.abs().max().item()
    colscale = tr.abs().amax(dim=0)
    assert ((r - tr).abs().amax(dim=0) / colscale).max().item() <= 1e-10
    assert (q - tq).abs().max().item() <= 1e-9


def test_errors(solver):
    import paper_2110_03423_b200 as P
    with pytest.raises(P.DimensionError):
        solver.householder_qr(np.ones((3, 5)))
    with pytest.raises(P.DimensionError):
        solver.householder_qr(np.ones((0, 0)))
