"""FP32 input path (BASELINE config C4: FP32 A, k=256, p=16, q=4) against the FP64 oracle.

The oracle runs the reference algorithm in FP64 on the very same (FP32-rounded) matrix, so
the comparison measures the 3xTF32 tensor-core pipeline, not the input rounding. Parity bar
for FP32 (BASELINE.json north_star): singular values within 1e-4 relative, U and V principal
angles <= 1e-3. Spectra are kept to sigma_1/sigma_s <= 1e2..1e3 (SURVEY.md §7 hard part 6:
1e-4 relative in FP32 needs sigma_1/sigma_k <~ 1e3).
"""
import threading

import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu

SIG_RTOL = 1e-4
ANGLE_TOL = 1e-3


def planted32(m, n, decay, seed):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    uu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return ((uu * decay(np.arange(r))) @ vv.T).astype(np.float32)


def check(res, ref, lead=None):
    k = ref.sigma.shape[0]
    lead = k if lead is None else lead
    rel = np.abs(res.factors.sigma[:lead] - ref.sigma[:lead]) / ref.sigma[:lead]
    assert rel.max() <= SIG_RTOL, rel.max()
    assert principal_angle(res.factors.u[:, :lead], ref.u[:, :lead]) <= ANGLE_TOL
    assert principal_angle(res.factors.v[:, :lead], ref.v[:, :lead]) <= ANGLE_TOL
    f = res.factors
    assert np.abs(f.u.T @ f.u - np.eye(k)).max() <= 1e-4
    assert np.abs(f.v.T @ f.v - np.eye(k)).max() <= 1e-4
    assert np.all(np.diff(f.sigma) <= 0)


@pytest.mark.parametrize("m,n,k,p,q", [(3000, 700, 40, 10, 2), (4000, 1024, 256, 16, 4),
                                       (2500, 900, 100, 10, 1), (777, 333, 17, 10, 3),
                                       (600, 1500, 30, 10, 2)])
def test_f32_vs_oracle(solver, port, m, n, k, p, q):
    import paper_2110_03423_b200 as P
    a = planted32(m, n, lambda i: np.exp(-i * np.log(1e2) / (k + p)), m + n)
    cfg = P.RsvdConfig(k=k, oversample=p, power_q=q, seed=42)
    res = solver.randomized_ksvd_f32(a, cfg)
    assert res.sketch_width == min(k + p, m, n)
    assert solver.last_info("robust_reruns") == 0
    ref = port.randomized_ksvd(a.astype(np.float64), k, p, q, 42)
    check(res, ref)


def test_f32_device_matches_host(solver):
    torch = pytest.importorskip("torch")
    import paper_2110_03423_b200 as P
    a = planted32(3000, 800, lambda i: 1.0 / (1.0 + i) ** 1.5, 5)
    cfg = P.RsvdConfig(k=32, power_q=2, seed=3)
    host = solver.randomized_ksvd_f32(a, cfg)
    u, s, v, sw = solver.randomized_ksvd_f32_device(torch.from_numpy(a).cuda(), cfg)
    assert np.array_equal(s.cpu().numpy(), host.factors.sigma)  # same kernels, same bits
    assert np.array_equal(u.cpu().numpy(), host.factors.u)
    _, s2, _, _ = solver.randomized_ksvd_f32_device(torch.from_numpy(a).cuda(), cfg,
                                                    values_only=True)
    assert torch.equal(s, s2)


def test_f32_chunked_upload_bit_identical(solver, monkeypatch):
    """FP32 host solves upload A in row chunks the tf32 sketch consumes as they land; chunks
    are whole tile pairs, so the result equals the device-resident solve bit for bit."""
    torch = pytest.importorskip("torch")
    import paper_2110_03423_b200 as P
    a = planted32(5000, 256, lambda i: 1.0 / (1.0 + i) ** 1.5, 6)
    cfg = P.RsvdConfig(k=16, power_q=2, seed=8)
    monkeypatch.setenv("RSVD_B200_UPLOAD_CHUNK_MB", "1")  # 1024-row chunks: 5 of them
    host = solver.randomized_ksvd_f32(a, cfg)
    u, s, v, sw = solver.randomized_ksvd_f32_device(torch.from_numpy(a).cuda(), cfg)
    assert np.array_equal(s.cpu().numpy(), host.factors.sigma)
    assert np.array_equal(u.cpu().numpy(), host.factors.u)
    assert np.array_equal(v.cpu().numpy(), host.factors.v)


def test_f32_fallback_ill_conditioned(solver, port):
    """cond(Y) ~ 1e6 >> 300: the 3xTF32 CholeskyQR aborts and the robust rerun's FP64
    Householder QR takes over; the leading singular triplets still meet the FP32 bar."""
    import paper_2110_03423_b200 as P
    m, n, k = 1500, 600, 20
    a = planted32(m, n, lambda i: 10.0 ** (-i * 6.0 / 29), 11)
    cfg = P.RsvdConfig(k=k, power_q=0, seed=4)
    res = solver.randomized_ksvd_f32(a, cfg)
    assert solver.last_info("robust_reruns") == 1
    assert solver.last_info("householder_fallbacks") >= 1
    ref = port.randomized_ksvd(a.astype(np.float64), k, power_q=0, seed=4)
    check(res, ref, lead=6)


def test_f32_nan_rejected(solver):
    import paper_2110_03423_b200 as P
    a = planted32(400, 200, lambda i: 1.0 / (1 + i), 1)
    a[33, 44] = np.inf
    with pytest.raises(P.ArgumentError, match="NaN or Inf"):
        solver.randomized_ksvd_f32(a, P.RsvdConfig(k=5))


def test_f32_sharded_local_group(port):
    import paper_2110_03423_b200 as P
    m, n, k = 4000, 800, 60
    a = planted32(m, n, lambda i: np.exp(-i * np.log(1e2) / (k + 10)), 8)
    cfg = P.RsvdConfig(k=k, power_q=2, seed=42)
    world = 2
    group = P.LocalGroup(world)
    solvers = [P.Solver(0) for _ in range(world)]
    for r, s in enumerate(solvers):
        s.attach_local(group, r)
    out, err = [None] * world, [None] * world

    def work(r):
        r0, r1 = P.shard_rows(m, world, r)
        try:
            out[r] = solvers[r].randomized_ksvd_sharded_f32(a[r0:r1], m, cfg)
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not any(err), err
    ref = port.randomized_ksvd(a.astype(np.float64), k, 10, 2, 42)
    u = np.vstack([out[r].factors.u for r in range(world)])
    res = P.RsvdResult(P.SvdFactors(u, out[0].factors.sigma, out[0].factors.v), out[0].sketch_width)
    check(res, ref)
    assert np.array_equal(out[0].factors.v, out[1].factors.v)
    for s in solvers:
        s.detach()


def test_f32_upload_time_aty_bit_identical(solver, monkeypatch):
    """Chunks that hold whole splits of the first power iteration's (A^T Y0)^T (here 2048-row
    splits, 4096-row chunks): its slabs are produced during the upload, and the result still
    equals the device-resident solve bit for bit."""
    torch = pytest.importorskip("torch")
    import paper_2110_03423_b200 as P
    a = planted32(163840, 256, lambda i: 1.0 / (1.0 + i) ** 1.5, 9)
    cfg = P.RsvdConfig(k=16, power_q=2, seed=3)
    monkeypatch.setenv("RSVD_B200_UPLOAD_CHUNK_MB", "4")  # 4096 rows of 1 KB
    host = solver.randomized_ksvd_f32(a, cfg)
    assert solver.last_info("upload_aty_splits") == 80
    u, s, v, sw = solver.randomized_ksvd_f32_device(torch.from_numpy(a).cuda(), cfg)
    assert solver.last_info("upload_aty_splits") == 0
    assert np.array_equal(s.cpu().numpy(), host.factors.sigma)
    assert np.array_equal(u.cpu().numpy(), host.factors.u)
    assert np.array_equal(v.cpu().numpy(), host.factors.v)
