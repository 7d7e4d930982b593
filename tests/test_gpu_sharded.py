"""Row-sharded rSVD on the GPU, on one B200.

The sharded pipeline is the same CUDA path the multi-GPU run uses, driven here by
`world` handles on cuda:0 from `world` host threads that reduce through an in-process
group (fixed-order device sums) — or through NCCL itself at world size 1. Tolerances are
the FP64 parity bar of BASELINE.json: sigma 1e-10 relative, principal angles 1e-8.
"""
import threading

import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu

SIG_RTOL = 1e-10
ANGLE_TOL = 1e-8


def planted(m, n, decay, seed):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    uu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (uu * decay(np.arange(r))) @ vv.T


def run_group(a, world, cfg, robust=False, m_total=None, spans=None, device=False):
    import paper_2110_03423_b200 as P
    m = a.shape[0]
    m_total = m if m_total is None else m_total
    spans = spans or [P.shard_rows(m, world, r) for r in range(world)]
    group = P.LocalGroup(world)
    solvers = [P.Solver(0) for _ in range(world)]
    for r, s in enumerate(solvers):
        s.attach_local(group, r)
        s.set_robust(robust)
    out, err = [None] * world, [None] * world

    def work(r):
        r0, r1 = spans[r]
        try:
            if device:
                import torch
                t = torch.from_numpy(np.ascontiguousarray(a[r0:r1])).cuda()
                u, s, v, sw = solvers[r].randomized_ksvd_sharded_device(t, m_total, cfg)
                torch.cuda.synchronize()
                out[r] = P.RsvdResult(P.SvdFactors(u.cpu().numpy(), s.cpu().numpy(),
                                                   v.cpu().numpy()), sw)
            else:
                out[r] = solvers[r].randomized_ksvd_sharded(a[r0:r1], m_total, cfg)
        except Exception as e:  # noqa: BLE001 — collected and re-raised by the test
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not any(t.is_alive() for t in th), "sharded solve hung"
    info = [(s.last_info("householder_fallbacks"), s.last_info("robust_reruns")) for s in solvers]
    for s in solvers:
        s.detach()
    return out, err, info


def gather(out, world, m, k):
    u = np.zeros((m, k))
    r0 = 0
    for r in range(world):
        ur = out[r].factors.u
        u[r0:r0 + ur.shape[0]] = ur
        r0 += ur.shape[0]
    return u


def check(out, world, ref, m, lead=None):
    k = ref.sigma.shape[0]
    lead = k if lead is None else lead
    for r in range(world):
        f = out[r].factors
        rel = np.abs(f.sigma[:lead] - ref.sigma[:lead]) / ref.sigma[:lead]
        assert rel.max() <= SIG_RTOL, (r, rel.max())
        # sigma and V are replicated bit-identically on every rank
        assert np.array_equal(f.sigma, out[0].factors.sigma)
        assert np.array_equal(f.v, out[0].factors.v)
    u = gather(out, world, m, k)
    assert principal_angle(u[:, :lead], ref.u[:, :lead]) <= ANGLE_TOL
    assert principal_angle(out[0].factors.v[:, :lead], ref.v[:, :lead]) <= ANGLE_TOL
    assert np.abs(u.T @ u - np.eye(k)).max() <= 1e-10
    v = out[0].factors.v
    assert np.abs(v.T @ v - np.eye(k)).max() <= 1e-10


@pytest.mark.parametrize("world,m,n,k,q", [(2, 3000, 700, 40, 2), (3, 2001, 512, 17, 1),
                                           (4, 4096, 1024, 64, 2)])
def test_sharded_matches_oracle(port, world, m, n, k, q):
    import paper_2110_03423_b200 as P
    a = planted(m, n, lambda i: np.exp(-i * np.log(1e4) / (k + 10)), m + world)
    cfg = P.RsvdConfig(k=k, power_q=q, seed=42)
    out, err, info = run_group(a, world, cfg)
    assert not any(err), err
    assert all(o.sketch_width == min(k + 10, n) for o in out)
    ref = port.randomized_ksvd(a, k, power_q=q, seed=42)
    check(out, world, ref, m)
    assert all(fb == 0 and rr == 0 for fb, rr in info)


def test_sharded_device_buffers(port):
    import paper_2110_03423_b200 as P
    m, n, k = 2500, 600, 30
    a = planted(m, n, lambda i: 1.0 / (1.0 + i) ** 2, 3)
    cfg = P.RsvdConfig(k=k, power_q=2, seed=5)
    out, err, _ = run_group(a, 2, cfg, device=True)
    assert not any(err), err
    check(out, 2, port.randomized_ksvd(a, k, power_q=2, seed=5), m)


def test_sharded_uneven_spans(port):
    import paper_2110_03423_b200 as P
    m, n, k = 1500, 400, 20
    a = planted(m, n, lambda i: np.exp(-i / 8.0), 9)
    cfg = P.RsvdConfig(k=k, power_q=2, seed=1)
    spans = [(0, 100), (100, 1400), (1400, 1500)]
    out, err, _ = run_group(a, 3, cfg, spans=spans)
    assert not any(err), err
    check(out, 3, port.randomized_ksvd(a, k, power_q=2, seed=1), m)


def test_sharded_tsqr_fallback(port):
    """Ill-conditioned sketch (q = 0): the optimistic run aborts, the robust rerun takes
    the TSQR Householder fallback on every rank, and still matches the reference."""
    import paper_2110_03423_b200 as P
    m, n, k = 600, 300, 20
    a = planted(m, n, lambda i: 10.0 ** (-i * 12.0 / 29), 5)
    cfg = P.RsvdConfig(k=k, power_q=0, seed=4)
    out, err, info = run_group(a, 2, cfg)
    assert not any(err), err
    assert all(fb >= 1 and rr == 1 for fb, rr in info), info
    check(out, 2, port.randomized_ksvd(a, k, power_q=0, seed=4), m, lead=8)


def test_sharded_errors_are_collective():
    import paper_2110_03423_b200 as P
    a = planted(400, 100, lambda i: 1.0 / (1 + i), 1)
    cfg = P.RsvdConfig(k=5, seed=2)
    # rows do not add up to m_total: every rank raises DimensionError
    _, err, _ = run_group(a, 2, cfg, m_total=401)
    assert all(isinstance(e, P.DimensionError) for e in err), err
    # a shard thinner than the sketch width
    _, err, _ = run_group(a, 2, cfg, spans=[(0, 10), (10, 400)])
    assert all(isinstance(e, P.DimensionError) for e in err), err
    # NaN in one shard is seen by every rank
    b = a.copy()
    b[350, 7] = np.nan
    _, err, _ = run_group(b, 2, cfg)
    assert all(isinstance(e, P.ArgumentError) and "NaN" in str(e) for e in err), err
    # wide input is rejected (row-sharding needs m_total >= n)
    _, err, _ = run_group(np.ascontiguousarray(a[:80]), 2, cfg)
    assert all(isinstance(e, P.DimensionError) for e in err), err


def test_nccl_world1_equals_single_device(solver):
    """Through NCCL itself (world size 1) the sharded solve is the single-device solve
    bit for bit: every all-reduce is the identity."""
    import paper_2110_03423_b200 as P
    a = planted(3000, 500, lambda i: np.exp(-i / 10.0), 4)
    cfg = P.RsvdConfig(k=25, power_q=2, seed=9)
    ref = solver.randomized_ksvd(a, cfg)
    s = P.Solver(0)
    s.attach_nccl(P.nccl_unique_id(), 0, 1)
    assert s.comm_info() == (0, 1)
    res = s.randomized_ksvd_sharded(a, a.shape[0], cfg)
    assert np.array_equal(res.factors.sigma, ref.factors.sigma)
    assert np.array_equal(res.factors.u, ref.factors.u)
    assert np.array_equal(res.factors.v, ref.factors.v)
    s.detach()
    assert s.comm_info() == (0, 1)


def test_nccl_sharded_solve_replays_as_graph():
    """With NCCL (capturable all-reduces) the sharded device-resident solve is captured
    once and replayed as one CUDA graph — all-reduces, the on-device flag reduction and
    the optimistic pipeline included — and the replay is the eager solve bit for bit."""
    import torch
    import paper_2110_03423_b200 as P
    a = planted(6000, 700, lambda i: np.exp(-i / 12.0), 8)
    cfg = P.RsvdConfig(k=30, power_q=2, seed=5)
    s = P.Solver(0)
    s.attach_nccl(P.nccl_unique_id(), 0, 1)
    t = torch.from_numpy(a).cuda()
    g0 = s.last_info("graph_launches")
    outs = [s.randomized_ksvd_sharded_device(t, a.shape[0], cfg) for _ in range(3)]
    torch.cuda.synchronize()
    assert s.last_info("graph_launches") - g0 >= 2  # second and third solve are replays
    s.set_graphs(False)
    eager = s.randomized_ksvd_sharded_device(t, a.shape[0], cfg)
    torch.cuda.synchronize()
    for o in outs:
        for x, y in zip(o[:3], eager[:3]):
            assert torch.equal(x, y)
    s.set_graphs(True)
    # an aborting (ill-conditioned) replay still reruns robustly and matches the oracle path
    rng = np.random.default_rng(3)
    m, n = 3000, 400
    uu, _ = np.linalg.qr(rng.standard_normal((m, n)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, n)))
    b = (uu * np.maximum(10.0 ** (-np.arange(n) / 3.0), 1e-15)) @ vv.T
    tb = torch.from_numpy(b).cuda()
    cfg2 = P.RsvdConfig(k=20, power_q=1, seed=2)
    r1 = s.randomized_ksvd_sharded_device(tb, m, cfg2)
    r2 = s.randomized_ksvd_sharded_device(tb, m, cfg2)
    torch.cuda.synchronize()
    assert s.last_info("robust_reruns") == 1
    assert torch.equal(r1[1], r2[1])
    s.detach()


@pytest.mark.parametrize("f32", [False, True])
def test_sharded_chunked_upload_world2(monkeypatch, f32):
    """Host-buffer sharded solves upload each shard in chunks that the sketch (and the
    first A^T Y0) consume as they land; forced into many small chunks at world 2 the
    result is bit-identical to the same shards solved from device buffers. (Shapes whose
    device-resident sketch runs un-split — 296+ row tiles per shard, like the BASELINE
    shards — as the chunked sketch always does; the FP32 chunks hold whole 2048-row
    splits of the first A^T Y0.)"""
    import torch
    import paper_2110_03423_b200 as P
    if f32:
        monkeypatch.setenv("RSVD_B200_UPLOAD_CHUNK_MB", "4")  # 4096 rows of 1 KB
        m, n, world = 2 * 163840, 256, 2  # 80 splits of 2048 rows per shard
        a = planted(m, n, lambda i: 1.0 / (1.0 + i) ** 1.5, 12).astype(np.float32)
        cfg = P.RsvdConfig(k=16, power_q=2, seed=3)
    else:
        monkeypatch.setenv("RSVD_B200_UPLOAD_CHUNK_MB", "1")  # 1024 rows of 1 KB
        m, n, world = 2 * 37888, 128, 2
        a = planted(m, n, lambda i: np.exp(-i / 15.0), 12)
        cfg = P.RsvdConfig(k=32, power_q=2, seed=7)
    group = P.LocalGroup(world)
    solvers = [P.Solver(0) for _ in range(world)]
    for r, s in enumerate(solvers):
        s.attach_local(group, r)
    spans = [P.shard_rows(m, world, r) for r in range(world)]
    host, dev, err = [None] * world, [None] * world, [None] * world

    def work(r):
        r0, r1 = spans[r]
        s = solvers[r]
        try:
            shard = np.ascontiguousarray(a[r0:r1])
            if f32:
                host[r] = s.randomized_ksvd_sharded_f32(shard, m, cfg)
                host[r] = (host[r], s.last_info("upload_aty_splits"))
                u, sg, v, _ = s.randomized_ksvd_sharded_f32_device(torch.from_numpy(shard).cuda(), m, cfg)
            else:
                host[r] = s.randomized_ksvd_sharded(shard, m, cfg)
                host[r] = (host[r], s.last_info("upload_aty_splits"))
                u, sg, v, _ = s.randomized_ksvd_sharded_device(torch.from_numpy(shard).cuda(), m, cfg)
            torch.cuda.synchronize()
            dev[r] = (u.cpu().numpy(), sg.cpu().numpy(), v.cpu().numpy())
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    for s in solvers:
        s.detach()
    assert not any(t.is_alive() for t in th)
    assert err == [None] * world, err
    for r in range(world):
        res, splits = host[r]
        assert splits > 0, r
        assert np.array_equal(res.factors.sigma, dev[r][1]), r
        assert np.array_equal(res.factors.u, dev[r][0]), r
        assert np.array_equal(res.factors.v, dev[r][2]), r
