"""CUDA-graph replay of repeated device-resident solves (solve_tall_graph in
csrc/rsvd_b200.cpp): the first solve of a shape/config/buffer set is captured, later ones
replay the graph. Replays must be bit-identical to the eager pipeline, reset their device
flags (NaN/Inf, Cholesky abort) every time, and fall back to the robust rerun exactly like
an eager optimistic attempt."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _synth(m, n, decay, seed, torch, dev):
    g = torch.Generator(device="cpu").manual_seed(seed)
    uu, _ = torch.linalg.qr(torch.randn(m, n, generator=g, dtype=torch.float64))
    vv, _ = torch.linalg.qr(torch.randn(n, n, generator=g, dtype=torch.float64))
    sig = torch.tensor(decay(np.arange(n)), dtype=torch.float64)
    return ((uu * sig) @ vv.T).to(dev).contiguous()


@pytest.fixture(scope="module")
def pair():
    import paper_2110_03423_b200 as P
    eager, graphed = P.Solver(0), P.Solver(0)
    eager.set_graphs(False)
    return eager, graphed


def _same(r1, r2):
    for x, y in zip(r1[:3], r2[:3]):
        assert np.array_equal(x.cpu().numpy(), y.cpu().numpy())


@pytest.mark.parametrize("m,n,k,q", [(3000, 700, 40, 2), (5000, 1200, 100, 1), (2048, 2048, 64, 2)])
def test_replay_bit_identical(pair, m, n, k, q):
    import torch
    import paper_2110_03423_b200 as P
    eager, graphed = pair
    a = _synth(m, n, lambda i: np.exp(-i / 30.0), 11, torch, torch.device("cuda", 0))
    cfg = P.RsvdConfig(k=k, power_q=q, seed=7)
    ref = eager.randomized_ksvd_device(a, cfg)
    g0 = graphed.last_info("graph_launches")
    outs = [graphed.randomized_ksvd_device(a, cfg) for _ in range(4)]
    # the first solve on a fresh workspace may run eagerly (lazy allocations inside the
    # pipeline invalidate its capture); every later one is a graph launch
    assert graphed.last_info("graph_launches") - g0 >= 3
    assert eager.last_info("graph_launches") == 0
    for r in outs:
        _same(ref, r)
    assert graphed.last_launch_count() == eager.last_launch_count()


def test_replay_f32_bit_identical(pair):
    import torch
    import paper_2110_03423_b200 as P
    eager, graphed = pair
    a = _synth(4000, 600, lambda i: np.exp(-i / 40.0), 3, torch, torch.device("cuda", 0)).float()
    cfg = P.RsvdConfig(k=48, oversample=16, power_q=2, seed=5)
    ref = eager.randomized_ksvd_f32_device(a, cfg)
    for _ in range(3):
        _same(ref, graphed.randomized_ksvd_f32_device(a, cfg))


def test_replay_resets_nonfinite_flag(pair):
    """A replay of a cached graph on data that now holds a NaN must raise, and the next
    clean replay must succeed (the flag memset is part of the graph)."""
    import torch
    import paper_2110_03423_b200 as P
    _, graphed = pair
    a = _synth(1500, 400, lambda i: 1.0 / (1 + i), 2, torch, torch.device("cuda", 0))
    cfg = P.RsvdConfig(k=20, power_q=1, seed=1)
    good = graphed.randomized_ksvd_device(a, cfg)
    graphed.randomized_ksvd_device(a, cfg)
    a[17, 33] = float("nan")
    with pytest.raises(P.ArgumentError):
        graphed.randomized_ksvd_device(a, cfg)
    a[17, 33] = 0.0
    a.copy_(_synth(1500, 400, lambda i: 1.0 / (1 + i), 2, torch, torch.device("cuda", 0)))
    _same(good, graphed.randomized_ksvd_device(a, cfg))


def test_replay_abort_reruns_robust(pair, port):
    """Cholesky breakdown inside a replayed graph: the abort flag sends the solve to the
    robust path (Householder fallback), same results as the eager solver."""
    import torch
    import paper_2110_03423_b200 as P
    eager, graphed = pair
    dev = torch.device("cuda", 0)
    a = _synth(600, 300, lambda i: 10.0 ** (-i * 12.0 / 29), 5, torch, dev)
    cfg = P.RsvdConfig(k=20, power_q=0, seed=4)
    ref = eager.randomized_ksvd_device(a, cfg)
    assert eager.last_info("robust_reruns") == 1
    for _ in range(2):
        r = graphed.randomized_ksvd_device(a, cfg)
        assert graphed.last_info("robust_reruns") == 1
        assert graphed.last_info("householder_fallbacks") >= 1
        _same(ref, r)


def test_graph_cache_alternating_outputs(pair):
    """Fresh output tensors per call (torch's allocator alternates buffer sets): every key
    is served from the small LRU cache, results stay identical."""
    import torch
    import paper_2110_03423_b200 as P
    eager, graphed = pair
    dev = torch.device("cuda", 0)
    a1 = _synth(2500, 500, lambda i: np.exp(-i / 20.0), 8, torch, dev)
    a2 = _synth(2500, 500, lambda i: np.exp(-i / 25.0), 9, torch, dev)
    cfg = P.RsvdConfig(k=30, power_q=2, seed=3)
    r1, r2 = eager.randomized_ksvd_device(a1, cfg), eager.randomized_ksvd_device(a2, cfg)
    keep = []
    for i in range(6):
        a, r = (a1, r1) if i % 2 == 0 else (a2, r2)
        out = graphed.randomized_ksvd_device(a, cfg)
        _same(r, out)
        keep.append(out)


def test_profiling_runs_eagerly(pair):
    """Per-launch timing (profiling level 2, bench.py's roofline numbers) needs eager launches:
    events recorded by graph nodes cannot be timed, so profiled solves bypass the graph."""
    import torch
    import paper_2110_03423_b200 as P
    _, graphed = pair
    a = _synth(20000, 1024, lambda i: np.exp(-i / 50.0), 4, torch, torch.device("cuda", 0))
    cfg = P.RsvdConfig(k=64, power_q=2, seed=42)
    ref = graphed.randomized_ksvd_device(a, cfg)
    graphed.randomized_ksvd_device(a, cfg)
    g0 = graphed.last_info("graph_launches")
    graphed.set_profiling(2)
    try:
        graphed.reset_stats()
        for _ in range(3):
            _same(ref, graphed.randomized_ksvd_device(a, cfg))
        st = graphed.kernel_stats("gemm_A")
    finally:
        graphed.set_profiling(0)
    assert graphed.last_info("graph_launches") == g0
    assert st["count"] == 3 * 6  # 2q + 2 passes over A per solve
    assert st["ms"] > 0
