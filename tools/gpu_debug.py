"""Ad-hoc GPU bring-up script: exercises each stage against the oracle and prints errors."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
from oracle.oracle import Oracle  # noqa: E402
import paper_2110_03423_b200 as P  # noqa: E402

O = Oracle("port")
S = P.Solver(0)


def angle(x, y):
    xty = x.T @ y
    res = y - x @ xty
    sine = np.linalg.svd(res, compute_uv=False)[0] if res.size else 0.0
    cosine = min(max(np.linalg.svd(xty, compute_uv=False)[-1], 0.0), 1.0)
    return float(np.arctan2(sine, cosine))


def run(name, f):
    t = time.time()
    try:
        f()
        print(f"[ok] {name} ({time.time()-t:.2f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def words():
    w = S.splitmix_words(0, 4)
    print("  words", [hex(x) for x in w], "ref", [hex(x) for x in O.words(0, 4)])
    u = S.uniforms(42, 1000)
    print("  uniforms bit-eq", np.array_equal(u, O.uniforms(42, 1000)))


def omega():
    for (r, c, seed) in [(4096, 74, 42), (5, 2, 3), (1001, 7, 9)]:
        g = S.gaussian_matrix(seed, r, c)
        ref = O.gaussian_matrix(seed, r, c)
        diff = g != ref
        ulps = np.abs(g.view(np.int64) - ref.view(np.int64))
        print(f"  omega {r}x{c}: mismatch frac {diff.mean():.5f}, max ulp {ulps.max()}")


def omega_cr():
    from mpmath import mp, mpf
    import math
    mp.prec = 200
    seed, count = 42, 4000
    w = O.uniforms(seed, 2 * count)
    g = S.gaussian_matrix(seed, 1, 2 * count).ravel()
    ref = O.gaussian_matrix(seed, 1, 2 * count).ravel()
    exact = np.empty(2 * count)
    for p in range(count):
        u1, u2 = w[2 * p], w[2 * p + 1]
        lg = float(mp.log(mpf(u1)))
        radius = math.sqrt(-2.0 * lg)
        angle = (2.0 * math.pi) * u2
        exact[2 * p] = radius * float(mp.cos(mpf(angle)))
        exact[2 * p + 1] = radius * float(mp.sin(mpf(angle)))
    print(f"  device vs correctly-rounded: mismatch {np.mean(g != exact):.5f}; glibc vs CR: {np.mean(ref != exact):.5f}; device vs glibc {np.mean(g != ref):.5f}")


def sketch():
    rng = np.random.default_rng(1)
    for (m, n, s) in [(300, 200, 12), (4096, 512, 74), (37, 29, 5)]:
        a = rng.standard_normal((m, n))
        y = S.sketch(a, s, 7)
        yr = O.sketch(a, s, 7)
        print(f"  sketch {m}x{n} s={s}: max rel err {np.abs(y-yr).max()/np.abs(yr).max():.3e}")
    I = np.eye(5)
    y = S.sketch(I, 2, 3)
    print("  sketch(I) == omega:", np.array_equal(y, O.gaussian_matrix(3, 5, 2)),
          np.abs(y - O.gaussian_matrix(3, 5, 2)).max())


def qr_paths():
    rng = np.random.default_rng(2)
    for (m, s) in [(500, 20), (5000, 74), (64, 64)]:
        y = rng.standard_normal((m, s))
        q = S.range_basis(y)
        qr = O.range_basis(y)
        print(f"  range_basis {m}x{s}: cols {q.shape[1]} vs {qr.shape[1]}, max diff "
              f"{np.abs(q-qr).max():.3e}, orth {np.abs(q.T@q-np.eye(q.shape[1])).max():.2e}")
    col = rng.standard_normal((15, 1))
    y = np.hstack([col, col])
    q = S.range_basis(y)
    print("  duplicate column ->", q.shape, O.range_basis(y).shape)


def full(m, n, k, p=10, q=2, seed=42, spectrum="exp"):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    if spectrum == "exp":
        sig = np.exp(-np.arange(r) / (r / 8))
    elif spectrum == "gauss":
        sig = None
    if sig is None:
        a = rng.standard_normal((m, n))
    else:
        u, _ = np.linalg.qr(rng.standard_normal((m, r)))
        v, _ = np.linalg.qr(rng.standard_normal((n, r)))
        a = (u * sig) @ v.T
    cfg = P.RsvdConfig(k=k, oversample=p, power_q=q, seed=seed)
    t = time.time()
    res = S.randomized_ksvd(a, cfg)
    tg = time.time() - t
    t = time.time()
    ref = O.randomized_ksvd(a, k, p, q, seed)
    tc = time.time() - t
    rel = np.abs(res.factors.sigma - ref.sigma) / np.abs(ref.sigma)
    au = angle(res.factors.u, ref.u)
    av = angle(res.factors.v, ref.v)
    print(f"  rsvd {m}x{n} k={k} q={q}: sigma max rel {rel.max():.3e}, angle U {au:.2e} V {av:.2e}, "
          f"elementwise U {np.abs(res.factors.u-ref.u).max():.2e} V {np.abs(res.factors.v-ref.v).max():.2e} "
          f"sw {res.sketch_width}/{ref.sketch_width} gpu {tg:.2f}s cpu {tc:.2f}s")
    # validation mode: bit-exact omega
    s = cfg.sketch_width(m, n)
    S.set_omega(O.gaussian_matrix(seed, min(m, n), s))
    res2 = S.randomized_ksvd(a, cfg)
    S.set_omega(None)
    rel2 = np.abs(res2.factors.sigma - ref.sigma) / np.abs(ref.sigma)
    print(f"    validation-mode sigma max rel {rel2.max():.3e}")


def timing():
    import torch
    m, n, k = 202599, 4096, 64
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    cfg = P.RsvdConfig(k=k, oversample=10, power_q=2, seed=42)
    S.set_profiling(True)
    for i in range(3):
        torch.cuda.synchronize()
        t = time.time()
        u, s, v, sw = S.randomized_ksvd_device(a, cfg)
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"  C2 device solve {dt*1e3:.1f} ms, launches {S.last_launch_count()}, sweeps {S.last_info('jacobi_sweeps')}, reruns {S.last_info('robust_reruns')}")
    print("  profile:", {k2: round(v2, 3) for k2, v2 in S.last_profile().items()})


import sys as _s
if len(_s.argv) > 1 and _s.argv[1] == "timing":
    run("timing C2", lambda: timing())
    raise SystemExit
run("words", words)
run("omega", omega)
run("omega_cr", omega_cr)
run("sketch", sketch)
run("qr", qr_paths)
run("full small", lambda: full(200, 150, 10))
run("full wide", lambda: full(150, 300, 10))
run("full gauss", lambda: full(1000, 400, 20, spectrum="gauss"))
run("full C1", lambda: full(4096, 4096, 64))
run("full q0", lambda: full(2000, 500, 16, q=0))
run("lowrank", lambda: (lambda a: print("  lowrank sigma", S.randomized_ksvd(a, P.RsvdConfig(k=6, seed=8)).factors.sigma,
                                        O.randomized_ksvd(a, 6, seed=8).sigma))(
    np.random.default_rng(3).standard_normal((80, 4)) @ np.random.default_rng(4).standard_normal((4, 50))))


run("timing C2", timing)
