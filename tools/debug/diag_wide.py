"""Per-index sigma errors of wide-sketch solves vs the oracle, under kernel-path overrides
(RSVD_B200_CHOL_MAX / RSVD_B200_JACOBI_SMEM_MAX force the blocked Cholesky / block Jacobi)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2110_03423_b200 as P
    from oracle.oracle import Oracle
    m, n, k, q = (int(x) for x in sys.argv[2:6])
    rng = np.random.default_rng(m + n)
    r = min(m, n)
    uu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    sig = np.exp(-np.arange(r) * (np.log(1e4) / (k + 10)))
    a = (uu * sig) @ vv.T
    S = P.Solver(0)
    res = S.randomized_ksvd(a, P.RsvdConfig(k=k, power_q=q, seed=42))
    ref = Oracle("port").randomized_ksvd(a, k, power_q=q, seed=42)
    rel = np.abs(res.factors.sigma - ref.sigma) / ref.sigma
    absr = np.abs(res.factors.sigma - ref.sigma) / ref.sigma[0]
    truth = sig[:k]
    print(f"{os.environ.get('TAG','')}: max rel {rel.max():.2e} at {rel.argmax()} (abs/s1 {absr.max():.2e}); "
          f"ours-vs-truth {np.max(np.abs(res.factors.sigma-truth)/truth):.2e} ref-vs-truth {np.max(np.abs(ref.sigma-truth)/truth):.2e} "
          f"sweeps {S.last_info('jacobi_sweeps')}", flush=True)
    sys.exit(0)
for (m, n, k, q) in [(3000, 1000, 150, 2), (2800, 1100, 190, 1), (2800, 1100, 190, 2), (2600, 1200, 262, 2)]:
    for tag, env in [("default", {}), ("chol1", {"RSVD_B200_CHOL_MAX": "100000"}),
                     ("blockchol", {"RSVD_B200_CHOL_MAX": "64"}), ("blockjac", {"RSVD_B200_JACOBI_SMEM_MAX": "32"})]:
        e = dict(os.environ, TAG=f"{m}x{n} k={k} q={q} {tag}", **env)
        subprocess.run([sys.executable, __file__, "child", str(m), str(n), str(k), str(q)], env=e)
