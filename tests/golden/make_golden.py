"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libranddsvd_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on small seeded inputs and stores inputs and
outputs as .npz. Only this container has /root/reference; the GPU box uses the committed
fixtures. Re-run with `python tests/golden/make_golden.py` after changing the case list.

Inputs are built with the reference's own Gaussian stream (GaussianSampler via
ref_gaussian_matrix) and simple deterministic constructions, mirroring the reference's
tests (test_rsvd.cpp, test_dense_core.cpp).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle  # noqa: E402


def planted(R, m, n, sigma, seed):
    """U diag(sigma) V^T with U, V the Householder Q of reference Gaussian draws
    (the reference's test_helpers.hpp planted_matrix recipe, restated)."""
    g1 = R.gaussian_matrix(seed, m, n)
    u, _ = R.householder_qr(g1)
    # second draw continues the same stream in the reference; use seed+1 here instead
    g2 = R.gaussian_matrix(seed + 1, n, n)
    v, _ = R.householder_qr(g2)
    f = np.array([sigma[j] if j < len(sigma) else 0.0 for j in range(n)])
    return R.gemm(1.0, u * f, False, v, True)


def main():
    R = Oracle("reference")
    out = {}
    # ---- sampler known answers (rng.cpp; test_dense_core.cpp:277-282)
    kat = {
        "words_seed0": [int(x) for x in R.words(0, 8)],
        "words_seed42": [int(x) for x in R.words(42, 8)],
        "uniforms_seed42": R.uniforms(42, 8).tolist(),
    }
    import hashlib
    kat["omega_s42_4096x74_sha256"] = hashlib.sha256(R.gaussian_matrix(42, 4096, 74).tobytes()).hexdigest()
    np.savez_compressed(os.path.join(HERE, "sampler.npz"),
                        words_seed0=R.words(0, 1024), words_seed42=R.words(42, 1024),
                        uniforms_seed7=R.uniforms(7, 4096),
                        omega_s42_1024x74=R.gaussian_matrix(42, 1024, 74),
                        omega_s3_5x2=R.gaussian_matrix(3, 5, 2),
                        omega_s9_1001x7=R.gaussian_matrix(9, 1001, 7))

    cases = []

    def add(name, a, k, p=10, q=2, seed=0, eps=0.5, eps_mode=False):
        cfg = dict(k=k, oversample=p, power_q=q, seed=seed, epsilon=eps, epsilon_mode=eps_mode)
        r = R.randomized_ksvd(a, k, p, q, seed, eps, eps_mode)
        sv = R.randomized_ksvd(a, k, p, q, seed, eps, eps_mode, values_only=True)
        assert np.array_equal(sv.sigma, r.sigma)
        np.savez_compressed(os.path.join(HERE, f"rsvd_{name}.npz"), a=a, u=r.u, sigma=r.sigma,
                            v=r.v, sketch_width=r.sketch_width,
                            omega=R.gaussian_matrix(seed, min(a.shape),
                                                    R.sketch_width(k, p, eps, eps_mode, *a.shape)))
        cases.append(dict(name=name, shape=list(a.shape), **cfg))

    fast = np.diag([1.0 / (i + 1) ** 2 for i in range(100)])
    add("fastdiag100_k5", fast, 5, seed=1)                           # test_rsvd.cpp:177-187
    add("identity12_k3", np.eye(12), 3, seed=2)                      # test_rsvd.cpp:189-196
    add("diag321_k2", np.diag([3.0, 2.0, 1.0]), 2, seed=3)           # test_rsvd.cpp:249-256
    add("planted_fast_200x150_k10_q12",
        planted(R, 200, 150, [1.0 / (i + 1) ** 2 for i in range(150)], 31), 10, q=12, seed=5)
    add("planted_slow_80x50_k7", planted(R, 80, 50, [1.0 / (i + 1) ** 0.1 for i in range(50)], 21),
        7, seed=1234)
    add("planted_fast_40x25_k5", planted(R, 40, 25, [1.0 / (i + 1) ** 2 for i in range(25)], 13),
        5, seed=11)
    add("planted_fast_25x40_wide_k5",
        planted(R, 40, 25, [1.0 / (i + 1) ** 2 for i in range(25)], 13).T.copy(), 5, seed=11)
    lr = R.gemm(1.0, R.gaussian_matrix(55, 80, 4), False, R.gaussian_matrix(56, 4, 50), False)
    add("lowrank4_80x50_k4", lr, 4, seed=8)                          # test_rsvd.cpp:288-307
    add("lowrank4_80x50_k6", lr, 6, seed=8)
    add("gauss_200x120_k10_q0", R.gaussian_matrix(77, 200, 120), 10, q=0, seed=19)
    add("gauss_200x120_k10_q1", R.gaussian_matrix(77, 200, 120), 10, q=1, seed=19)
    add("eps_mode_120x80_k5", planted(R, 120, 80, [np.exp(-i / 8) for i in range(80)], 4), 5,
        seed=6, eps=0.25, eps_mode=True)
    add("expdecay_256x192_k24", planted(R, 256, 192, [np.exp(-i / 20) for i in range(192)], 42),
        24, seed=42)

    # ---- step functions (test_rsvd.cpp:46-136)
    col = R.gaussian_matrix(33, 15, 1)
    dup = np.hstack([col, col])
    y_rand = R.gaussian_matrix(2, 50, 6)
    a20 = R.gaussian_matrix(8, 20, 20)
    y0 = R.sketch(a20, 6, 9)
    np.savez_compressed(
        os.path.join(HERE, "steps.npz"),
        sketch_identity=R.sketch(np.eye(5), 2, 3),
        dup=dup, dup_basis=R.range_basis(dup),
        y_rand=y_rand, y_rand_basis=R.range_basis(y_rand),
        a20=a20, y0=y0, w_q1=R.power_iterate(a20, y0, 1), w_q0=R.power_iterate(a20, y0, 0))

    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(dict(kat={k: ([hex(x) for x in v] if k.startswith("words") else v)
                            for k, v in kat.items()}, cases=cases), f, indent=1)
    print(f"wrote {len(cases)} rsvd cases")


if __name__ == "__main__":
    main()
