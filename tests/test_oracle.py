"""CPU: pin the oracle restatement (oracle/rsvd_oracle.c) to the reference.

* bit-exact against the committed golden fixtures (made from the reference library);
* bit-exact against the live reference library where it can be built (this container);
* the reference's own known answers (test_dense_core.cpp:277-282).
"""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, principal_angle


def test_splitmix_known_answer(port, kat):
    # test_dense_core.cpp:281 — first word for seed 0
    assert int(port.words(0, 1)[0]) == 0xE220A8397B1DCDAF
    assert [hex(int(x)) for x in port.words(0, 8)] == kat["words_seed0"]
    assert [hex(int(x)) for x in port.words(42, 8)] == kat["words_seed42"]


def test_sampler_golden(port):
    g = np.load(os.path.join(GOLDEN, "sampler.npz"))
    assert np.array_equal(port.words(0, 1024), g["words_seed0"])
    assert np.array_equal(port.words(42, 1024), g["words_seed42"])
    assert np.array_equal(port.uniforms(7, 4096), g["uniforms_seed7"])
    for key, (seed, r, c) in {"omega_s42_1024x74": (42, 1024, 74), "omega_s3_5x2": (3, 5, 2),
                              "omega_s9_1001x7": (9, 1001, 7)}.items():
        # normals go through the host libm (same glibc on both sides)
        assert np.array_equal(port.gaussian_matrix(seed, r, c), g[key]), key


def test_normals_known_answer(port):
    # SURVEY.md Appendix A (reference run on this host)
    want = [0.41471975043153003, 0.65268122215194302, -0.89188621362775733,
            1.3268335628141055, 1.7295930879374031, -1.8834167889028144]
    assert port.gaussian_matrix(42, 1, 6).ravel().tolist() == want


def test_omega_c2_digest(port, kat):
    om = port.gaussian_matrix(42, 4096, 74)
    assert hashlib.sha256(om.tobytes()).hexdigest() == kat["omega_s42_4096x74_sha256"]


def test_oracle_matches_golden_rsvd(port, golden_cases):
    for c, d in golden_cases:
        r = port.randomized_ksvd(d["a"], c["k"], c["oversample"], c["power_q"], c["seed"],
                                 c["epsilon"], c["epsilon_mode"])
        assert np.array_equal(r.sigma, d["sigma"]), c["name"]
        assert np.array_equal(r.u, d["u"]), c["name"]
        assert np.array_equal(r.v, d["v"]), c["name"]
        assert r.sketch_width == int(d["sketch_width"]), c["name"]
        sv = port.randomized_ksvd(d["a"], c["k"], c["oversample"], c["power_q"], c["seed"],
                                  c["epsilon"], c["epsilon_mode"], values_only=True)
        assert np.array_equal(sv.sigma, d["sigma"]), c["name"]


def test_oracle_steps_golden(port):
    s = np.load(os.path.join(GOLDEN, "steps.npz"))
    assert np.array_equal(port.sketch(np.eye(5), 2, 3), s["sketch_identity"])
    assert np.array_equal(port.sketch(np.eye(5), 2, 3), port.gaussian_matrix(3, 5, 2))
    assert np.array_equal(port.range_basis(s["dup"]), s["dup_basis"])
    assert port.range_basis(s["dup"]).shape == (15, 1)
    assert np.array_equal(port.range_basis(s["y_rand"]), s["y_rand_basis"])
    assert np.array_equal(port.power_iterate(s["a20"], s["y0"], 1), s["w_q1"])
    assert np.array_equal(port.power_iterate(s["a20"], s["y0"], 0), s["w_q0"])


@pytest.mark.parametrize("shape", [(50, 30), (200, 150), (30, 50), (64, 64), (7, 3)])
def test_oracle_bit_exact_vs_reference(port, reference, shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.standard_normal(shape)
    if shape[0] >= shape[1]:
        qp, rp = port.householder_qr(a)
        qr, rr = reference.householder_qr(a)
        assert np.array_equal(qp, qr) and np.array_equal(rp, rr)
    up, sp, vp = port.dense_svd(a)
    ur, sr, vr = reference.dense_svd(a)
    assert np.array_equal(up, ur) and np.array_equal(sp, sr) and np.array_equal(vp, vr)
    k = min(shape) // 2
    rp = port.randomized_ksvd(a, k, seed=3)
    rr = reference.randomized_ksvd(a, k, seed=3)
    assert np.array_equal(rp.u, rr.u) and np.array_equal(rp.sigma, rr.sigma)
    assert np.array_equal(rp.v, rr.v) and rp.sketch_width == rr.sketch_width
    x = rng.standard_normal((shape[1], 4))
    assert np.array_equal(port.gemm(1.0, a, False, x, False), reference.gemm(1.0, a, False, x, False))
    assert np.array_equal(port.gemm(1.0, a, True, a, False), reference.gemm(1.0, a, True, a, False))


def test_oracle_errors(port):
    from oracle.oracle import OracleError
    a = np.eye(10)
    for k in (0, 11):
        with pytest.raises(OracleError, match="ArgumentError"):
            port.randomized_ksvd(a, k)
    with pytest.raises(OracleError, match="ArgumentError"):
        port.randomized_ksvd(a, 1, epsilon=1.0)
    b = a.copy()
    b[3, 4] = np.nan
    with pytest.raises(OracleError, match="ArgumentError"):
        port.randomized_ksvd(b, 2)
    with pytest.raises(OracleError, match="ArgumentError"):
        port.sketch(np.zeros((10, 6)), 7, 0)
    with pytest.raises(OracleError, match="DimensionError"):
        port.householder_qr(np.zeros((3, 5)))


def test_oracle_properties(port):
    # exact low-rank recovery incl. k beyond the rank (test_rsvd.cpp:288-307)
    a = port.gemm(1.0, port.gaussian_matrix(55, 80, 4), False, port.gaussian_matrix(56, 4, 50), False)
    r = port.randomized_ksvd(a, 6, seed=8)
    assert r.sigma[4] <= 1e-13 * r.sigma[0] and r.sigma[5] <= 1e-13 * r.sigma[0]
    assert port.residual_fro(a, r.u, r.sigma, r.v) / np.linalg.norm(a) <= 1e-10
    assert np.abs(r.u.T @ r.u - np.eye(6)).max() <= 1e-10
    # transpose consistency is bit-equal (test_rsvd.cpp:351-362)
    g = port.gaussian_matrix(13, 40, 25)
    t = port.randomized_ksvd(g, 5, seed=11)
    w = port.randomized_ksvd(g.T.copy(), 5, seed=11)
    assert np.array_equal(w.u, t.v) and np.array_equal(w.v, t.u)
    assert principal_angle(t.u, t.u) < 1e-12
