"""PCA on the GPU (§8f row 3): randsvd::pca (pca.hpp:13-28, pca.cpp:10-52) — centering,
randomized k-SVD of the centered data, explained variance sigma^2/(N-1), projection —
against the oracle's rSVD of the host-centered data."""
import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu


def data(n, d, seed):
    rng = np.random.default_rng(seed)
    r = min(n, d)
    uu, _ = np.linalg.qr(rng.standard_normal((n, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((d, r)))
    x = (uu * (10.0 * np.exp(-np.arange(r) / 6.0))) @ vv.T
    return x + rng.uniform(50, 100, size=d)  # a large per-feature offset, as in image data


@pytest.mark.parametrize("n,d,k", [(500, 120, 8), (2000, 700, 30), (60, 200, 5)])
def test_fit_pca_vs_oracle(solver, port, n, d, k):
    import paper_2110_03423_b200 as P
    from paper_2110_03423_b200 import pca
    x = data(n, d, n + d)
    model = pca.fit_pca(x, k, P.RsvdConfig(seed=3), solver)
    xc = x - x.mean(axis=0)
    ref = port.randomized_ksvd(xc, k, seed=3)
    np.testing.assert_allclose(model.mean, x.mean(axis=0), rtol=1e-13)
    var_ref = ref.sigma ** 2 / (n - 1)
    assert np.max(np.abs(model.explained_variance - var_ref) / var_ref) <= 2e-10
    assert np.all(np.diff(model.explained_variance) <= 0)
    assert principal_angle(model.components, ref.v) <= 1e-8
    assert np.abs(model.components.T @ model.components - np.eye(k)).max() <= 1e-10
    proj = pca.transform(model, x, solver)
    np.testing.assert_allclose(proj, xc @ model.components, rtol=0, atol=1e-9 * np.abs(xc).max())


def test_pca_errors(solver):
    import paper_2110_03423_b200 as P
    from paper_2110_03423_b200 import pca
    with pytest.raises(P.ArgumentError):
        pca.fit_pca(np.ones((1, 5)), 1, solver=solver)
    x = data(50, 20, 1)
    for k in (0, 21):
        with pytest.raises(P.ArgumentError):
            pca.fit_pca(x, k, solver=solver)
    model = pca.fit_pca(x, 3, solver=solver)
    with pytest.raises(P.DimensionError):
        pca.transform(model, np.ones((4, 19)), solver)
