"""PCA on the B200 rSVD — the host mirror of the reference's randsvd::pca
(/root/reference/proj/include/randsvd/pca.hpp:13-28, src/pca.cpp:10-52), the paper's CelebA
application. Same names, fields and error behaviour; centering, the solve and the
projection run on the GPU (rsvd_b200_fit_pca / rsvd_b200_pca_transform)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .rsvd import ArgumentError, DimensionError, RsvdConfig, Solver, _arr, _check, _dp, default_solver


@dataclass
class PcaModel:
    """randsvd::pca::PcaModel (pca.hpp:13-17)."""
    mean: np.ndarray                # d
    components: np.ndarray          # d x k, orthonormal columns
    explained_variance: np.ndarray  # sigma_i^2 / (N - 1), non-increasing


def fit_pca(x, k: int, cfg: RsvdConfig | None = None, solver: Solver | None = None) -> PcaModel:
    """randsvd::pca::fit_pca (pca.cpp:28-41): randomized k-SVD of the centered data."""
    s = solver or default_solver()
    x = _arr(x)
    n, d = x.shape
    cfg = cfg or RsvdConfig()
    if n < 2:
        raise ArgumentError(f"center_columns needs at least 2 rows, got {n}")
    mean, comp, var = np.empty(d), np.empty((d, max(k, 1))), np.empty(max(k, 1))
    c = cfg._c()
    _check(s.lib, s.lib.rsvd_b200_fit_pca(s.h, _dp(x), n, d, k, C.byref(c), _dp(mean), _dp(comp),
                                          _dp(var)))
    return PcaModel(mean, comp[:, :k], var[:k])


def transform(model: PcaModel, x, solver: Solver | None = None) -> np.ndarray:
    """randsvd::pca::transform (pca.cpp:43-52): (x - mean) components."""
    s = solver or default_solver()
    x = _arr(x)
    d, k = model.components.shape
    if x.shape[1] != d:
        raise DimensionError(f"transform: data has {x.shape[1]} features, model has {d}")
    out = np.empty((x.shape[0], k))
    mean = np.ascontiguousarray(model.mean, dtype=np.float64)
    comp = np.ascontiguousarray(model.components, dtype=np.float64)
    _check(s.lib, s.lib.rsvd_b200_pca_transform(s.h, _dp(x), x.shape[0], d, _dp(mean), _dp(comp),
                                                k, _dp(out)))
    return out
