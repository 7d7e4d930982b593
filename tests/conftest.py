import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        try:
            from oracle.oracle import build
            build()
        except Exception:
            pass
    if not available("reference"):
        pytest.skip("reference library (oracle/_ref) not built on this host")
    return Oracle("reference")


@pytest.fixture(scope="session")
def solver():
    import paper_2110_03423_b200 as P
    return P.Solver(int(os.environ.get("RSVD_B200_DEVICE", "0")))


@pytest.fixture(scope="session")
def golden_cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        meta = json.load(f)
    out = []
    for c in meta["cases"]:
        d = dict(np.load(os.path.join(GOLDEN, f"rsvd_{c['name']}.npz")))
        out.append((c, d))
    return out


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)["kat"]


def principal_angle(x, y):
    """Largest principal angle between column spans, as test_helpers.hpp:66-73 computes it:
    atan2(sigma_max(y - x x^T y), sigma_min(x^T y))."""
    xty = x.T @ y
    res = y - x @ xty
    sine = np.linalg.svd(res, compute_uv=False)[0]
    cosine = min(max(np.linalg.svd(xty, compute_uv=False)[-1], 0.0), 1.0)
    return float(np.arctan2(sine, cosine))
