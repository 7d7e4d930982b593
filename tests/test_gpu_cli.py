"""The C++ drop-in end to end on the GPU: `randsvd_b200` (csrc/cli_rsvd.cpp) is written
against include/randsvd/*.hpp exactly as a reference caller would be, and mirrors the
reference CLI's rsvd / pca subcommands (cli.cpp:81-306): DMAT in, DMAT out, the one-line
summary, exit codes 1/2/3. Results are checked against the oracle; the pinned DMAT->HBM
loader is checked against the file."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, principal_angle
from paper_2110_03423_b200.dmat import read_dmat, write_dmat

pytestmark = pytest.mark.gpu

CLI = os.path.join(ROOT, "paper_2110_03423_b200", "_lib", "randsvd_b200")


def run(*args):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)


def planted(m, n, seed):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    uu, _ = np.linalg.qr(rng.standard_normal((m, r)))
    vv, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (uu * np.exp(-np.arange(r) / 5.0)) @ vv.T


def test_cli_rsvd_matches_oracle(tmp_path, port):
    a = planted(700, 300, 1)
    src = str(tmp_path / "a.dmat")
    write_dmat(src, a)
    pfx = str(tmp_path / "out")
    r = run("rsvd", src, "--k", 12, "--oversample", 8, "--power-q", 2, "--seed", 7,
            "--threads", 4, "--out", pfx)
    assert r.returncode == 0, r.stderr
    assert r.stderr.startswith("rsvd: shape=700x300 k=12 s=20 q=2 seed=7 residual=")
    u, s, v = (read_dmat(f"{pfx}.{x}.dmat") for x in ("u", "sigma", "v"))
    ref = port.randomized_ksvd(a, 12, 8, 2, 7)
    assert np.max(np.abs(s[:, 0] - ref.sigma) / ref.sigma) <= 1e-10
    assert principal_angle(u, ref.u) <= 1e-8 and principal_angle(v, ref.v) <= 1e-8
    # values-only and --k-frac (k = ceil(0.04 * 300) = 12), wide input transposed internally
    r = run("rsvd", src, "--k-frac", 0.04, "--oversample", 8, "--seed", 7, "--values-only",
            "--out", pfx + "2")
    assert r.returncode == 0, r.stderr
    assert "residual=n/a" in r.stderr
    assert np.array_equal(read_dmat(pfx + "2.sigma.dmat"), s)  # bit-identical sigma


def test_cli_pca(tmp_path, port):
    rng = np.random.default_rng(2)
    x = planted(400, 90, 3) + rng.uniform(10, 20, size=90)
    src = str(tmp_path / "x.dmat")
    write_dmat(src, x)
    r = run("pca", src, "--k", 6, "--seed", 1, "--out", str(tmp_path / "p"))
    assert r.returncode == 0, r.stderr
    comp = read_dmat(str(tmp_path / "p.components.dmat"))
    var = read_dmat(str(tmp_path / "p.variance.dmat"))[:, 0]
    ref = port.randomized_ksvd(x - x.mean(axis=0), 6, seed=1)
    assert np.max(np.abs(var - ref.sigma ** 2 / 399) / var) <= 2e-10
    assert principal_angle(comp, ref.v) <= 1e-8


def test_cli_exit_codes(tmp_path):
    assert run("rsvd").returncode == 1                                   # usage
    assert run("rsvd", "x.dmat", "--k", 3).returncode == 1               # no --out
    assert run("rsvd", str(tmp_path / "missing.dmat"), "--k", 3, "--out", "o").returncode == 2
    bad = str(tmp_path / "bad.dmat")
    open(bad, "wb").write(b"NOPE")
    assert run("rsvd", bad, "--k", 3, "--out", str(tmp_path / "o")).returncode == 2
    src = str(tmp_path / "a.dmat")
    write_dmat(src, planted(30, 20, 4))
    r = run("rsvd", src, "--k", 25, "--out", str(tmp_path / "o"))       # k > min(m, n)
    assert r.returncode == 3 and "error:" in r.stderr


def test_load_dmat_device_shards(tmp_path):
    torch = pytest.importorskip("torch")
    from paper_2110_03423_b200.dmat import load_dmat_device
    a = np.random.default_rng(5).standard_normal((1000, 333))
    src = str(tmp_path / "a.dmat")
    write_dmat(src, a)
    full = load_dmat_device(src)
    assert torch.equal(full.cpu(), torch.from_numpy(a))
    part = load_dmat_device(src, 400, 250)
    assert torch.equal(part.cpu(), torch.from_numpy(a[400:650]))
