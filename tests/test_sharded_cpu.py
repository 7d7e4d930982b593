"""Row-sharded solve, host side, on CPU (gloo, world_size 2) — SURVEY.md §8e.

The GPU kernels cannot run here, so these tests pin the two host-side pieces of the
multi-GPU path:
  * the reduction plan: a numpy model of the sharded pipeline that all-reduces exactly
    the sums the CUDA path all-reduces (Gram of each CholeskyQR pass, (A_g^T Q_g)^T,
    Q_g^T A_g, the TSQR R stack) reproduces the single-process oracle's rSVD;
  * the communicator bootstrap: rank 0's NCCL unique id reaches every rank intact over
    a gloo process group, and shard_rows tiles [0, m).
The same pipeline on the GPU is covered by tests/test_gpu_sharded.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import principal_angle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _chol_upper(g):
    return np.linalg.cholesky(g).T  # G = R^T R, R upper, diag > 0


def _sign_fix(ub, v):
    """svd.cpp:237-254: the largest-|.| entry of each V column (first on ties) positive."""
    for c in range(v.shape[1]):
        j = int(np.argmax(np.abs(v[:, c])))
        if v[j, c] < 0:
            v[:, c] *= -1
            ub[:, c] *= -1
    return ub, v


def sharded_model(a_local, omega, k, q, allreduce, tsqr=False):
    """The CUDA path's reduction plan in numpy (rsvd_b200.cpp: tall_qr, tsqr,
    power_iterate_dev, project_and_solve_dev) for one rank's rows."""

    def tall_qr(y):
        if tsqr:  # Householder fallback: local QR, stack R over ranks, QR of the stack
            world, rank = dist.get_world_size(), dist.get_rank()
            qg, rg = np.linalg.qr(y)
            d = np.sign(np.diag(rg))
            qg, rg = qg * d, rg * d[:, None]
            s = y.shape[1]
            stack = np.zeros((world * s, s))
            stack[rank * s:(rank + 1) * s] = rg
            stack = allreduce(stack)
            qs, r = np.linalg.qr(stack)
            d = np.sign(np.diag(r))
            qs = qs * d
            return qg @ qs[rank * s:(rank + 1) * s]
        r1 = _chol_upper(allreduce(y.T @ y))  # CholeskyQR2, Grams all-reduced
        q1 = y @ np.linalg.inv(r1)
        r2 = _chol_upper(allreduce(q1.T @ q1))
        return q1 @ np.linalg.inv(r2)

    w = tall_qr(a_local @ omega)
    for _ in range(q):
        z = allreduce(a_local.T @ w)            # n x s partials
        z = np.linalg.qr(z)[0]                   # replicated wide QR
        w = tall_qr(a_local @ z)
    b = allreduce(w.T @ a_local)                 # s x n partials
    ub, sig, vt = np.linalg.svd(b, full_matrices=False)
    ub, v = _sign_fix(ub[:, :k].copy(), vt[:k].T.copy())
    return w @ ub, sig[:k], v


def _worker(rank, world, port, a, omega, k, q, tsqr, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_03423_b200 import shard_rows

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        r0, r1 = shard_rows(a.shape[0], world, rank)
        u, s, v = sharded_model(a[r0:r1], omega, k, q, allreduce, tsqr)
        out[rank] = (r0, r1, u, s, v)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tsqr", [False, True])
def test_sharded_reduction_plan_matches_oracle(port, tsqr):
    world, k, p, q, seed = 2, 6, 4, 2, 7
    m, n = 301, 120
    g = port.gaussian_matrix(11, m, n)
    sig = np.exp(-np.arange(n) / 3.0)
    a = port.gemm(1.0, g * sig, False, np.linalg.qr(port.gaussian_matrix(12, n, n))[0], True)
    ref = port.randomized_ksvd(a, k, p, q, seed)
    omega = port.gaussian_matrix(seed, n, k + p)  # every rank regenerates the same Omega
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), a, omega, k, q, tsqr, out), nprocs=world,
             join=True)
    u = np.zeros((m, k))
    for r in range(world):
        r0, r1, ur, sr, vr = out[r]
        u[r0:r1] = ur
        np.testing.assert_allclose(sr, ref.sigma, rtol=1e-10)
        np.testing.assert_allclose(vr, out[0][4], rtol=0, atol=0)  # replicated bit-identically
        assert principal_angle(vr, ref.v) < 1e-8
    assert principal_angle(u, ref.u) < 1e-8
    assert np.abs(u.T @ u - np.eye(k)).max() < 1e-10


def _id_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2110_03423_b200 as P
        from paper_2110_03423_b200.dist import broadcast_unique_id
        uid = P.nccl_unique_id() if rank == 0 else None
        out[rank] = (uid, broadcast_unique_id(uid))
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_broadcast_over_gloo():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_id_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    uid0 = out[0][0]
    assert len(uid0) == 128
    for r in range(world):
        assert out[r][1] == uid0


def test_shard_rows_tiles_the_rows():
    from paper_2110_03423_b200 import ArgumentError, shard_rows
    for m, world in [(10, 3), (202599, 8), (8, 8), (1600000, 8)]:
        spans = [shard_rows(m, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ArgumentError):
        shard_rows(3, 4, 0)
    with pytest.raises(ArgumentError):
        shard_rows(10, 2, 2)
