"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU oracles.

* ``Oracle("port")``      -> oracle/_build/librsvd_oracle.so, the plain-C restatement
                             (oracle/rsvd_oracle.c) of the reference path.
* ``Oracle("reference")`` -> oracle/_ref/libranddsvd_ref.so, the unmodified reference
                             library (/root/reference/proj/src) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module, and
only as the checker / CPU baseline. The product package (paper_2110_03423_b200) never
imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "librsvd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libranddsvd_ref.so")

_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_u64 = C.c_uint64

ERRORS = {1: "ArgumentError", 2: "DimensionError", 3: "ConvergenceError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def build(quiet: bool = True) -> None:
    """Compile the oracles (port always; the reference only where its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


@dataclass
class Result:
    u: np.ndarray | None
    sigma: np.ndarray
    v: np.ndarray | None
    sketch_width: int


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build()
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = "orc_" if kind == "port" else "ref_"
        f = self._f
        f("last_error").restype = C.c_char_p
        f("gemm").argtypes = [C.c_double, _dp, _sz, _sz, C.c_int, _dp, _sz, _sz, C.c_int,
                              C.c_double, _dp, _dp]
        f("householder_qr").argtypes = [_dp, _sz, _sz, _dp, _dp]
        f("dense_svd").argtypes = [_dp, _sz, _sz, _dp, _dp, _dp]
        f("extend_orthonormal").argtypes = [_dp, _sz, _sz, _sz, _dp]
        f("sketch_width").argtypes = [_sz, _sz, C.c_double, C.c_int, _sz, _sz]
        f("sketch_width").restype = _sz
        f("sketch").argtypes = [_dp, _sz, _sz, _sz, _u64, _dp]
        f("power_iterate").argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, _dp]
        f("range_basis").argtypes = [_dp, _sz, _sz, _dp, C.POINTER(_sz)]
        f("project_and_solve").argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, _dp, _dp, _dp,
                                           C.POINTER(_sz)]
        f("randomized_ksvd").argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _u64, C.c_double, C.c_int,
                                         C.c_int, _dp, _dp, _dp, C.POINTER(_sz)]
        f("residual_fro").argtypes = [_dp, _sz, _sz, _dp, _dp, _dp, _sz]
        f("residual_fro").restype = C.c_double
        f("gaussian_matrix").argtypes = [_u64, _sz, _sz, _dp]
        if kind == "port":
            f("splitmix_words").argtypes = [_u64, _u64, _sz, C.POINTER(_u64)]
            f("uniforms").argtypes = [_u64, _u64, _sz, _dp]
        else:
            f("splitmix_words").argtypes = [_u64, _sz, C.POINTER(_u64)]
            f("uniforms").argtypes = [_u64, _sz, _dp]
            f("set_max_threads").argtypes = [C.c_uint]
            f("sampler_normals").argtypes = [_u64, _sz, _sz, _sz, _dp]
            f("synth_matrix").argtypes = [_sz, _sz, C.c_int, C.c_double, _u64, _dp]
            f("run_grid_csv").argtypes = [C.c_char_p, _sz, C.c_char_p, _sz]
            f("run_grid_csv").restype = C.c_long
            f("matrix_new").argtypes = [_dp, _sz, _sz]
            f("matrix_new").restype = C.c_void_p
            f("matrix_free").argtypes = [C.c_void_p]
            f("randomized_ksvd_prepared").argtypes = [C.c_void_p, _sz, _sz, _sz, _u64, _dp]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(ERRORS.get(rc, "Error"), self._f("last_error")().decode())

    # ------------------------------------------------------------------ rng
    def words(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        op = out.ctypes.data_as(C.POINTER(_u64))
        if self.kind == "port":
            self._f("splitmix_words")(seed, 1, count, op)
        else:
            self._f("splitmix_words")(seed, count, op)
        return out

    def uniforms(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        if self.kind == "port":
            self._f("uniforms")(seed, 1, count, _ptr(out))
        else:
            self._f("uniforms")(seed, count, _ptr(out))
        return out

    def gaussian_matrix(self, seed: int, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64)
        self._f("gaussian_matrix")(seed, rows, cols, _ptr(out))
        return out

    def sampler_normals(self, seed: int, count: int, skip_words: int = 0,
                        skip_normals: int = 0) -> np.ndarray:
        """Reference only: `count` normals of GaussianSampler(seed) after `skip_words`
        next_u64() calls and `skip_normals` normal() calls (rng.cpp:22-46)."""
        out = np.empty(count, dtype=np.float64)
        self._f("sampler_normals")(seed, skip_words, skip_normals, count, _ptr(out))
        return out

    def synth_matrix(self, rows: int, cols: int, kind: str = "fast", beta: float = 1.0,
                     seed: int = 0) -> np.ndarray:
        """Reference only: synth::synth_matrix (synth.cpp:58-71)."""
        out = np.empty((rows, cols))
        k = {"fast": 0, "sharp": 1, "slow": 2}[kind]
        self._check(self._f("synth_matrix")(rows, cols, k, float(beta), seed % 2**64, _ptr(out)))
        return out

    def run_grid_csv(self, preset: str, reps: int = 1) -> str:
        """Reference only: bench::run_grid(preset) written by bench::write_csv."""
        buf = C.create_string_buffer(1 << 20)
        n = self._f("run_grid_csv")(preset.encode(), reps, buf, len(buf))
        if n < 0:
            raise RuntimeError(self._f("last_error")().decode() if n == -1 else "buffer")
        return buf.value.decode()

    # ------------------------------------------------------------ dense core
    def gemm(self, alpha, a, ta, b, tb, beta=0.0, c=None) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        out = np.empty((m, n))
        cc = None if c is None else np.ascontiguousarray(c, dtype=np.float64)
        self._check(self._f("gemm")(alpha, _ptr(a), a.shape[0], a.shape[1], int(ta), _ptr(b),
                                    b.shape[0], b.shape[1], int(tb), beta, _ptr(cc), _ptr(out)))
        return out

    def householder_qr(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, n = a.shape
        q = np.empty((m, n))
        r = np.empty((n, n))
        self._check(self._f("householder_qr")(_ptr(a), m, n, _ptr(q), _ptr(r)))
        return q, r

    def dense_svd(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, n = a.shape
        p = min(m, n)
        u, s, v = np.empty((m, p)), np.empty(p), np.empty((n, p))
        self._check(self._f("dense_svd")(_ptr(a), m, n, _ptr(u), _ptr(s), _ptr(v)))
        return u, s, v

    def extend_orthonormal(self, u, target):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty((u.shape[0], target))
        self._check(self._f("extend_orthonormal")(_ptr(u), u.shape[0], u.shape[1], target,
                                                  _ptr(out)))
        return out

    # ------------------------------------------------------------- rsvd steps
    def sketch_width(self, k, oversample, epsilon, epsilon_mode, m, n) -> int:
        return int(self._f("sketch_width")(k, oversample, epsilon, int(epsilon_mode), m, n))

    def sketch(self, a, s, seed):
        a = np.ascontiguousarray(a, dtype=np.float64)
        y = np.empty((a.shape[0], s))
        self._check(self._f("sketch")(_ptr(a), a.shape[0], a.shape[1], s, seed, _ptr(y)))
        return y

    def power_iterate(self, a, y0, q):
        a = np.ascontiguousarray(a, dtype=np.float64)
        y0 = np.ascontiguousarray(y0, dtype=np.float64)
        w = np.empty_like(y0)
        self._check(self._f("power_iterate")(_ptr(a), a.shape[0], a.shape[1], _ptr(y0),
                                             y0.shape[1], q, _ptr(w)))
        return w

    def range_basis(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        q = np.empty_like(y)
        cols = _sz(0)
        self._check(self._f("range_basis")(_ptr(y), y.shape[0], y.shape[1], _ptr(q),
                                           C.byref(cols)))
        return np.ascontiguousarray(q.reshape(-1)[: y.shape[0] * cols.value]
                                    .reshape(y.shape[0], cols.value))

    def project_and_solve(self, a, qb, k) -> Result:
        a = np.ascontiguousarray(a, dtype=np.float64)
        qb = np.ascontiguousarray(qb, dtype=np.float64)
        m, n = a.shape
        sq = qb.shape[1]
        kk = max(1, min(k, sq, n))
        u, s, v = np.empty((m, kk)), np.empty(kk), np.empty((n, kk))
        sw = _sz(0)
        self._check(self._f("project_and_solve")(_ptr(a), m, n, _ptr(qb), sq, k, _ptr(u),
                                                 _ptr(s), _ptr(v), C.byref(sw)))
        return Result(u, s, v, sw.value)

    def randomized_ksvd(self, a, k, oversample=10, power_q=2, seed=0, epsilon=0.5,
                        epsilon_mode=False, values_only=False) -> Result:
        a = np.ascontiguousarray(a, dtype=np.float64)
        m, n = a.shape
        kk = max(k, 1)
        u = None if values_only else np.empty((m, kk))
        v = None if values_only else np.empty((n, kk))
        s = np.empty(kk)
        sw = _sz(0)
        self._check(self._f("randomized_ksvd")(_ptr(a), m, n, k, oversample, power_q, seed,
                                               epsilon, int(epsilon_mode), int(values_only),
                                               _ptr(u), _ptr(s), _ptr(v), C.byref(sw)))
        return Result(u, s, v, sw.value)

    def residual_fro(self, a, u, sigma, v) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        return float(self._f("residual_fro")(_ptr(a), a.shape[0], a.shape[1], _ptr(u),
                                             _ptr(sigma), _ptr(v), len(sigma)))

    # ---------------------------------------------------- reference-only timing
    def set_max_threads(self, n: int) -> None:
        if self.kind == "reference":
            self._f("set_max_threads")(n)

    def timed_solve(self, a, k, oversample, power_q, seed, reps=1):
        """Wall-clock seconds of randsvd::randomized_ksvd on a prebuilt DenseMatrix
        (the timed region of cli.cpp:256-266). Reference library only."""
        import time
        assert self.kind == "reference"
        a = np.ascontiguousarray(a, dtype=np.float64)
        h = self._f("matrix_new")(_ptr(a), a.shape[0], a.shape[1])
        try:
            sig = np.empty(k)
            times = []
            for _ in range(reps):
                t0 = time.perf_counter()
                self._check(self._f("randomized_ksvd_prepared")(h, k, oversample, power_q, seed,
                                                                _ptr(sig)))
                times.append(time.perf_counter() - t0)
            return times, sig
        finally:
            self._f("matrix_free")(h)
