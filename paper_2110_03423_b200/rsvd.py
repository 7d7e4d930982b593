"""Python host mirror of the reference API over the C-ABI (include/rsvd_b200.h).

Same names, argument meaning and error behaviour as the reference's C++ entry points
(/root/reference/proj/include/randsvd/rsvd.hpp:13-63): ``RsvdConfig``,
``randomized_ksvd``, ``singular_values_only``, ``sketch``, ``power_iterate``,
``range_basis``, ``project_and_solve``; failures raise ``ArgumentError``,
``DimensionError`` or ``ConvergenceError`` like errors.hpp:16-37. Matrices are
row-major float64 numpy arrays (host) or CUDA torch tensors (device path).

Every call runs the sm_100a kernels in ``_lib/librsvd_b200.so``; there is no CPU
fallback. If the library or a B200 is missing the call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class Error(RuntimeError):
    """randsvd::Error"""


class ArgumentError(Error):
    """randsvd::ArgumentError"""


class DimensionError(Error):
    """randsvd::DimensionError"""


class ConvergenceError(Error):
    """randsvd::ConvergenceError"""


class DeviceError(Error):
    """CUDA / NCCL / allocation failure (no reference counterpart)."""


_STATUS = {1: ArgumentError, 2: DimensionError, 3: ConvergenceError}


def _check(lib, st: int) -> None:
    if st != 0:
        msg = lib.rsvd_b200_last_error().decode()
        raise _STATUS.get(st, DeviceError)(msg)


@dataclass
class RsvdConfig:
    """randsvd::RsvdConfig (rsvd.hpp:13-23) with the reference defaults."""
    k: int = 1
    oversample: int = 10
    power_q: int = 2
    seed: int = 0
    epsilon: float = 0.5
    epsilon_mode: bool = False

    def sketch_width(self, m: int, n: int) -> int:
        cap = min(m, n)
        if self.epsilon_mode:
            import math
            return min(int(math.ceil(self.k / self.epsilon)), cap)
        return min(self.k + self.oversample, cap)

    def _c(self) -> _lib.Config:
        return _lib.Config(self.k, self.oversample, self.power_q, self.seed & (2**64 - 1),
                           self.epsilon, int(bool(self.epsilon_mode)))


@dataclass
class SvdFactors:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray


@dataclass
class RsvdResult:
    factors: SvdFactors
    sketch_width: int = 0

    def residual_fro(self, a, solver: "Solver | None" = None) -> float:
        """||a - u diag(sigma) v^T||_F (rsvd.hpp:31-32, rsvd.cpp:37-49), on the GPU
        (rsvd_b200_residual_fro: fused GEMM epilogue, the product is never formed)."""
        a = _arr(a)
        f = self.factors
        if f.u.shape[0] != a.shape[0] or f.v.shape[0] != a.shape[1]:
            raise DimensionError(f"residual_fro: factors for {f.u.shape[0]}x{f.v.shape[0]} "
                                 f"against input {a.shape[0]}x{a.shape[1]}")
        return (solver or default_solver()).residual_fro(a, f.u, f.sigma, f.v)


def _arr(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise DimensionError(f"DenseMatrix requires rows >= 1 and cols >= 1, got shape {a.shape}")
    return a


def _dp(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _outputs(out, rows_u: int, n: int, k: int):
    """Output arrays (u rows_u x k, v n x k, sigma k): fresh numpy arrays, or the caller's
    preallocated ones (out=(u, sigma, v), C-contiguous float64 of those shapes) - e.g. views
    of pinned host memory reused across calls, which the device-to-host copies write at full
    PCIe speed and without first-touch page faults."""
    if out is None:
        return np.empty((rows_u, k)), np.empty((n, k)), np.empty(k)
    u, s, v = out
    for arr, shape, name in ((u, (rows_u, k), "u"), (s, (k,), "sigma"), (v, (n, k), "v")):
        if (not isinstance(arr, np.ndarray) or arr.dtype != np.float64 or arr.shape != shape
                or not arr.flags.c_contiguous or not arr.flags.writeable):
            raise ArgumentError(f"out {name} must be a writeable C-contiguous float64 array of "
                                f"shape {shape}")
    return u, v, s


class Solver:
    """One rsvd_b200_handle: a CUDA device, its stream and HBM workspace."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        _check(self.lib, self.lib.rsvd_b200_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.rsvd_b200_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- options
    def set_omega(self, omega: np.ndarray | None) -> None:
        """Validation mode: consume this Omega (n x s) instead of the device generator."""
        if omega is None:
            _check(self.lib, self.lib.rsvd_b200_set_omega(self.h, None, 0, 0))
            return
        om = _arr(omega)
        _check(self.lib, self.lib.rsvd_b200_set_omega(self.h, _dp(om), om.shape[0], om.shape[1]))

    def set_profiling(self, level: int) -> None:
        self.lib.rsvd_b200_set_profiling(self.h, int(level))

    def kernel_stats(self, tag: str = "gemm_A") -> dict:
        cnt, ms, fl = C.c_long(0), C.c_double(0), C.c_double(0)
        self.lib.rsvd_b200_kernel_stats(self.h, tag.encode(), C.byref(cnt), C.byref(ms),
                                        C.byref(fl))
        return {"count": cnt.value, "ms": ms.value, "flops": fl.value}

    def reset_stats(self) -> None:
        self.lib.rsvd_b200_reset_stats(self.h)

    def last_info(self, key: str) -> int:
        return int(self.lib.rsvd_b200_last_info(self.h, key.encode()))

    def set_robust(self, on: bool) -> None:
        """Force the host-checked robust path (Householder fallback) for every solve."""
        self.lib.rsvd_b200_set_robust(self.h, int(on))

    def set_graphs(self, on: bool) -> None:
        """Enable (default) / disable the CUDA-graph replay of repeated device-resident solves."""
        self.lib.rsvd_b200_set_graphs(self.h, int(on))

    def last_profile(self) -> dict:
        names = (C.c_char_p * 32)()
        ms = (C.c_double * 32)()
        n = self.lib.rsvd_b200_last_profile(self.h, names, ms, 32)
        return {names[i].decode(): ms[i] for i in range(n)}

    def dmma_peak_tflops(self) -> float:
        """Measured FP64 tensor-core peak of this GPU (rsvd_b200_dmma_peak)."""
        t = C.c_double(0)
        _check(self.lib, self.lib.rsvd_b200_dmma_peak(self.h, C.byref(t)))
        return t.value

    def imma_peak_tops(self) -> float:
        """Measured INT8 tensor-core peak of this GPU (rsvd_b200_imma_peak)."""
        t = C.c_double(0)
        _check(self.lib, self.lib.rsvd_b200_imma_peak(self.h, C.byref(t)))
        return t.value

    def last_launch_count(self) -> int:
        return int(self.lib.rsvd_b200_last_launch_count(self.h))

    def wait_for_torch(self, device=None) -> None:
        """Order this solver's stream after the work already queued on torch's current
        stream (device tensors handed to the _device entry points are produced there)."""
        import torch
        st = torch.cuda.current_stream(device)
        _check(self.lib, self.lib.rsvd_b200_wait_stream(self.h, C.c_void_p(st.cuda_stream)))

    @property
    def stream(self) -> int:
        return int(self.lib.rsvd_b200_stream(self.h) or 0)

    # --------------------------------------------------------------- hot path
    def randomized_ksvd(self, a, cfg: RsvdConfig, out=None) -> RsvdResult:
        a = _arr(a)
        m, n = a.shape
        k = max(int(cfg.k), 1)
        u, v, s = _outputs(out, m, n, k)
        sw = C.c_size_t(0)
        c = cfg._c()
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd(self.h, _dp(a), m, n, C.byref(c),
                                                            _dp(u), _dp(s), _dp(v), C.byref(sw)))
        return RsvdResult(SvdFactors(u, s, v), sw.value)

    def singular_values_only(self, a, cfg: RsvdConfig) -> np.ndarray:
        a = _arr(a)
        m, n = a.shape
        s = np.empty(max(int(cfg.k), 1))
        c = cfg._c()
        _check(self.lib, self.lib.rsvd_b200_singular_values_only(self.h, _dp(a), m, n, C.byref(c),
                                                                 _dp(s)))
        return s[: cfg.k]

    def randomized_ksvd_device(self, a, cfg: RsvdConfig, values_only: bool = False):
        """A already resident in HBM (a CUDA float64 torch tensor, row-major, possibly with a
        leading-dimension stride). Returns (u, sigma, v, sketch_width) as CUDA tensors."""
        import torch
        assert a.is_cuda and a.dtype == torch.float64 and a.dim() == 2 and a.stride(1) == 1
        self.wait_for_torch(a.device)
        m, n = a.shape
        k = int(cfg.k)
        dev = a.device
        sig = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        u = None if values_only else torch.empty((m, max(k, 1)), dtype=torch.float64, device=dev)
        v = None if values_only else torch.empty((n, max(k, 1)), dtype=torch.float64, device=dev)
        sw = C.c_size_t(0)
        c = cfg._c()
        dptr = lambda t: None if t is None else C.cast(t.data_ptr(), C.POINTER(C.c_double))
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd_device(
            self.h, dptr(a), m, n, a.stride(0), C.byref(c), dptr(u), dptr(sig), dptr(v),
            C.byref(sw)))
        return u, sig[:k], v, sw.value

    def residual_fro(self, a, u, sigma, v) -> float:
        """||a - u diag(sigma) v^T||_F on the device (host arrays)."""
        a, u, v = _arr(a), _arr(u), _arr(v)
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        k = sigma.shape[0]
        if u.shape != (a.shape[0], k) or v.shape != (a.shape[1], k):
            raise DimensionError("residual_fro: factor shapes do not match the input")
        out = C.c_double(0.0)
        _check(self.lib, self.lib.rsvd_b200_residual_fro(self.h, _dp(a), a.shape[0], a.shape[1],
                                                         _dp(u), _dp(sigma), _dp(v), k,
                                                         C.byref(out)))
        return out.value

    def residual_fro_device(self, a, u, sigma, v) -> float:
        """Same with CUDA float64 tensors (a may have a row stride)."""
        import torch
        for t in (a, u, sigma, v):
            assert t.is_cuda and t.dtype == torch.float64
        u, v, sigma = u.contiguous(), v.contiguous(), sigma.contiguous()  # may copy on torch's
        self.wait_for_torch(a.device)  # stream: order the solver's stream after those copies
        out = C.c_double(0.0)
        dptr = lambda t: C.cast(t.data_ptr(), C.POINTER(C.c_double))
        _check(self.lib, self.lib.rsvd_b200_residual_fro_device(
            self.h, dptr(a), a.shape[0], a.shape[1], a.stride(0), dptr(u), dptr(sigma), dptr(v),
            sigma.shape[0], C.byref(out)))
        return out.value

    # ------------------------------------------------------------- FP32 input
    def randomized_ksvd_f32(self, a, cfg: RsvdConfig, out=None) -> RsvdResult:
        """FP32 A (host): 3xTF32 tensor-core products, FP64 outputs (BASELINE config C4)."""
        a = np.ascontiguousarray(a, dtype=np.float32)
        if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
            raise DimensionError(f"DenseMatrix requires rows >= 1 and cols >= 1, got {a.shape}")
        m, n = a.shape
        k = max(int(cfg.k), 1)
        u, v, s = _outputs(out, m, n, k)
        sw = C.c_size_t(0)
        c = cfg._c()
        fp = a.ctypes.data_as(C.POINTER(C.c_float))
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd_f32(self.h, fp, m, n, C.byref(c),
                                                                _dp(u), _dp(s), _dp(v),
                                                                C.byref(sw)))
        return RsvdResult(SvdFactors(u, s, v), sw.value)

    def _device_f32(self, fn, a, extra, cfg, values_only):
        import torch
        assert a.is_cuda and a.dtype == torch.float32 and a.dim() == 2 and a.stride(1) == 1
        self.wait_for_torch(a.device)
        ml, n = a.shape
        k = int(cfg.k)
        dev = a.device
        sig = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        u = None if values_only else torch.empty((ml, max(k, 1)), dtype=torch.float64, device=dev)
        v = None if values_only else torch.empty((n, max(k, 1)), dtype=torch.float64, device=dev)
        sw = C.c_size_t(0)
        c = cfg._c()
        dptr = lambda t: None if t is None else C.cast(t.data_ptr(), C.POINTER(C.c_double))
        fptr = C.cast(a.data_ptr(), C.POINTER(C.c_float))
        _check(self.lib, fn(self.h, fptr, ml, *extra, n, a.stride(0), C.byref(c), dptr(u),
                            dptr(sig), dptr(v), C.byref(sw)))
        return u, sig[:k], v, sw.value

    def randomized_ksvd_f32_device(self, a, cfg: RsvdConfig, values_only: bool = False):
        """FP32 A resident in HBM (CUDA float32 tensor); returns FP64 (u, sigma, v, s)."""
        return self._device_f32(self.lib.rsvd_b200_randomized_ksvd_f32_device, a, (), cfg,
                                values_only)

    def randomized_ksvd_sharded_f32_device(self, a_local, m_total: int, cfg: RsvdConfig,
                                           values_only: bool = False):
        return self._device_f32(self.lib.rsvd_b200_randomized_ksvd_sharded_f32_device, a_local,
                                (m_total,), cfg, values_only)

    def randomized_ksvd_sharded_f32(self, a_local, m_total: int, cfg: RsvdConfig,
                                    out=None) -> RsvdResult:
        a = np.ascontiguousarray(a_local, dtype=np.float32)
        ml, n = a.shape
        k = max(int(cfg.k), 1)
        u, v, s = _outputs(out, ml, n, k)
        sw = C.c_size_t(0)
        c = cfg._c()
        fp = a.ctypes.data_as(C.POINTER(C.c_float))
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd_sharded_f32(
            self.h, fp, ml, m_total, n, C.byref(c), _dp(u), _dp(s), _dp(v), C.byref(sw)))
        return RsvdResult(SvdFactors(u, s, v), sw.value)

    # ------------------------------------------------------- row-sharded solves
    def attach_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        """Attach an NCCL communicator (rank 0 made `unique_id` with nccl_unique_id())."""
        if len(unique_id) != 128:
            raise ArgumentError("NCCL unique id must be 128 bytes")
        _check(self.lib, self.lib.rsvd_b200_comm_init_nccl(self.h, unique_id, rank, world))

    def attach_local(self, group: "LocalGroup", rank: int) -> None:
        """Join an in-process group (one thread per rank, buffers mutually addressable)."""
        _check(self.lib, self.lib.rsvd_b200_comm_init_local(self.h, group.g, rank))

    def detach(self) -> None:
        self.lib.rsvd_b200_comm_free(self.h)

    def comm_info(self) -> tuple[int, int]:
        r, w = C.c_int(0), C.c_int(1)
        self.lib.rsvd_b200_comm_info(self.h, C.byref(r), C.byref(w))
        return r.value, w.value

    def randomized_ksvd_sharded(self, a_local, m_total: int, cfg: RsvdConfig,
                                out=None) -> RsvdResult:
        """Collective row-sharded solve from host buffers: this rank's rows of A in, its
        rows of U and the replicated sigma, V out."""
        a = _arr(a_local)
        ml, n = a.shape
        k = max(int(cfg.k), 1)
        u, v, s = _outputs(out, ml, n, k)
        sw = C.c_size_t(0)
        c = cfg._c()
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd_sharded(
            self.h, _dp(a), ml, m_total, n, C.byref(c), _dp(u), _dp(s), _dp(v), C.byref(sw)))
        return RsvdResult(SvdFactors(u, s, v), sw.value)

    def randomized_ksvd_sharded_device(self, a_local, m_total: int, cfg: RsvdConfig,
                                       values_only: bool = False):
        """Collective row-sharded solve with this rank's rows resident in HBM (CUDA float64
        tensor). Returns (u_local, sigma, v, sketch_width) as CUDA tensors."""
        import torch
        a = a_local
        assert a.is_cuda and a.dtype == torch.float64 and a.dim() == 2 and a.stride(1) == 1
        self.wait_for_torch(a.device)
        ml, n = a.shape
        k = int(cfg.k)
        dev = a.device
        sig = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        u = None if values_only else torch.empty((ml, max(k, 1)), dtype=torch.float64, device=dev)
        v = None if values_only else torch.empty((n, max(k, 1)), dtype=torch.float64, device=dev)
        sw = C.c_size_t(0)
        c = cfg._c()
        dptr = lambda t: None if t is None else C.cast(t.data_ptr(), C.POINTER(C.c_double))
        _check(self.lib, self.lib.rsvd_b200_randomized_ksvd_sharded_device(
            self.h, dptr(a), ml, m_total, n, a.stride(0), C.byref(c), dptr(u), dptr(sig),
            dptr(v), C.byref(sw)))
        return u, sig[:k], v, sw.value

    # ---------------------------------------------------------- step functions
    def gaussian_matrix(self, seed: int, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols))
        _check(self.lib, self.lib.rsvd_b200_gaussian_matrix(self.h, seed & (2**64 - 1), rows,
                                                            cols, _dp(out)))
        return out

    def gaussian_stream(self, seed: int, counter: int, rows: int, cols: int,
                        cached: float | None = None) -> np.ndarray:
        """rows x cols normals from a GaussianSampler(seed) that has drawn `counter` words and
        holds `cached` (a pending sine half) or nothing (rng.cpp:22-53)."""
        out = np.empty((rows, cols))
        _check(self.lib, self.lib.rsvd_b200_gaussian_stream(
            self.h, seed & (2**64 - 1), counter, int(cached is not None),
            0.0 if cached is None else float(cached), rows, cols, _dp(out)))
        return out

    def sketch_stream(self, a, s: int, seed: int, counter: int,
                      cached: float | None = None) -> np.ndarray:
        """sketch() from a sampler part-way through its stream (see gaussian_stream)."""
        a = _arr(a)
        y = np.empty((a.shape[0], max(int(s), 1)))
        _check(self.lib, self.lib.rsvd_b200_sketch_stream(
            self.h, _dp(a), a.shape[0], a.shape[1], s, seed & (2**64 - 1), counter,
            int(cached is not None), 0.0 if cached is None else float(cached), _dp(y)))
        return y

    def splitmix_words(self, seed: int, count: int, first_counter: int = 1) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        _check(self.lib, self.lib.rsvd_b200_splitmix_words(
            self.h, seed & (2**64 - 1), first_counter, count,
            out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def uniforms(self, seed: int, count: int, first_counter: int = 1) -> np.ndarray:
        out = np.empty(count)
        _check(self.lib, self.lib.rsvd_b200_uniforms(self.h, seed & (2**64 - 1), first_counter,
                                                     count, _dp(out)))
        return out

    def sketch(self, a, s: int, seed: int) -> np.ndarray:
        a = _arr(a)
        y = np.empty((a.shape[0], max(int(s), 1)))
        _check(self.lib, self.lib.rsvd_b200_sketch(self.h, _dp(a), a.shape[0], a.shape[1], s,
                                                   seed & (2**64 - 1), _dp(y)))
        return y

    def power_iterate(self, a, y0, q: int) -> np.ndarray:
        a, y0 = _arr(a), _arr(y0)
        if y0.shape[0] != a.shape[0]:
            raise DimensionError(f"power_iterate: y0 has {y0.shape[0]} rows, a has {a.shape[0]}")
        w = np.empty_like(y0)
        _check(self.lib, self.lib.rsvd_b200_power_iterate(self.h, _dp(a), a.shape[0], a.shape[1],
                                                          _dp(y0), y0.shape[1], q, _dp(w)))
        return w

    _SPECTRA = {"fast": 0, "sharp": 1, "slow": 2}

    def synth_matrix(self, rows: int, cols: int, kind: str = "fast", beta: float = 1.0,
                     seed: int = 0) -> np.ndarray:
        """randsvd::synth::synth_matrix (synth.cpp:58-71) generated on the device."""
        out = np.empty((rows, cols))
        _check(self.lib, self.lib.rsvd_b200_synth_matrix(self.h, rows, cols, self._SPECTRA[kind],
                                                         float(beta), seed % 2**64, _dp(out)))
        return out

    def synth_matrix_device(self, rows: int, cols: int, kind: str = "fast", beta: float = 1.0,
                            seed: int = 0, device=None):
        """Same, into a new CUDA float64 tensor (stream-ordered before return)."""
        import torch
        out = torch.empty((rows, cols), dtype=torch.float64,
                          device=device if device is not None else f"cuda:{self.device}")
        self.wait_for_torch(out.device)
        _check(self.lib, self.lib.rsvd_b200_synth_matrix_device(
            self.h, rows, cols, self._SPECTRA[kind], float(beta), seed % 2**64, out.data_ptr(),
            cols))
        return out

    def householder_qr(self, a):
        """Thin QR (qr.cpp:27-102) on the device: (q m x n, r n x n, diag r >= 0)."""
        a = _arr(a)
        m, n = a.shape
        q, r = np.empty((m, n)), np.empty((n, n))
        _check(self.lib, self.lib.rsvd_b200_householder_qr(self.h, _dp(a), m, n, _dp(q), _dp(r)))
        return q, r

    def householder_qr_device(self, a):
        """Same on a CUDA float64 tensor (row stride allowed); returns CUDA tensors."""
        import torch
        assert a.is_cuda and a.dtype == torch.float64 and a.dim() == 2 and a.stride(1) == 1
        self.wait_for_torch(a.device)
        m, n = a.shape
        q = torch.empty((m, n), dtype=torch.float64, device=a.device)
        r = torch.empty((n, n), dtype=torch.float64, device=a.device)
        _check(self.lib, self.lib.rsvd_b200_householder_qr_device(
            self.h, a.data_ptr(), a.stride(0), m, n, q.data_ptr(), n, r.data_ptr(), n))
        return q, r

    def range_basis(self, y) -> np.ndarray:
        y = _arr(y)
        q = np.empty(y.size)
        cols = C.c_size_t(0)
        _check(self.lib, self.lib.rsvd_b200_range_basis(self.h, _dp(y), y.shape[0], y.shape[1],
                                                        _dp(q), C.byref(cols)))
        return q[: y.shape[0] * cols.value].reshape(y.shape[0], cols.value)

    def project_and_solve(self, a, qbasis, k: int) -> RsvdResult:
        a, qb = _arr(a), _arr(qbasis)
        m, n = a.shape
        kk = max(int(k), 1)
        u, s, v = np.empty((m, kk)), np.empty(kk), np.empty((n, kk))
        sw = C.c_size_t(0)
        _check(self.lib, self.lib.rsvd_b200_project_and_solve(
            self.h, _dp(a), m, n, _dp(qb), qb.shape[1], k, _dp(u), _dp(s), _dp(v), C.byref(sw)))
        return RsvdResult(SvdFactors(u, s, v), sw.value)


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0), to broadcast to the other ranks."""
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    _check(lib, lib.rsvd_b200_nccl_unique_id(buf))
    return buf.raw


class LocalGroup:
    """In-process communicator group (rsvd_b200_local_group): `world` handles driven from
    `world` host threads reduce through fixed-order device sums."""

    def __init__(self, world: int):
        self.lib = _lib.load()
        g = C.c_void_p()
        _check(self.lib, self.lib.rsvd_b200_local_group_create(world, C.byref(g)))
        self.g = g
        self.world = world

    def __del__(self):
        try:
            if self.g:
                self.lib.rsvd_b200_local_group_destroy(self.g)
                self.g = None
        except Exception:
            pass


_default: Solver | None = None


def default_solver() -> Solver:
    global _default
    if _default is None:
        _default = Solver(int(os.environ.get("RSVD_B200_DEVICE", "0")))
    return _default


def randomized_ksvd(a, cfg: RsvdConfig) -> RsvdResult:
    """randsvd::randomized_ksvd (rsvd.hpp:58) on the B200."""
    return default_solver().randomized_ksvd(a, cfg)


def singular_values_only(a, cfg: RsvdConfig) -> np.ndarray:
    """randsvd::singular_values_only (rsvd.hpp:62-63) on the B200."""
    return default_solver().singular_values_only(a, cfg)


def sketch(a, s: int, seed: int) -> np.ndarray:
    return default_solver().sketch(a, s, seed)


def power_iterate(a, y0, q: int) -> np.ndarray:
    return default_solver().power_iterate(a, y0, q)


def range_basis(y) -> np.ndarray:
    return default_solver().range_basis(y)


def householder_qr(a):
    return default_solver().householder_qr(a)


def project_and_solve(a, qbasis, k: int) -> RsvdResult:
    return default_solver().project_and_solve(a, qbasis, k)
