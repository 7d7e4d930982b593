"""Loader for the in-tree C-ABI library paper_2110_03423_b200/_lib/librsvd_b200.so.

Fails loudly when the library is missing: the product path never falls back to CPU.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "librsvd_b200.so")

# Every symbol include/rsvd_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "rsvd_b200_config_default", "rsvd_b200_sketch_width", "rsvd_b200_create",
    "rsvd_b200_destroy", "rsvd_b200_last_error", "rsvd_b200_stream", "rsvd_b200_set_omega",
    "rsvd_b200_randomized_ksvd", "rsvd_b200_singular_values_only",
    "rsvd_b200_randomized_ksvd_device", "rsvd_b200_gaussian_matrix", "rsvd_b200_sketch",
    "rsvd_b200_gaussian_stream", "rsvd_b200_sketch_stream",
    "rsvd_b200_power_iterate", "rsvd_b200_range_basis", "rsvd_b200_project_and_solve",
    "rsvd_b200_householder_qr", "rsvd_b200_householder_qr_device",
    "rsvd_b200_synth_matrix", "rsvd_b200_synth_matrix_device",
    "rsvd_b200_splitmix_words", "rsvd_b200_uniforms", "rsvd_b200_last_profile",
    "rsvd_b200_set_profiling", "rsvd_b200_last_launch_count", "rsvd_b200_version",
    "rsvd_b200_kernel_stats", "rsvd_b200_reset_stats", "rsvd_b200_last_info",
    "rsvd_b200_set_robust", "rsvd_b200_set_graphs", "rsvd_b200_nccl_unique_id", "rsvd_b200_comm_init_nccl",
    "rsvd_b200_local_group_create", "rsvd_b200_local_group_destroy", "rsvd_b200_comm_init_local",
    "rsvd_b200_comm_info", "rsvd_b200_comm_free", "rsvd_b200_randomized_ksvd_sharded",
    "rsvd_b200_randomized_ksvd_sharded_device", "rsvd_b200_dmma_peak", "rsvd_b200_imma_peak",
    "rsvd_b200_debug_gemm_tf32", "rsvd_b200_debug_cholesky", "rsvd_b200_debug_jacobi",
    "rsvd_b200_debug_gemm_oz", "rsvd_b200_debug_gemm_ozd",
    "rsvd_b200_randomized_ksvd_f32",
    "rsvd_b200_randomized_ksvd_f32_device", "rsvd_b200_randomized_ksvd_sharded_f32",
    "rsvd_b200_randomized_ksvd_sharded_f32_device", "rsvd_b200_wait_stream",
    "rsvd_b200_residual_fro", "rsvd_b200_residual_fro_device", "rsvd_b200_fit_pca",
    "rsvd_b200_pca_transform", "rsvd_b200_dmat_shape", "rsvd_b200_load_dmat_device",
    "rsvd_b200_dmat_last_error",
]


class Config(C.Structure):
    """rsvd_b200_config (include/rsvd_b200.h)."""
    _fields_ = [("k", C.c_size_t), ("oversample", C.c_size_t), ("power_q", C.c_size_t),
                ("seed", C.c_uint64), ("epsilon", C.c_double), ("epsilon_mode", C.c_int)]


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_sz = C.c_size_t
_vp = C.c_void_p
_LIB = None


def load() -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2110_03423_b200.build` "
                          "(the rSVD has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    cfgp = C.POINTER(Config)
    sig = {
        "rsvd_b200_config_default": (None, [cfgp]),
        "rsvd_b200_sketch_width": (_sz, [cfgp, _sz, _sz]),
        "rsvd_b200_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
        "rsvd_b200_destroy": (C.c_int, [_vp]),
        "rsvd_b200_last_error": (C.c_char_p, []),
        "rsvd_b200_stream": (_vp, [_vp]),
        "rsvd_b200_wait_stream": (C.c_int, [_vp, _vp]),
        "rsvd_b200_dmat_shape": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64)]),
        "rsvd_b200_load_dmat_device": (C.c_int, [_vp, C.c_char_p, C.c_uint64, C.c_uint64, _dp,
                                                 _sz]),
        "rsvd_b200_dmat_last_error": (C.c_char_p, []),
        "rsvd_b200_fit_pca": (C.c_int, [_vp, _dp, _sz, _sz, _sz, cfgp, _dp, _dp, _dp]),
        "rsvd_b200_pca_transform": (C.c_int, [_vp, _dp, _sz, _sz, _dp, _dp, _sz, _dp]),
        "rsvd_b200_residual_fro": (C.c_int, [_vp, _dp, _sz, _sz, _dp, _dp, _dp, _sz, _dp]),
        "rsvd_b200_residual_fro_device": (C.c_int, [_vp, _dp, _sz, _sz, _sz, _dp, _dp, _dp, _sz,
                                                    _dp]),
        "rsvd_b200_set_omega": (C.c_int, [_vp, _dp, _sz, _sz]),
        "rsvd_b200_randomized_ksvd": (C.c_int, [_vp, _dp, _sz, _sz, cfgp, _dp, _dp, _dp,
                                                C.POINTER(_sz)]),
        "rsvd_b200_singular_values_only": (C.c_int, [_vp, _dp, _sz, _sz, cfgp, _dp]),
        "rsvd_b200_randomized_ksvd_device": (C.c_int, [_vp, _dp, _sz, _sz, _sz, cfgp, _dp, _dp,
                                                       _dp, C.POINTER(_sz)]),
        "rsvd_b200_gaussian_matrix": (C.c_int, [_vp, C.c_uint64, _sz, _sz, _dp]),
        "rsvd_b200_sketch": (C.c_int, [_vp, _dp, _sz, _sz, _sz, C.c_uint64, _dp]),
        "rsvd_b200_gaussian_stream": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                                _sz, _sz, _dp]),
        "rsvd_b200_sketch_stream": (C.c_int, [_vp, _dp, _sz, _sz, _sz, C.c_uint64, C.c_uint64,
                                              C.c_int, C.c_double, _dp]),
        "rsvd_b200_power_iterate": (C.c_int, [_vp, _dp, _sz, _sz, _dp, _sz, _sz, _dp]),
        "rsvd_b200_range_basis": (C.c_int, [_vp, _dp, _sz, _sz, _dp, C.POINTER(_sz)]),
        "rsvd_b200_householder_qr": (C.c_int, [_vp, _dp, _sz, _sz, _dp, _dp]),
        "rsvd_b200_synth_matrix": (C.c_int, [_vp, _sz, _sz, C.c_int, C.c_double, C.c_uint64,
                                             _dp]),
        "rsvd_b200_synth_matrix_device": (C.c_int, [_vp, _sz, _sz, C.c_int, C.c_double,
                                                    C.c_uint64, _vp, _sz]),
        "rsvd_b200_householder_qr_device": (C.c_int, [_vp, _vp, _sz, _sz, _sz, _vp, _sz, _vp,
                                                      _sz]),
        "rsvd_b200_project_and_solve": (C.c_int, [_vp, _dp, _sz, _sz, _dp, _sz, _sz, _dp, _dp,
                                                  _dp, C.POINTER(_sz)]),
        "rsvd_b200_splitmix_words": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _sz,
                                               C.POINTER(C.c_uint64)]),
        "rsvd_b200_uniforms": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _sz, _dp]),
        "rsvd_b200_last_profile": (C.c_int, [_vp, C.POINTER(C.c_char_p), _dp, C.c_int]),
        "rsvd_b200_set_profiling": (None, [_vp, C.c_int]),
        "rsvd_b200_last_launch_count": (C.c_long, [_vp]),
        "rsvd_b200_version": (C.c_char_p, []),
        "rsvd_b200_kernel_stats": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_long), _dp, _dp]),
        "rsvd_b200_reset_stats": (None, [_vp]),
        "rsvd_b200_last_info": (C.c_long, [_vp, C.c_char_p]),
        "rsvd_b200_set_robust": (None, [_vp, C.c_int]),
        "rsvd_b200_set_graphs": (None, [_vp, C.c_int]),
        "rsvd_b200_nccl_unique_id": (C.c_int, [C.c_char_p]),
        "rsvd_b200_dmma_peak": (C.c_int, [_vp, _dp]),
        "rsvd_b200_imma_peak": (C.c_int, [_vp, _dp]),
        "rsvd_b200_randomized_ksvd_f32": (C.c_int, [_vp, _fp, _sz, _sz, cfgp, _dp, _dp, _dp,
                                                    C.POINTER(_sz)]),
        "rsvd_b200_randomized_ksvd_f32_device": (C.c_int, [_vp, _fp, _sz, _sz, _sz, cfgp, _dp,
                                                           _dp, _dp, C.POINTER(_sz)]),
        "rsvd_b200_randomized_ksvd_sharded_f32": (C.c_int, [_vp, _fp, _sz, _sz, _sz, cfgp, _dp,
                                                            _dp, _dp, C.POINTER(_sz)]),
        "rsvd_b200_randomized_ksvd_sharded_f32_device": (C.c_int, [_vp, _fp, _sz, _sz, _sz, _sz,
                                                                   cfgp, _dp, _dp, _dp,
                                                                   C.POINTER(_sz)]),
        "rsvd_b200_debug_gemm_tf32": (C.c_int, [_vp, C.c_int, _vp, C.c_long, C.c_long, C.c_long,
                                                _vp, C.c_long, C.c_int, _vp, C.c_long, C.c_int,
                                                C.c_int, C.c_int]),
        "rsvd_b200_debug_gemm_oz": (C.c_int, [_vp, C.c_int, _vp, C.c_long, C.c_long, C.c_long,
                                              _vp, C.c_long, C.c_int, C.c_int, _vp, C.c_long,
                                              C.c_int, C.c_int]),
        "rsvd_b200_debug_gemm_ozd": (C.c_int, [_vp, C.c_int, _vp, C.c_long, C.c_long, C.c_long,
                                               _vp, C.c_long, C.c_int, C.c_int, _vp, C.c_long,
                                               C.c_int, C.c_int]),
        "rsvd_b200_debug_cholesky": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp, C.c_double,
                                               C.POINTER(C.c_int)]),
        "rsvd_b200_debug_jacobi": (C.c_int, [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp,
                                             C.POINTER(C.c_int)]),
        "rsvd_b200_comm_init_nccl": (C.c_int, [_vp, C.c_char_p, C.c_int, C.c_int]),
        "rsvd_b200_local_group_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
        "rsvd_b200_local_group_destroy": (None, [_vp]),
        "rsvd_b200_comm_init_local": (C.c_int, [_vp, _vp, C.c_int]),
        "rsvd_b200_comm_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "rsvd_b200_comm_free": (None, [_vp]),
        "rsvd_b200_randomized_ksvd_sharded": (C.c_int, [_vp, _dp, _sz, _sz, _sz, cfgp, _dp, _dp,
                                                        _dp, C.POINTER(_sz)]),
        "rsvd_b200_randomized_ksvd_sharded_device": (C.c_int, [_vp, _dp, _sz, _sz, _sz, _sz,
                                                               cfgp, _dp, _dp, _dp,
                                                               C.POINTER(_sz)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _LIB = lib
    return lib
