"""B200-native randomized truncated SVD (arxiv 2110.03423, Algorithm 1).

Drop-in for the reference's `randsvd::randomized_ksvd` / `singular_values_only` path:
C-ABI in include/rsvd_b200.h, C++ API in include/randsvd/*.hpp, this Python mirror in
`paper_2110_03423_b200.rsvd`. Kernels: csrc/*.cu (sm_100a).
"""
from .rsvd import (ArgumentError, ConvergenceError, DeviceError, DimensionError, Error,  # noqa: F401
                   RsvdConfig, RsvdResult, Solver, SvdFactors, power_iterate, project_and_solve,
                   LocalGroup, nccl_unique_id, randomized_ksvd, range_basis, householder_qr,
                   singular_values_only, sketch)
from .dist import attach_process_group, shard_rows  # noqa: F401
