// Drop-in API of the B200 randomized k-SVD: the same entry points, parameters and
// output layout as the reference (/root/reference/proj/include/randsvd/rsvd.hpp:13-63),
// implemented over the C-ABI in include/rsvd_b200.h (csrc/randsvd_dropin.cpp).
// Every solve runs on the GPU (sm_100a); there is no CPU fallback.
#pragma once

#include <cstdint>
#include <vector>

#include "randsvd/errors.hpp"
#include "randsvd/matrix.hpp"
#include "randsvd/parallel.hpp"
#include "randsvd/rng.hpp"
#include "randsvd/svd.hpp"

namespace randsvd {

struct RsvdConfig {
    std::size_t k = 1;
    std::size_t oversample = 10;
    std::size_t power_q = 2;
    std::uint64_t seed = 0;
    double epsilon = 0.5;
    bool epsilon_mode = false;
    std::size_t sketch_width(std::size_t m, std::size_t n) const;
};

struct RsvdResult {
    SvdFactors factors;
    std::size_t sketch_width = 0;
    /// ||a - u diag(sigma) v^T||_F (rsvd.cpp:37-49), evaluated on the GPU by a fused GEMM.
    double residual_fro(const DenseMatrix& a) const;
};

DenseMatrix sketch(const DenseMatrix& a, std::size_t s, GaussianSampler& sampler);
DenseMatrix power_iterate(const DenseMatrix& a, const DenseMatrix& y0, std::size_t q);
DenseMatrix range_basis(const DenseMatrix& y);
RsvdResult project_and_solve(const DenseMatrix& a, const DenseMatrix& qbasis, std::size_t k);
RsvdResult randomized_ksvd(const DenseMatrix& a, const RsvdConfig& cfg);
std::vector<double> singular_values_only(const DenseMatrix& a, const RsvdConfig& cfg);

/// Select the CUDA device used by this thread's solver (default: $RSVD_B200_DEVICE or 0).
void set_device(int device);

}  // namespace randsvd
