// Drop-in Gaussian sampler (reference: include/randsvd/rng.hpp:21-47, rng.cpp:9-53): the
// same counter-based SplitMix64 stream, uniforms in (0, 1] and Box-Muller normals with the
// sine half cached, with the same members and layout. Scalar draws (next_u64, uniform01,
// normal) run on the host exactly as the reference's do; gaussian_matrix and sketch()
// draw their matrices on the device (csrc/omega.cu) from the sampler's CURRENT state —
// counter and cached half — and advance it as the reference's row-major loop of normal()
// calls would, so mixed scalar/matrix use of one sampler continues the same stream.
#pragma once

#include <cstdint>

#include "randsvd/matrix.hpp"

namespace randsvd {

namespace detail {
struct SamplerAccess;
}

class GaussianSampler {
public:
    explicit GaussianSampler(std::uint64_t seed) : seed_(seed) {}

    std::uint64_t seed() const noexcept { return seed_; }
    std::uint64_t counter() const noexcept { return counter_; }

    /// Next raw 64-bit word: mix64(seed + (++counter) * golden ratio).
    std::uint64_t next_u64();
    /// Uniform in (0, 1]: the top 53 bits of a word, plus one, times 2^-53.
    double uniform01();
    /// Standard normal (Box-Muller; cosine half first, sine half cached).
    double normal();

private:
    friend struct detail::SamplerAccess;
    std::uint64_t seed_;
    std::uint64_t counter_ = 0;
    double cached_ = 0.0;
    bool has_cached_ = false;
};

/// rows x cols standard normals in row-major order, drawn on the device from the
/// sampler's current state (which advances by rows * cols normals).
DenseMatrix gaussian_matrix(GaussianSampler& sampler, std::size_t rows, std::size_t cols);

}  // namespace randsvd
