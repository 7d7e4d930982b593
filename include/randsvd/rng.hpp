// Drop-in Gaussian sampler handle (reference: include/randsvd/rng.hpp:21-47). On the
// B200 path the stream is generated on the device (SplitMix64 counter words + Box-Muller,
// csrc/omega.cu); this class only carries the seed into sketch(), whose Omega is the
// first n*s normals of a fresh sampler, as in the reference (rsvd.cpp:51-59).
#pragma once

#include <cstdint>

#include "randsvd/matrix.hpp"

namespace randsvd {

class GaussianSampler {
public:
    explicit GaussianSampler(std::uint64_t seed) : seed_(seed) {}
    std::uint64_t seed() const noexcept { return seed_; }
    std::uint64_t counter() const noexcept { return counter_; }
    /// Advance by `words` counter steps (what drawing a matrix consumes on the host).
    void advance(std::uint64_t words) noexcept { counter_ += words; }

private:
    std::uint64_t seed_;
    std::uint64_t counter_ = 0;
};

/// rows x cols standard normals in row-major order, drawn on the device from the
/// sampler's current position (must be a fresh sampler: counter 0).
DenseMatrix gaussian_matrix(GaussianSampler& sampler, std::size_t rows, std::size_t cols);

}  // namespace randsvd
