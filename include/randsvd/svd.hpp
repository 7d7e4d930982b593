// Drop-in factor record (reference: include/randsvd/svd.hpp:13-17): u m x r and
// v n x r with orthonormal columns, sigma non-increasing and non-negative.
#pragma once

#include <vector>

#include "randsvd/matrix.hpp"

namespace randsvd {

struct SvdFactors {
    DenseMatrix u;
    std::vector<double> sigma;
    DenseMatrix v;
};

inline constexpr int kSvdMaxSweeps = 30;

}  // namespace randsvd
