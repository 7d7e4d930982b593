// Drop-in thin QR (reference: include/randsvd/qr.hpp:8-18): q m x n with orthonormal
// columns, r n x n upper triangular with a non-negative diagonal and exact zeros below it.
// Computed on the B200 by the blocked Householder kernel (rsvd_b200_householder_qr).
#pragma once

#include "randsvd/matrix.hpp"

namespace randsvd {

struct QrFactors {
    DenseMatrix q;
    DenseMatrix r;
};

/// Householder thin QR of a; requires a.rows >= a.cols (DimensionError otherwise).
QrFactors householder_qr(const DenseMatrix& a);

}  // namespace randsvd
