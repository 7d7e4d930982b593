// TEST INFRASTRUCTURE ONLY (see tests/doctest_shim/doctest.h). The drop-in's svd.hpp
// carries the factor record the hot path returns; the reference's test helpers also call
// its full dense SVD (svd.hpp:19-29), which is not part of the B200 path (SURVEY.md §2
// rows 9-13: the whole-matrix dense_svd is out of scope). For the reference-suite binaries
// those two oracles come from the reference's own svd.cpp, compiled unmodified next to
// the tests (oracle/Makefile).
#pragma once
#include_next "randsvd/svd.hpp"

namespace randsvd {
SvdFactors dense_svd(const DenseMatrix& a);
DenseMatrix extend_orthonormal(const DenseMatrix& u, std::size_t target_cols);
}  // namespace randsvd
