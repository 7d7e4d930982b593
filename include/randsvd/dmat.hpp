// Drop-in DMAT I/O (reference: /root/reference/proj/include/randsvd/dmat.hpp:10-19):
// "DMAT1\n", rows and cols as u64 little-endian, then rows*cols binary64 little-endian
// values in row-major order. Errors throw IoError with the failing byte offset.
#pragma once

#include <iosfwd>
#include <string>

#include "randsvd/matrix.hpp"

namespace randsvd {

DenseMatrix read_dmat(const std::string& path);
void write_dmat(const std::string& path, const DenseMatrix& m);
DenseMatrix read_dmat(std::istream& in, const std::string& name);
void write_dmat(std::ostream& out, const DenseMatrix& m, const std::string& name);

}  // namespace randsvd
