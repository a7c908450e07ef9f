// saitprec/kernels.hpp — drop-in for the reference's kernels.hpp (:12-40).
// spmv / spgemm / add_identity / drop_* / scale_columns run on the B200 and
// return bitwise the reference's results; so does trisolve, the exact solve
// the SAIT pair replaces (synchronization-free substitution on the device).
#pragma once

#include <span>
#include <vector>

#include "saitprec/csr.hpp"

namespace saitprec {

void spmv(const CsrMatrix& a, std::span<const double> x, std::span<double> y);
std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x);
CsrMatrix spgemm(const CsrMatrix& a, const CsrMatrix& b);
CsrMatrix add_identity(const CsrMatrix& m);
CsrMatrix drop_by_threshold(const CsrMatrix& m, double tau);
CsrMatrix drop_by_pattern(const CsrMatrix& m, const SparsityPattern& s);
std::vector<double> trisolve(const CsrMatrix& t, TriangularKind kind, std::span<const double> b);
CsrMatrix scale_columns(const CsrMatrix& m, std::span<const double> d);

}  // namespace saitprec
