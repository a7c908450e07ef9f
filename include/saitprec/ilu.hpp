// saitprec/ilu.hpp — drop-in for the reference's ilu.hpp (:10-30).  The
// factors are bitwise the reference's (host IKJ elimination in the library).
#pragma once

#include "saitprec/csr.hpp"

namespace saitprec {

struct IluFactors {
  CsrMatrix lower;  // unit lower, diagonal stored
  CsrMatrix upper;
  int level = 0;
};

IluFactors ilu_k(const CsrMatrix& a, int level);
double ilu_residual_on_pattern(const CsrMatrix& a, const IluFactors& f);

}  // namespace saitprec
