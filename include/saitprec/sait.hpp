// saitprec/sait.hpp — drop-in for the reference's sait.hpp (:14-74): the SAIT
// builders, computed by the B200 column-form fused-drop SpGEMM recursion.
#pragma once

#include <functional>
#include <span>
#include <vector>

#include "saitprec/csr.hpp"

namespace saitprec {

struct SaitThrParams {  // reference sait.hpp:14-17
  double threshold = 0.0;
  int steps = 1;
};

struct SaitPatParams {  // reference sait.hpp:24-27
  int pattern_steps = 1;
  int refine_steps = 1;
};

struct JacobiSplit {  // reference sait.hpp:32-36
  std::vector<double> inv_diag;
  CsrMatrix iteration_matrix;
  TriangularKind kind;
};

JacobiSplit jacobi_split(const CsrMatrix& t, TriangularKind kind);

using DropRule = std::function<CsrMatrix(const CsrMatrix&)>;

// With an empty DropRule the undropped recursion runs on the device.  A
// non-empty rule is arbitrary host code and cannot run on the device:
// std::invalid_argument (use sait_thr / sait_pat / sait_thr_cap instead).
CsrMatrix sait_polynomial(const JacobiSplit& split, int steps, const DropRule& drop);
CsrMatrix sait_thr(const CsrMatrix& t, TriangularKind kind, const SaitThrParams& params);
SparsityPattern sait_pat_capture_pattern(const CsrMatrix& t, TriangularKind kind, int pattern_steps);
CsrMatrix sait_pat(const CsrMatrix& t, TriangularKind kind, const SaitPatParams& params);
std::vector<double> jacobi_sweeps_apply(const CsrMatrix& t, TriangularKind kind, std::span<const double> b,
                                        int sweeps);

// Extension (BASELINE.json config 4): sait_thr with a per-column fill cap of
// floor(cap_factor * nnz(T[:, j])) entries.
CsrMatrix sait_thr_cap(const CsrMatrix& t, TriangularKind kind, const SaitThrParams& params, double cap_factor);

}  // namespace saitprec
