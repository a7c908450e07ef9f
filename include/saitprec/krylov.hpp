// saitprec/krylov.hpp — the solver module of SPEC.md:282-351 (absent from the
// reference code) over the device loops of sait_c.h.  The preconditioner is a
// SaitPairPreconditioner (device resident) or nullptr (identity).
#pragma once

#include <span>
#include <vector>

#include "saitprec/csr.hpp"
#include "saitprec/dense.hpp"
#include "saitprec/preconditioner.hpp"

namespace saitprec {

struct SolveStats {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;  // history[0] = 1
  double true_relres = 0.0;
  double seconds = 0.0;
  double precond_seconds = 0.0;  // device time of the preconditioner applies
};

SolveStats pcg(const CsrMatrix& a, std::span<const double> b, const SaitPairPreconditioner* p, double tol,
               int maxit, std::vector<double>& x);
SolveStats gmres(const CsrMatrix& a, std::span<const double> b, const SaitPairPreconditioner* p, int restart,
                 double tol, int maxit, std::vector<double>& x);

struct EigResult {  // SPEC.md EigResult
  std::vector<double> eigenvalues;     // ascending
  DenseMatrix eigenvectors;            // n x nev
  std::vector<std::vector<double>> residual_history;
  int iterations = 0;
};

EigResult lobpcg(const CsrMatrix& a, const SaitPairPreconditioner* p, int nev, double tol, int maxit,
                 std::uint64_t seed);

}  // namespace saitprec
