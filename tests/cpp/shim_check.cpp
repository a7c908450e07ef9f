// shim_check.cpp — a program written against the reference's saitprec:: API
// (include/saitprec/*.hpp), linked against libsaitprec_b200.so instead of the
// reference library.  It runs the SAIT path end to end and dumps the results
// (tests/test_gpu_shim.py compares them bitwise with the reference's golden
// outputs and the oracle).  Usage: shim_check <out.bin>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "sait_c.h"
#include "saitprec/csr.hpp"
#include "saitprec/dense.hpp"
#include "saitprec/ilu.hpp"
#include "saitprec/kernels.hpp"
#include "saitprec/krylov.hpp"
#include "saitprec/preconditioner.hpp"
#include "saitprec/sait.hpp"

using namespace saitprec;

static FILE* out = nullptr;

static void put(const std::string& name, const std::vector<double>& v) {
  int32_t l = static_cast<int32_t>(name.size());
  int64_t n = static_cast<int64_t>(v.size());
  char t = 'd';
  fwrite(&l, 4, 1, out);
  fwrite(name.data(), 1, l, out);
  fwrite(&t, 1, 1, out);
  fwrite(&n, 8, 1, out);
  fwrite(v.data(), 8, n, out);
}
static void put(const std::string& name, const std::vector<int64_t>& v) {
  int32_t l = static_cast<int32_t>(name.size());
  int64_t n = static_cast<int64_t>(v.size());
  char t = 'q';
  fwrite(&l, 4, 1, out);
  fwrite(name.data(), 1, l, out);
  fwrite(&t, 1, 1, out);
  fwrite(&n, 8, 1, out);
  fwrite(v.data(), 8, n, out);
}
static void put(const std::string& name, const CsrMatrix& m) {
  put(name + "/row_ptr", m.row_ptr);
  put(name + "/col_idx", m.col_idx);
  put(name + "/values", m.values);
}
static void put_msg(const std::string& name, const std::string& msg) {
  std::vector<int64_t> bytes(msg.begin(), msg.end());
  put(name, bytes);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  out = std::fopen(argv[1], "wb");
  // 64 x 64 5-point Poisson through from_triplets (BASELINE config 1)
  const index_t nx = 64, n = nx * nx;
  std::vector<Triplet> tr;
  for (index_t y = 0; y < nx; ++y)
    for (index_t x = 0; x < nx; ++x) {
      const index_t i = y * nx + x;
      tr.push_back({i, i, 4.0});
      if (x > 0) tr.push_back({i, i - 1, -1.0});
      if (x + 1 < nx) tr.push_back({i, i + 1, -1.0});
      if (y > 0) tr.push_back({i, i - nx, -1.0});
      if (y + 1 < nx) tr.push_back({i, i + nx, -1.0});
    }
  const CsrMatrix A = from_triplets(n, n, tr);
  validate(A);
  const IluFactors f = ilu_k(A, 0);
  check_triangular(f.lower, unit_lower_triangular);
  const CsrMatrix ML = sait_thr(f.lower, lower_triangular, {1e-2, 4});
  const CsrMatrix MU = sait_thr(f.upper, upper_triangular, {1e-2, 4});
  put("A", A);
  put("ML", ML);
  put("MU", MU);
  std::vector<double> r(n);
  sait_fill_uniform_pm1(1, n, r.data());
  SaitPairPreconditioner P(ML, MU);
  put("z", apply_precond(P, r));
  put("pair_nnz", std::vector<int64_t>{P.nnz()});
  std::vector<double> x;
  const SolveStats st = gmres(A, r, &P, 30, 1e-8, 3000, x);
  put("gmres_x", x);
  put("gmres_hist", st.residual_history);
  put("gmres_iters", std::vector<int64_t>{st.iterations});
  // other builders and kernels
  put("pat_2_3", sait_pat(f.lower, lower_triangular, {2, 3}));
  put("cap", sait_thr_cap(f.upper, upper_triangular, {1e-2, 4}, 1.5));
  const SparsityPattern S = sait_pat_capture_pattern(f.lower, lower_triangular, 2);
  put("patcap_2/row_ptr", S.row_ptr);
  put("patcap_2/col_idx", S.col_idx);
  put("sweeps", jacobi_sweeps_apply(f.lower, unit_lower_triangular, r, 4));
  put("spgemm", spgemm(f.lower, f.upper));
  put("ilu_res", std::vector<double>{ilu_residual_on_pattern(A, f)});
  const JacobiSplit sp = jacobi_split(f.upper, upper_triangular);
  put("poly", sait_polynomial(sp, 3, {}));
  put("transpose", transpose(ML));
  {  // dense.hpp:41 spmm on an n x 11 block (slabs of 8 + 2 + 1 on the device)
    DenseMatrix X(n, 11);
    for (index_t j = 0; j < 11; ++j) sait_fill_uniform_pm1(40 + j, n, X.col(j).data());
    const DenseMatrix Y = spmm(ML, X);
    put("spmm11", std::vector<double>(Y.data().begin(), Y.data().end()));
    std::vector<double> cols;
    for (index_t j = 0; j < 11; ++j) {
      std::vector<double> xj(X.col(j).begin(), X.col(j).end());
      const std::vector<double> yj = spmv(ML, xj);
      cols.insert(cols.end(), yj.begin(), yj.end());
    }
    put("spmm11_cols", cols);
  }
  {
    ExactIluPreconditioner E(f);
    put("exact_z", apply_precond(E, r));
    put("exact_nnz", std::vector<int64_t>{E.nnz()});
    JacobiSweepsPreconditioner J(f, 3);
    put("jacobi3_z", apply_precond(J, r));
  }
  try {
    IluFactors g = f;
    g.upper.values[g.upper.row_ptr[9]] = 0.0;  // diagonal of row 9 (first entry of an upper row)
    trisolve(g.upper, upper_triangular, r);
  } catch (const std::runtime_error& e) {
    put_msg("err_trisolve", e.what());
  }
  // exceptions keep the reference's types and messages
  try {
    sait_thr(f.lower, lower_triangular, {1.5, 2});
  } catch (const std::invalid_argument& e) {
    put_msg("err_thr", e.what());
  }
  try {
    CsrMatrix z = f.lower;
    z.values[z.row_ptr[6] - 1] = 0.0;  // diagonal of row 5
    sait_thr(z, lower_triangular, {0.1, 2});
  } catch (const std::runtime_error& e) {
    put_msg("err_diag", e.what());
  }
  try {
    std::vector<double> bad(5);
    P.apply(bad, r);
  } catch (const std::invalid_argument& e) {
    put_msg("err_apply", e.what());
  }
  try {
    sait_polynomial(sp, 3, [](const CsrMatrix& m) { return m; });
  } catch (const std::invalid_argument& e) {
    put_msg("err_droprule", e.what());
  }
  std::fclose(out);
  std::printf("shim_check ok: nnz(ML)=%lld gmres iterations=%d\n", static_cast<long long>(ML.nnz()), st.iterations);
  return 0;
}
