// saitprec_shim.cpp — the reference's C++ API (namespace saitprec, headers in
// include/saitprec/) implemented over the C ABI of libsait_b200.so.
//
// Layering: saitprec:: (this file, host C++) -> sait_c.h (plain C) -> CUDA.
// Host value types keep the reference layout; every call that does
// arithmetic on the SAIT path uploads to the B200, runs the device kernels and
// brings the result back, so a program written against the reference
// re-links against libsaitprec_b200.so unchanged.  C ABI status codes become
// the reference's exception types with the reference's messages.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>

#include "sait_c.h"
#include "saitprec/csr.hpp"
#include "saitprec/dense.hpp"
#include "saitprec/ilu.hpp"
#include "saitprec/kernels.hpp"
#include "saitprec/krylov.hpp"
#include "saitprec/preconditioner.hpp"
#include "saitprec/sait.hpp"

namespace saitprec {
namespace {

void check(int rc) {
  if (rc == SAIT_OK) return;
  const std::string msg = sait_last_error();
  if (rc == SAIT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// One stream per calling thread: the device pair keeps per-stream scratch, so
// concurrent const apply() calls from different threads never share it.
sait_stream_t thread_stream() {
  struct Holder {
    sait_stream_t s = nullptr;
    ~Holder() {
      if (s) sait_stream_destroy(s);
    }
  };
  thread_local Holder h;
  if (!h.s) check(sait_stream_create(&h.s));
  return h.s;
}

sait_host_csr view(const CsrMatrix& m) {
  sait_host_csr c;
  c.nrows = m.nrows;
  c.ncols = m.ncols;
  c.row_ptr = const_cast<int64_t*>(m.row_ptr.data());
  c.col_idx = const_cast<int64_t*>(m.col_idx.data());
  c.values = const_cast<double*>(m.values.data());
  return c;
}

sait_host_csr view(const SparsityPattern& m) {
  sait_host_csr c;
  c.nrows = m.nrows;
  c.ncols = m.ncols;
  c.row_ptr = const_cast<int64_t*>(m.row_ptr.data());
  c.col_idx = const_cast<int64_t*>(m.col_idx.data());
  c.values = nullptr;
  return c;
}

struct Dev {  // owning device CSR handle
  sait_dcsr_t h = nullptr;
  Dev() = default;
  explicit Dev(sait_dcsr_t x) : h(x) {}
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : h(o.h) { o.h = nullptr; }
  ~Dev() {
    if (h) sait_csr_free(h);
  }
  sait_dcsr_t release() {
    sait_dcsr_t r = h;
    h = nullptr;
    return r;
  }
};

template <class M>
Dev upload(const M& m) {
  sait_host_csr c = view(m);
  sait_dcsr_t h = nullptr;
  check(sait_csr_upload(&c, thread_stream(), &h));
  return Dev(h);
}

CsrMatrix download(sait_dcsr_t h) {
  CsrMatrix m;
  int64_t nr = 0, nc = 0, nz = 0;
  check(sait_csr_info(h, &nr, &nc, &nz));
  m.nrows = nr;
  m.ncols = nc;
  m.row_ptr.assign(nr + 1, 0);
  m.col_idx.assign(nz, 0);
  m.values.assign(nz, 0.0);
  check(sait_csr_download(h, m.row_ptr.data(), m.col_idx.data(), m.values.data(), thread_stream()));
  return m;
}

SparsityPattern download_pattern(sait_dcsr_t h) {
  SparsityPattern p;
  int64_t nr = 0, nc = 0, nz = 0;
  check(sait_csr_info(h, &nr, &nc, &nz));
  p.nrows = nr;
  p.ncols = nc;
  p.row_ptr.assign(nr + 1, 0);
  p.col_idx.assign(nz, 0);
  check(sait_csr_download(h, p.row_ptr.data(), p.col_idx.data(), nullptr, thread_stream()));
  return p;
}

struct DevVec {  // owning device buffer of doubles
  double* p = nullptr;
  size_t n = 0;
  explicit DevVec(size_t count) : n(count) {
    void* q = nullptr;
    check(sait_device_alloc(sizeof(double) * (count ? count : 1), &q));
    p = static_cast<double*>(q);
  }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
  ~DevVec() { sait_device_free(p); }
  void put(const double* h, size_t count) { check(sait_memcpy(p, h, sizeof(double) * count, 1)); }
  void get(double* h, size_t count) const { check(sait_memcpy(h, p, sizeof(double) * count, 2)); }
};

int lower_flag(TriangularKind k) { return k.side == TriangularKind::Side::Lower ? 1 : 0; }

CsrMatrix run_build(const CsrMatrix& t, TriangularKind kind, const sait_drop_spec& spec) {
  Dev dt = upload(t);
  sait_dcsr_t out = nullptr;
  check(sait_build(dt.h, lower_flag(kind), &spec, thread_stream(), &out, nullptr));
  Dev o(out);
  return download(o.h);
}

}  // namespace

// ------------------------------------------------------------------- csr.hpp

CsrMatrix from_triplets(index_t nrows, index_t ncols, std::span<const Triplet> triplets) {
  if (nrows < 0 || ncols < 0) throw std::invalid_argument("from_triplets: negative dimension");
  for (std::size_t k = 0; k < triplets.size(); ++k) {
    const Triplet& t = triplets[k];
    if (t.row < 0 || t.row >= nrows || t.col < 0 || t.col >= ncols)
      throw std::invalid_argument("from_triplets: triplet " + std::to_string(k) + " (row " + std::to_string(t.row) +
                                  ", col " + std::to_string(t.col) + ", value " + std::to_string(t.value) +
                                  ") out of range for " + std::to_string(nrows) + "x" + std::to_string(ncols) +
                                  " matrix");
  }
  std::vector<std::size_t> ord(triplets.size());
  std::iota(ord.begin(), ord.end(), std::size_t{0});
  std::stable_sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
    return triplets[a].row != triplets[b].row ? triplets[a].row < triplets[b].row : triplets[a].col < triplets[b].col;
  });
  CsrMatrix m;
  m.nrows = nrows;
  m.ncols = ncols;
  m.row_ptr.assign(nrows + 1, 0);
  index_t lr = -1, lc = -1;
  for (std::size_t k : ord) {  // duplicates summed in input order
    const Triplet& t = triplets[k];
    if (t.row == lr && t.col == lc) {
      m.values.back() += t.value;
      continue;
    }
    m.col_idx.push_back(t.col);
    m.values.push_back(t.value);
    ++m.row_ptr[t.row + 1];
    lr = t.row;
    lc = t.col;
  }
  std::partial_sum(m.row_ptr.begin(), m.row_ptr.end(), m.row_ptr.begin());
  return m;
}

CsrMatrix identity(index_t n) {
  CsrMatrix m;
  m.nrows = m.ncols = n;
  m.row_ptr.resize(n + 1);
  std::iota(m.row_ptr.begin(), m.row_ptr.end(), index_t{0});
  m.col_idx.resize(n);
  std::iota(m.col_idx.begin(), m.col_idx.end(), index_t{0});
  m.values.assign(n, 1.0);
  return m;
}

CsrMatrix transpose(const CsrMatrix& a) {
  Dev d = upload(a);
  sait_dcsr_t out = nullptr;
  check(sait_transpose(d.h, thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

void validate(const CsrMatrix& a) {
  if (a.nrows < 0 || a.ncols < 0) throw std::invalid_argument("validate: negative dimension");
  if (a.row_ptr.size() != static_cast<std::size_t>(a.nrows) + 1 || a.row_ptr[0] != 0)
    throw std::invalid_argument("validate: bad row_ptr head");
  for (index_t i = 0; i < a.nrows; ++i) {
    if (a.row_ptr[i + 1] < a.row_ptr[i])
      throw std::invalid_argument("validate: row_ptr decreasing at row " + std::to_string(i));
    index_t prev = -1;
    for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const index_t j = a.col_idx[k];
      if (j < 0 || j >= a.ncols)
        throw std::invalid_argument("validate: column out of range in row " + std::to_string(i));
      if (j <= prev)
        throw std::invalid_argument("validate: columns not strictly increasing in row " + std::to_string(i));
      prev = j;
    }
  }
  if (a.col_idx.size() != static_cast<std::size_t>(a.nnz()) || a.values.size() != static_cast<std::size_t>(a.nnz()))
    throw std::invalid_argument("validate: index/value array length mismatch");
}

void check_triangular(const CsrMatrix& a, TriangularKind kind) {
  const bool lower = kind.side == TriangularKind::Side::Lower;
  for (index_t i = 0; i < a.nrows; ++i)
    for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const index_t j = a.col_idx[k];
      if (lower ? j > i : j < i)
        throw std::invalid_argument("check_triangular: entry (" + std::to_string(i) + ", " + std::to_string(j) +
                                    ") outside stated triangle");
      if (kind.unit_diagonal && j == i && a.values[k] != 1.0)
        throw std::invalid_argument("check_triangular: non-unit diagonal at row " + std::to_string(i));
    }
}

SparsityPattern pattern_of(const CsrMatrix& m) {
  SparsityPattern s;
  s.nrows = m.nrows;
  s.ncols = m.ncols;
  s.row_ptr = m.row_ptr;
  s.col_idx = m.col_idx;
  return s;
}

CsrMatrix purge_zeros(const CsrMatrix& m) {
  CsrMatrix r;
  r.nrows = m.nrows;
  r.ncols = m.ncols;
  r.row_ptr.assign(m.nrows + 1, 0);
  for (index_t i = 0; i < m.nrows; ++i) {
    for (index_t k = m.row_ptr[i]; k < m.row_ptr[i + 1]; ++k)
      if (m.values[k] != 0.0) {
        r.col_idx.push_back(m.col_idx[k]);
        r.values.push_back(m.values[k]);
      }
    r.row_ptr[i + 1] = static_cast<index_t>(r.col_idx.size());
  }
  return r;
}

double nnz_ratio(const CsrMatrix& m, const CsrMatrix& t) {
  if (t.nnz() == 0) throw std::invalid_argument("nnz_ratio: reference matrix has no stored entries");
  return static_cast<double>(m.nnz()) / static_cast<double>(t.nnz());
}

// --------------------------------------------------------------- kernels.hpp

void spmv(const CsrMatrix& a, std::span<const double> x, std::span<double> y) {
  if (static_cast<index_t>(x.size()) != a.ncols)
    throw std::invalid_argument("spmv: vector length " + std::to_string(x.size()) + " does not match ncols " +
                                std::to_string(a.ncols));
  if (static_cast<index_t>(y.size()) != a.nrows) throw std::invalid_argument("spmv: output length mismatch");
  Dev d = upload(a);
  DevVec dx(x.size()), dy(y.size());
  dx.put(x.data(), x.size());
  check(sait_spmv(d.h, dx.p, static_cast<int64_t>(x.size()), dy.p, static_cast<int64_t>(y.size()), thread_stream()));
  check(sait_device_synchronize());
  dy.get(y.data(), y.size());
}

std::vector<double> spmv(const CsrMatrix& a, std::span<const double> x) {
  std::vector<double> y(a.nrows);
  spmv(a, x, y);
  return y;
}

CsrMatrix spgemm(const CsrMatrix& a, const CsrMatrix& b) {
  if (a.ncols != b.nrows)
    throw std::invalid_argument("spgemm: inner dimensions " + std::to_string(a.ncols) + " and " +
                                std::to_string(b.nrows) + " do not match");
  Dev da = upload(a), db = upload(b);
  sait_dcsr_t out = nullptr;
  check(sait_spgemm(da.h, db.h, thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

CsrMatrix add_identity(const CsrMatrix& m) {
  if (m.nrows != m.ncols) throw std::invalid_argument("add_identity: matrix is not square");
  Dev d = upload(m);
  sait_dcsr_t out = nullptr;
  check(sait_add_identity(d.h, thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

CsrMatrix drop_by_threshold(const CsrMatrix& m, double tau) {
  if (!(tau >= 0.0 && tau < 1.0))
    throw std::invalid_argument("drop_by_threshold: tau must be in [0, 1), got " + std::to_string(tau));
  if (tau == 0.0) return m;
  Dev d = upload(m);
  sait_dcsr_t out = nullptr;
  check(sait_drop_by_threshold(d.h, tau, thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

CsrMatrix drop_by_pattern(const CsrMatrix& m, const SparsityPattern& s) {
  if (m.nrows != s.nrows || m.ncols != s.ncols) throw std::invalid_argument("drop_by_pattern: shape mismatch");
  Dev d = upload(m), ds = upload(s);
  sait_dcsr_t out = nullptr;
  check(sait_drop_by_pattern(d.h, ds.h, thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

// The exact solve SAIT replaces, on the device (synchronization-free
// substitution, bitwise the sequential result).
std::vector<double> trisolve(const CsrMatrix& t, TriangularKind kind, std::span<const double> b) {
  if (t.nrows != t.ncols) throw std::invalid_argument("trisolve: matrix is not square");
  if (static_cast<index_t>(b.size()) != t.nrows) throw std::invalid_argument("trisolve: right-hand side length mismatch");
  Dev d = upload(t);
  DevVec db(b.size()), dx(b.size());
  db.put(b.data(), b.size());
  check(sait_trisolve(d.h, lower_flag(kind), db.p, static_cast<int64_t>(b.size()), dx.p, thread_stream()));
  std::vector<double> x(b.size());
  dx.get(x.data(), x.size());
  return x;
}

CsrMatrix scale_columns(const CsrMatrix& m, std::span<const double> d) {
  if (static_cast<index_t>(d.size()) != m.ncols) throw std::invalid_argument("scale_columns: scale vector length mismatch");
  Dev dm = upload(m);
  DevVec dd(d.size());
  dd.put(d.data(), d.size());
  sait_dcsr_t out = nullptr;
  check(sait_scale_columns(dm.h, dd.p, static_cast<int64_t>(d.size()), thread_stream(), &out));
  Dev o(out);
  return download(o.h);
}

// ------------------------------------------------------------------ sait.hpp

JacobiSplit jacobi_split(const CsrMatrix& t, TriangularKind kind) {
  if (t.nrows != t.ncols) throw std::invalid_argument("jacobi_split: matrix is not square");
  Dev d = upload(t);
  DevVec inv(t.nrows);
  sait_dcsr_t out = nullptr;
  check(sait_jacobi_split(d.h, lower_flag(kind), inv.p, thread_stream(), &out));
  Dev o(out);
  JacobiSplit s;
  s.kind = kind;
  s.inv_diag.assign(t.nrows, 0.0);
  inv.get(s.inv_diag.data(), t.nrows);
  s.iteration_matrix = download(o.h);
  return s;
}

CsrMatrix sait_polynomial(const JacobiSplit& split, int steps, const DropRule& drop) {
  if (steps < 1) throw std::invalid_argument("sait_polynomial: steps must be >= 1");
  if (drop)
    throw std::invalid_argument(
        "sait_polynomial: a custom DropRule cannot run on the device; use sait_thr, sait_pat or sait_thr_cap");
  Dev d = upload(split.iteration_matrix);
  sait_dcsr_t out = nullptr;
  check(sait_polynomial(d.h, steps, thread_stream(), &out, nullptr));
  Dev o(out);
  return download(o.h);
}

CsrMatrix sait_thr(const CsrMatrix& t, TriangularKind kind, const SaitThrParams& params) {
  sait_drop_spec spec{SAIT_DROP_THRESHOLD, params.threshold, params.steps, 0, 0, 0.0};
  return run_build(t, kind, spec);
}

CsrMatrix sait_thr_cap(const CsrMatrix& t, TriangularKind kind, const SaitThrParams& params, double cap_factor) {
  sait_drop_spec spec{SAIT_DROP_THRESHOLD_CAP, params.threshold, params.steps, 0, 0, cap_factor};
  return run_build(t, kind, spec);
}

CsrMatrix sait_pat(const CsrMatrix& t, TriangularKind kind, const SaitPatParams& params) {
  sait_drop_spec spec{SAIT_DROP_PATTERN, 0.0, 0, params.pattern_steps, params.refine_steps, 0.0};
  return run_build(t, kind, spec);
}

SparsityPattern sait_pat_capture_pattern(const CsrMatrix& t, TriangularKind kind, int pattern_steps) {
  if (pattern_steps < 0) throw std::invalid_argument("sait_pat_capture_pattern: pattern_steps must be >= 0");
  Dev d = upload(t);
  sait_dcsr_t out = nullptr;
  check(sait_pat_capture_pattern(d.h, lower_flag(kind), pattern_steps, thread_stream(), &out));
  Dev o(out);
  return download_pattern(o.h);
}

std::vector<double> jacobi_sweeps_apply(const CsrMatrix& t, TriangularKind kind, std::span<const double> b,
                                        int sweeps) {
  if (sweeps < 1) throw std::invalid_argument("jacobi_sweeps_apply: sweeps must be >= 1");
  if (static_cast<index_t>(b.size()) != t.nrows)
    throw std::invalid_argument("jacobi_sweeps_apply: right-hand side length mismatch");
  Dev d = upload(t);
  DevVec db(b.size()), dx(b.size());
  db.put(b.data(), b.size());
  check(sait_jacobi_sweeps_apply(d.h, lower_flag(kind), db.p, sweeps, dx.p, thread_stream()));
  std::vector<double> x(b.size());
  dx.get(x.data(), x.size());
  return x;
}

// ----------------------------------------------------------------- dense.hpp

DenseMatrix spmm(const CsrMatrix& a, const DenseMatrix& x) {
  if (a.ncols != x.nrows()) throw std::invalid_argument("spmm: dimension mismatch");
  DenseMatrix y(a.nrows, x.ncols());
  if (x.ncols() == 0) return y;
  Dev d = upload(a);
  DevVec dx(static_cast<size_t>(x.nrows() * x.ncols())), dy(static_cast<size_t>(a.nrows * x.ncols()));
  dx.put(x.data().data(), x.data().size());
  // one block product (the matrix read once per 8 columns), not a spmv per column
  check(sait_spmm(d.h, dx.p, dy.p, x.ncols(), thread_stream()));
  check(sait_device_synchronize());
  dy.get(y.data().data(), y.data().size());
  return y;
}

DenseMatrix transpose_times(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.nrows() != b.nrows()) throw std::invalid_argument("transpose_times: dimension mismatch");
  DenseMatrix c(a.ncols(), b.ncols());
  for (index_t j = 0; j < b.ncols(); ++j)
    for (index_t i = 0; i < a.ncols(); ++i) c(i, j) = dot(a.col(i), b.col(j));
  return c;
}

DenseMatrix times(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.ncols() != b.nrows()) throw std::invalid_argument("times: dimension mismatch");
  DenseMatrix c(a.nrows(), b.ncols());
  for (index_t j = 0; j < b.ncols(); ++j) {
    auto cj = c.col(j);
    for (index_t k = 0; k < a.ncols(); ++k) {
      const double bkj = b(k, j);
      if (bkj == 0.0) continue;
      auto ak = a.col(k);
      for (index_t i = 0; i < a.nrows(); ++i) cj[i] += ak[i] * bkj;
    }
  }
  return c;
}

double dot(std::span<const double> a, std::span<const double> b) {
  double acc = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) acc += a[i] * b[i];
  return acc;
}

double norm2(std::span<const double> a) { return std::sqrt(dot(a, a)); }

// ------------------------------------------------------------------- ilu.hpp

IluFactors ilu_k(const CsrMatrix& a, int level) {
  // Large matrices at fill levels 0 and 1 factorize on the device
  // (sait_ilu_device: the same factors bit for bit, the same errors);
  // SAIT_SHIM_DEVICE_ILU_MIN overrides the size threshold (stored entries).
  static const int64_t device_min = [] {
    const char* e = std::getenv("SAIT_SHIM_DEVICE_ILU_MIN");
    return e ? std::atoll(e) : int64_t{1} << 20;
  }();
  if ((level == 0 || level == 1) && a.nrows == a.ncols && a.nnz() >= device_min) {
    Dev d = upload(a);
    sait_dcsr_t lo = nullptr, up = nullptr;
    check(sait_ilu_device(d.h, level, thread_stream(), &lo, &up));
    Dev l(lo), u(up);
    IluFactors f;
    f.lower = download(l.h);
    f.upper = download(u.h);
    f.level = level;
    return f;
  }
  sait_host_csr c = view(a), lo{}, up{};
  check(sait_ilu_k(&c, level, &lo, &up));
  auto take = [](sait_host_csr& h) {
    CsrMatrix m;
    m.nrows = h.nrows;
    m.ncols = h.ncols;
    const int64_t nnz = h.row_ptr[h.nrows];
    m.row_ptr.assign(h.row_ptr, h.row_ptr + h.nrows + 1);
    m.col_idx.assign(h.col_idx, h.col_idx + nnz);
    m.values.assign(h.values, h.values + nnz);
    sait_host_csr_free(&h);
    return m;
  };
  IluFactors f;
  f.lower = take(lo);
  f.upper = take(up);
  f.level = level;
  return f;
}

double ilu_residual_on_pattern(const CsrMatrix& a, const IluFactors& f) {
  if (a.nrows != f.lower.nrows || a.ncols != f.upper.ncols)
    throw std::invalid_argument("ilu_residual_on_pattern: shape mismatch");
  const CsrMatrix prod = spgemm(f.lower, f.upper);
  double worst = 0.0;
  for (index_t i = 0; i < a.nrows; ++i) {
    index_t kp = prod.row_ptr[i];
    const index_t ep = prod.row_ptr[i + 1];
    for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const index_t j = a.col_idx[k];
      while (kp < ep && prod.col_idx[kp] < j) ++kp;
      const double pv = (kp < ep && prod.col_idx[kp] == j) ? prod.values[kp] : 0.0;
      worst = std::max(worst, std::abs(pv - a.values[k]));
    }
  }
  return worst;
}

// ------------------------------------------------------- preconditioner.hpp

DenseMatrix Preconditioner::apply_block(const DenseMatrix& r) const {
  DenseMatrix z(r.nrows(), r.ncols());
  for (index_t j = 0; j < r.ncols(); ++j) apply(r.col(j), z.col(j));
  return z;
}

void IdentityPreconditioner::apply(std::span<const double> r, std::span<double> z) const {
  std::copy(r.begin(), r.end(), z.begin());
}

ExactIluPreconditioner::ExactIluPreconditioner(IluFactors factors) : factors_(std::move(factors)) {
  Dev dl = upload(factors_.lower), du = upload(factors_.upper);
  sait_exact_t h = nullptr;
  check(sait_exact_ilu_create(dl.h, du.h, 1, &h));
  dl.release();
  du.release();
  exact_ = h;
}

ExactIluPreconditioner::~ExactIluPreconditioner() { sait_exact_ilu_destroy(static_cast<sait_exact_t>(exact_)); }

void ExactIluPreconditioner::apply(std::span<const double> r, std::span<double> z) const {
  DevVec dr(r.size()), dz(z.size());
  dr.put(r.data(), r.size());
  check(sait_exact_ilu_apply(static_cast<sait_exact_t>(exact_), dr.p, static_cast<int64_t>(r.size()), dz.p,
                             static_cast<int64_t>(z.size()), thread_stream()));
  dz.get(z.data(), z.size());
}

SaitPairPreconditioner::SaitPairPreconditioner(CsrMatrix lower_inverse, CsrMatrix upper_inverse)
    : lower_inv_(std::move(lower_inverse)), upper_inv_(std::move(upper_inverse)) {
  if (lower_inv_.nrows != upper_inv_.ncols)
    throw std::invalid_argument("SaitPairPreconditioner: factor shapes do not chain");
  Dev dl = upload(lower_inv_), du = upload(upper_inv_);
  sait_pair_t p = nullptr;
  check(sait_pair_create(dl.h, du.h, 1, &p));
  dl.release();
  du.release();
  pair_ = p;
}

SaitPairPreconditioner::~SaitPairPreconditioner() {
  if (pair_) sait_pair_destroy(static_cast<sait_pair_t>(pair_));
}

void SaitPairPreconditioner::apply(std::span<const double> r, std::span<double> z) const {
  check(sait_pair_apply_host(static_cast<sait_pair_t>(pair_), r.data(), static_cast<int64_t>(r.size()), z.data(),
                             static_cast<int64_t>(z.size()), thread_stream()));
}

DenseMatrix SaitPairPreconditioner::apply_block(const DenseMatrix& r) const {
  if (r.nrows() != lower_inv_.ncols) throw std::invalid_argument("spmm: dimension mismatch");
  DenseMatrix z(upper_inv_.nrows, r.ncols());
  check(sait_pair_apply_block_host(static_cast<sait_pair_t>(pair_), r.data().data(), z.data().data(), r.nrows(),
                                   r.ncols(), 0, thread_stream()));
  return z;
}

JacobiSweepsPreconditioner::JacobiSweepsPreconditioner(IluFactors factors, int sweeps)
    : factors_(std::move(factors)), sweeps_(sweeps) {
  if (sweeps_ < 1) throw std::invalid_argument("JacobiSweepsPreconditioner: sweeps must be >= 1");
}

void JacobiSweepsPreconditioner::apply(std::span<const double> r, std::span<double> z) const {
  const std::vector<double> y = jacobi_sweeps_apply(factors_.lower, unit_lower_triangular, r, sweeps_);
  const std::vector<double> x = jacobi_sweeps_apply(factors_.upper, upper_triangular, y, sweeps_);
  std::copy(x.begin(), x.end(), z.begin());
}

void TimedPreconditioner::apply(std::span<const double> r, std::span<double> z) const {
  const auto t0 = std::chrono::steady_clock::now();
  inner_.apply(r, z);
  seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

DenseMatrix TimedPreconditioner::apply_block(const DenseMatrix& r) const {
  const auto t0 = std::chrono::steady_clock::now();
  DenseMatrix z = inner_.apply_block(r);
  seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return z;
}

std::vector<double> apply_precond(const Preconditioner& p, std::span<const double> r) {
  std::vector<double> z(r.size());
  p.apply(r, z);
  return z;
}

// ---------------------------------------------------------------- krylov.hpp

namespace {
template <class Fn>
SolveStats run_solver(const CsrMatrix& a, std::span<const double> b, std::vector<double>& x, int maxit, Fn&& fn) {
  if (static_cast<index_t>(b.size()) != a.nrows) throw std::invalid_argument("solver: right-hand side length mismatch");
  Dev d = upload(a);
  DevVec db(b.size()), dx(b.size());
  db.put(b.data(), b.size());
  std::vector<double> hist(static_cast<size_t>(maxit) + 1, 0.0);
  sait_solve_stats st{};
  check(fn(d.h, db.p, dx.p, hist.data(), &st));
  x.assign(b.size(), 0.0);
  dx.get(x.data(), x.size());
  SolveStats out;
  out.iterations = st.iterations;
  out.converged = st.converged != 0;
  out.true_relres = st.true_relres;
  out.seconds = st.seconds;
  out.precond_seconds = st.precond_seconds;
  out.residual_history.assign(hist.begin(), hist.begin() + st.iterations + 1);
  return out;
}
}  // namespace

SolveStats pcg(const CsrMatrix& a, std::span<const double> b, const SaitPairPreconditioner* p, double tol, int maxit,
               std::vector<double>& x) {
  return run_solver(a, b, x, maxit, [&](sait_dcsr_t h, double* db, double* dx, double* hist, sait_solve_stats* st) {
    return sait_pcg(h, p ? static_cast<sait_pair_t>(p->device_handle()) : nullptr, db, dx, a.nrows, tol, maxit, hist,
                    st, thread_stream());
  });
}

SolveStats gmres(const CsrMatrix& a, std::span<const double> b, const SaitPairPreconditioner* p, int restart,
                 double tol, int maxit, std::vector<double>& x) {
  return run_solver(a, b, x, maxit, [&](sait_dcsr_t h, double* db, double* dx, double* hist, sait_solve_stats* st) {
    return sait_gmres(h, p ? static_cast<sait_pair_t>(p->device_handle()) : nullptr, db, dx, a.nrows, restart, tol,
                      maxit, hist, st, thread_stream());
  });
}

EigResult lobpcg(const CsrMatrix& a, const SaitPairPreconditioner* p, int nev, double tol, int maxit,
                 std::uint64_t seed) {
  Dev d = upload(a);
  EigResult r;
  r.eigenvalues.assign(nev, 0.0);
  DevVec vecs(static_cast<size_t>(a.nrows) * static_cast<size_t>(nev > 0 ? nev : 1));
  std::vector<double> res((static_cast<size_t>(maxit) + 1) * static_cast<size_t>(nev > 0 ? nev : 1));
  int its = 0;
  check(sait_lobpcg(d.h, p ? static_cast<sait_pair_t>(p->device_handle()) : nullptr, nev, tol, maxit, seed,
                    r.eigenvalues.data(), vecs.p, res.data(), &its, thread_stream()));
  r.iterations = its;
  r.eigenvectors = DenseMatrix(a.nrows, nev);
  vecs.get(r.eigenvectors.data().data(), r.eigenvectors.data().size());
  for (int it = 0; it <= its; ++it)
    r.residual_history.emplace_back(res.begin() + static_cast<size_t>(it) * nev,
                                    res.begin() + static_cast<size_t>(it + 1) * nev);
  return r;
}

}  // namespace saitprec
