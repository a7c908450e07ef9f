// ref_wrapper.cpp — extern "C" entry points over the UNMODIFIED reference
// saitprec:: library, compiled together with the reference sources where they
// lie (/root/reference/proj/core/src/*.cpp) by oracle/Makefile into
// oracle/_ref/libsaitref.so.  TEST / BASELINE INFRASTRUCTURE ONLY: used by
// tests/ to pin the C restatement and by bench.py --impl reference / the
// cpu_baseline leg to time the reference's own CPU path.
//
// Results are returned in malloc'd arrays (free with ref_free / ref_csr_free).
// Exceptions become status codes: 1 = std::invalid_argument,
// 2 = std::runtime_error; the message is kept for ref_last_error().
#include <omp.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "saitprec/csr.hpp"
#include "saitprec/dense.hpp"
#include "saitprec/ilu.hpp"
#include "saitprec/kernels.hpp"
#include "saitprec/preconditioner.hpp"
#include "saitprec/sait.hpp"

using saitprec::CsrMatrix;

extern "C" {
struct ref_csr {
  int64_t nrows, ncols;
  int64_t* row_ptr;
  int64_t* col_idx;
  double* values;  // NULL for a pattern
};
}

namespace {
thread_local std::string g_err;

CsrMatrix to_ref(const ref_csr* m) {
  CsrMatrix r;
  r.nrows = m->nrows;
  r.ncols = m->ncols;
  int64_t nnz = m->row_ptr[m->nrows];
  r.row_ptr.assign(m->row_ptr, m->row_ptr + m->nrows + 1);
  r.col_idx.assign(m->col_idx, m->col_idx + nnz);
  if (m->values) r.values.assign(m->values, m->values + nnz);
  else r.values.assign(nnz, 0.0);
  return r;
}

saitprec::SparsityPattern to_pattern(const ref_csr* m) {
  saitprec::SparsityPattern s;
  s.nrows = m->nrows;
  s.ncols = m->ncols;
  int64_t nnz = m->row_ptr[m->nrows];
  s.row_ptr.assign(m->row_ptr, m->row_ptr + m->nrows + 1);
  s.col_idx.assign(m->col_idx, m->col_idx + nnz);
  return s;
}

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

void from_ref(const CsrMatrix& m, ref_csr* out) {
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->row_ptr = dup(m.row_ptr);
  out->col_idx = dup(m.col_idx);
  out->values = dup(m.values);
}

void from_pattern(const saitprec::SparsityPattern& s, ref_csr* out) {
  out->nrows = s.nrows;
  out->ncols = s.ncols;
  out->row_ptr = dup(s.row_ptr);
  out->col_idx = dup(s.col_idx);
  out->values = nullptr;
}

saitprec::TriangularKind kind_of(int lower) {
  return lower ? saitprec::lower_triangular : saitprec::upper_triangular;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// BASELINE config 4 fill cap, attached through the
// reference's own DropRule hook (sait.hpp:43).  Column j keeps its diagonal
// plus the cap[j]-1 largest-|v| off-diagonals, ties to the smaller row.
CsrMatrix cap_columns(const CsrMatrix& m, const std::vector<int64_t>& cap) {
  CsrMatrix mt = saitprec::transpose(m);
  std::vector<char> keep(mt.col_idx.size(), 0);
  std::vector<int64_t> off;
  for (int64_t j = 0; j < mt.nrows; ++j) {
    off.clear();
    for (int64_t e = mt.row_ptr[j]; e < mt.row_ptr[j + 1]; ++e) {
      if (mt.col_idx[e] == j) keep[e] = 1;
      else off.push_back(e);
    }
    int64_t room = cap[j] - 1 < 0 ? 0 : cap[j] - 1;
    if (static_cast<int64_t>(off.size()) > room) {
      std::stable_sort(off.begin(), off.end(), [&](int64_t a, int64_t b) {
        double fa = std::fabs(mt.values[a]), fb = std::fabs(mt.values[b]);
        if (fa != fb) return fa > fb;
        return mt.col_idx[a] < mt.col_idx[b];
      });
      off.resize(room);
    }
    for (int64_t e : off) keep[e] = 1;
  }
  CsrMatrix kt;
  kt.nrows = mt.nrows;
  kt.ncols = mt.ncols;
  kt.row_ptr.assign(mt.nrows + 1, 0);
  for (int64_t j = 0; j < mt.nrows; ++j) {
    for (int64_t e = mt.row_ptr[j]; e < mt.row_ptr[j + 1]; ++e) {
      if (!keep[e]) continue;
      kt.col_idx.push_back(mt.col_idx[e]);
      kt.values.push_back(mt.values[e]);
    }
    kt.row_ptr[j + 1] = static_cast<int64_t>(kt.col_idx.size());
  }
  return saitprec::transpose(kt);
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }
void ref_csr_free(ref_csr* m) {
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->values);
  m->row_ptr = nullptr;
  m->col_idx = nullptr;
  m->values = nullptr;
}
int ref_max_threads(void) { return omp_get_max_threads(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }

int ref_transpose(const ref_csr* a, ref_csr* out) {
  return guarded([&] { from_ref(saitprec::transpose(to_ref(a)), out); });
}
int ref_spmv(const ref_csr* a, const double* x, int64_t xlen, double* y, int64_t ylen) {
  return guarded([&] {
    saitprec::spmv(to_ref(a), std::span<const double>(x, xlen), std::span<double>(y, ylen));
  });
}
int ref_spgemm(const ref_csr* a, const ref_csr* b, ref_csr* out) {
  return guarded([&] { from_ref(saitprec::spgemm(to_ref(a), to_ref(b)), out); });
}
int ref_add_identity(const ref_csr* a, ref_csr* out) {
  return guarded([&] { from_ref(saitprec::add_identity(to_ref(a)), out); });
}
int ref_drop_by_threshold(const ref_csr* a, double tau, ref_csr* out) {
  return guarded([&] { from_ref(saitprec::drop_by_threshold(to_ref(a), tau), out); });
}
int ref_drop_by_pattern(const ref_csr* a, const ref_csr* s, ref_csr* out) {
  return guarded([&] { from_ref(saitprec::drop_by_pattern(to_ref(a), to_pattern(s)), out); });
}
int ref_scale_columns(const ref_csr* a, const double* d, int64_t dlen, ref_csr* out) {
  return guarded([&] {
    from_ref(saitprec::scale_columns(to_ref(a), std::span<const double>(d, dlen)), out);
  });
}
int ref_jacobi_split(const ref_csr* t, int lower, double** inv_diag, ref_csr* tt) {
  return guarded([&] {
    saitprec::JacobiSplit s = saitprec::jacobi_split(to_ref(t), kind_of(lower));
    *inv_diag = dup(s.inv_diag);
    from_ref(s.iteration_matrix, tt);
  });
}
int ref_sait_thr(const ref_csr* t, int lower, double tau, int steps, ref_csr* out) {
  return guarded([&] {
    from_ref(saitprec::sait_thr(to_ref(t), kind_of(lower), {tau, steps}), out);
  });
}
int ref_sait_pat(const ref_csr* t, int lower, int p, int m, ref_csr* out) {
  return guarded([&] {
    from_ref(saitprec::sait_pat(to_ref(t), kind_of(lower), {p, m}), out);
  });
}
int ref_sait_pat_capture_pattern(const ref_csr* t, int lower, int p, ref_csr* out) {
  return guarded([&] {
    from_pattern(saitprec::sait_pat_capture_pattern(to_ref(t), kind_of(lower), p), out);
  });
}
int ref_sait_polynomial_nodrop(const ref_csr* t, int lower, int steps, ref_csr* out) {
  return guarded([&] {
    saitprec::JacobiSplit s = saitprec::jacobi_split(to_ref(t), kind_of(lower));
    from_ref(saitprec::sait_polynomial(s, steps, {}), out);
  });
}
// sait_polynomial on a caller-supplied iteration matrix (any square matrix,
// e.g. with a stored diagonal): the reference's recursion, no drop rule.
int ref_sait_polynomial_tt(const ref_csr* tt, int steps, ref_csr* out) {
  return guarded([&] {
    saitprec::JacobiSplit s;
    s.iteration_matrix = to_ref(tt);
    s.inv_diag.assign(static_cast<size_t>(s.iteration_matrix.nrows), 1.0);
    s.kind = kind_of(1);
    from_ref(saitprec::sait_polynomial(s, steps, {}), out);
  });
}
int ref_sait_thr_cap(const ref_csr* t, int lower, double tau, int steps, double cap_factor,
                     ref_csr* out) {
  return guarded([&] {
    if (!(tau >= 0.0 && tau < 1.0))
      throw std::invalid_argument("sait_thr: threshold must be in [0, 1), got " +
                                  std::to_string(tau));
    CsrMatrix tm = to_ref(t);
    saitprec::JacobiSplit s = saitprec::jacobi_split(tm, kind_of(lower));
    std::vector<int64_t> cap(tm.ncols, 0);
    for (int64_t c : tm.col_idx) cap[c]++;
    for (auto& c : cap) c = static_cast<int64_t>(std::floor(cap_factor * static_cast<double>(c)));
    CsrMatrix m = saitprec::sait_polynomial(s, steps, [&](const CsrMatrix& x) {
      return cap_columns(saitprec::drop_by_threshold(x, tau), cap);
    });
    from_ref(saitprec::scale_columns(m, s.inv_diag), out);
  });
}
int ref_jacobi_sweeps_apply(const ref_csr* t, int lower, const double* b, int sweeps, double* x) {
  return guarded([&] {
    std::vector<double> r = saitprec::jacobi_sweeps_apply(
        to_ref(t), kind_of(lower), std::span<const double>(b, t->nrows), sweeps);
    std::memcpy(x, r.data(), sizeof(double) * r.size());
  });
}
int ref_trisolve(const ref_csr* t, int lower, const double* b, double* x) {
  return guarded([&] {
    std::vector<double> r =
        saitprec::trisolve(to_ref(t), kind_of(lower), std::span<const double>(b, t->nrows));
    std::memcpy(x, r.data(), sizeof(double) * r.size());
  });
}
int ref_ilu_k(const ref_csr* a, int level, ref_csr* lower, ref_csr* upper) {
  return guarded([&] {
    saitprec::IluFactors f = saitprec::ilu_k(to_ref(a), level);
    from_ref(f.lower, lower);
    from_ref(f.upper, upper);
  });
}
int ref_pair_apply(const ref_csr* ml, const ref_csr* mu, const double* r, double* z) {
  return guarded([&] {
    saitprec::SaitPairPreconditioner p(to_ref(ml), to_ref(mu));
    p.apply(std::span<const double>(r, ml->ncols), std::span<double>(z, mu->nrows));
  });
}
int ref_pair_apply_block(const ref_csr* ml, const ref_csr* mu, const double* r, int64_t nvec,
                         double* z) {
  return guarded([&] {
    saitprec::SaitPairPreconditioner p(to_ref(ml), to_ref(mu));
    saitprec::DenseMatrix rb(ml->ncols, nvec);
    std::memcpy(rb.data().data(), r, sizeof(double) * ml->ncols * nvec);
    saitprec::DenseMatrix zb = p.apply_block(rb);
    std::memcpy(z, zb.data().data(), sizeof(double) * mu->nrows * nvec);
  });
}

// ---- baseline timing helpers (bench.py --impl reference / cpu_baseline) ----

// A persistent SaitPairPreconditioner so repeated applies time only apply().
void* ref_pair_create(const ref_csr* ml, const ref_csr* mu) {
  try {
    return new saitprec::SaitPairPreconditioner(to_ref(ml), to_ref(mu));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_pair_destroy(void* p) { delete static_cast<saitprec::SaitPairPreconditioner*>(p); }
// Applies the pair to `nvec` vectors (r: nvec*n contiguous) one after the
// other through SaitPairPreconditioner::apply; returns elapsed seconds
// (std::chrono::steady_clock, as in TimedPreconditioner).
double ref_pair_time_apply(void* p, const double* r, double* z, int64_t n, int64_t nvec) {
  auto* pc = static_cast<saitprec::SaitPairPreconditioner*>(p);
  auto t0 = std::chrono::steady_clock::now();
  for (int64_t v = 0; v < nvec; ++v)
    pc->apply(std::span<const double>(r + v * n, n), std::span<double>(z + v * n, n));
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
// The same loop with y preallocated once: saitprec::spmv (kernels.hpp) into
// caller storage, separating the reference's per-call allocation of y
// (preconditioner.cpp:42-45 via kernels.cpp:28-32) from its SpMV time.
double ref_pair_time_apply_prealloc(void* p, const double* r, double* z, int64_t n, int64_t nvec) {
  auto* pc = static_cast<saitprec::SaitPairPreconditioner*>(p);
  std::vector<double> y(pc->lower_inverse().nrows);
  auto t0 = std::chrono::steady_clock::now();
  for (int64_t v = 0; v < nvec; ++v) {
    saitprec::spmv(pc->lower_inverse(), std::span<const double>(r + v * n, n), std::span<double>(y));
    saitprec::spmv(pc->upper_inverse(), std::span<const double>(y), std::span<double>(z + v * n, n));
  }
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
double ref_pair_time_apply_block(void* p, const double* r, double* z, int64_t n, int64_t nvec) {
  auto* pc = static_cast<saitprec::SaitPairPreconditioner*>(p);
  saitprec::DenseMatrix rb(n, nvec);
  std::memcpy(rb.data().data(), r, sizeof(double) * n * nvec);
  auto t0 = std::chrono::steady_clock::now();
  saitprec::DenseMatrix zb = pc->apply_block(rb);
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::memcpy(z, zb.data().data(), sizeof(double) * n * nvec);
  return s;
}
// Times saitprec::sait_thr on T; returns seconds, writes the built nnz.
double ref_time_sait_thr(const ref_csr* t, int lower, double tau, int steps, int64_t* nnz_out) {
  CsrMatrix tm = to_ref(t);
  auto t0 = std::chrono::steady_clock::now();
  CsrMatrix m = saitprec::sait_thr(tm, kind_of(lower), {tau, steps});
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *nnz_out = m.nnz();
  return s;
}

}  // extern "C"
