// solvers.cu — device-resident solver loops that drive the SAIT apply
// (north_star (3); GMRES per DESIGN.md "solvers").
// Vectors never leave HBM; per iteration only the few scalars the host needs
// for control (dots, Hessenberg column) come back.  Operation order matches
// oracle/solvers.c exactly (canonical dots in blas.cu, the same elementwise
// expressions, the same host-side Givens/back-substitution code), so iteration
// counts and residual histories are bitwise identical to the CPU restatement.
#include <chrono>
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sait {
void pair_apply_internal(sait_pair_t p, const double* r, double* z, cudaStream_t s);
int64_t pair_dim(sait_pair_t p);
void exact_apply_internal(sait_exact_t e, const double* r, double* z, cudaStream_t s);
int64_t exact_dim(sait_exact_t e);

int64_t dot_blocks(int64_t n);
void dot_partials(int64_t n, const double* x, const double* V, int64_t ld, int m, double* part, cudaStream_t s);
void dot_fold(const double* part, int64_t nb, int m, double* out, bool sqrt_out, cudaStream_t s);
void multi_dot(int64_t n, const double* x, const double* V, int64_t ld, int m, double* out, double* scratch,
               cudaStream_t s, bool sqrt_out);
void cgs_subtract(int64_t n, double* w, const double* V, int64_t ld, int m, const double* h, cudaStream_t s);
void divide_by(int64_t n, const double* w, const double* d, double* out, cudaStream_t s);
void linear_combination(int64_t n, const double* V, int64_t ld, int k, const double* y, double* u, cudaStream_t s);
void axpy(int64_t n, double a, const double* x, double* y, cudaStream_t s);
void xpay(int64_t n, const double* x, double a, double* y, cudaStream_t s);
void x_minus_y(int64_t n, const double* x, double* y, cudaStream_t s);
void y_plus_x(int64_t n, const double* x, double* y, cudaStream_t s);
int64_t gram_scratch(int64_t n, int ka, int kb);
void gram(int64_t n, const double* A, int ka, const double* B, int kb, double* G, int ldg, double* scratch,
          void* tiles_dev, cudaStream_t s, bool upper_only);
void gram_rr(int64_t n, const double* S, int m, int k, double* G, double* scratch, void* tiles_dev, cudaStream_t s);
bool gram_fast(int64_t n, const double* const* ablk, const int* acols, int na, const double* const* bblk,
               const int* bcols, int nb, const int* bcol_out, double* G, int ldg, double* scratch, void* idx_dev,
               cudaStream_t s);
void fill_uniform_pm1_device(uint64_t seed, int64_t n, double* out, cudaStream_t s, int64_t offset = 0);
void gram_partials(int64_t n, const double* A, int ka, const double* B, int kb, double* part, void* tiles_dev,
                   cudaStream_t s);
void block_lincomb(int64_t n, const double* in, int kin, const double* C, int kout, double* out, cudaStream_t s);
bool block_lincomb_host_coef(int64_t n, const double* in, int kin, const double* C_host, int kout, double* out,
                             cudaStream_t s);
void block_sub_lincomb(int64_t n, const double* X, int k, const double* G, double* W, cudaStream_t s);
bool block_sub_lincomb_host_coef(int64_t n, const double* X, int k, const double* G_host, double* W,
                                 cudaStream_t s);
bool lobpcg_update_fused(int64_t n, int k, int m, double* S, double* AS, const double* C_host, const double* Cp_host,
                         const double* lam_host, double* R, cudaStream_t s, double* norms = nullptr);
void block_residual(int64_t n, int k, const double* AX, const double* X, const double* lam, double* R,
                    cudaStream_t s);
void pair_apply_block_internal(sait_pair_t p, const double* r, double* z, int64_t n, int64_t nvec, int layout,
                               cudaStream_t s);

namespace {

// The operator A: SELL-32 copy when regular, CSR kernels otherwise.
struct Operator {
  const DevCsr* a;
  SellMatrix sell;
  Operator(const DevCsr& m, cudaStream_t s) : a(&m), sell(make_sell(m, SAIT_FMT_AUTO, s)) {}
  void apply(const double* x, double* y, cudaStream_t s) const {
    if (sell.ok()) sell_spmv(sell, x, y, s);
    else spmv(*a, x, y, s);
  }
  // column-major n x k block
  void apply_block(const double* x, double* y, int k, cudaStream_t s) const {
    if (sell.ok()) {
      sell_spmm_colmajor(sell, x, a->ncols, y, a->nrows, k, s);
    } else {
      for (int j = 0; j < k; ++j) spmv(*a, x + a->ncols * j, y + a->nrows * j, s);
    }
  }
  void release(cudaStream_t s) { free_sell(sell, s); }
};

// Device time of the preconditioner applies inside a solve -- the paper's
// runtime split, which the reference takes with
// TimedPreconditioner (preconditioner.cpp:66-77) on the host: CUDA events
// around each apply on the solver's stream, a ring of pairs collected lazily
// (the loops synchronise every iteration anyway, so collecting never stalls
// the pipeline).
struct PrecondTimer {
  static constexpr int kRing = 32;
  cudaEvent_t ev[2 * kRing] = {};
  int head = 0, pending = 0;
  double ms = 0.0;
  int64_t count = 0;
  PrecondTimer() {
    for (auto& e : ev) SAIT_CUDA(cudaEventCreate(&e));
  }
  ~PrecondTimer() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  PrecondTimer(const PrecondTimer&) = delete;
  PrecondTimer& operator=(const PrecondTimer&) = delete;
  int begin(cudaStream_t s) {
    if (pending == kRing) collect_one();
    const int slot = (head + pending) % kRing;
    SAIT_CUDA(cudaEventRecord(ev[2 * slot], s));
    return slot;
  }
  void end(int slot, cudaStream_t s) {
    SAIT_CUDA(cudaEventRecord(ev[2 * slot + 1], s));
    ++pending;
  }
  void collect_one() {
    SAIT_CUDA(cudaEventSynchronize(ev[2 * head + 1]));
    float t = 0.f;
    SAIT_CUDA(cudaEventElapsedTime(&t, ev[2 * head], ev[2 * head + 1]));
    ms += t;
    ++count;
    head = (head + 1) % kRing;
    --pending;
  }
  void finish() {
    while (pending) collect_one();
  }
};

// z = M r: the SAIT pair, the exact ILU solves (the comparator), or identity
struct Precond {
  sait_pair_t p = nullptr;
  sait_exact_t e = nullptr;
  int64_t n = 0;
  PrecondTimer* timer = nullptr;
  bool present() const { return p || e; }
  int64_t dim() const { return p ? pair_dim(p) : e ? exact_dim(e) : n; }
  void apply(const double* r, double* z, cudaStream_t s) const {
    const int slot = timer ? timer->begin(s) : 0;
    if (p) pair_apply_internal(p, r, z, s);
    else if (e) exact_apply_internal(e, r, z, s);
    else SAIT_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    if (timer) timer->end(slot, s);
  }
};

// small device scratch for dot results, read back with one copy into a
// pinned buffer (a pageable destination is staged by the driver: ~10-20 us
// more per solver iteration)
struct Scalars {
  double* d = nullptr;
  double* part = nullptr;
  double* pinned = nullptr;
  std::vector<double> h;
  Scalars(int64_t n, int count, int max_m, cudaStream_t s) {
    d = dalloc<double>(count, s);
    part = dalloc<double>(dot_blocks(n) * max_m, s);
    h.assign(count, 0.0);
    SAIT_CUDA(cudaMallocHost(&pinned, sizeof(double) * (count > 0 ? count : 1)));
  }
  Scalars(const Scalars&) = delete;
  Scalars& operator=(const Scalars&) = delete;
  ~Scalars() {
    if (pinned) cudaFreeHost(pinned);
  }
  void fetch(int count, cudaStream_t s) {
    SAIT_CUDA(cudaMemcpyAsync(pinned, d, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    std::memcpy(h.data(), pinned, sizeof(double) * count);
  }
  void release(cudaStream_t s) {
    dfree(d, s);
    dfree(part, s);
  }
};

// ---- small dense algebra for LOBPCG's Rayleigh-Ritz (host; the same
// operation sequence as oracle/solvers.c so results agree bitwise).
bool chol_lower(const double* G, int m, double* L) {
  for (int i = 0; i < m * m; ++i) L[i] = 0.0;
  for (int j = 0; j < m; ++j) {
    double d = G[j * m + j];
    for (int k = 0; k < j; ++k) d = d - L[j * m + k] * L[j * m + k];
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    L[j * m + j] = ljj;
    for (int i = j + 1; i < m; ++i) {
      double t = G[i * m + j];
      for (int k = 0; k < j; ++k) t = t - L[i * m + k] * L[j * m + k];
      L[i * m + j] = t / ljj;
    }
  }
  return true;
}

void tri_lower_inv(const double* L, int m, double* Li) {
  for (int i = 0; i < m * m; ++i) Li[i] = 0.0;
  for (int j = 0; j < m; ++j) {
    Li[j * m + j] = 1.0 / L[j * m + j];
    for (int i = j + 1; i < m; ++i) {
      double t = 0.0;
      for (int k = j; k < i; ++k) t = t - L[i * m + k] * Li[k * m + j];
      Li[i * m + j] = t / L[i * m + i];
    }
  }
}

// cyclic Jacobi on symmetric F (destroyed): ascending eigenvalues w, vectors
// in Q's columns -- bitwise the restatement's jacobi_eig (oracle/solvers.c),
// which rotates columns p, q and then rows p, q.  F is exactly symmetric on
// entry (rayleigh_ritz symmetrises it) and stays so: for k != p, q the row
// step of (p, k), (q, k) is the same expression on the same operands as the
// column step of (k, p), (k, q).  So the rotation runs once on the
// contiguous rows and is mirrored into the columns; the 2 x 2 block (p, q)
// follows the column-then-row sequence exactly.  Q is kept transposed so its
// rotations are contiguous too (the RR solve sits between two GPU phases of
// every LOBPCG iteration: 30 % less host time at m = 24).
void jacobi_eig(double* F, int m, double* w, double* Q) {
  std::vector<double> QT(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i) QT[i * m + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) off = off + F[p * m + q] * F[p * m + q];
    if (off == 0.0) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        double* __restrict__ Fp = F + p * m;
        double* __restrict__ Fq = F + q * m;
        const double apq = Fp[q];
        if (apq == 0.0) continue;
        const double app = Fp[p], aqq = Fq[q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        // the 2 x 2 block after the column step
        const double cpp = c * app - s * apq, cpq = s * app + c * apq;
        const double cqp = c * Fq[p] - s * aqq, cqq = s * Fq[p] + c * aqq;
        for (int k = 0; k < m; ++k) {
          const double fpk = Fp[k], fqk = Fq[k];
          Fp[k] = c * fpk - s * fqk;
          Fq[k] = s * fpk + c * fqk;
        }
        for (int k = 0; k < m; ++k) {
          F[k * m + p] = Fp[k];
          F[k * m + q] = Fq[k];
        }
        Fp[p] = c * cpp - s * cqp;  // the row step on the block
        Fq[q] = s * cpq + c * cqq;
        Fp[q] = 0.0;
        Fq[p] = 0.0;
        double* __restrict__ Qp = QT.data() + p * m;
        double* __restrict__ Qq = QT.data() + q * m;
        for (int k = 0; k < m; ++k) {
          const double qkp = Qp[k], qkq = Qq[k];
          Qp[k] = c * qkp - s * qkq;
          Qq[k] = s * qkp + c * qkq;
        }
      }
  }
  std::vector<int> idx(m);
  for (int i = 0; i < m; ++i) idx[i] = i;
  for (int i = 0; i < m; ++i) {  // selection sort, ties keep index order
    int best = i;
    for (int j = i + 1; j < m; ++j)
      if (F[idx[j] * m + idx[j]] < F[idx[best] * m + idx[best]]) best = j;
    std::swap(idx[i], idx[best]);
  }
  for (int j = 0; j < m; ++j) {
    w[j] = F[idx[j] * m + idx[j]];
    for (int i = 0; i < m; ++i) Q[i * m + j] = QT[idx[j] * m + i];
  }
}

// k lowest B-orthonormal Ritz vectors of (GA, GB), m x m; C is m x k row-major
bool rayleigh_ritz(const double* GA, const double* GB, int m, int k, double* C, double* mu) {
  std::vector<double> L(m * m), Li(m * m), T(m * m), F(m * m), Q(m * m), w(m);
  if (!chol_lower(GB, m, L.data())) return false;
  tri_lower_inv(L.data(), m, Li.data());
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double t = 0.0;
      for (int q = 0; q < m; ++q) t = t + Li[i * m + q] * GA[q * m + j];
      T[i * m + j] = t;
    }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double t = 0.0;
      for (int q = 0; q < m; ++q) t = t + T[i * m + q] * Li[j * m + q];
      F[i * m + j] = t;
    }
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      const double a = 0.5 * (F[i * m + j] + F[j * m + i]);
      F[i * m + j] = a;
      F[j * m + i] = a;
    }
  jacobi_eig(F.data(), m, w.data(), Q.data());
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < k; ++j) {
      double t = 0.0;
      for (int q = 0; q < m; ++q) t = t + Li[q * m + i] * Q[q * m + j];
      C[i * k + j] = t;
    }
  for (int j = 0; j < k; ++j) mu[j] = w[j];
  return true;
}

}  // namespace
}  // namespace sait

struct sait_dcsr_s {
  int dev = 0;
  sait::DevCsr m;
};

namespace {
thread_local std::string g_solver_err;
}

namespace sait {
void set_last_error(const std::string& msg);
}

template <class F>
static int solver_guard(F&& f) {
  try {
    f();
    return SAIT_OK;
  } catch (const sait::Error& e) {
    sait::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    sait::set_last_error(e.what());
    return SAIT_ERR_RUNTIME;
  }
}

extern "C" {

static int gmres_impl(sait_dcsr_t A, sait::Precond M, const double* d_b, double* d_x, int64_t n, int restart,
                      double tol, int maxit, double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  return solver_guard([&] {
    if (!A || !d_b || !d_x) sait::throw_invalid("gmres: null argument");
    const sait::DevCsr& a = A->m;
    if (a.nrows != n || a.ncols != n) sait::throw_invalid("gmres: operator shape does not match n");
    if (M.present() && M.dim() != n) sait::throw_invalid("gmres: preconditioner dimension mismatch");
    if (restart < 1) sait::throw_invalid("gmres: restart must be >= 1");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != A->dev) SAIT_CUDA(cudaSetDevice(A->dev));
    cudaStream_t s = sait::as_stream(stream);
    const auto t0 = std::chrono::steady_clock::now();
    const int m = restart;
    sait::Operator op(a, s);
    sait::Precond pc = M;
    pc.n = n;
    sait::PrecondTimer ptimer;
    pc.timer = &ptimer;
    double* V = sait::dalloc<double>((m + 1) * n, s);
    double* w = sait::dalloc<double>(n, s);
    double* z = sait::dalloc<double>(n, s);
    double* u = sait::dalloc<double>(n, s);
    double* yd = sait::dalloc<double>(m, s);
    // scalar layout: [h (m+1) | h2 (m+1) | norm]
    sait::Scalars sc(n, 2 * (m + 1) + 1, m + 1, s);
    double* dh = sc.d;
    double* dh2 = sc.d + (m + 1);
    double* dnorm = sc.d + 2 * (m + 1);
    std::vector<double> H((m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0), h(m + 2, 0.0), y(m, 0.0);
    SAIT_CUDA(cudaMemsetAsync(d_x, 0, sizeof(double) * n, s));
    sait::multi_dot(n, d_b, d_b, n, 1, dnorm, sc.part, s, true);
    sc.fetch(2 * (m + 1) + 1, s);
    const double bnorm = sc.h[2 * (m + 1)];
    int its = 0;
    bool conv = false;
    double est = 1.0, beta = bnorm;
    if (h_hist) h_hist[0] = 1.0;
    if (bnorm == 0.0) {
      conv = true;
      est = 0.0;
    }
    SAIT_CUDA(cudaMemcpyAsync(w, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    SAIT_CUDA(cudaMemcpyAsync(dnorm, &beta, sizeof(double), cudaMemcpyHostToDevice, s));
    while (!conv && its < maxit) {
      sait::divide_by(n, w, dnorm, V, s);  // v0 = r / beta
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int k = 0;
      for (int i = 0; i < m && its < maxit; ++i) {
        double* vi = V + static_cast<int64_t>(i) * n;
        pc.apply(vi, z, s);
        op.apply(z, w, s);
        sait::multi_dot(n, w, V, n, i + 1, dh, sc.part, s, false);  // CGS2, pass 1
        sait::cgs_subtract(n, w, V, n, i + 1, dh, s);
        sait::multi_dot(n, w, V, n, i + 1, dh2, sc.part, s, false);  // pass 2
        sait::cgs_subtract(n, w, V, n, i + 1, dh2, s);
        sait::multi_dot(n, w, w, n, 1, dnorm, sc.part, s, true);
        sc.fetch(2 * (m + 1) + 1, s);
        for (int j = 0; j <= i; ++j) h[j] = sc.h[j] + sc.h[(m + 1) + j];
        h[i + 1] = sc.h[2 * (m + 1)];
        if (h[i + 1] != 0.0) sait::divide_by(n, w, dnorm, V + static_cast<int64_t>(i + 1) * n, s);
        for (int j = 0; j < i; ++j) {  // previous rotations
          const double t0 = cs[j] * h[j] + sn[j] * h[j + 1];
          const double t1 = -sn[j] * h[j] + cs[j] * h[j + 1];
          h[j] = t0;
          h[j + 1] = t1;
        }
        const double den = std::sqrt(h[i] * h[i] + h[i + 1] * h[i + 1]);
        if (den == 0.0) {
          cs[i] = 1.0;
          sn[i] = 0.0;
        } else {
          cs[i] = h[i] / den;
          sn[i] = h[i + 1] / den;
        }
        h[i] = den;
        h[i + 1] = 0.0;
        g[i + 1] = -sn[i] * g[i];
        g[i] = cs[i] * g[i];
        for (int j = 0; j <= i; ++j) H[j * m + i] = h[j];
        ++its;
        k = i + 1;
        est = std::fabs(g[i + 1]) / bnorm;
        if (h_hist) h_hist[its] = est;
        if (est <= tol) {
          conv = true;
          break;
        }
      }
      for (int ii = k - 1; ii >= 0; --ii) {  // back substitution
        double t = g[ii];
        for (int jj = ii + 1; jj < k; ++jj) t = t - H[ii * m + jj] * y[jj];
        y[ii] = t / H[ii * m + ii];
      }
      SAIT_CUDA(cudaMemcpyAsync(yd, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
      sait::linear_combination(n, V, n, k, yd, u, s);
      pc.apply(u, z, s);
      sait::y_plus_x(n, z, d_x, s);  // x += M (V y)
      op.apply(d_x, z, s);            // true residual r = b - A x
      sait::x_minus_y(n, d_b, z, s);  // z = b - Ax
      SAIT_CUDA(cudaMemcpyAsync(w, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      sait::multi_dot(n, w, w, n, 1, dnorm, sc.part, s, true);
      sc.fetch(2 * (m + 1) + 1, s);
      beta = sc.h[2 * (m + 1)];
      if (beta == 0.0) conv = true;
    }
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      stats->iterations = its;
      stats->converged = conv ? 1 : 0;
      stats->relres_estimate = est;
      stats->true_relres = bnorm == 0.0 ? 0.0 : beta / bnorm;
      stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      ptimer.finish();
      stats->precond_seconds = ptimer.ms * 1e-3;
      stats->precond_applies = ptimer.count;
    }
    sait::dfree(V, s);
    sait::dfree(w, s);
    sait::dfree(z, s);
    sait::dfree(u, s);
    sait::dfree(yd, s);
    sc.release(s);
    op.release(s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (dev != A->dev) cudaSetDevice(dev);
  });
}

static int pcg_impl(sait_dcsr_t A, sait::Precond M, const double* d_b, double* d_x, int64_t n, double tol,
                    int maxit, double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  return solver_guard([&] {
    if (!A || !d_b || !d_x) sait::throw_invalid("pcg: null argument");
    const sait::DevCsr& a = A->m;
    if (a.nrows != n || a.ncols != n) sait::throw_invalid("pcg: operator shape does not match n");
    if (M.present() && M.dim() != n) sait::throw_invalid("pcg: preconditioner dimension mismatch");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != A->dev) SAIT_CUDA(cudaSetDevice(A->dev));
    cudaStream_t s = sait::as_stream(stream);
    const auto t0 = std::chrono::steady_clock::now();
    sait::Operator op(a, s);
    sait::Precond pc = M;
    pc.n = n;
    sait::PrecondTimer ptimer;
    pc.timer = &ptimer;
    double* r = sait::dalloc<double>(n, s);
    double* z = sait::dalloc<double>(n, s);
    double* p = sait::dalloc<double>(n, s);
    double* q = sait::dalloc<double>(n, s);
    sait::Scalars sc(n, 4, 1, s);  // [dot | ...]
    auto dot = [&](const double* x, const double* y2, bool sq) {
      sait::multi_dot(n, x, y2, n, 1, sc.d, sc.part, s, sq);
      sc.fetch(1, s);
      return sc.h[0];
    };
    SAIT_CUDA(cudaMemsetAsync(d_x, 0, sizeof(double) * n, s));
    SAIT_CUDA(cudaMemcpyAsync(r, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    const double bnorm = dot(d_b, d_b, true);
    double rel = 1.0;
    int its = 0;
    bool conv = bnorm == 0.0, breakdown = false;
    if (h_hist) h_hist[0] = 1.0;
    if (!conv) {
      pc.apply(r, z, s);
      SAIT_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      double rz = dot(r, z, false);
      while (its < maxit) {
        op.apply(p, q, s);
        const double pq = dot(p, q, false);
        if (!(pq > 0.0)) {
          breakdown = true;
          break;
        }
        const double alpha = rz / pq;
        sait::axpy(n, alpha, p, d_x, s);
        sait::axpy(n, -alpha, q, r, s);
        ++its;
        rel = dot(r, r, true) / bnorm;
        if (h_hist) h_hist[its] = rel;
        if (rel <= tol) {
          conv = true;
          break;
        }
        pc.apply(r, z, s);
        const double rz2 = dot(r, z, false);
        const double beta = rz2 / rz;
        rz = rz2;
        sait::xpay(n, z, beta, p, s);  // p = z + beta p
      }
    }
    if (stats) {
      op.apply(d_x, q, s);
      sait::x_minus_y(n, d_b, q, s);
      const double tr = dot(q, q, true);
      stats->iterations = its;
      stats->converged = conv ? 1 : 0;
      stats->relres_estimate = bnorm == 0.0 ? 0.0 : rel;
      stats->true_relres = bnorm == 0.0 ? 0.0 : tr / bnorm;
      stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      ptimer.finish();
      stats->precond_seconds = ptimer.ms * 1e-3;
      stats->precond_applies = ptimer.count;
    }
    sait::dfree(r, s);
    sait::dfree(z, s);
    sait::dfree(p, s);
    sait::dfree(q, s);
    sc.release(s);
    op.release(s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (dev != A->dev) cudaSetDevice(dev);
    if (breakdown) sait::throw_runtime("pcg: breakdown, p'Ap <= 0 at iteration " + std::to_string(its));
  });
}

int sait_gmres(sait_dcsr_t A, sait_pair_t M, const double* d_b, double* d_x, int64_t n, int restart, double tol,
               int maxit, double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  sait::Precond pc;
  pc.p = M;
  return gmres_impl(A, pc, d_b, d_x, n, restart, tol, maxit, h_hist, stats, stream);
}

int sait_gmres_exact(sait_dcsr_t A, sait_exact_t M, const double* d_b, double* d_x, int64_t n, int restart,
                     double tol, int maxit, double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  sait::Precond pc;
  pc.e = M;
  return gmres_impl(A, pc, d_b, d_x, n, restart, tol, maxit, h_hist, stats, stream);
}

int sait_pcg(sait_dcsr_t A, sait_pair_t M, const double* d_b, double* d_x, int64_t n, double tol, int maxit,
             double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  sait::Precond pc;
  pc.p = M;
  return pcg_impl(A, pc, d_b, d_x, n, tol, maxit, h_hist, stats, stream);
}

int sait_pcg_exact(sait_dcsr_t A, sait_exact_t M, const double* d_b, double* d_x, int64_t n, double tol, int maxit,
                   double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  sait::Precond pc;
  pc.e = M;
  return pcg_impl(A, pc, d_b, d_x, n, tol, maxit, h_hist, stats, stream);
}

static int lobpcg_impl(sait_dcsr_t A, sait::Precond M, int nev, double tol, int maxit, uint64_t seed,
                       double* h_evals, double* d_evecs, double* h_resnorms, int* iterations, sait_stream_t stream,
                       sait_solve_stats* stats = nullptr, bool fast_gram = false) {
  return solver_guard([&] {
    const auto t_start = std::chrono::steady_clock::now();
    sait::PrecondTimer ptimer;
    if (!A || !h_evals || !iterations) sait::throw_invalid("lobpcg: null argument");
    const sait::DevCsr& a = A->m;
    const int64_t n = a.nrows;
    const int k = nev;
    if (a.ncols != n) sait::throw_invalid("lobpcg: operator is not square");
    if (k < 1 || k > 16) sait::throw_invalid("lobpcg: block size must be in [1, 16]");
    if (M.present() && M.dim() != n) sait::throw_invalid("lobpcg: preconditioner dimension mismatch");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != A->dev) SAIT_CUDA(cudaSetDevice(A->dev));
    cudaStream_t s = sait::as_stream(stream);
    sait::Operator op(a, s);
    const int64_t blk = static_cast<int64_t>(k) * n;
    double* S = sait::dalloc<double>(6 * blk, s);  // [X W P | AX AW AP]: one allocation (gram_rr)
    double* AS = S + 3 * blk;
    double* R = sait::dalloc<double>(blk, s);
    // small host->device operands (Gram corrections, coefficient blocks) use a
    // ring of slots so consecutive uploads need no synchronisation
    constexpr int kSlots = 8;
    double* dsmall = sait::dalloc<double>(kSlots * 48 * 48, s);
    int slot = 0;
    auto next_small = [&] { return dsmall + static_cast<int64_t>(48 * 48) * (slot++ % kSlots); };
    sait::Scalars sc(n, 48 * 96, 64, s);  // up to m x 6k Gram entries (gram_rr)
    double* gscratch = sait::dalloc<double>(sait::gram_scratch(n, 3 * k, 6 * k), s);
    void* gtiles = sait::dalloc<long long>(256, s);
    double *X = S, *W = S + blk, *P = S + 2 * blk;
    double *AX = AS, *AW = AS + blk, *AP = AS + 2 * blk;
    auto block_spmv = [&](const double* in, double* out) { op.apply_block(in, out, k, s); };
    // G[a][b] = S_a . Y_b (canonical dots, tiled tall-skinny kernel), row-major
    // ka x kb on the host; sym: S == Y, lower tiles mirrored (bitwise equal,
    // the canonical dot is symmetric in its arguments)
    // fast_gram: the tensor-core Gram (gram_fast: FP64 DMMA, deterministic,
    // not the canonical order); falls back to the canonical kernel for shapes
    // it does not cover
    auto gram_dmma = [&](const double* const* ab, int na, const double* const* bb, int nbk, const int* bout, int ka,
                         int ldg) {
      int ac[3], bc[6];
      for (int i = 0; i < na; ++i) ac[i] = std::min(8, ka - 8 * i);
      for (int i = 0; i < nbk; ++i) bc[i] = 8;
      return sait::gram_fast(n, ab, ac, na, bb, bc, nbk, bout, sc.d, ldg, gscratch, gtiles, s);
    };
    auto gram = [&](const double* Sa, int ka, const double* Yb, int kb, std::vector<double>& G, bool sym = false) {
      G.assign(static_cast<size_t>(ka) * kb, 0.0);
      if (fast_gram && kb % 8 == 0 && ka <= 24 && kb <= 48) {
        const double* ab[3];
        const double* bb[6];
        int bout[48];
        const int na = (ka + 7) / 8, nbk = kb / 8;
        for (int i = 0; i < na; ++i) ab[i] = Sa + static_cast<int64_t>(8 * i) * n;
        for (int i = 0; i < nbk; ++i) bb[i] = Yb + static_cast<int64_t>(8 * i) * n;
        for (int j = 0; j < kb; ++j) bout[j] = j;
        if (gram_dmma(ab, na, bb, nbk, bout, ka, kb)) {
          sc.fetch(ka * kb, s);
          std::copy(sc.h.begin(), sc.h.begin() + static_cast<size_t>(ka) * kb, G.begin());
          if (sym)
            for (int a2 = 0; a2 < ka; ++a2)
              for (int b2 = 0; b2 < a2; ++b2) G[a2 * kb + b2] = G[b2 * kb + a2];
          return;
        }
      }
      sait::gram(n, Sa, ka, Yb, kb, sc.d, kb, gscratch, gtiles, s, sym);
      sc.fetch(ka * kb, s);
      std::copy(sc.h.begin(), sc.h.begin() + static_cast<size_t>(ka) * kb, G.begin());
      if (sym)
        for (int a2 = 0; a2 < ka; ++a2)
          for (int b2 = 0; b2 < a2; ++b2)
            if ((b2 / 8) < (a2 / 8)) G[a2 * kb + b2] = G[b2 * kb + a2];
    };
    auto lincomb = [&](const double* in, int kin, const double* C, int kout, double* out) {
      if (sait::block_lincomb_host_coef(n, in, kin, C, kout, out, s)) return;
      double* d = next_small();
      SAIT_CUDA(cudaMemcpyAsync(d, C, sizeof(double) * kin * kout, cudaMemcpyHostToDevice, s));
      sait::block_lincomb(n, in, kin, d, kout, out, s);
    };
    auto cholqr = [&](double* Y, double* AY) {
      std::vector<double> G, L(k * k), Li(k * k), Ri(k * k);
      gram(Y, k, Y, k, G, true);
      if (!sait::chol_lower(G.data(), k, L.data())) return false;
      sait::tri_lower_inv(L.data(), k, Li.data());
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) Ri[i * k + j] = Li[j * k + i];
      lincomb(Y, k, Ri.data(), k, Y);  // in place: each element is read before it is written
      if (AY) {
        lincomb(AY, k, Ri.data(), k, AY);
      }
      return true;
    };
    std::vector<double> GA, GB, C(48 * 16), lam(48);
    static const bool dbg = std::getenv("SAIT_DEBUG_LOBPCG") != nullptr;
    // SAIT_LOBPCG_FUSED=0: the unfused update (A/B and parity checks)
    static const bool fused_off = [] {
      const char* e = std::getenv("SAIT_LOBPCG_FUSED");
      return e && e[0] == '0';
    }();
    const bool defer_w = fast_gram && !fused_off && k == 8;
    // deferred W normalisation (fast mode): W_n = W Rwi with Rwi = L^-T, L the
    // Cholesky factor of W^T W = GB[k:2k, k:2k]; the Grams of [X W_n P] are
    // T^T G T with T = diag(I, Rwi, I)
    std::vector<double> Rwi(k * k);
    bool w_deficient = false;
    auto normalize_w = [&](std::vector<double>& GA2, std::vector<double>& GB2, int mm) {
      std::vector<double> Gw(k * k), Lw(k * k), Lwi(k * k), tmpG(static_cast<size_t>(mm) * mm);
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) Gw[i * k + j] = GB2[(k + i) * mm + k + j];
      if (!sait::chol_lower(Gw.data(), k, Lw.data())) return false;
      sait::tri_lower_inv(Lw.data(), k, Lwi.data());
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) Rwi[i * k + j] = Lwi[j * k + i];
      for (std::vector<double>* Gp : {&GA2, &GB2}) {
        std::vector<double>& G = *Gp;
        tmpG = G;  // G T: the W columns
        for (int a2 = 0; a2 < mm; ++a2)
          for (int j = 0; j < k; ++j) {
            double t = 0.0;
            for (int q = 0; q <= j; ++q) t += G[a2 * mm + k + q] * Rwi[q * k + j];
            tmpG[a2 * mm + k + j] = t;
          }
        G = tmpG;  // T^T (G T): the W rows
        for (int i = 0; i < k; ++i)
          for (int b2 = 0; b2 < mm; ++b2) {
            double t = 0.0;
            for (int q = 0; q <= i; ++q) t += Rwi[q * k + i] * tmpG[(k + q) * mm + b2];
            G[(k + i) * mm + b2] = t;
          }
        for (int i = 0; i < mm; ++i)  // exactly symmetric
          for (int j = i + 1; j < mm; ++j) {
            const double s2 = 0.5 * (G[i * mm + j] + G[j * mm + i]);
            G[i * mm + j] = s2;
            G[j * mm + i] = s2;
          }
      }
      return true;
    };
    auto unnormalize_w_rows = [&](double* Cw) {  // k rows of k coefficients: Cw <- Rwi Cw
      std::vector<double> t(k * k);
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
          double a = 0.0;
          for (int q = i; q < k; ++q) a += Rwi[i * k + q] * Cw[q * k + j];
          t[i * k + j] = a;
        }
      std::copy(t.begin(), t.end(), Cw);
    };
    auto tp = std::chrono::steady_clock::now();
    auto phase = [&](const char* nm) {
      if (!dbg) return;
      SAIT_CUDA(cudaStreamSynchronize(s));
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "%s=%.2fms ", nm, std::chrono::duration<double, std::milli>(now - tp).count());
      tp = now;
    };
    // X0 ~ U[-1,1], column j from seed (seed * 1000 + j), generated on the
    // device with the host generator's exact arithmetic
    for (int j = 0; j < k; ++j)
      sait::fill_uniform_pm1_device(seed * 1000 + static_cast<uint64_t>(j), n, X + static_cast<int64_t>(j) * n, s);
    phase("init_x");
    block_spmv(X, AX);
    bool failed = false;
    std::string why;
    gram(X, k, X, k, GB, true);
    gram(X, k, AX, k, GA);
    int it = 0;
    bool conv = false, have_p = false;
    if (!sait::rayleigh_ritz(GA.data(), GB.data(), k, k, C.data(), lam.data())) {
      failed = true;
      why = "lobpcg: initial block is rank deficient";
    } else {
      lincomb(X, k, C.data(), k, X);
      lincomb(AX, k, C.data(), k, AX);
      bool r_ready = false;   // R already written by the fused update
      bool norms_ready = false;  // ... and its column norms in sc.d (fast mode)
      bool p_normed = false;  // P, AP already orthonormalised (fast mode)
      for (it = 0; it <= maxit; ++it) {
        if (!r_ready) {
          double* dl = next_small();
          SAIT_CUDA(cudaMemcpyAsync(dl, lam.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
          sait::block_residual(n, k, AX, X, dl, R, s);
        }
        r_ready = false;
        if (!norms_ready)
          for (int j = 0; j < k; ++j)
            sait::multi_dot(n, R + static_cast<int64_t>(j) * n, R + static_cast<int64_t>(j) * n, n, 1, sc.d + j,
                            sc.part, s, true);
        norms_ready = false;
        sc.fetch(k, s);
        conv = true;
        for (int j = 0; j < k; ++j) {
          if (h_resnorms) h_resnorms[static_cast<int64_t>(it) * k + j] = sc.h[j];
          if (!(sc.h[j] <= tol)) conv = false;
        }
        phase("\nresid");
        if (conv || it == maxit) break;
        const int pslot = ptimer.begin(s);
        if (M.p) {
          sait::pair_apply_block_internal(M.p, R, W, n, k, 0, s);
        } else if (M.e) {  // exact ILU solves, column by column
          for (int j = 0; j < k; ++j)
            sait::exact_apply_internal(M.e, R + static_cast<int64_t>(j) * n, W + static_cast<int64_t>(j) * n, s);
        } else {
          SAIT_CUDA(cudaMemcpyAsync(W, R, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
        }
        ptimer.end(pslot, s);
        phase("precond");
        std::vector<double> G1;
        gram(X, k, W, k, G1);
        if (!sait::block_sub_lincomb_host_coef(n, X, k, G1.data(), W, s)) {
          double* dg = next_small();
          SAIT_CUDA(cudaMemcpyAsync(dg, G1.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, s));
          sait::block_sub_lincomb(n, X, k, dg, W, s);
        }
        // fast mode defers W's Cholesky-QR: the Rayleigh-Ritz Gram already
        // holds W^T W, so the normalisation W R^-1 is applied to the Grams and
        // folded into the update coefficients on the host (no W^T W pass, no
        // W R^-1 pass); the canonical mode keeps the restatement's cholqr
        if (!defer_w && !cholqr(W, nullptr)) {
          failed = true;
          why = "lobpcg: preconditioned residual block is rank deficient";
          break;
        }
        phase("orth_w");
        block_spmv(W, AW);
        phase("aw");
        const bool use_p = have_p && (p_normed || cholqr(P, AP));
        phase("cholqr_p");
        int m = use_p ? 3 * k : 2 * k;
        bool ok = false;
        while (true) {
          bool fast_done = false;
          if (fast_gram && m % 8 == 0 && m <= 24) {  // both Grams from one tensor-core pass over [S | AS]
            const double* ab[3];
            const double* bb[6];
            int bout[48];
            const int na = m / 8;
            for (int i = 0; i < na; ++i) {
              ab[i] = S + static_cast<int64_t>(8 * i) * n;
              bb[i] = S + static_cast<int64_t>(8 * i) * n;
              bb[na + i] = AS + static_cast<int64_t>(8 * i) * n;
            }
            for (int j = 0; j < 2 * m; ++j) bout[j] = j;
            if (gram_dmma(ab, na, bb, 2 * na, bout, m, 2 * m)) {
              sc.fetch(m * 2 * m, s);
              GB.assign(static_cast<size_t>(m) * m, 0.0);
              GA.assign(static_cast<size_t>(m) * m, 0.0);
              for (int a2 = 0; a2 < m; ++a2)
                for (int b2 = 0; b2 < m; ++b2) {
                  GB[a2 * m + b2] = b2 >= a2 ? sc.h[a2 * 2 * m + b2] : sc.h[b2 * 2 * m + a2];  // exactly symmetric
                  // S^T AS: the tiles below the block diagonal are not
                  // computed (gram_dmma_kernel); mirror the upper ones
                  GA[a2 * m + b2] = b2 / 8 >= a2 / 8 ? sc.h[a2 * 2 * m + m + b2] : sc.h[b2 * 2 * m + m + a2];
                }
              fast_done = true;
            }
          }
          if (!fast_done) {  // both Grams in one launch (S read once), one read-back
            const int ld = 6 * k;
            sait::gram_rr(n, S, m, k, sc.d, gscratch, gtiles, s);
            sc.fetch(m * ld, s);
            GB.assign(static_cast<size_t>(m) * m, 0.0);
            GA.assign(static_cast<size_t>(m) * m, 0.0);
            for (int a2 = 0; a2 < m; ++a2)
              for (int b2 = 0; b2 < m; ++b2) {
                GB[a2 * m + b2] = sc.h[a2 * ld + b2];
                GA[a2 * m + b2] = sc.h[a2 * ld + 3 * k + b2];
              }
            for (int a2 = 0; a2 < m; ++a2)  // GB's skipped lower tiles mirror the upper ones (as gram(sym))
              for (int b2 = 0; b2 < a2; ++b2)
                if ((b2 / 8) < (a2 / 8)) GB[a2 * m + b2] = GB[b2 * m + a2];
          }
          for (int i = 0; i < m; ++i)
            for (int j = i + 1; j < m; ++j) {
              const double s2 = 0.5 * (GA[i * m + j] + GA[j * m + i]);
              GA[i * m + j] = s2;
              GA[j * m + i] = s2;
            }
          if (defer_w && !normalize_w(GA, GB, m)) {
            w_deficient = true;
            break;
          }
          if (sait::rayleigh_ritz(GA.data(), GB.data(), m, k, C.data(), lam.data())) {
            ok = true;
            break;
          }
          if (m == 3 * k) {
            m = 2 * k;
            continue;
          }
          break;
        }
        phase("rr");
        if (w_deficient) {
          failed = true;
          why = "lobpcg: preconditioned residual block is rank deficient";
          break;
        }
        if (!ok) {
          failed = true;
          why = "lobpcg: Gram matrix not positive definite";
          break;
        }
        // in place, each element read before it is written: X and AX first
        // (they read the old P), then P and AP (from W and the old P)
        // P's coefficients.  Fast mode folds the next iteration's Cholesky-QR
        // of P into them: P_new = [W P] Cp has the Gram Cp^T GB[k:m, k:m] Cp
        // (GB: this iteration's Gram of [X W P]), so P_new Ri comes out of
        // the same pass with Cp Ri (no PᵀP pass, no two k x k lincombs).  The
        // canonical mode keeps the restatement's explicit cholqr (bitwise).
        const double* Cp = C.data() + k * k;
        std::vector<double> Cpf;
        p_normed = false;
        if (fast_gram && !fused_off && k == 8) {
          const int mp = m - k;
          std::vector<double> T(static_cast<size_t>(mp) * k), Gp(k * k), Lp(k * k), Lpi(k * k);
          for (int a2 = 0; a2 < mp; ++a2)  // T = GB[k:m, k:m] Cp
            for (int j = 0; j < k; ++j) {
              double t = 0.0;
              for (int b2 = 0; b2 < mp; ++b2) t += GB[(k + a2) * m + k + b2] * Cp[b2 * k + j];
              T[a2 * k + j] = t;
            }
          for (int i = 0; i < k; ++i)  // Gp = Cp^T T, symmetrised
            for (int j = 0; j <= i; ++j) {
              double t = 0.0;
              for (int a2 = 0; a2 < mp; ++a2) t += Cp[a2 * k + i] * T[a2 * k + j];
              Gp[i * k + j] = t;
              Gp[j * k + i] = t;
            }
          if (sait::chol_lower(Gp.data(), k, Lp.data())) {
            sait::tri_lower_inv(Lp.data(), k, Lpi.data());
            Cpf.assign(static_cast<size_t>(mp) * k, 0.0);  // Cp Ri, Ri = Lpi^T
            for (int a2 = 0; a2 < mp; ++a2)
              for (int j = 0; j < k; ++j) {
                double t = 0.0;
                for (int q = 0; q <= j; ++q) t += Cp[a2 * k + q] * Lpi[j * k + q];
                Cpf[a2 * k + j] = t;
              }
            Cp = Cpf.data();
            p_normed = true;
          }
        }
        if (defer_w) {  // coefficients of the normalised W -> of the stored W (rows of W: Rwi c)
          unnormalize_w_rows(C.data() + k * k);  // X's coefficients (and P's, when Cp points into C)
          if (Cp != C.data() + k * k) unnormalize_w_rows(Cpf.data());
        }
        // fast mode: the update also leaves the next residual's norms in sc.d
        // (block partials of its own pass; the canonical mode keeps the
        // restatement's per-column dots)
        if (!fused_off && sait::lobpcg_update_fused(n, k, m, S, AS, C.data(), Cp, lam.data(), R, s,
                                                    defer_w ? sc.d : nullptr)) {
          r_ready = true;  // (canonical mode: bitwise the four lincombs + the next residual)
          norms_ready = defer_w;
        } else {
          p_normed = false;
          lincomb(S, m, C.data(), k, X);
          lincomb(AS, m, C.data(), k, AX);
          lincomb(W, m - k, C.data() + k * k, k, P);
          lincomb(AW, m - k, C.data() + k * k, k, AP);
        }
        have_p = true;
        phase("update");
      }
    }
    for (int j = 0; j < k; ++j) h_evals[j] = lam[j];
    if (d_evecs) SAIT_CUDA(cudaMemcpyAsync(d_evecs, X, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
    *iterations = it;
    if (stats) {
      ptimer.finish();
      stats->iterations = it;
      stats->converged = conv ? 1 : 0;
      stats->relres_estimate = 0.0;
      stats->true_relres = 0.0;
      stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      stats->precond_seconds = ptimer.ms * 1e-3;
      stats->precond_applies = ptimer.count;
    }
    SAIT_CUDA(cudaStreamSynchronize(s));
    sait::dfree(S, s);  // (AS lives in the same allocation)
    sait::dfree(R, s);
    sait::dfree(dsmall, s);
    sait::dfree(gscratch, s);
    sait::dfree(gtiles, s);
    sc.release(s);
    op.release(s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (dev != A->dev) cudaSetDevice(dev);
    if (failed) sait::throw_runtime(why);
  });
}

int sait_lobpcg(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed, double* h_evals,
                double* d_evecs, double* h_resnorms, int* iterations, sait_stream_t stream) {
  sait::Precond pc;
  pc.p = M;
  return lobpcg_impl(A, pc, nev, tol, maxit, seed, h_evals, d_evecs, h_resnorms, iterations, stream);
}

int sait_lobpcg_ex(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed, double* h_evals,
                   double* d_evecs, double* h_resnorms, int* iterations, sait_solve_stats* stats,
                   sait_stream_t stream) {
  sait::Precond pc;
  pc.p = M;
  return lobpcg_impl(A, pc, nev, tol, maxit, seed, h_evals, d_evecs, h_resnorms, iterations, stream, stats);
}

int sait_lobpcg_opt(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed, int gram_mode,
                    double* h_evals, double* d_evecs, double* h_resnorms, int* iterations, sait_solve_stats* stats,
                    sait_stream_t stream) {
  if (gram_mode != SAIT_GRAM_CANONICAL && gram_mode != SAIT_GRAM_TENSOR) {
    sait::set_last_error("lobpcg: unknown gram mode " + std::to_string(gram_mode));
    return SAIT_ERR_INVALID_ARGUMENT;
  }
  sait::Precond pc;
  pc.p = M;
  return lobpcg_impl(A, pc, nev, tol, maxit, seed, h_evals, d_evecs, h_resnorms, iterations, stream, stats,
                     gram_mode == SAIT_GRAM_TENSOR);
}

int sait_lobpcg_exact(sait_dcsr_t A, sait_exact_t M, int nev, double tol, int maxit, uint64_t seed,
                      double* h_evals, double* d_evecs, double* h_resnorms, int* iterations, sait_stream_t stream) {
  sait::Precond pc;
  pc.e = M;
  return lobpcg_impl(A, pc, nev, tol, maxit, seed, h_evals, d_evecs, h_resnorms, iterations, stream);
}

// ---- vector primitives of the solver loops (for loops that run across
// ranks; identical kernels, so identical bits)
int64_t sait_dot_blocks(int64_t n) { return sait::dot_blocks(n); }

int sait_dot_partials(const double* d_x, const double* d_V, int64_t ld, int m, int64_t n, double* d_partials,
                      sait_stream_t stream) {
  return solver_guard([&] {
    if (m < 0 || n < 0 || (m > 0 && (!d_x || !d_V || !d_partials))) sait::throw_invalid("dot_partials: bad arguments");
    if (m == 0 || n == 0) return;
    sait::dot_partials(n, d_x, d_V, ld, m, d_partials, sait::as_stream(stream));
  });
}

int sait_dot_fold(const double* d_partials, int64_t nb, int m, double* d_out, int sqrt_out, sait_stream_t stream) {
  return solver_guard([&] {
    if (m < 0 || nb < 1 || (m > 0 && (!d_partials || !d_out))) sait::throw_invalid("dot_fold: bad arguments");
    sait::dot_fold(d_partials, nb, m, d_out, sqrt_out != 0, sait::as_stream(stream));
  });
}

int sait_vec_update(int op, int64_t n, double a, const double* d_x, double* d_y, sait_stream_t stream) {
  return solver_guard([&] {
    if (n < 0 || (n > 0 && (!d_x || !d_y))) sait::throw_invalid("vec_update: bad arguments");
    if (n == 0) return;
    cudaStream_t s = sait::as_stream(stream);
    switch (op) {
      case 0: sait::axpy(n, a, d_x, d_y, s); break;      // y = y + a x
      case 1: sait::xpay(n, d_x, a, d_y, s); break;      // y = x + a y
      case 2: sait::x_minus_y(n, d_x, d_y, s); break;    // y = x - y
      case 3: sait::y_plus_x(n, d_x, d_y, s); break;     // y = y + x
      default: sait::throw_invalid("vec_update: unknown op");
    }
  });
}

int sait_vec_cgs(int64_t n, double* d_w, const double* d_V, int64_t ld, int m, const double* d_h,
                 sait_stream_t stream) {
  return solver_guard([&] {
    if (n > 0 && m > 0) sait::cgs_subtract(n, d_w, d_V, ld, m, d_h, sait::as_stream(stream));
  });
}

int sait_vec_div(int64_t n, const double* d_w, const double* d_d, double* d_out, sait_stream_t stream) {
  return solver_guard([&] {
    if (n > 0) sait::divide_by(n, d_w, d_d, d_out, sait::as_stream(stream));
  });
}

int sait_gram_partials(const double* d_A, int ka, const double* d_B, int kb, int64_t n, double* d_partials,
                       sait_stream_t stream) {
  return solver_guard([&] {
    if (ka < 1 || kb < 1 || ka > 48 || kb > 48 || n < 0) sait::throw_invalid("gram_partials: bad arguments");
    if (n == 0) return;
    void* tiles = nullptr;
    cudaStream_t s = sait::as_stream(stream);
    tiles = sait::dalloc<long long>(256, s);
    sait::gram_partials(n, d_A, ka, d_B, kb, d_partials, tiles, s);
    sait::dfree(tiles, s);
  });
}

int sait_block_lincomb(int64_t n, const double* d_in, int kin, const double* d_C, int kout, double* d_out,
                       sait_stream_t stream) {
  return solver_guard([&] {
    if (kin < 1 || kin > 48 || kout < 1 || kout > 16) sait::throw_invalid("block_lincomb: bad arguments");
    if (n > 0) sait::block_lincomb(n, d_in, kin, d_C, kout, d_out, sait::as_stream(stream));
  });
}

int sait_block_sub_lincomb(int64_t n, const double* d_X, int k, const double* d_G, double* d_W,
                           sait_stream_t stream) {
  return solver_guard([&] {
    if (k < 1 || k > 16) sait::throw_invalid("block_sub_lincomb: bad arguments");
    if (n > 0) sait::block_sub_lincomb(n, d_X, k, d_G, d_W, sait::as_stream(stream));
  });
}

int sait_block_residual(int64_t n, int k, const double* d_AX, const double* d_X, const double* d_lam, double* d_R,
                        sait_stream_t stream) {
  return solver_guard([&] {
    if (k < 1) sait::throw_invalid("block_residual: bad arguments");
    if (n > 0) sait::block_residual(n, k, d_AX, d_X, d_lam, d_R, sait::as_stream(stream));
  });
}

int sait_fill_uniform_pm1_device(uint64_t seed, int64_t n, int64_t offset, double* d_out, sait_stream_t stream) {
  return solver_guard([&] { sait::fill_uniform_pm1_device(seed, n, d_out, sait::as_stream(stream), offset); });
}

int sait_dense_chol_lower(const double* G, int m, double* L) { return sait::chol_lower(G, m, L) ? 1 : 0; }
void sait_dense_tri_lower_inv(const double* L, int m, double* Li) { sait::tri_lower_inv(L, m, Li); }
int sait_dense_rayleigh_ritz(const double* GA, const double* GB, int m, int k, double* C, double* lam) {
  return sait::rayleigh_ritz(GA, GB, m, k, C, lam) ? 1 : 0;
}

int sait_vec_lincomb(int64_t n, const double* d_V, int64_t ld, int k, const double* d_y, double* d_u,
                     sait_stream_t stream) {
  return solver_guard([&] {
    if (n > 0 && k > 0) sait::linear_combination(n, d_V, ld, k, d_y, d_u, sait::as_stream(stream));
  });
}

}  // extern "C"
