// solvers.cu — device-resident solver loops that drive the SAIT apply
// (north_star (3); GMRES per DESIGN.md "solvers").
// Vectors never leave HBM; per iteration only the few scalars the host needs
// for control (dots, Hessenberg column) come back.  Operation order matches
// oracle/solvers.c exactly (canonical dots in blas.cu, the same elementwise
// expressions, the same host-side Givens/back-substitution code), so iteration
// counts and residual histories are bitwise identical to the CPU restatement.
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace sait {
void pair_apply_internal(sait_pair_t p, const double* r, double* z, cudaStream_t s);
int64_t pair_dim(sait_pair_t p);

int64_t dot_blocks(int64_t n);
void multi_dot(int64_t n, const double* x, const double* V, int64_t ld, int m, double* out, double* scratch,
               cudaStream_t s, bool sqrt_out);
void cgs_subtract(int64_t n, double* w, const double* V, int64_t ld, int m, const double* h, cudaStream_t s);
void divide_by(int64_t n, const double* w, const double* d, double* out, cudaStream_t s);
void linear_combination(int64_t n, const double* V, int64_t ld, int k, const double* y, double* u, cudaStream_t s);
void axpy(int64_t n, double a, const double* x, double* y, cudaStream_t s);
void xpay(int64_t n, const double* x, double a, double* y, cudaStream_t s);
void x_minus_y(int64_t n, const double* x, double* y, cudaStream_t s);
void y_plus_x(int64_t n, const double* x, double* y, cudaStream_t s);

namespace {

// The operator A: SELL-32 copy when regular, CSR kernels otherwise.
struct Operator {
  const DevCsr* a;
  SellMatrix sell;
  Operator(const DevCsr& m, cudaStream_t s) : a(&m), sell(make_sell(m, s)) {}
  void apply(const double* x, double* y, cudaStream_t s) const {
    if (sell.ok()) sell_spmv(sell, x, y, s);
    else spmv(*a, x, y, s);
  }
  void release(cudaStream_t s) { free_sell(sell, s); }
};

struct Precond {
  sait_pair_t p;
  int64_t n;
  void apply(const double* r, double* z, cudaStream_t s) const {
    if (p) pair_apply_internal(p, r, z, s);
    else SAIT_CUDA(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
};

// small device scratch for dot results, read back with one copy
struct Scalars {
  double* d = nullptr;
  double* part = nullptr;
  std::vector<double> h;
  Scalars(int64_t n, int count, int max_m, cudaStream_t s) {
    d = dalloc<double>(count, s);
    part = dalloc<double>(dot_blocks(n) * max_m, s);
    h.assign(count, 0.0);
  }
  void fetch(int count, cudaStream_t s) {
    SAIT_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
  }
  void release(cudaStream_t s) {
    dfree(d, s);
    dfree(part, s);
  }
};

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

int sait_gmres(sait_dcsr_t A, sait_pair_t M, const double* d_b, double* d_x, int64_t n, int restart, double tol,
               int maxit, double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  return solver_guard([&] {
    if (!A || !d_b || !d_x) sait::throw_invalid("gmres: null argument");
    const sait::DevCsr& a = A->m;
    if (a.nrows != n || a.ncols != n) sait::throw_invalid("gmres: operator shape does not match n");
    if (M && sait::pair_dim(M) != n) sait::throw_invalid("gmres: preconditioner dimension mismatch");
    if (restart < 1) sait::throw_invalid("gmres: restart must be >= 1");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != A->dev) SAIT_CUDA(cudaSetDevice(A->dev));
    cudaStream_t s = sait::as_stream(stream);
    const auto t0 = std::chrono::steady_clock::now();
    const int m = restart;
    sait::Operator op(a, s);
    sait::Precond pc{M, n};
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

int sait_pcg(sait_dcsr_t A, sait_pair_t M, const double* d_b, double* d_x, int64_t n, double tol, int maxit,
             double* h_hist, sait_solve_stats* stats, sait_stream_t stream) {
  return solver_guard([&] {
    if (!A || !d_b || !d_x) sait::throw_invalid("pcg: null argument");
    const sait::DevCsr& a = A->m;
    if (a.nrows != n || a.ncols != n) sait::throw_invalid("pcg: operator shape does not match n");
    if (M && sait::pair_dim(M) != n) sait::throw_invalid("pcg: preconditioner dimension mismatch");
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != A->dev) SAIT_CUDA(cudaSetDevice(A->dev));
    cudaStream_t s = sait::as_stream(stream);
    const auto t0 = std::chrono::steady_clock::now();
    sait::Operator op(a, s);
    sait::Precond pc{M, n};
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

}  // extern "C"
