/*
 * solvers.c — CPU restatement of the solver loops that drive the SAIT apply
 * (TEST INFRASTRUCTURE ONLY, see sait_oracle.h).
 *
 * The reference has no solver code: PCG / LOBPCG exist only in SPEC.md:282-351
 * and GMRES is not specified at all (SPEC.md:347 lists it as a non-goal while
 * BASELINE.json configs 1 and 3 require GMRES(30)).  Iteration-count parity is
 * therefore UNPINNED against the reference; these restatements fix the
 * algorithms and define the canonical reduction order
 * that the device kernels reproduce, so GPU and CPU agree bit for bit.  The
 * solvers' own vector arithmetic (dots, Gram blocks, axpy-type updates,
 * Gram-Schmidt and block linear combinations) uses fused multiply-adds (C99
 * fma, correctly rounded, = the device's __fma_rn); the SAIT path itself
 * (spmv / spgemm in sait_oracle.c) keeps the reference's unfused order.
 *
 * Canonical dot (orc_dot): blocks of 2048 elements; in block b, "thread" t
 * (0..255) accumulates s = fma(a[i], b[i], s) for i = 2048 b + t + 256 k,
 * k = 0..7 in order, starting from 0.0; the 256 per-thread sums are combined by a butterfly
 * within each 32-lane warp (offsets 16,8,4,2,1: v[l] += v[l^off], result at
 * lane 0) and then across the 8 warp results (offsets 4,2,1).  The block
 * partials P_b are reduced the same way by one 256-thread block whose thread
 * t first sums P_t, P_{t+256}, ... in order from 0.0.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "sait_oracle.h"

#define DOT_T 256
#define DOT_K 8
#define DOT_B (DOT_T * DOT_K)

/* butterfly over 32 lanes then over 8 warp leaders; v has DOT_T entries */
static double block_tree(double *v) {
  double w[8];
  for (int warp = 0; warp < 8; ++warp) {
    double l[32];
    memcpy(l, v + 32 * warp, sizeof l);
    for (int off = 16; off >= 1; off >>= 1) {
      double nl[32];
      for (int i = 0; i < 32; ++i) nl[i] = l[i] + l[i ^ off];
      memcpy(l, nl, sizeof l);
    }
    w[warp] = l[0];
  }
  for (int off = 4; off >= 1; off >>= 1) {
    double nw[8];
    for (int i = 0; i < 8; ++i) nw[i] = w[i] + w[i ^ off];
    memcpy(w, nw, sizeof w);
  }
  return w[0];
}

/* partial of one 2048-element block (the canonical per-block order) */
static double block_partial(const double *a, const double *b, int64_t n, int64_t blk) {
  double v[DOT_T];
  for (int t = 0; t < DOT_T; ++t) {
    double s = 0.0;
    for (int k = 0; k < DOT_K; ++k) {
      int64_t i = blk * DOT_B + t + (int64_t)DOT_T * k;
      if (i < n) s = fma(a[i], b[i], s);
    }
    v[t] = s;
  }
  return block_tree(v);
}

/* fold of the block partials (one 256-thread block, then the tree) */
static double fold_partials(const double *part, int64_t nb, int64_t stride) {
  double v[DOT_T];
  for (int t = 0; t < DOT_T; ++t) {
    double s = 0.0;
    for (int64_t q = t; q < nb; q += DOT_T) s = s + part[q * stride];
    v[t] = s;
  }
  return block_tree(v);
}

static int64_t dot_blocks(int64_t n) {
  int64_t nb = (n + DOT_B - 1) / DOT_B;
  return nb < 1 ? 1 : nb;
}

/* The blocks are independent, so they are computed in parallel (OpenMP);
 * every partial and the fold keep the canonical order: bitwise the serial
 * restatement for any thread count. */
double orc_dot(const double *a, const double *b, int64_t n) {
  int64_t nb = dot_blocks(n);
  double *part = (double *)malloc((size_t)nb * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t blk = 0; blk < nb; ++blk) part[blk] = block_partial(a, b, n, blk);
  double r = fold_partials(part, nb, 1);
  free(part);
  return r;
}

/* G[a * ld + b] = orc_dot(S_a, Y_b) for a < ka, b < kb (column-major blocks
 * of n rows): the same canonical dots, computed block by block so that each
 * 2048-row slab of S and Y is read once from memory. */
static void multi_dot(const double *S, int ka, const double *Y, int kb, int64_t n, double *G, int ld) {
  int64_t nb = dot_blocks(n);
  const int np = ka * kb;
  double *part = (double *)malloc((size_t)nb * (size_t)np * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t blk = 0; blk < nb; ++blk)
    for (int a = 0; a < ka; ++a)
      for (int b = 0; b < kb; ++b)
        part[blk * np + a * kb + b] = block_partial(S + (int64_t)a * n, Y + (int64_t)b * n, n, blk);
  for (int a = 0; a < ka; ++a)
    for (int b = 0; b < kb; ++b) G[a * ld + b] = fold_partials(part + a * kb + b, nb, np);
  free(part);
}

static double nrm(const double *a, int64_t n) { return sqrt(orc_dot(a, a, n)); }

static int fail_solver(const char *msg) {
  extern int orc_set_error(const char *m);
  return orc_set_error(msg);
}

/* How (ml, mu) precondition GMRES / PCG: 0 = the SAIT pair z = M_U (M_L r);
 * 1 = the exact ILU solves z = U^-1 (L^-1 r) (ExactIluPreconditioner,
 * preconditioner.cpp:28-32) with ml = L, mu = U. */
static int g_precond_exact = 0;
void orc_solver_precond_exact(int on) { g_precond_exact = on; }

/* z = M r, or a copy when no preconditioner */
static void precond(const orc_csr *ml, const orc_csr *mu, const double *r, double *z, int64_t n) {
  if (ml && mu && g_precond_exact) {
    double *y = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    memset(z, 0, (size_t)n * sizeof(double));
    orc_trisolve(ml, 1, r, y);
    orc_trisolve(mu, 0, y, z);
    free(y);
  } else if (ml && mu) {
    orc_pair_apply(ml, mu, r, z);
  } else {
    memcpy(z, r, (size_t)n * sizeof(double));
  }
}

/*
 * Right-preconditioned restarted GMRES(m) from x0 = 0:
 * Arnoldi on A M with classical Gram-Schmidt applied twice (CGS2), Givens
 * rotations on the Hessenberg column, stop when the Arnoldi residual estimate
 * |g_{i+1}| / ||b|| <= tol (checked every iteration), x += M (V y) at the end
 * of each cycle, true residual recomputed at every restart and at exit.
 * hist[k] = relative residual estimate after k iterations (hist[0] = 1).
 */
int orc_gmres(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, const double *b, int m,
              double tol, int maxit, double *x, double *hist, orc_solve_stats *st) {
  int64_t n = a->nrows;
  double *V = (double *)calloc((size_t)(m + 1) * (size_t)n, sizeof(double));
  double *w = (double *)malloc((size_t)n * sizeof(double));
  double *z = (double *)malloc((size_t)n * sizeof(double));
  double *u = (double *)malloc((size_t)n * sizeof(double));
  double *H = (double *)calloc((size_t)(m + 1) * (size_t)m, sizeof(double)); /* H[row * m + col] */
  double *cs = (double *)calloc((size_t)m, sizeof(double));
  double *sn = (double *)calloc((size_t)m, sizeof(double));
  double *g = (double *)calloc((size_t)m + 1, sizeof(double));
  double *h = (double *)calloc((size_t)m + 2, sizeof(double));
  double *h2 = (double *)calloc((size_t)m + 2, sizeof(double));
  double *y = (double *)calloc((size_t)m, sizeof(double));
  memset(x, 0, (size_t)n * sizeof(double));
  double bnorm = nrm(b, n);
  int its = 0, conv = 0;
  double est = 1.0;
  if (hist) hist[0] = 1.0;
  if (bnorm == 0.0) {
    conv = 1;
    est = 0.0;
  }
  memcpy(w, b, (size_t)n * sizeof(double)); /* r0 = b - A*0 */
  double beta = bnorm;
  while (!conv && its < maxit) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) V[e] = w[e] / beta;
    memset(g, 0, (size_t)(m + 1) * sizeof(double));
    g[0] = beta;
    int k = 0;
    for (int i = 0; i < m && its < maxit; ++i) {
      double *vi = V + (int64_t)i * n;
      precond(ml, mu, vi, z, n);
      orc_spmv(a, z, n, w, n);
      /* CGS2 */
      for (int pass = 0; pass < 2; ++pass) {
        double *hh = pass == 0 ? h : h2;
        multi_dot(V, i + 1, w, 1, n, hh, 1); /* hh[j] = orc_dot(V_j, w) */
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n; ++e) {
          double t = w[e];
          for (int j = 0; j <= i; ++j) t = fma(-hh[j], V[(int64_t)j * n + e], t);
          w[e] = t;
        }
      }
      for (int j = 0; j <= i; ++j) h[j] = h[j] + h2[j];
      h[i + 1] = nrm(w, n);
      if (h[i + 1] != 0.0) {
        double *vn = V + (int64_t)(i + 1) * n;
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n; ++e) vn[e] = w[e] / h[i + 1];
      }
      /* Givens */
      for (int j = 0; j < i; ++j) {
        double t0 = cs[j] * h[j] + sn[j] * h[j + 1];
        double t1 = -sn[j] * h[j] + cs[j] * h[j + 1];
        h[j] = t0;
        h[j + 1] = t1;
      }
      double den = sqrt(h[i] * h[i] + h[i + 1] * h[i + 1]);
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
      est = fabs(g[i + 1]) / bnorm;
      if (hist) hist[its] = est;
      if (est <= tol) {
        conv = 1;
        break;
      }
    }
    /* y = H(0:k,0:k) \ g(0:k), back substitution */
    for (int ii = k - 1; ii >= 0; --ii) {
      double t = g[ii];
      for (int jj = ii + 1; jj < k; ++jj) t = t - H[ii * m + jj] * y[jj];
      y[ii] = t / H[ii * m + ii];
    }
    /* x += M (V y) */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) {
      double t = y[0] * V[e];
      for (int j = 1; j < k; ++j) t = fma(y[j], V[(int64_t)j * n + e], t);
      u[e] = t;
    }
    precond(ml, mu, u, z, n);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) x[e] = x[e] + z[e];
    /* true residual */
    orc_spmv(a, x, n, z, n);
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; ++e) w[e] = b[e] - z[e];
    beta = nrm(w, n);
    if (beta == 0.0) conv = 1;
  }
  if (st) {
    st->iterations = its;
    st->converged = conv;
    st->final_relres = est;
    st->true_relres = bnorm == 0.0 ? 0.0 : beta / bnorm;
  }
  free(V); free(w); free(z); free(u); free(H); free(cs); free(sn); free(g); free(h); free(h2); free(y);
  return ORC_OK;
}

/*
 * PCG from x0 = 0, stop when ||r_k|| / ||b|| <= tol on the
 * recurrence residual; breakdown p'Ap <= 0 -> runtime error.  hist as GMRES.
 */
int orc_pcg(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, const double *b, double tol,
            int maxit, double *x, double *hist, orc_solve_stats *st) {
  int64_t n = a->nrows;
  double *r = (double *)malloc((size_t)n * sizeof(double));
  double *z = (double *)malloc((size_t)n * sizeof(double));
  double *p = (double *)malloc((size_t)n * sizeof(double));
  double *q = (double *)malloc((size_t)n * sizeof(double));
  memset(x, 0, (size_t)n * sizeof(double));
  memcpy(r, b, (size_t)n * sizeof(double));
  double bnorm = nrm(b, n), rel = 1.0;
  int its = 0, conv = bnorm == 0.0, rc = ORC_OK;
  if (hist) hist[0] = 1.0;
  if (!conv) {
    precond(ml, mu, r, z, n);
    memcpy(p, z, (size_t)n * sizeof(double));
    double rz = orc_dot(r, z, n);
    while (its < maxit) {
      orc_spmv(a, p, n, q, n);
      double pq = orc_dot(p, q, n);
      if (!(pq > 0.0)) {
        rc = ORC_RUNTIME_ERROR;
        break;
      }
      double alpha = rz / pq;
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < n; ++e) {
        x[e] = fma(alpha, p[e], x[e]);
        r[e] = fma(-alpha, q[e], r[e]);
      }
      ++its;
      rel = nrm(r, n) / bnorm;
      if (hist) hist[its] = rel;
      if (rel <= tol) {
        conv = 1;
        break;
      }
      precond(ml, mu, r, z, n);
      double rz2 = orc_dot(r, z, n);
      double beta = rz2 / rz;
      rz = rz2;
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < n; ++e) p[e] = fma(beta, p[e], z[e]);
    }
  }
  if (st) {
    orc_spmv(a, x, n, q, n);
    for (int64_t e = 0; e < n; ++e) q[e] = b[e] - q[e];
    st->iterations = its;
    st->converged = conv;
    st->final_relres = bnorm == 0.0 ? 0.0 : rel;
    st->true_relres = bnorm == 0.0 ? 0.0 : nrm(q, n) / bnorm;
  }
  free(r); free(z); free(p); free(q);
  return rc;
}

/* ------------------------------------------------------------------ LOBPCG
 * Block LOBPCG (Knyazev 2001) for the nev smallest eigenpairs of SPD A with
 * the SAIT pair as preconditioner.  Fixed choices (DESIGN.md
 * "solvers"): X0 ~ U[-1,1] column j from seed (seed, j); W = T R is
 * orthogonalised against X and Cholesky-QR normalised, P is Cholesky-QR
 * normalised; Rayleigh-Ritz on S = [X W P] with B-Gram S'S and symmetrised
 * S'AS; the small generalized problem is solved by Cholesky + cyclic Jacobi;
 * if S'S is not positive definite the P block is dropped for that iteration.
 * Converged when every ||A x_j - lambda_j x_j|| <= tol (unit x_j).
 * Block vectors are column-major n x k.  Gram entries use orc_dot.  */

/* G[a][b] = S_a . Y_b for a in [0,ka), b in [0,kb) */
static void gram(const double *S, int ka, const double *Y, int kb, int64_t n, double *G, int ld) {
  multi_dot(S, ka, Y, kb, n, G, ld);
}

/* out[:, j] = sum_q in[:, q] C[q][j] (sequential q, first term a product) */
static void lincomb_cols(const double *in, int kin, const double *C, int ldc, int kout, int64_t n, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < kout; ++j) {
      double t = in[i] * C[0 * ldc + j];
      for (int q = 1; q < kin; ++q) t = fma(in[(int64_t)q * n + i], C[q * ldc + j], t);
      out[(int64_t)j * n + i] = t;
    }
}

/* Cholesky of SPD m x m (row-major) into lower L; returns 0 if not PD */
static int chol_lower(const double *G, int m, double *L) {
  for (int i = 0; i < m * m; ++i) L[i] = 0.0;
  for (int j = 0; j < m; ++j) {
    double d = G[j * m + j];
    for (int k = 0; k < j; ++k) d = d - L[j * m + k] * L[j * m + k];
    if (!(d > 0.0)) return 0;
    double ljj = sqrt(d);
    L[j * m + j] = ljj;
    for (int i = j + 1; i < m; ++i) {
      double t = G[i * m + j];
      for (int k = 0; k < j; ++k) t = t - L[i * m + k] * L[j * m + k];
      L[i * m + j] = t / ljj;
    }
  }
  return 1;
}

/* inverse of lower-triangular L (forward substitution per column) */
static void tri_lower_inv(const double *L, int m, double *Li) {
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

/* cyclic Jacobi eigen-decomposition of symmetric F (m x m, destroyed);
 * eigenvalues ascending in w, eigenvectors in columns of Q (row-major) */
static void jacobi_eig(double *F, int m, double *w, double *Q) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) Q[i * m + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) off = off + F[p * m + q] * F[p * m + q];
    if (off == 0.0) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        double apq = F[p * m + q];
        if (apq == 0.0) continue;
        double app = F[p * m + p], aqq = F[q * m + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < m; ++k) { /* columns p, q */
          double fkp = F[k * m + p], fkq = F[k * m + q];
          F[k * m + p] = c * fkp - s * fkq;
          F[k * m + q] = s * fkp + c * fkq;
        }
        for (int k = 0; k < m; ++k) { /* rows p, q */
          double fpk = F[p * m + k], fqk = F[q * m + k];
          F[p * m + k] = c * fpk - s * fqk;
          F[q * m + k] = s * fpk + c * fqk;
        }
        F[p * m + q] = 0.0;
        F[q * m + p] = 0.0;
        for (int k = 0; k < m; ++k) {
          double qkp = Q[k * m + p], qkq = Q[k * m + q];
          Q[k * m + p] = c * qkp - s * qkq;
          Q[k * m + q] = s * qkp + c * qkq;
        }
      }
  }
  /* selection sort ascending (stable on ties by index) */
  int idx[64];
  for (int i = 0; i < m; ++i) idx[i] = i;
  for (int i = 0; i < m; ++i) {
    int best = i;
    for (int j = i + 1; j < m; ++j)
      if (F[idx[j] * m + idx[j]] < F[idx[best] * m + idx[best]]) best = j;
    int tmp = idx[i];
    idx[i] = idx[best];
    idx[best] = tmp;
  }
  double *Qs = (double *)malloc((size_t)m * m * sizeof(double));
  for (int j = 0; j < m; ++j) {
    w[j] = F[idx[j] * m + idx[j]];
    for (int i = 0; i < m; ++i) Qs[i * m + j] = Q[i * m + idx[j]];
  }
  memcpy(Q, Qs, (size_t)m * m * sizeof(double));
  free(Qs);
}

/* Rayleigh-Ritz: given GB (SPD) and GA (sym) of size m, fill C (m x k, row
 * major, ldc = k) with the k lowest B-orthonormal Ritz vectors, mu with their
 * values.  Returns 0 when GB is not positive definite. */
static int rayleigh_ritz(const double *GA, const double *GB, int m, int k, double *C, double *mu) {
  double L[64 * 64], Li[64 * 64], T[64 * 64], F[64 * 64], Q[64 * 64], w[64];
  if (!chol_lower(GB, m, L)) return 0;
  tri_lower_inv(L, m, Li);
  /* F = Li GA Li^T */
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
      double a = 0.5 * (F[i * m + j] + F[j * m + i]);
      F[i * m + j] = a;
      F[j * m + i] = a;
    }
  jacobi_eig(F, m, w, Q);
  /* C = Li^T Q[:, :k] */
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < k; ++j) {
      double t = 0.0;
      for (int q = 0; q < m; ++q) t = t + Li[q * m + i] * Q[q * m + j];
      C[i * k + j] = t;
    }
  for (int j = 0; j < k; ++j) mu[j] = w[j];
  return 1;
}

/* Y <- Y R^-1 with G = Y'Y = R'R (Cholesky-QR); AY transformed alike when
 * given.  Returns 0 if G is not PD. */
static int cholqr(double *Y, double *AY, int k, int64_t n, double *tmp) {
  double G[32 * 32], L[32 * 32], Li[32 * 32], Ri[32 * 32];
  gram(Y, k, Y, k, n, G, k);
  if (!chol_lower(G, k, L)) return 0;
  tri_lower_inv(L, k, Li);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) Ri[i * k + j] = Li[j * k + i]; /* R^-1 = (L^-1)^T */
  lincomb_cols(Y, k, Ri, k, k, n, tmp);
  memcpy(Y, tmp, (size_t)k * n * sizeof(double));
  if (AY) {
    lincomb_cols(AY, k, Ri, k, k, n, tmp);
    memcpy(AY, tmp, (size_t)k * n * sizeof(double));
  }
  return 1;
}

static void block_spmv(const orc_csr *a, const double *X, int k, double *Y) {
  int64_t n = a->nrows;
  for (int j = 0; j < k; ++j) orc_spmv(a, X + (int64_t)j * n, n, Y + (int64_t)j * n, n);
}

int orc_lobpcg(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, int k, double tol, int maxit,
               uint64_t seed, double *evals, double *evecs, int *iters, double *resnorms) {
  int64_t n = a->nrows;
  if (k < 1 || k > 16 || 3 * k > 64) return fail_solver("lobpcg: block size must be in [1, 16]");
  size_t blk = (size_t)k * (size_t)n;
  double *S = (double *)calloc(3 * blk, sizeof(double));  /* [X W P] */
  double *AS = (double *)calloc(3 * blk, sizeof(double)); /* [AX AW AP] */
  double *R = (double *)malloc(blk * sizeof(double));
  double *tmp = (double *)malloc(4 * blk * sizeof(double));
  double *X = S, *W = S + blk, *P = S + 2 * blk;
  double *AX = AS, *AW = AS + blk, *AP = AS + 2 * blk;
  double GA[48 * 48], GB[48 * 48], C[48 * 16], lam[48];
  for (int j = 0; j < k; ++j) orc_fill_uniform_pm1(seed * 1000 + (uint64_t)j, n, X + (size_t)j * n);
  block_spmv(a, X, k, AX);
  int rc = ORC_OK, have_p = 0, it = 0, conv = 0;
  /* initial Rayleigh-Ritz on X */
  gram(X, k, X, k, n, GB, k);
  gram(X, k, AX, k, n, GA, k);
  if (!rayleigh_ritz(GA, GB, k, k, C, lam)) {
    rc = fail_solver("lobpcg: initial block is rank deficient");
    goto done;
  }
  lincomb_cols(X, k, C, k, k, n, tmp);
  memcpy(X, tmp, blk * sizeof(double));
  lincomb_cols(AX, k, C, k, k, n, tmp);
  memcpy(AX, tmp, blk * sizeof(double));
  for (it = 0; it <= maxit; ++it) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < k; ++j) R[(size_t)j * n + i] = fma(-lam[j], X[(size_t)j * n + i], AX[(size_t)j * n + i]);
    conv = 1;
    for (int j = 0; j < k; ++j) {
      resnorms[(size_t)it * k + j] = sqrt(orc_dot(R + (size_t)j * n, R + (size_t)j * n, n));
      if (!(resnorms[(size_t)it * k + j] <= tol)) conv = 0;
    }
    if (conv || it == maxit) break;
    /* W = T R, orthogonalised against X, normalised */
    for (int j = 0; j < k; ++j) precond(ml, mu, R + (size_t)j * n, W + (size_t)j * n, n);
    {
      double G1[16 * 16];
      gram(X, k, W, k, n, G1, k);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i)
        for (int j = 0; j < k; ++j) {
          double t = W[(size_t)j * n + i];
          for (int q = 0; q < k; ++q) t = fma(-X[(size_t)q * n + i], G1[q * k + j], t);
          W[(size_t)j * n + i] = t;
        }
    }
    if (!cholqr(W, NULL, k, n, tmp)) {
      rc = fail_solver("lobpcg: preconditioned residual block is rank deficient");
      break;
    }
    block_spmv(a, W, k, AW);
    int use_p = have_p && cholqr(P, AP, k, n, tmp);
    int m = use_p ? 3 * k : 2 * k;
    for (;;) {
      gram(S, m, S, m, n, GB, m);
      gram(S, m, AS, m, n, GA, m);
      for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j) {
          double s2 = 0.5 * (GA[i * m + j] + GA[j * m + i]);
          GA[i * m + j] = s2;
          GA[j * m + i] = s2;
        }
      if (rayleigh_ritz(GA, GB, m, k, C, lam)) break;
      if (m == 3 * k) {
        m = 2 * k; /* drop P */
        use_p = 0;
        continue;
      }
      rc = fail_solver("lobpcg: Gram matrix not positive definite");
      goto done;
    }
    /* P = [W P] C[k:, :], AP likewise; X = S C, AX = AS C */
    lincomb_cols(W, m - k, C + k * k, k, k, n, tmp);
    lincomb_cols(AW, m - k, C + k * k, k, k, n, tmp + blk);
    lincomb_cols(S, m, C, k, k, n, tmp + 2 * blk);
    lincomb_cols(AS, m, C, k, k, n, tmp + 3 * blk);
    memcpy(P, tmp, blk * sizeof(double));
    memcpy(AP, tmp + blk, blk * sizeof(double));
    memcpy(X, tmp + 2 * blk, blk * sizeof(double));
    memcpy(AX, tmp + 3 * blk, blk * sizeof(double));
    have_p = 1;
  }
done:
  for (int j = 0; j < k; ++j) evals[j] = lam[j];
  if (evecs) memcpy(evecs, X, blk * sizeof(double));
  *iters = it;
  free(S);
  free(AS);
  free(R);
  free(tmp);
  if (rc == ORC_OK && !conv) rc = ORC_OK; /* not converged: caller checks residuals */
  return rc;
}
