/*
 * sait_oracle.h — CPU restatement of the reference SAIT path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2106_12836_b200/,
 * include/) may include, link or call this file.  Only tests/, the
 * smoke() checker in __graft_entry__.py and the cpu_baseline / --impl
 * reference legs of bench.py use it, and only as the checker.
 *
 * Every function names the reference file:line it restates (paths are
 * relative to /root/reference/proj/core/).  The restatement is plain C11,
 * single threaded, compiled with -ffp-contract=off so every multiply and add
 * rounds separately, exactly like the reference built with the pinned flags
 * (SURVEY.md §8c).  It is pinned against oracle/_ref (the reference compiled
 * from its own sources) and against tests/golden/ fixtures.
 *
 * Errors mirror the reference exceptions: functions return ORC_OK,
 * ORC_INVALID_ARGUMENT (std::invalid_argument) or ORC_RUNTIME_ERROR
 * (std::runtime_error) and leave the exception text in orc_last_error().
 */
#ifndef SAIT_ORACLE_H
#define SAIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_RUNTIME_ERROR = 2 };

/* Same layout as saitprec::CsrMatrix (include/saitprec/csr.hpp:24-43):
 * int64 row_ptr/col_idx, fp64 values.  values == NULL means a pattern. */
typedef struct {
  int64_t nrows;
  int64_t ncols;
  int64_t *row_ptr;
  int64_t *col_idx;
  double *values;
} orc_csr;

const char *orc_last_error(void);
void orc_csr_free(orc_csr *m);
void orc_free(void *p);
int64_t orc_nnz(const orc_csr *m);

/* csr.cpp */
int orc_identity(int64_t n, orc_csr *out);                         /* csr.cpp:60-70  */
int orc_transpose(const orc_csr *a, orc_csr *out);                 /* csr.cpp:72-92  */
int orc_check_triangular(const orc_csr *a, int lower, int unit);   /* csr.cpp:124-139 */
int orc_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t *rows,
                      const int64_t *cols, const double *vals, orc_csr *out); /* csr.cpp:10-58 */

/* kernels.cpp */
int orc_spmv(const orc_csr *a, const double *x, int64_t xlen, double *y, int64_t ylen); /* :10-26 */
int orc_spgemm(const orc_csr *a, const orc_csr *b, orc_csr *out);        /* :34-102  */
int orc_add_identity(const orc_csr *m, orc_csr *out);                    /* :104-134 */
int orc_drop_by_threshold(const orc_csr *m, double tau, orc_csr *out);   /* :136-160 */
int orc_drop_by_pattern(const orc_csr *m, const orc_csr *s, orc_csr *out); /* :162-194 */
int orc_scale_columns(const orc_csr *m, const double *d, int64_t dlen, orc_csr *out); /* :236-246 */
int orc_trisolve(const orc_csr *t, int lower, const double *b, double *x); /* :196-234 */

/* sait.cpp */
int orc_jacobi_split(const orc_csr *t, int lower, double **inv_diag, orc_csr *tt); /* :32-73 */
int orc_stabilized(const orc_csr *prev, const orc_csr *cur);                       /* :18-28 */

/* drop rule selector for the polynomial recursion (sait.hpp:43 DropRule) */
enum { ORC_DROP_NONE = 0, ORC_DROP_THRESHOLD = 1, ORC_DROP_PATTERN = 2, ORC_DROP_THRESHOLD_CAP = 3 };
typedef struct {
  int kind;
  double tau;               /* THRESHOLD / THRESHOLD_CAP */
  const orc_csr *pattern;   /* PATTERN */
  const int64_t *cap;       /* THRESHOLD_CAP: max entries (incl. diagonal) per column of M */
} orc_drop;

int orc_sait_polynomial(const orc_csr *tt, int steps, const orc_drop *drop, orc_csr *out,
                        int *steps_run); /* sait.cpp:75-88 */
int orc_sait_thr(const orc_csr *t, int lower, double tau, int steps, orc_csr *out,
                 int *steps_run); /* sait.cpp:90-101 */
int orc_sait_pat_capture_pattern(const orc_csr *t, int lower, int pattern_steps,
                                 orc_csr *out); /* sait.cpp:103-111 */
int orc_sait_pat(const orc_csr *t, int lower, int pattern_steps, int refine_steps, orc_csr *out,
                 int *steps_run); /* sait.cpp:113-136 */
/* BASELINE config 4 "fill cap": no reference counterpart.
 * Restated through the reference's DropRule hook: drop = cap(threshold(M)),
 * cap keeps the diagonal plus the (cap_j - 1) largest-|v| off-diagonals of
 * column j, ties to the smaller row index; cap_j = floor(factor * nnz(T[:,j])). */
int orc_drop_cap_columns(const orc_csr *m, const int64_t *cap, orc_csr *out);
int orc_sait_thr_cap(const orc_csr *t, int lower, double tau, int steps, double cap_factor,
                     orc_csr *out, int *steps_run);
int orc_jacobi_sweeps_apply(const orc_csr *t, int lower, const double *b, int sweeps,
                            double *x); /* sait.cpp:138-159 */

/* preconditioner.cpp / dense.cpp */
int orc_pair_apply(const orc_csr *ml, const orc_csr *mu, const double *r, double *z); /* :42-45 */
int orc_pair_apply_block(const orc_csr *ml, const orc_csr *mu, const double *r, int64_t nvec,
                         double *z); /* preconditioner.cpp:47-49 + dense.cpp:10-19, column-major */

/* ilu.cpp */
int orc_ilu_k(const orc_csr *a, int level, orc_csr *lower, orc_csr *upper); /* ilu.cpp:98-173 */
int orc_ilu_residual_on_pattern(const orc_csr *a, const orc_csr *l, const orc_csr *u,
                                double *out); /* ilu.cpp:175-192 */

/* Problem generators (SPEC.md:353-408 restated) */
uint64_t orc_rng_u64(uint64_t seed, uint64_t counter);
double orc_rng_uniform(uint64_t seed, uint64_t counter); /* U[0,1) with 53 bits */
void orc_fill_uniform_pm1(uint64_t seed, int64_t n, double *out); /* U[-1,1) */
int orc_laplacian_2d(int64_t nx, orc_csr *out);
int orc_laplacian_3d(int64_t n, orc_csr *out);
int orc_convdiff_2d(int64_t nx, double bx, double by, orc_csr *out);
int orc_synthetic_lower(int64_t n, int64_t draws, double p, uint64_t seed, orc_csr *out);

/* Solvers (SPEC.md:282-351 restated; GMRES per DESIGN.md).  All reductions
 * use the canonical order of orc_dot (shared with the device kernels). */
double orc_dot(const double *a, const double *b, int64_t n);
typedef struct {
  int iterations;
  int converged;
  double final_relres;    /* estimate at exit */
  double true_relres;     /* ||b - A x|| / ||b|| recomputed at exit */
} orc_solve_stats;
/* precond: 0 none, 1 SAIT pair (ml, mu) */
/* solvers.c: 1 = GMRES/PCG apply (ml, mu) as exact ILU factors (two trisolves) */
void orc_solver_precond_exact(int on);
int orc_gmres(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, const double *b, int restart,
              double tol, int maxit, double *x, double *hist, orc_solve_stats *st);
int orc_pcg(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, const double *b, double tol,
            int maxit, double *x, double *hist, orc_solve_stats *st);
int orc_lobpcg(const orc_csr *a, const orc_csr *ml, const orc_csr *mu, int nev, double tol,
               int maxit, uint64_t seed, double *evals, double *evecs, int *iters,
               double *resnorms);

#ifdef __cplusplus
}
#endif
#endif
