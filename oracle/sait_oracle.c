/*
 * sait_oracle.c — CPU restatement of the reference SAIT path (test infrastructure only;
 * see sait_oracle.h for the rules).  Reference paths are relative to
 * /root/reference/proj/core/.  Compile with -ffp-contract=off.
 */
#include "sait_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char *orc_last_error(void) { return g_err; }

int orc_set_error(const char *m) { return fail(ORC_RUNTIME_ERROR, "%s", m); }

void orc_free(void *p) { free(p); }

void orc_csr_free(orc_csr *m) {
  if (!m) return;
  free(m->row_ptr);
  free(m->col_idx);
  free(m->values);
  m->row_ptr = NULL;
  m->col_idx = NULL;
  m->values = NULL;
}

int64_t orc_nnz(const orc_csr *m) { return m->row_ptr ? m->row_ptr[m->nrows] : 0; }

/* allocate a CSR with capacity for cap entries (row_ptr zeroed) */
static void csr_alloc(orc_csr *m, int64_t nrows, int64_t ncols, int64_t cap, int with_values) {
  m->nrows = nrows;
  m->ncols = ncols;
  m->row_ptr = (int64_t *)calloc((size_t)nrows + 1, sizeof(int64_t));
  m->col_idx = (int64_t *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int64_t));
  m->values = with_values ? (double *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(double)) : NULL;
}

static void csr_shrink(orc_csr *m) {
  int64_t nnz = m->row_ptr[m->nrows];
  m->col_idx = (int64_t *)realloc(m->col_idx, (size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
  if (m->values) m->values = (double *)realloc(m->values, (size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
}

static void csr_copy(const orc_csr *a, orc_csr *out) {
  int64_t nnz = orc_nnz(a);
  csr_alloc(out, a->nrows, a->ncols, nnz, a->values != NULL);
  memcpy(out->row_ptr, a->row_ptr, ((size_t)a->nrows + 1) * sizeof(int64_t));
  if (nnz) memcpy(out->col_idx, a->col_idx, (size_t)nnz * sizeof(int64_t));
  if (nnz && a->values) memcpy(out->values, a->values, (size_t)nnz * sizeof(double));
}

/* ------------------------------------------------------------------ csr.cpp */

/* csr.cpp:60-70 */
int orc_identity(int64_t n, orc_csr *out) {
  csr_alloc(out, n, n, n, 1);
  for (int64_t i = 0; i < n; ++i) {
    out->row_ptr[i + 1] = i + 1;
    out->col_idx[i] = i;
    out->values[i] = 1.0;
  }
  return ORC_OK;
}

/* csr.cpp:72-92 — counting-sort transpose; entries of each output row come
 * out in increasing source-row order. */
int orc_transpose(const orc_csr *a, orc_csr *out) {
  int64_t nnz = orc_nnz(a);
  csr_alloc(out, a->ncols, a->nrows, nnz, a->values != NULL);
  for (int64_t e = 0; e < nnz; ++e) out->row_ptr[a->col_idx[e] + 1]++;
  for (int64_t j = 0; j < a->ncols; ++j) out->row_ptr[j + 1] += out->row_ptr[j];
  int64_t *cursor = (int64_t *)malloc(((size_t)a->ncols + 1) * sizeof(int64_t));
  memcpy(cursor, out->row_ptr, ((size_t)a->ncols + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < a->nrows; ++i) {
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      int64_t pos = cursor[a->col_idx[e]]++;
      out->col_idx[pos] = i;
      if (a->values) out->values[pos] = a->values[e];
    }
  }
  free(cursor);
  return ORC_OK;
}

/* csr.cpp:124-139 */
int orc_check_triangular(const orc_csr *a, int lower, int unit) {
  for (int64_t i = 0; i < a->nrows; ++i) {
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      int64_t j = a->col_idx[e];
      int off = lower ? (j > i) : (j < i);
      if (off)
        return fail(ORC_INVALID_ARGUMENT,
                    "check_triangular: entry (%lld, %lld) outside stated triangle",
                    (long long)i, (long long)j);
      if (unit && j == i && a->values[e] != 1.0)
        return fail(ORC_INVALID_ARGUMENT, "check_triangular: non-unit diagonal at row %lld",
                    (long long)i);
    }
  }
  return ORC_OK;
}

/* csr.cpp:10-58 — stable (row, col) ordering, duplicates summed in input order. */
typedef struct {
  int64_t r, c, k;
} trip_key;

static int trip_cmp(const void *pa, const void *pb) {
  const trip_key *a = (const trip_key *)pa, *b = (const trip_key *)pb;
  if (a->r != b->r) return a->r < b->r ? -1 : 1;
  if (a->c != b->c) return a->c < b->c ? -1 : 1;
  return a->k < b->k ? -1 : (a->k > b->k); /* stability via original index */
}

int orc_from_triplets(int64_t nrows, int64_t ncols, int64_t count, const int64_t *rows,
                      const int64_t *cols, const double *vals, orc_csr *out) {
  if (nrows < 0 || ncols < 0) return fail(ORC_INVALID_ARGUMENT, "from_triplets: negative dimension");
  for (int64_t k = 0; k < count; ++k) {
    if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
      return fail(ORC_INVALID_ARGUMENT,
                  "from_triplets: triplet %lld (row %lld, col %lld, value %f) out of range for "
                  "%lldx%lld matrix",
                  (long long)k, (long long)rows[k], (long long)cols[k], vals[k],
                  (long long)nrows, (long long)ncols);
  }
  trip_key *ord = (trip_key *)malloc((size_t)(count > 0 ? count : 1) * sizeof(trip_key));
  for (int64_t k = 0; k < count; ++k) {
    ord[k].r = rows[k];
    ord[k].c = cols[k];
    ord[k].k = k;
  }
  qsort(ord, (size_t)count, sizeof(trip_key), trip_cmp);
  csr_alloc(out, nrows, ncols, count, 1);
  int64_t nnz = 0, cr = -1, cc = -1;
  for (int64_t q = 0; q < count; ++q) {
    const trip_key *t = &ord[q];
    if (t->r == cr && t->c == cc) {
      out->values[nnz - 1] += vals[t->k];
    } else {
      out->col_idx[nnz] = t->c;
      out->values[nnz] = vals[t->k];
      ++nnz;
      cr = t->r;
      cc = t->c;
      out->row_ptr[t->r + 1]++;
    }
  }
  for (int64_t i = 0; i < nrows; ++i) out->row_ptr[i + 1] += out->row_ptr[i];
  free(ord);
  csr_shrink(out);
  return ORC_OK;
}

/* -------------------------------------------------------------- kernels.cpp */

/* kernels.cpp:10-26 — row-sequential accumulation in stored order, from 0.0 */
int orc_spmv(const orc_csr *a, const double *x, int64_t xlen, double *y, int64_t ylen) {
  if (xlen != a->ncols)
    return fail(ORC_INVALID_ARGUMENT, "spmv: vector length %lld does not match ncols %lld",
                (long long)xlen, (long long)a->ncols);
  if (ylen != a->nrows) return fail(ORC_INVALID_ARGUMENT, "spmv: output length mismatch");
  /* rows are independent: parallel over rows, each row in stored order */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < a->nrows; ++i) {
    double acc = 0.0;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) acc += a->values[e] * x[a->col_idx[e]];
    y[i] = acc;
  }
  return ORC_OK;
}

static int cmp_i64(const void *pa, const void *pb) {
  int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
  return (a > b) - (a < b);
}

/* kernels.cpp:34-102 — Gustavson: per output (i,j) the first product is
 * assigned, later ones added, in increasing order of A's row; columns sorted. */
int orc_spgemm(const orc_csr *a, const orc_csr *b, orc_csr *out) {
  if (a->ncols != b->nrows)
    return fail(ORC_INVALID_ARGUMENT, "spgemm: inner dimensions %lld and %lld do not match",
                (long long)a->ncols, (long long)b->nrows);
  int64_t n = a->nrows, m = b->ncols;
  int64_t *mark = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  double *acc = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
  int64_t *cols = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  for (int64_t j = 0; j < m; ++j) mark[j] = -1;
  /* structural count */
  out->nrows = n;
  out->ncols = m;
  out->row_ptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    int64_t cnt = 0;
    for (int64_t ea = a->row_ptr[i]; ea < a->row_ptr[i + 1]; ++ea) {
      int64_t k = a->col_idx[ea];
      for (int64_t eb = b->row_ptr[k]; eb < b->row_ptr[k + 1]; ++eb) {
        int64_t j = b->col_idx[eb];
        if (mark[j] != i) {
          mark[j] = i;
          ++cnt;
        }
      }
    }
    out->row_ptr[i + 1] = out->row_ptr[i] + cnt;
  }
  int64_t nnz = out->row_ptr[n];
  out->col_idx = (int64_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
  out->values = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  for (int64_t j = 0; j < m; ++j) mark[j] = -1;
  for (int64_t i = 0; i < n; ++i) {
    int64_t nc = 0;
    for (int64_t ea = a->row_ptr[i]; ea < a->row_ptr[i + 1]; ++ea) {
      int64_t k = a->col_idx[ea];
      double av = a->values[ea];
      for (int64_t eb = b->row_ptr[k]; eb < b->row_ptr[k + 1]; ++eb) {
        int64_t j = b->col_idx[eb];
        double prod = av * b->values[eb];
        if (mark[j] != i) {
          mark[j] = i;
          acc[j] = prod;
          cols[nc++] = j;
        } else {
          acc[j] = acc[j] + prod;
        }
      }
    }
    qsort(cols, (size_t)nc, sizeof(int64_t), cmp_i64);
    int64_t pos = out->row_ptr[i];
    for (int64_t q = 0; q < nc; ++q) {
      out->col_idx[pos] = cols[q];
      out->values[pos] = acc[cols[q]];
      ++pos;
    }
  }
  free(mark);
  free(acc);
  free(cols);
  return ORC_OK;
}

/* kernels.cpp:104-134 — diagonal inserted (1.0) or incremented (v + 1.0) */
int orc_add_identity(const orc_csr *m, orc_csr *out) {
  if (m->nrows != m->ncols) return fail(ORC_INVALID_ARGUMENT, "add_identity: matrix is not square");
  csr_alloc(out, m->nrows, m->ncols, orc_nnz(m) + m->nrows, 1);
  int64_t pos = 0;
  for (int64_t i = 0; i < m->nrows; ++i) {
    int have = 0;
    for (int64_t e = m->row_ptr[i]; e < m->row_ptr[i + 1]; ++e) {
      int64_t j = m->col_idx[e];
      if (!have && j > i) {
        out->col_idx[pos] = i;
        out->values[pos++] = 1.0;
        have = 1;
      }
      out->col_idx[pos] = j;
      out->values[pos++] = (j == i) ? m->values[e] + 1.0 : m->values[e];
      if (j == i) have = 1;
    }
    if (!have) {
      out->col_idx[pos] = i;
      out->values[pos++] = 1.0;
    }
    out->row_ptr[i + 1] = pos;
  }
  csr_shrink(out);
  return ORC_OK;
}

/* kernels.cpp:136-160 — keep j == i or |v| >= tau; tau == 0 returns a copy */
int orc_drop_by_threshold(const orc_csr *m, double tau, orc_csr *out) {
  if (!(tau >= 0.0 && tau < 1.0))
    return fail(ORC_INVALID_ARGUMENT, "drop_by_threshold: tau must be in [0, 1), got %f", tau);
  if (tau == 0.0) {
    csr_copy(m, out);
    return ORC_OK;
  }
  csr_alloc(out, m->nrows, m->ncols, orc_nnz(m), 1);
  int64_t pos = 0;
  for (int64_t i = 0; i < m->nrows; ++i) {
    for (int64_t e = m->row_ptr[i]; e < m->row_ptr[i + 1]; ++e) {
      int64_t j = m->col_idx[e];
      if (j == i || fabs(m->values[e]) >= tau) {
        out->col_idx[pos] = j;
        out->values[pos++] = m->values[e];
      }
    }
    out->row_ptr[i + 1] = pos;
  }
  csr_shrink(out);
  return ORC_OK;
}

/* kernels.cpp:162-194 — sorted merge of the row against the pattern row */
int orc_drop_by_pattern(const orc_csr *m, const orc_csr *s, orc_csr *out) {
  if (m->nrows != s->nrows || m->ncols != s->ncols)
    return fail(ORC_INVALID_ARGUMENT, "drop_by_pattern: shape mismatch");
  csr_alloc(out, m->nrows, m->ncols, orc_nnz(m), 1);
  int64_t pos = 0;
  for (int64_t i = 0; i < m->nrows; ++i) {
    int64_t em = m->row_ptr[i], es = s->row_ptr[i];
    while (em < m->row_ptr[i + 1] && es < s->row_ptr[i + 1]) {
      int64_t jm = m->col_idx[em], js = s->col_idx[es];
      if (jm == js) {
        out->col_idx[pos] = jm;
        out->values[pos++] = m->values[em];
        ++em;
        ++es;
      } else if (jm < js) {
        ++em;
      } else {
        ++es;
      }
    }
    out->row_ptr[i + 1] = pos;
  }
  csr_shrink(out);
  return ORC_OK;
}

/* kernels.cpp:236-246 — v * d[col] */
int orc_scale_columns(const orc_csr *m, const double *d, int64_t dlen, orc_csr *out) {
  if (dlen != m->ncols)
    return fail(ORC_INVALID_ARGUMENT, "scale_columns: scale vector length mismatch");
  csr_copy(m, out);
  for (int64_t e = 0; e < orc_nnz(out); ++e) out->values[e] *= d[out->col_idx[e]];
  return ORC_OK;
}

/* kernels.cpp:196-234 */
int orc_trisolve(const orc_csr *t, int lower, const double *b, double *x) {
  if (t->nrows != t->ncols) return fail(ORC_INVALID_ARGUMENT, "trisolve: matrix is not square");
  int64_t n = t->nrows;
  for (int64_t s = 0; s < n; ++s) {
    int64_t i = lower ? s : n - 1 - s;
    double acc = b[i], diag = 0.0;
    int have = 0;
    for (int64_t e = t->row_ptr[i]; e < t->row_ptr[i + 1]; ++e) {
      int64_t j = t->col_idx[e];
      if (j == i) {
        diag = t->values[e];
        have = 1;
      } else {
        acc -= t->values[e] * x[j];
      }
    }
    if (!have || diag == 0.0)
      return fail(ORC_RUNTIME_ERROR, "trisolve: singular matrix, zero diagonal at row %lld",
                  (long long)i);
    x[i] = acc / diag;
  }
  return ORC_OK;
}

/* ----------------------------------------------------------------- sait.cpp */

/* sait.cpp:32-73 — inv = 1/d (IEEE division), tT[i,j] = (-t) * inv, no diagonal */
int orc_jacobi_split(const orc_csr *t, int lower, double **inv_diag, orc_csr *tt) {
  if (t->nrows != t->ncols) return fail(ORC_INVALID_ARGUMENT, "jacobi_split: matrix is not square");
  int rc = orc_check_triangular(t, lower, 0);
  if (rc) return rc;
  int64_t n = t->nrows;
  double *inv = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  csr_alloc(tt, n, n, orc_nnz(t), 1);
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    double diag = 0.0;
    int have = 0;
    for (int64_t e = t->row_ptr[i]; e < t->row_ptr[i + 1]; ++e) {
      if (t->col_idx[e] == i) {
        diag = t->values[e];
        have = 1;
        break;
      }
    }
    if (!have || diag == 0.0) {
      free(inv);
      orc_csr_free(tt);
      return fail(ORC_RUNTIME_ERROR, "jacobi_split: singular matrix, zero diagonal at row %lld",
                  (long long)i);
    }
    inv[i] = 1.0 / diag;
    for (int64_t e = t->row_ptr[i]; e < t->row_ptr[i + 1]; ++e) {
      int64_t j = t->col_idx[e];
      if (j == i) continue;
      tt->col_idx[pos] = j;
      tt->values[pos++] = -t->values[e] * inv[i];
    }
    tt->row_ptr[i + 1] = pos;
  }
  csr_shrink(tt);
  *inv_diag = inv;
  return ORC_OK;
}

/* sait.cpp:18-28 — same pattern and |b-a| <= 1e-15 * max(|a|,|b|) for all values.
 * std::max(x, y) is (x < y) ? y : x, restated literally for NaN behaviour. */
int orc_stabilized(const orc_csr *prev, const orc_csr *cur) {
  if (prev->nrows != cur->nrows) return 0;
  if (memcmp(prev->row_ptr, cur->row_ptr, ((size_t)prev->nrows + 1) * sizeof(int64_t)) != 0) return 0;
  int64_t nnz = orc_nnz(cur);
  if (nnz && memcmp(prev->col_idx, cur->col_idx, (size_t)nnz * sizeof(int64_t)) != 0) return 0;
  for (int64_t e = 0; e < nnz; ++e) {
    double a = prev->values[e], b = cur->values[e];
    double fa = fabs(a), fb = fabs(b);
    double mx = (fa < fb) ? fb : fa;
    if (fabs(b - a) > 1e-15 * mx) return 0;
  }
  return 1;
}

/* A15 extension: per-column cap after threshold (see header). */
typedef struct {
  double mag;
  int64_t row;
  int64_t src;
} cap_item;

static int cap_cmp(const void *pa, const void *pb) {
  const cap_item *a = (const cap_item *)pa, *b = (const cap_item *)pb;
  if (a->mag != b->mag) return a->mag > b->mag ? -1 : 1; /* larger |v| first */
  return a->row < b->row ? -1 : (a->row > b->row);      /* tie: smaller row first */
}

int orc_drop_cap_columns(const orc_csr *m, const int64_t *cap, orc_csr *out) {
  orc_csr mt;
  orc_transpose(m, &mt); /* row j of mt = column j of m, rows ascending */
  int64_t nnz = orc_nnz(&mt);
  char *keep = (char *)calloc((size_t)(nnz > 0 ? nnz : 1), 1);
  cap_item *items = (cap_item *)malloc((size_t)(m->nrows > 0 ? m->nrows : 1) * sizeof(cap_item));
  for (int64_t j = 0; j < mt.nrows; ++j) {
    int64_t nd = 0;
    for (int64_t e = mt.row_ptr[j]; e < mt.row_ptr[j + 1]; ++e) {
      if (mt.col_idx[e] == j) {
        keep[e] = 1;
      } else {
        items[nd].mag = fabs(mt.values[e]);
        items[nd].row = mt.col_idx[e];
        items[nd].src = e;
        ++nd;
      }
    }
    int64_t room = cap[j] - 1;
    if (room < 0) room = 0;
    if (nd > room) qsort(items, (size_t)nd, sizeof(cap_item), cap_cmp);
    for (int64_t q = 0; q < nd && q < room; ++q) keep[items[q].src] = 1;
  }
  /* compact mt then transpose back */
  orc_csr kt;
  csr_alloc(&kt, mt.nrows, mt.ncols, nnz, 1);
  int64_t pos = 0;
  for (int64_t j = 0; j < mt.nrows; ++j) {
    for (int64_t e = mt.row_ptr[j]; e < mt.row_ptr[j + 1]; ++e) {
      if (!keep[e]) continue;
      kt.col_idx[pos] = mt.col_idx[e];
      kt.values[pos++] = mt.values[e];
    }
    kt.row_ptr[j + 1] = pos;
  }
  orc_transpose(&kt, out);
  orc_csr_free(&kt);
  orc_csr_free(&mt);
  free(keep);
  free(items);
  return ORC_OK;
}

static int apply_drop(const orc_csr *next, const orc_drop *drop, orc_csr *out) {
  switch (drop ? drop->kind : ORC_DROP_NONE) {
    case ORC_DROP_THRESHOLD:
      return orc_drop_by_threshold(next, drop->tau, out);
    case ORC_DROP_PATTERN:
      return orc_drop_by_pattern(next, drop->pattern, out);
    case ORC_DROP_THRESHOLD_CAP: {
      orc_csr t1;
      int rc = orc_drop_by_threshold(next, drop->tau, &t1);
      if (rc) return rc;
      rc = orc_drop_cap_columns(&t1, drop->cap, out);
      orc_csr_free(&t1);
      return rc;
    }
    default:
      csr_copy(next, out);
      return ORC_OK;
  }
}

/* one recursion step: add_identity(spgemm(tT, M)) (sait.cpp:81) */
static int poly_step(const orc_csr *tt, const orc_csr *m, orc_csr *out) {
  orc_csr prod;
  int rc = orc_spgemm(tt, m, &prod);
  if (rc) return rc;
  rc = orc_add_identity(&prod, out);
  orc_csr_free(&prod);
  return rc;
}

/* sait.cpp:75-88 */
int orc_sait_polynomial(const orc_csr *tt, int steps, const orc_drop *drop, orc_csr *out,
                        int *steps_run) {
  if (steps < 1) return fail(ORC_INVALID_ARGUMENT, "sait_polynomial: steps must be >= 1");
  orc_csr m;
  orc_identity(tt->nrows, &m);
  int k = 0;
  for (k = 0; k < steps; ++k) {
    orc_csr raw, next;
    int rc = poly_step(tt, &m, &raw);
    if (rc) {
      orc_csr_free(&m);
      return rc;
    }
    rc = apply_drop(&raw, drop, &next);
    orc_csr_free(&raw);
    if (rc) {
      orc_csr_free(&m);
      return rc;
    }
    int done = orc_stabilized(&m, &next);
    orc_csr_free(&m);
    m = next;
    if (done) {
      ++k;
      break;
    }
  }
  if (steps_run) *steps_run = k;
  *out = m;
  return ORC_OK;
}

/* sait.cpp:90-101 */
int orc_sait_thr(const orc_csr *t, int lower, double tau, int steps, orc_csr *out, int *steps_run) {
  if (!(tau >= 0.0 && tau < 1.0))
    return fail(ORC_INVALID_ARGUMENT, "sait_thr: threshold must be in [0, 1), got %f", tau);
  double *inv;
  orc_csr tt, m;
  int rc = orc_jacobi_split(t, lower, &inv, &tt);
  if (rc) return rc;
  orc_drop d = {ORC_DROP_THRESHOLD, tau, NULL, NULL};
  rc = orc_sait_polynomial(&tt, steps, &d, &m, steps_run);
  if (!rc) {
    rc = orc_scale_columns(&m, inv, t->nrows, out);
    orc_csr_free(&m);
  }
  orc_csr_free(&tt);
  free(inv);
  return rc;
}

/* sait.cpp:103-111 */
int orc_sait_pat_capture_pattern(const orc_csr *t, int lower, int pattern_steps, orc_csr *out) {
  if (pattern_steps < 0)
    return fail(ORC_INVALID_ARGUMENT, "sait_pat_capture_pattern: pattern_steps must be >= 0");
  double *inv;
  orc_csr tt, m;
  int rc = orc_jacobi_split(t, lower, &inv, &tt);
  if (rc) return rc;
  if (pattern_steps == 0) {
    orc_identity(t->nrows, &m);
  } else {
    rc = orc_sait_polynomial(&tt, pattern_steps, NULL, &m, NULL);
  }
  orc_csr_free(&tt);
  free(inv);
  if (rc) return rc;
  free(m.values);
  m.values = NULL;
  *out = m;
  return ORC_OK;
}

/* sait.cpp:113-136 */
int orc_sait_pat(const orc_csr *t, int lower, int pattern_steps, int refine_steps, orc_csr *out,
                 int *steps_run) {
  if (pattern_steps < 0) return fail(ORC_INVALID_ARGUMENT, "sait_pat: pattern_steps must be >= 0");
  if (refine_steps < 1) return fail(ORC_INVALID_ARGUMENT, "sait_pat: refine_steps must be >= 1");
  double *inv;
  orc_csr tt, m;
  int rc = orc_jacobi_split(t, lower, &inv, &tt);
  if (rc) return rc;
  orc_identity(t->nrows, &m);
  for (int k = 0; k < pattern_steps; ++k) {
    orc_csr next;
    poly_step(&tt, &m, &next);
    orc_csr_free(&m);
    m = next;
  }
  orc_csr pattern;
  csr_copy(&m, &pattern);
  free(pattern.values);
  pattern.values = NULL;
  int k;
  for (k = 0; k < refine_steps; ++k) {
    orc_csr raw, next;
    poly_step(&tt, &m, &raw);
    orc_drop_by_pattern(&raw, &pattern, &next);
    orc_csr_free(&raw);
    int done = orc_stabilized(&m, &next);
    orc_csr_free(&m);
    m = next;
    if (done) {
      ++k;
      break;
    }
  }
  if (steps_run) *steps_run = pattern_steps + k;
  rc = orc_scale_columns(&m, inv, t->nrows, out);
  orc_csr_free(&m);
  orc_csr_free(&pattern);
  orc_csr_free(&tt);
  free(inv);
  return rc;
}

/* A15: sait_polynomial(split, steps, cap∘threshold) then scale_columns */
int orc_sait_thr_cap(const orc_csr *t, int lower, double tau, int steps, double cap_factor,
                     orc_csr *out, int *steps_run) {
  if (!(tau >= 0.0 && tau < 1.0))
    return fail(ORC_INVALID_ARGUMENT, "sait_thr: threshold must be in [0, 1), got %f", tau);
  if (!(cap_factor >= 1.0))
    return fail(ORC_INVALID_ARGUMENT, "sait_thr_cap: cap factor must be >= 1, got %f", cap_factor);
  double *inv;
  orc_csr tt, m;
  int rc = orc_jacobi_split(t, lower, &inv, &tt);
  if (rc) return rc;
  int64_t n = t->nrows;
  int64_t *cap = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  for (int64_t e = 0; e < orc_nnz(t); ++e) cap[t->col_idx[e]]++;
  for (int64_t j = 0; j < n; ++j) cap[j] = (int64_t)floor(cap_factor * (double)cap[j]);
  orc_drop d = {ORC_DROP_THRESHOLD_CAP, tau, NULL, cap};
  rc = orc_sait_polynomial(&tt, steps, &d, &m, steps_run);
  if (!rc) {
    rc = orc_scale_columns(&m, inv, n, out);
    orc_csr_free(&m);
  }
  free(cap);
  orc_csr_free(&tt);
  free(inv);
  return rc;
}

/* sait.cpp:138-159 */
int orc_jacobi_sweeps_apply(const orc_csr *t, int lower, const double *b, int sweeps, double *x) {
  if (sweeps < 1) return fail(ORC_INVALID_ARGUMENT, "jacobi_sweeps_apply: sweeps must be >= 1");
  double *inv;
  orc_csr tt;
  int rc = orc_jacobi_split(t, lower, &inv, &tt);
  if (rc) return rc;
  int64_t n = t->nrows;
  double *scaled = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double *tmp = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int64_t i = 0; i < n; ++i) scaled[i] = inv[i] * b[i];
  memcpy(x, scaled, (size_t)n * sizeof(double));
  for (int k = 1; k < sweeps; ++k) {
    orc_spmv(&tt, x, n, tmp, n);
    for (int64_t i = 0; i < n; ++i) x[i] = tmp[i] + scaled[i];
  }
  free(scaled);
  free(tmp);
  free(inv);
  orc_csr_free(&tt);
  return ORC_OK;
}

/* -------------------------------------------------------- preconditioner.cpp */

/* preconditioner.cpp:34-45 */
int orc_pair_apply(const orc_csr *ml, const orc_csr *mu, const double *r, double *z) {
  if (ml->nrows != mu->ncols)
    return fail(ORC_INVALID_ARGUMENT, "SaitPairPreconditioner: factor shapes do not chain");
  double *y = (double *)malloc((size_t)(ml->nrows > 0 ? ml->nrows : 1) * sizeof(double));
  int rc = orc_spmv(ml, r, ml->ncols, y, ml->nrows);
  if (!rc) rc = orc_spmv(mu, y, ml->nrows, z, mu->nrows);
  free(y);
  return rc;
}

/* preconditioner.cpp:47-49, dense.cpp:10-19; column-major blocks */
int orc_pair_apply_block(const orc_csr *ml, const orc_csr *mu, const double *r, int64_t nvec,
                         double *z) {
  for (int64_t c = 0; c < nvec; ++c) {
    int rc = orc_pair_apply(ml, mu, r + c * ml->ncols, z + c * mu->nrows);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ ilu.cpp */

/* ilu.cpp:28-94 (symbolic) and :98-173 (numeric IKJ).  Level-of-fill rule
 * lev(i,j) = min_k lev(i,k) + lev(k,j) + 1 over the pivot rows k < i in
 * increasing order, kept when <= level; then IKJ elimination on that pattern. */
int orc_ilu_k(const orc_csr *a, int level, orc_csr *lower, orc_csr *upper) {
  if (a->nrows != a->ncols) return fail(ORC_INVALID_ARGUMENT, "ilu_k: matrix is not square");
  if (level < 0) return fail(ORC_INVALID_ARGUMENT, "ilu_k: negative fill level");
  int64_t n = a->nrows;
  double max_abs = 0.0;
  for (int64_t e = 0; e < orc_nnz(a); ++e) {
    double v = fabs(a->values[e]);
    if (v > max_abs) max_abs = v;
  }
  double tol = 1e-14 * max_abs;

  /* symbolic: per row a sorted singly linked list over column ids */
  const int64_t END = -1;
  int64_t *link = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int *lev = (int *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int));
  int64_t *seen = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  for (int64_t j = 0; j < n; ++j) seen[j] = -1;
  int64_t lcap = orc_nnz(a) + 16, ucap = orc_nnz(a) + 16, ln = 0, un = 0;
  int64_t *lptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *uptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t *lcol = (int64_t *)malloc((size_t)lcap * sizeof(int64_t));
  int64_t *ucol = (int64_t *)malloc((size_t)ucap * sizeof(int64_t));
  int *ulev = (int *)malloc((size_t)ucap * sizeof(int));
  for (int64_t i = 0; i < n; ++i) {
    int64_t head = END, tail = END;
    int diag = 0;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      int64_t j = a->col_idx[e];
      diag |= (j == i);
      if (tail == END) head = j; else link[tail] = j;
      link[j] = END;
      lev[j] = 0;
      seen[j] = i;
      tail = j;
    }
    if (!diag) {
      free(link); free(lev); free(seen); free(lptr); free(uptr); free(lcol); free(ucol); free(ulev);
      return fail(ORC_INVALID_ARGUMENT, "ilu_k: structurally zero diagonal at row %lld", (long long)i);
    }
    for (int64_t k = head; k != END && k < i; k = link[k]) {
      int64_t cur = k; /* insertion cursor: U(k,:) columns ascend */
      for (int64_t q = uptr[k]; q < uptr[k + 1]; ++q) {
        int64_t j = ucol[q];
        if (j == k) continue;
        int nl = lev[k] + ulev[q] + 1;
        if (nl > level) continue;
        if (seen[j] == i) {
          if (nl < lev[j]) lev[j] = nl;
        } else {
          while (link[cur] != END && link[cur] < j) cur = link[cur];
          link[j] = link[cur];
          link[cur] = j;
          lev[j] = nl;
          seen[j] = i;
        }
      }
    }
    for (int64_t j = head; j != END; j = link[j]) {
      if (j < i) {
        if (ln == lcap) { lcap *= 2; lcol = (int64_t *)realloc(lcol, (size_t)lcap * sizeof(int64_t)); }
        lcol[ln++] = j;
      } else {
        if (un == ucap) {
          ucap *= 2;
          ucol = (int64_t *)realloc(ucol, (size_t)ucap * sizeof(int64_t));
          ulev = (int *)realloc(ulev, (size_t)ucap * sizeof(int));
        }
        ucol[un] = j;
        ulev[un++] = lev[j];
      }
    }
    lptr[i + 1] = ln;
    uptr[i + 1] = un;
  }

  /* numeric IKJ */
  csr_alloc(lower, n, n, ln + n, 1);
  csr_alloc(upper, n, n, un, 1);
  double *w = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double *udiag = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t j = 0; j < n; ++j) seen[j] = -1;
  int64_t lpos = 0, upos = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = lptr[i]; p < lptr[i + 1]; ++p) { w[lcol[p]] = 0.0; seen[lcol[p]] = i; }
    for (int64_t p = uptr[i]; p < uptr[i + 1]; ++p) { w[ucol[p]] = 0.0; seen[ucol[p]] = i; }
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) w[a->col_idx[e]] = a->values[e];
    for (int64_t p = lptr[i]; p < lptr[i + 1]; ++p) {
      int64_t k = lcol[p];
      double f = w[k] / udiag[k];
      w[k] = f;
      for (int64_t q = upper->row_ptr[k]; q < upper->row_ptr[k + 1]; ++q) {
        int64_t j = upper->col_idx[q];
        if (j == k) continue;
        if (seen[j] == i) w[j] -= f * upper->values[q];
      }
    }
    for (int64_t p = lptr[i]; p < lptr[i + 1]; ++p) {
      lower->col_idx[lpos] = lcol[p];
      lower->values[lpos++] = w[lcol[p]];
    }
    lower->col_idx[lpos] = i;
    lower->values[lpos++] = 1.0;
    lower->row_ptr[i + 1] = lpos;
    double piv = w[i];
    if (piv == 0.0 || fabs(piv) < tol) {
      int64_t row = i;
      double mag = fabs(piv);
      free(link); free(lev); free(seen); free(lptr); free(uptr); free(lcol); free(ucol); free(ulev);
      free(w); free(udiag);
      orc_csr_free(lower);
      orc_csr_free(upper);
      return fail(ORC_RUNTIME_ERROR, "ilu_k: pivot breakdown at row %lld (|pivot| = %f)",
                  (long long)row, mag);
    }
    udiag[i] = piv;
    for (int64_t p = uptr[i]; p < uptr[i + 1]; ++p) {
      upper->col_idx[upos] = ucol[p];
      upper->values[upos++] = w[ucol[p]];
    }
    upper->row_ptr[i + 1] = upos;
  }
  free(link); free(lev); free(seen); free(lptr); free(uptr); free(lcol); free(ucol); free(ulev);
  free(w); free(udiag);
  return ORC_OK;
}

/* ilu.cpp:175-192 */
int orc_ilu_residual_on_pattern(const orc_csr *a, const orc_csr *l, const orc_csr *u, double *out) {
  if (a->nrows != l->nrows || a->ncols != u->ncols)
    return fail(ORC_INVALID_ARGUMENT, "ilu_residual_on_pattern: shape mismatch");
  orc_csr prod;
  orc_spgemm(l, u, &prod);
  double mx = 0.0;
  for (int64_t i = 0; i < a->nrows; ++i) {
    int64_t kp = prod.row_ptr[i], ep = prod.row_ptr[i + 1];
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      int64_t j = a->col_idx[e];
      while (kp < ep && prod.col_idx[kp] < j) ++kp;
      double pv = (kp < ep && prod.col_idx[kp] == j) ? prod.values[kp] : 0.0;
      double d = fabs(pv - a->values[e]);
      if (d > mx) mx = d;
    }
  }
  orc_csr_free(&prod);
  *out = mx;
  return ORC_OK;
}

/* ------------------------------------------------------------ generators */

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* counter-based stream: value #counter of stream `seed` */
uint64_t orc_rng_u64(uint64_t seed, uint64_t counter) { return splitmix64(seed ^ splitmix64(counter)); }

double orc_rng_uniform(uint64_t seed, uint64_t counter) {
  return (double)(orc_rng_u64(seed, counter) >> 11) * 0x1.0p-53;
}

void orc_fill_uniform_pm1(uint64_t seed, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * orc_rng_uniform(seed, (uint64_t)i) - 1.0;
}

/* 2D 5-point (diag 4, neighbours -1), lexicographic, x fastest, Dirichlet */
int orc_laplacian_2d(int64_t nx, orc_csr *out) {
  if (nx < 1) return fail(ORC_INVALID_ARGUMENT, "laplacian_2d: nx must be >= 1");
  int64_t n = nx * nx;
  csr_alloc(out, n, n, 5 * n, 1);
  int64_t pos = 0;
  for (int64_t y = 0; y < nx; ++y)
    for (int64_t x = 0; x < nx; ++x) {
      int64_t i = x + nx * y;
      if (y > 0) { out->col_idx[pos] = i - nx; out->values[pos++] = -1.0; }
      if (x > 0) { out->col_idx[pos] = i - 1; out->values[pos++] = -1.0; }
      out->col_idx[pos] = i; out->values[pos++] = 4.0;
      if (x + 1 < nx) { out->col_idx[pos] = i + 1; out->values[pos++] = -1.0; }
      if (y + 1 < nx) { out->col_idx[pos] = i + nx; out->values[pos++] = -1.0; }
      out->row_ptr[i + 1] = pos;
    }
  csr_shrink(out);
  return ORC_OK;
}

/* 3D 7-point (diag 6, neighbours -1) */
int orc_laplacian_3d(int64_t m, orc_csr *out) {
  if (m < 1) return fail(ORC_INVALID_ARGUMENT, "laplacian_3d: n must be >= 1");
  int64_t n = m * m * m, s2 = m * m;
  csr_alloc(out, n, n, 7 * n, 1);
  int64_t pos = 0;
  for (int64_t z = 0; z < m; ++z)
    for (int64_t y = 0; y < m; ++y)
      for (int64_t x = 0; x < m; ++x) {
        int64_t i = x + m * y + s2 * z;
        if (z > 0) { out->col_idx[pos] = i - s2; out->values[pos++] = -1.0; }
        if (y > 0) { out->col_idx[pos] = i - m; out->values[pos++] = -1.0; }
        if (x > 0) { out->col_idx[pos] = i - 1; out->values[pos++] = -1.0; }
        out->col_idx[pos] = i; out->values[pos++] = 6.0;
        if (x + 1 < m) { out->col_idx[pos] = i + 1; out->values[pos++] = -1.0; }
        if (y + 1 < m) { out->col_idx[pos] = i + m; out->values[pos++] = -1.0; }
        if (z + 1 < m) { out->col_idx[pos] = i + s2; out->values[pos++] = -1.0; }
        out->row_ptr[i + 1] = pos;
      }
  csr_shrink(out);
  return ORC_OK;
}

/* 2D convection-diffusion on the unit square, nx*nx interior points, h = 1/(nx+1),
 * scaled by h^2: isotropic 9-point diffusion (1/6)[-1 -4 -1; -4 20 -4; -1 -4 -1]
 * plus first-order upwind convection h*(bx d/dx + by d/dy).  See DESIGN.md. */
int orc_convdiff_2d(int64_t nx, double bx, double by, orc_csr *out) {
  if (nx < 1) return fail(ORC_INVALID_ARGUMENT, "convdiff_2d: nx must be >= 1");
  double h = 1.0 / (double)(nx + 1);
  double st[3][3]; /* st[dy+1][dx+1] */
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) st[a][b] = 0.0;
  st[0][0] = st[0][2] = st[2][0] = st[2][2] = -1.0 / 6.0;
  st[0][1] = st[1][0] = st[1][2] = st[2][1] = -4.0 / 6.0;
  st[1][1] = 20.0 / 6.0;
  double cx = h * bx, cy = h * by;
  if (cx >= 0) { st[1][1] += cx; st[1][0] -= cx; } else { st[1][1] -= cx; st[1][2] += cx; }
  if (cy >= 0) { st[1][1] += cy; st[0][1] -= cy; } else { st[1][1] -= cy; st[2][1] += cy; }
  int64_t n = nx * nx;
  csr_alloc(out, n, n, 9 * n, 1);
  int64_t pos = 0;
  for (int64_t y = 0; y < nx; ++y)
    for (int64_t x = 0; x < nx; ++x) {
      int64_t i = x + nx * y;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int64_t xx = x + dx, yy = y + dy;
          if (xx < 0 || xx >= nx || yy < 0 || yy >= nx) continue;
          out->col_idx[pos] = xx + nx * yy;
          out->values[pos++] = st[dy + 1][dx + 1];
        }
      out->row_ptr[i + 1] = pos;
    }
  csr_shrink(out);
  return ORC_OK;
}

/* BASELINE config 4: lower T, `draws` off-diagonal draws per row at offset
 * 1 + floor(log(u)/log(1-p)) (u in (0,1]), capped at i; duplicates summed in
 * draw order; values N(0,1) (Box-Muller); d_i = 1.5 * sum_j |t_ij| + 1. */
int orc_synthetic_lower(int64_t n, int64_t draws, double p, uint64_t seed, orc_csr *out) {
  if (n < 1 || draws < 0 || !(p > 0.0 && p < 1.0))
    return fail(ORC_INVALID_ARGUMENT, "synthetic_lower: bad parameters");
  csr_alloc(out, n, n, n * (draws + 1), 1);
  int64_t *cols = (int64_t *)malloc((size_t)(draws + 1) * sizeof(int64_t));
  double *vals = (double *)malloc((size_t)(draws + 1) * sizeof(double));
  double lq = log1p(-p);
  uint64_t s_off = seed * 2 + 1, s_val = seed * 2 + 2;
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t nc = 0;
    if (i > 0) {
      for (int64_t d = 0; d < draws; ++d) {
        uint64_t ctr = (uint64_t)i * (uint64_t)draws + (uint64_t)d;
        double u = (double)((orc_rng_u64(s_off, ctr) >> 11) + 1) * 0x1.0p-53; /* (0,1] */
        double g = floor(log(u) / lq);
        int64_t off = g >= (double)i ? i : 1 + (int64_t)g;
        if (off > i) off = i;
        double u1 = (double)((orc_rng_u64(s_val, 2 * ctr) >> 11) + 1) * 0x1.0p-53;
        double u2 = orc_rng_uniform(s_val, 2 * ctr + 1);
        double v = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        int64_t c = i - off;
        /* insert keeping cols ascending, summing duplicates in draw order */
        int64_t q = 0;
        while (q < nc && cols[q] < c) ++q;
        if (q < nc && cols[q] == c) {
          vals[q] += v;
        } else {
          for (int64_t r = nc; r > q; --r) { cols[r] = cols[r - 1]; vals[r] = vals[r - 1]; }
          cols[q] = c;
          vals[q] = v;
          ++nc;
        }
      }
    }
    double s = 0.0;
    for (int64_t q = 0; q < nc; ++q) s += fabs(vals[q]);
    for (int64_t q = 0; q < nc; ++q) { out->col_idx[pos] = cols[q]; out->values[pos++] = vals[q]; }
    out->col_idx[pos] = i;
    out->values[pos++] = 1.5 * s + 1.0;
    out->row_ptr[i + 1] = pos;
  }
  free(cols);
  free(vals);
  csr_shrink(out);
  return ORC_OK;
}
