/*
 * sait_c.h — C ABI of the B200 SAIT library (libsait_b200.so).
 *
 * This is the drop-in boundary for the reference's SAIT hot path: every entry
 * point below names the reference interface it replaces (paths relative to
 * /root/reference/proj/core/).  Plain C types only: int64 sizes, raw host or
 * device pointers, opaque handles.  A `sait_stream_t` is a cudaStream_t
 * (NULL = the legacy default stream); device-pointer entry points enqueue on
 * it and return without synchronising unless stated.
 *
 * Status: every function returning int returns SAIT_OK (0) or an error code;
 * the message is in sait_last_error() (thread-local).  The error kinds map to
 * the reference's exceptions:
 *   SAIT_ERR_INVALID_ARGUMENT  <->  std::invalid_argument
 *   SAIT_ERR_RUNTIME           <->  std::runtime_error
 * and the messages carry the same text as the reference's (e.g.
 * "jacobi_split: singular matrix, zero diagonal at row 7").
 *
 * Device storage: CSR with int32 row_ptr / col_idx and fp64 values
 * (nnz < 2^31 is checked at upload / build time).
 */
#ifndef SAIT_C_H
#define SAIT_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAIT_ABI_VERSION 1

enum sait_status {
  SAIT_OK = 0,
  SAIT_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  SAIT_ERR_RUNTIME = 2,          /* std::runtime_error */
  SAIT_ERR_CUDA = 3,             /* CUDA runtime failure (no reference counterpart) */
  SAIT_ERR_NOMEM = 4
};

typedef struct sait_dcsr_s *sait_dcsr_t; /* device CSR matrix */
typedef struct sait_pair_s *sait_pair_t; /* SAIT pair preconditioner on one device */
typedef void *sait_stream_t;             /* cudaStream_t */

/* Host CSR in the reference layout (csr.hpp:24-43: int64 indices, fp64
 * values).  When the library fills one, free it with sait_host_csr_free. */
typedef struct {
  int64_t nrows;
  int64_t ncols;
  int64_t *row_ptr; /* nrows + 1 */
  int64_t *col_idx; /* nnz */
  double *values;   /* nnz; NULL for a sparsity pattern (csr.hpp:46-60) */
} sait_host_csr;

const char *sait_last_error(void);
int sait_abi_version(void);
void sait_host_csr_free(sait_host_csr *m);

/* ---------------------------------------------------------- device CSR ---
 * Replaces the host-side storage of saitprec::CsrMatrix (csr.hpp:24-43). */

/* Copies a host CSR (int64 indices) to the current device. */
int sait_csr_upload(const sait_host_csr *m, sait_stream_t stream, sait_dcsr_t *out);
/* Shape and stored-entry count. */
int sait_csr_info(sait_dcsr_t m, int64_t *nrows, int64_t *ncols, int64_t *nnz);
/* Copies back into caller arrays sized from sait_csr_info (values may be NULL). Synchronous. */
int sait_csr_download(sait_dcsr_t m, int64_t *row_ptr, int64_t *col_idx, double *values,
                      sait_stream_t stream);
/* Copies back into a library-allocated host CSR. Synchronous. */
int sait_csr_to_host(sait_dcsr_t m, sait_stream_t stream, sait_host_csr *out);
/* Raw device arrays (int32 row_ptr/col_idx, fp64 values; values NULL for a pattern). */
int sait_csr_device_arrays(sait_dcsr_t m, const int32_t **row_ptr, const int32_t **col_idx,
                           const double **values);
void sait_csr_free(sait_dcsr_t m);

/* ------------------------------------------------------------- kernels ---
 * kernels.hpp:12-40 on device matrices.  Results are new device matrices with
 * the reference's exact patterns and (bitwise) values. */

/* kernels.hpp:14 / kernels.cpp:10-26: y = A x, device vectors; row-sequential
 * accumulation in stored order (bitwise equal to the reference).  xlen/ylen are
 * checked like the reference's span sizes. */
int sait_spmv(sait_dcsr_t a, const double *d_x, int64_t xlen, double *d_y, int64_t ylen,
              sait_stream_t stream);
/* dense.hpp:41 / dense.cpp:10-19: Y = A X for a column-major n x nvec block
 * (DenseMatrix layout; d_x holds ncols x nvec, d_y nrows x nvec).  The
 * reference runs one spmv per column; here the matrix is read once per slab
 * of up to 8 columns (each column's rows still summed in stored order:
 * bitwise the per-column spmv). */
int sait_spmm(sait_dcsr_t a, const double *d_x, double *d_y, int64_t nvec, sait_stream_t stream);
/* kernels.hpp:21 / kernels.cpp:34-102: C = A B (Gustavson, ascending-k accumulation). */
int sait_spgemm(sait_dcsr_t a, sait_dcsr_t b, sait_stream_t stream, sait_dcsr_t *out);
/* kernels.hpp:25 / kernels.cpp:104-134 */
int sait_add_identity(sait_dcsr_t m, sait_stream_t stream, sait_dcsr_t *out);
/* kernels.hpp:30 / kernels.cpp:136-160 */
int sait_drop_by_threshold(sait_dcsr_t m, double tau, sait_stream_t stream, sait_dcsr_t *out);
/* kernels.hpp:33 / kernels.cpp:162-194 (pattern: a device CSR whose values are ignored) */
int sait_drop_by_pattern(sait_dcsr_t m, sait_dcsr_t pattern, sait_stream_t stream,
                         sait_dcsr_t *out);
/* kernels.hpp:40 / kernels.cpp:236-246: M * diag(d), d a device vector of length ncols. */
int sait_scale_columns(sait_dcsr_t m, const double *d_d, int64_t dlen, sait_stream_t stream,
                       sait_dcsr_t *out);
/* csr.hpp:84 / csr.cpp:72-92 */
int sait_transpose(sait_dcsr_t m, sait_stream_t stream, sait_dcsr_t *out);

/* ---------------------------------------------------------------- SAIT ---
 * sait.hpp:14-74.  `lower` selects TriangularKind::Side (1 = Lower). */

enum sait_drop_kind {
  SAIT_DROP_THRESHOLD = 1,     /* sait_thr  (sait.cpp:90-101) */
  SAIT_DROP_PATTERN = 2,       /* sait_pat  (sait.cpp:113-136) */
  SAIT_DROP_THRESHOLD_CAP = 3, /* BASELINE config 4 fill cap */
  SAIT_DROP_NONE = 4           /* sait_polynomial(split, steps, {}) then M D^-1 */
};

/* SaitThrParams{threshold, steps} / SaitPatParams{pattern_steps, refine_steps}
 * (sait.hpp:14-27) plus the fill-cap factor. */
typedef struct {
  int kind;            /* sait_drop_kind */
  double tau;          /* THRESHOLD, THRESHOLD_CAP: in [0, 1) */
  int steps;           /* THRESHOLD, THRESHOLD_CAP, NONE: >= 1 */
  int pattern_steps;   /* PATTERN: >= 0 */
  int refine_steps;    /* PATTERN: >= 1 */
  double cap_factor;   /* THRESHOLD_CAP: >= 1; column j keeps <= floor(f * nnz(T[:,j])) entries */
} sait_drop_spec;

typedef struct {
  int steps_run;       /* recursion steps executed (early stop included) */
  int stabilized;      /* 1 if the 1e-15 early stop fired (sait.cpp:14-28) */
  int64_t nnz_out;     /* stored entries of the result */
  int64_t products;    /* multiply-adds executed by the SpGEMM steps (one pass) */
  double seconds;      /* device time of the whole build (CUDA events) */
} sait_build_stats;

/* Step-wise build over a block of COLUMNS [col0, col1) of M (multi-GPU column
 * sharding).  A column of M evolves independently of the
 * others, so a block needs no data from other blocks; only the reference's
 * global early stop (sait.cpp:84-85) couples them: after every step the
 * caller reduces `changed` across blocks (max) and calls ..._stop() when no
 * block changed.  finish(transposed = 0) returns M[:, col0:col1] as an
 * n x (col1 - col0) CSR (local column index = global - col0); transposed = 1
 * returns that block's rows of M^T, i.e. a (col1 - col0) x n CSR.
 * sait_build == one session over [0, n) with local early stop. */
typedef struct sait_build_session_s *sait_build_session_t;
int sait_build_session_create(sait_dcsr_t t, int lower, const sait_drop_spec *spec, int64_t col0,
                              int64_t col1, sait_stream_t stream, sait_build_session_t *out);
int sait_build_session_remaining(sait_build_session_t s);
int sait_build_session_step(sait_build_session_t s, int *changed);
int sait_build_session_stop(sait_build_session_t s);
int sait_build_session_finish(sait_build_session_t s, int transposed, sait_dcsr_t *out,
                              sait_build_stats *stats);
void sait_build_session_destroy(sait_build_session_t s);

/* sait.hpp:40 / sait.cpp:32-73: d_inv_diag (device, length n) receives 1/T[i,i];
 * *tt receives I - D^-1 T with no stored diagonal. */
int sait_jacobi_split(sait_dcsr_t t, int lower, double *d_inv_diag, sait_stream_t stream,
                      sait_dcsr_t *tt);
/* sait_thr / sait_pat / fill-capped sait_thr in one entry (sait.cpp:75-136):
 * returns the approximate inverse M = poly(tT) D^-1 of the triangular T. */
int sait_build(sait_dcsr_t t, int lower, const sait_drop_spec *spec, sait_stream_t stream,
               sait_dcsr_t *m_out, sait_build_stats *stats);
/* Both factors of an ILU pair with the same drop spec (the input of
 * SaitPairPreconditioner): M_L = build(lower) on `stream` and M_U =
 * build(upper) concurrently on an internal stream; bitwise the two separate
 * sait_build calls.  stats2 (may be NULL) receives [M_L, M_U]. */
int sait_build_pair(sait_dcsr_t lower, sait_dcsr_t upper, const sait_drop_spec *spec, sait_stream_t stream,
                    sait_dcsr_t *ml_out, sait_dcsr_t *mu_out, sait_build_stats *stats2);
/* sait.hpp:53 / sait.cpp:75-88 with an empty DropRule: the undropped
 * unit-diagonal polynomial in tT (no D^-1 scaling), from the iteration
 * matrix tt of a JacobiSplit. */
int sait_polynomial(sait_dcsr_t tt, int steps, sait_stream_t stream, sait_dcsr_t *m_out,
                    sait_build_stats *stats);
/* sait.hpp:64 / sait.cpp:103-111 (result: a pattern, values NULL). */
int sait_pat_capture_pattern(sait_dcsr_t t, int lower, int pattern_steps, sait_stream_t stream,
                             sait_dcsr_t *pattern_out);

/* sait.hpp:73 / sait.cpp:138-159: k Jacobi sweeps x <- tT x + D^-1 b from
 * x = 0 on device vectors (the paper's section 4.3 comparison variant). */
int sait_jacobi_sweeps_apply(sait_dcsr_t t, int lower, const double *d_b, int sweeps, double *d_x,
                             sait_stream_t stream);

/* ilu.hpp:27 / ilu.cpp:98-173 with level 0, on the device: the factors of
 * ilu_k(a, 0) bitwise (L with its explicit unit diagonal, U from the
 * diagonal on), computed in dependency-level order.  Errors as the
 * reference: "ilu_k: matrix is not square", "ilu_k: structurally zero
 * diagonal at row i" (SAIT_ERR_INVALID_ARGUMENT), "ilu_k: pivot breakdown at
 * row i (|pivot| = %f)" (SAIT_ERR_RUNTIME) for the first such row. */
int sait_ilu0(sait_dcsr_t a, sait_stream_t stream, sait_dcsr_t *lower, sait_dcsr_t *upper);
/* The same for fill level 0 or 1 (ilu_k(a, level)); level 1's pattern is the
 * structural product (tril(A,-1) + I)(triu(A,1) + I) computed by the device
 * SpGEMM.  Levels >= 2: SAIT_ERR_INVALID_ARGUMENT (use sait_ilu_k). */
int sait_ilu_device(sait_dcsr_t a, int level, sait_stream_t stream, sait_dcsr_t *lower, sait_dcsr_t *upper);

/* kernels.hpp:36 / kernels.cpp:196-234: x = T^-1 b by substitution (Lower:
 * rows ascending, Upper: descending; the stored diagonal is used, entries on
 * the wrong side of it read x as zero), device vectors, bitwise the
 * reference's result.  Synchronous; SAIT_ERR_RUNTIME "trisolve: singular
 * matrix, zero diagonal at row i" for the first such row in solve order. */
int sait_trisolve(sait_dcsr_t t, int lower, const double *d_b, int64_t blen, double *d_x,
                  sait_stream_t stream);

/* --------------------------------------- multi-GPU redistribution (K4) ---
 * The distributed form of transpose (csr.cpp:72-92) that turns the
 * column-sharded build's blocks M[:, C_r:C_{r+1}] into the row blocks of the
 * row-sharded apply without a host round trip. */

/* One received piece: rows [0, nrows) of a CSR whose entries of row i are
 * col_idx/values[row_ptr[i] - row_ptr[0] .. row_ptr[i+1] - row_ptr[0]) (device
 * pointers; row_ptr may start at any base), columns shifted by col_offset. */
typedef struct {
  const int32_t *row_ptr;
  const int32_t *col_idx;
  const double *values;
  int64_t col_offset;
} sait_row_piece;
/* Row i of *out = the pieces' rows i concatenated in part order.  Parts must
 * cover disjoint, ascending column ranges (then rows stay sorted). */
int sait_csr_assemble_rows(int nparts, const sait_row_piece *parts, int64_t nrows, int64_t ncols,
                           sait_stream_t stream, sait_dcsr_t *out);
/* [*lo, *hi) = the range of stored columns ((0, 0) when empty). */
int sait_csr_col_span(sait_dcsr_t m, int64_t *lo, int64_t *hi, sait_stream_t stream);
/* In place: every column index += offset; ncols = new_ncols. */
int sait_csr_shift_cols(sait_dcsr_t m, int64_t offset, int64_t new_ncols, sait_stream_t stream);
/* out[j] = row_ptr[rows[j]] for k host row indices (host in, host out). */
int sait_csr_row_ptr_at(sait_dcsr_t m, const int64_t *rows, int k, int64_t *out, sait_stream_t stream);
/* d_work[j] (device, n int64) = predicted products of column j's recursion
 * (its step-2 work: sum over the entries (k, j) of tT of nnz(tT[:, k]) + 1);
 * the column-sharded build balances its blocks on the prefix sums. */
int sait_column_work(sait_dcsr_t t, int64_t *d_work, sait_stream_t stream);

/* ------------------------------------------------------- SpMV operator ---
 * A prepared y = A x for a (possibly rectangular) device CSR: keeps the
 * SELL-32 copy when the rows are regular enough (the apply's kernel), else the
 * CSR kernels.  Bitwise equal to spmv (kernels.cpp:10-26).  Used for the
 * local row blocks of the multi-GPU apply. */
typedef struct sait_op_s *sait_op_t;
int sait_operator_create(sait_dcsr_t a, int take_ownership, sait_op_t *out);
int sait_operator_apply(sait_op_t op, const double *d_x, int64_t xlen, double *d_y, int64_t ylen,
                        sait_stream_t stream);
void sait_operator_destroy(sait_op_t op);

/* Row block of a sharded factor whose halo is read straight from the
 * neighbouring ranks' buffers (peer memory over NVLink): the
 * extended vector is [halo below | own | halo above]; columns c < own_lo read
 * lo_src[c + lo_shift], columns c >= own_hi read hi_src[c + hi_shift], after
 * the owner's flag (*lo_flag / *hi_flag) reached `epoch` (system-scope
 * acquire).  The local part of d_x_ext must already hold the own segment.
 * Needs the SELL copy (SAIT_ERR_INVALID_ARGUMENT otherwise). */
typedef struct {
  int64_t own_lo, own_hi;
  const double *lo_src;
  int64_t lo_shift;
  const double *hi_src;
  int64_t hi_shift;
  const int *lo_flag, *hi_flag;
  int epoch;
} sait_halo_t;
int sait_operator_apply_halo(sait_op_t op, const double *d_x_ext, int64_t ext_len, const sait_halo_t *halo,
                             double *d_y, int64_t ylen, sait_stream_t stream);
/* The row-sharded pair with peer-memory halos as one native object (the
 * data path of the multi-GPU apply): per factor this rank's two
 * parity copies of its extended vector, its epoch flag, the own segment, the
 * own rows its neighbours read (send ranges) and per parity the neighbours'
 * halo sources.  apply(r, z) on this rank's rows, epoch e += 1, parity e & 1:
 *   1. only the boundary slices of r the neighbours read are copied into M_L's
 *      extended vector, and the same kernel publishes flag_L = e;
 *   2. M_L's halo SpMV reads its own x straight from r and its halo over
 *      NVLink (after the owners' flags), writes y into M_U's own segment,
 *      and its last CTA publishes flag_U = e (no extra launch);
 *   3. M_U's halo SpMV (a programmatic dependent of M_L) -> z.
 * Without neighbours this is two kernels, like the single-GPU pair.  The
 * operators are borrowed (they must outlive the pair). */
typedef struct {
  double *ext[2];       /* extended vector, parity 0 / 1 (device) */
  int *flag;            /* this rank's published epoch for this factor */
  int64_t ext_len, own_offset, own_len;
  int64_t send_a0, send_n0, send_a1, send_n1; /* own rows [a, a + n) the neighbours read */
  sait_halo_t halo[2];  /* per parity (the epoch field is set per apply) */
} sait_peer_factor_desc;
typedef struct sait_peer_pair_s *sait_peer_pair_t;
int sait_peer_pair_create(sait_op_t ml, sait_op_t mu, const sait_peer_factor_desc *desc, sait_peer_pair_t *out);
int sait_peer_pair_apply(sait_peer_pair_t p, const double *d_r, double *d_z, sait_stream_t stream);
void sait_peer_pair_destroy(sait_peer_pair_t p);
/* *d_flag = epoch once everything queued before on `stream` has completed
 * (system-scope release: peers polling the flag then see the data). */
int sait_publish_epoch(int *d_flag, int epoch, sait_stream_t stream);
/* CUDA IPC for buffers from sait_device_alloc: a 64-byte handle another
 * process on the node opens to get a device pointer to the same memory. */
int sait_ipc_handle(const void *d_ptr, void *handle64);
int sait_ipc_open(const void *handle64, void **d_ptr);
int sait_ipc_close(void *d_ptr);

/* ------------------------------------------------ pair preconditioner ---
 * SaitPairPreconditioner (preconditioner.hpp:54-68, preconditioner.cpp:34-49). */

/* Takes ownership of ml and mu when take_ownership != 0 (the reference ctor
 * moves its matrices in); otherwise they must outlive the pair.  Shape check
 * of preconditioner.cpp:37-39. */
int sait_pair_create(sait_dcsr_t ml, sait_dcsr_t mu, int take_ownership, sait_pair_t *out);
/* Apply storage of a pair's factors.  AUTO (what sait_pair_create uses):
 * SELL-32 slices with shared slice patterns when the factor repeats a few
 * slice structures (stencil factors: only the values stream), else int16
 * column deltas, else int32 columns; rows too ragged for 32-row slices in
 * their natural order (padding > 25%) are sorted by length within 1024-row
 * windows; CSR when even that pads more than 25%.  A forced SELL format falls back down that
 * list when the matrix does not allow it; sait_pair_format reports what was
 * used.  Every format gives the same bits (rows summed in stored order). */
enum { SAIT_FMT_AUTO = 0, SAIT_FMT_CSR = 1, SAIT_FMT_SELL_I32 = 2, SAIT_FMT_SELL_I16 = 3, SAIT_FMT_SELL_DICT = 4 };
int sait_pair_create_ex(sait_dcsr_t ml, sait_dcsr_t mu, int take_ownership, int format, sait_pair_t *out);
typedef struct {
  int format;           /* SAIT_FMT_* in use (never AUTO) */
  int row_sorted;       /* SELL: 1 when the rows were sorted by length within
                         * 1024-row windows (SELL-C-sigma, for factors too
                         * ragged for 32-row slices in their natural order) */
  int64_t nrows, nnz;
  int64_t stored_slots; /* SELL: slots incl. padding; CSR: nnz */
  int64_t nslices, dict_elems;
  /* bytes one SpMV with this factor must move in this format: stored
   * values + indices (+ slice offsets, pattern offsets, dictionary) + x read
   * once + y written once -- the denominator of the apply roofline */
  int64_t stream_bytes;
} sait_factor_format;
/* which: 0 = M_L, 1 = M_U */
int sait_pair_format(sait_pair_t p, int which, sait_factor_format *out);
/* name() == "sait" and nnz() (preconditioner.hpp:62-63) */
int sait_pair_info(sait_pair_t p, int64_t *n, int64_t *nnz);
/* apply(r, z): z = M_U (M_L r), device vectors (preconditioner.cpp:42-45).
 * Enqueued on `stream`; safe to call concurrently from several threads/streams. */
int sait_pair_apply(sait_pair_t p, const double *d_r, int64_t rlen, double *d_z, int64_t zlen,
                    sait_stream_t stream);
/* Same with HOST vectors (any host memory; pinned is faster).  The copies are
 * pipelined with the two SpMVs.  Synchronous on return. */
int sait_pair_apply_host(sait_pair_t p, const double *h_r, int64_t rlen, double *h_z,
                         int64_t zlen, sait_stream_t stream);
/* apply_block (preconditioner.cpp:47-49): nvec vectors.  layout 0 = column-major
 * n x nvec (DenseMatrix, dense.hpp:12-38), 1 = row-major n x nvec. Device pointers. */
int sait_pair_apply_block(sait_pair_t p, const double *d_r, double *d_z, int64_t n,
                          int64_t nvec, int layout, sait_stream_t stream);
/* Same with HOST blocks; synchronous on return.  Column-major blocks are
 * pipelined vector group by vector group (copy in / pairs / copy out on three
 * streams), so with pinned buffers a vector costs max(H2D, D2H), not the sum. */
int sait_pair_apply_block_host(sait_pair_t p, const double *h_r, double *h_z, int64_t n,
                               int64_t nvec, int layout, sait_stream_t stream);
/* One factor's SpMV with the pair's planned kernel (which: 0 = M_L, 1 = M_U);
 * the building block of apply, exposed for per-kernel timing. */
int sait_pair_spmv_factor(sait_pair_t p, int which, const double *d_x, double *d_y,
                          sait_stream_t stream);
/* Borrowed handles of the two factors (owned by the pair). */
int sait_pair_factors(sait_pair_t p, sait_dcsr_t *ml, sait_dcsr_t *mu);
void sait_pair_destroy(sait_pair_t p);

/* ------------------------------------------ exact ILU preconditioner ---
 * ExactIluPreconditioner (preconditioner.hpp:39-49, preconditioner.cpp:25-32):
 * z = U^-1 (L^-1 r), the sequential baseline SAIT replaces, on the device.
 * name() == "exact", nnz() = nnz(L) + nnz(U).  Takes ownership of the
 * factors when take_ownership != 0.  apply is synchronous (it reports a zero
 * pivot like trisolve) and safe to call concurrently on different streams. */
typedef struct sait_exact_s *sait_exact_t;
int sait_exact_ilu_create(sait_dcsr_t lower, sait_dcsr_t upper, int take_ownership, sait_exact_t *out);
int sait_exact_ilu_info(sait_exact_t p, int64_t *n, int64_t *nnz);
int sait_exact_ilu_apply(sait_exact_t p, const double *d_r, int64_t rlen, double *d_z, int64_t zlen,
                         sait_stream_t stream);
void sait_exact_ilu_destroy(sait_exact_t p);

/* ------------------------------------------------------------ solvers ---
 * Device-resident loops driving the apply (north_star (3)); the reference has
 * them only as SPEC.md:282-351 (PCG, LOBPCG) and not at all for GMRES, so the
 * algorithms are fixed in DESIGN.md "solvers".  Vectors stay in HBM; b, x,
 * eigenvectors are device pointers on A's device.  M may be NULL (identity).
 * Reductions use a canonical order, so results are bitwise reproducible. */
typedef struct {
  int iterations;
  int converged;
  double relres_estimate; /* the stopping quantity at exit */
  double true_relres;     /* ||b - A x|| / ||b|| recomputed at exit */
  double seconds;         /* wall time of the solve */
  /* the paper's runtime split (TimedPreconditioner,
   * preconditioner.cpp:66-77): device time of the preconditioner applies
   * (CUDA events on the solver's stream) and their number; the rest of
   * `seconds` is the operator, the orthogonalisation and the control */
  double precond_seconds;
  int64_t precond_applies;
} sait_solve_stats;

/* Right-preconditioned restarted GMRES(restart) from x0 = 0, CGS2 Arnoldi,
 * stop when the Arnoldi residual estimate / ||b|| <= tol.  h_hist (host,
 * maxit + 1 entries, may be NULL) receives the estimate per iteration. */
int sait_gmres(sait_dcsr_t A, sait_pair_t M, const double *d_b, double *d_x, int64_t n, int restart,
               double tol, int maxit, double *h_hist, sait_solve_stats *stats, sait_stream_t stream);
/* PCG from x0 = 0: stop when ||r|| / ||b|| <= tol;
 * SAIT_ERR_RUNTIME on breakdown (p'Ap <= 0). */
int sait_pcg(sait_dcsr_t A, sait_pair_t M, const double *d_b, double *d_x, int64_t n, double tol,
             int maxit, double *h_hist, sait_solve_stats *stats, sait_stream_t stream);

/* The same loops preconditioned by the exact ILU solves (the comparator of
 * the paper's iteration tables). */
int sait_gmres_exact(sait_dcsr_t A, sait_exact_t M, const double *d_b, double *d_x, int64_t n,
                     int restart, double tol, int maxit, double *h_hist, sait_solve_stats *stats,
                     sait_stream_t stream);
int sait_pcg_exact(sait_dcsr_t A, sait_exact_t M, const double *d_b, double *d_x, int64_t n, double tol,
                   int maxit, double *h_hist, sait_solve_stats *stats, sait_stream_t stream);

/* Block LOBPCG for the nev (<= 16) smallest eigenpairs of
 * SPD A, preconditioned by the pair applied to the whole residual block
 * (apply_block, preconditioner.cpp:47-49).  X0 ~ U[-1,1] from `seed`.
 * h_evals: nev host values (ascending); d_evecs: n x nev column-major device
 * block (may be NULL); h_resnorms: host (maxit + 1) x nev residual norms per
 * iteration (may be NULL); converged when every ||A x - lambda x|| <= tol. */
int sait_lobpcg(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed,
                double *h_evals, double *d_evecs, double *h_resnorms, int *iterations,
                sait_stream_t stream);
/* The same, also filling stats (iterations, converged, seconds and the
 * preconditioner's share: precond_seconds / precond_applies, one apply per
 * block of nev vectors). */
int sait_lobpcg_ex(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed,
                   double *h_evals, double *d_evecs, double *h_resnorms, int *iterations,
                   sait_solve_stats *stats, sait_stream_t stream);
/* LOBPCG with a choice of Gram kernel.  SAIT_GRAM_CANONICAL: the canonical
 * reduction order (bitwise the restatement oracle/solvers.c; what sait_lobpcg
 * uses).  SAIT_GRAM_TENSOR: FP64 tensor-core (DMMA) Grams -- deterministic,
 * but the products inside an mma are summed in the hardware's order, so the
 * run agrees with the restatement to within the north_star's +-1 iteration
 * rather than bit for bit. */
enum { SAIT_GRAM_CANONICAL = 0, SAIT_GRAM_TENSOR = 1 };
int sait_lobpcg_opt(sait_dcsr_t A, sait_pair_t M, int nev, double tol, int maxit, uint64_t seed, int gram_mode,
                    double *h_evals, double *d_evecs, double *h_resnorms, int *iterations,
                    sait_solve_stats *stats, sait_stream_t stream);
/* The same with the exact ILU solves as preconditioner (column by column;
 * the comparator of SPEC.md acceptance #9). */
int sait_lobpcg_exact(sait_dcsr_t A, sait_exact_t M, int nev, double tol, int maxit, uint64_t seed,
                      double *h_evals, double *d_evecs, double *h_resnorms, int *iterations,
                      sait_stream_t stream);

/* Vector primitives of those loops, for solver loops driven across ranks
 * (the same kernels, so the same bits).  Dots: `sait_dot_partials` writes the
 * canonical per-2048-element-block partials of x . V_j (partials[j * nb + b],
 * nb = sait_dot_blocks(n)); `sait_dot_fold` folds nb partials per dot in the
 * canonical order (sqrt_out: square root of the result).  A row-sharded vector
 * aligned to 2048-element blocks gives each rank a contiguous run of the
 * global blocks, so folding every rank's partials reproduces the single-GPU
 * dot bitwise.  vec_update op: 0 y = y + a x, 1 y = x + a y, 2 y = x - y,
 * 3 y = y + x.  vec_cgs: w = w - sum_j h_j V_j (j ascending); vec_div:
 * out = w / d[0]; vec_lincomb: u = sum_j y_j V_j.  h, d, y are device. */
int64_t sait_dot_blocks(int64_t n);
int sait_dot_partials(const double *d_x, const double *d_V, int64_t ld, int m, int64_t n, double *d_partials,
                      sait_stream_t stream);
int sait_dot_fold(const double *d_partials, int64_t nb, int m, double *d_out, int sqrt_out,
                  sait_stream_t stream);
int sait_vec_update(int op, int64_t n, double a, const double *d_x, double *d_y, sait_stream_t stream);
int sait_vec_cgs(int64_t n, double *d_w, const double *d_V, int64_t ld, int m, const double *d_h,
                 sait_stream_t stream);
int sait_vec_div(int64_t n, const double *d_w, const double *d_d, double *d_out, sait_stream_t stream);
int sait_vec_lincomb(int64_t n, const double *d_V, int64_t ld, int k, const double *d_y, double *d_u,
                     sait_stream_t stream);
/* LOBPCG's pieces: canonical Gram partials of every A_a . B_b (a < ka <= 48,
 * b < kb <= 48; partials[(a * kb + b) * nb + blk], fold with sait_dot_fold,
 * m = ka * kb, to a row-major ka x kb Gram); column-major block kernels
 * (out = in C, W = W - X G, R_j = AX_j - lam_j X_j; C, G, lam on the device);
 * U[-1, 1] fill of global entries [offset, offset + n) of seed's sequence
 * (sait_fill_uniform_pm1 on the device); and the host dense algebra
 * (Cholesky, inverse of a lower triangle, Rayleigh-Ritz: returns 1 on success,
 * 0 if the matrix is not positive definite). */
int sait_gram_partials(const double *d_A, int ka, const double *d_B, int kb, int64_t n, double *d_partials,
                       sait_stream_t stream);
int sait_block_lincomb(int64_t n, const double *d_in, int kin, const double *d_C, int kout, double *d_out,
                       sait_stream_t stream);
int sait_block_sub_lincomb(int64_t n, const double *d_X, int k, const double *d_G, double *d_W,
                           sait_stream_t stream);
int sait_block_residual(int64_t n, int k, const double *d_AX, const double *d_X, const double *d_lam,
                        double *d_R, sait_stream_t stream);
int sait_fill_uniform_pm1_device(uint64_t seed, int64_t n, int64_t offset, double *d_out, sait_stream_t stream);
int sait_dense_chol_lower(const double *G, int m, double *L);
void sait_dense_tri_lower_inv(const double *L, int m, double *Li);
int sait_dense_rayleigh_ritz(const double *GA, const double *GB, int m, int k, double *C, double *lam);

/* ----------------------------------------------------- inputs (host) ---
 * Producers of the path's inputs.  ilu_k is ilu.hpp:27 / ilu.cpp:98-173
 * (bitwise identical factors); the generators fix BASELINE.json's synthetic
 * problems. */
int sait_ilu_k(const sait_host_csr *a, int level, sait_host_csr *lower, sait_host_csr *upper);
int sait_problem_laplacian_2d(int64_t nx, sait_host_csr *out);
int sait_problem_laplacian_3d(int64_t n, sait_host_csr *out);
int sait_problem_convdiff_2d(int64_t nx, double bx, double by, sait_host_csr *out);
int sait_problem_synthetic_lower(int64_t n, int64_t draws, double p, uint64_t seed,
                                 sait_host_csr *out);
void sait_fill_uniform_pm1(uint64_t seed, int64_t n, double *out);
/* SPEC.md:373-381 mm_read (spec only in the reference): Matrix Market
 * coordinate real/integer, general or symmetric (expanded to full storage),
 * 1-based, '%' comments; entries assembled like from_triplets (csr.cpp:10-58,
 * duplicates summed in file order).  Errors "mm_read: line N: ..."
 * (SAIT_ERR_INVALID_ARGUMENT).  mm_write emits the general form with %.17g
 * values: mm_read(mm_write(M)) == M bit for bit. */
int sait_mm_read(const char *path, sait_host_csr *out);
int sait_mm_write(const char *path, const sait_host_csr *m);
/* SPEC.md:382-389 make_rhs: mode 0 ones-solution b = A 1 (row sums in stored
 * order), mode 1 seeded-random unit vector uniform_pm1(seed) / ||.||_2. */
int sait_make_rhs(const sait_host_csr *a, int mode, uint64_t seed, double *out);

/* ------------------------------------------------------------ utility --- */
int sait_device_synchronize(void);
/* Device memory and streams for hosts that do not link the CUDA runtime
 * (e.g. the C++ saitprec:: shim).  kind: 1 H2D, 2 D2H, 3 D2D (synchronous). */
int sait_device_alloc(size_t bytes, void **ptr);
void sait_device_free(void *ptr);
int sait_memcpy(void *dst, const void *src, size_t bytes, int kind);
int sait_stream_create(sait_stream_t *stream);
void sait_stream_destroy(sait_stream_t stream);
/* Pinned host buffers for the host-vector entry points. */
int sait_host_alloc(size_t bytes, void **ptr);
void sait_host_free(void *ptr);
/* Counts kernels launched by this library on this process (all threads). */
int64_t sait_kernel_launch_count(void);
/* Grow the device's stream-ordered pool (which this library allocates its
 * scratch and results from, and never trims) by `bytes` up front, so the
 * first builds of a process do not pay for new device mappings.  Optional. */
int sait_device_pool_reserve(int device, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* SAIT_C_H */
