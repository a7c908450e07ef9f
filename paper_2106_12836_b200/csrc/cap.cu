// cap.cu — the A15 fill cap on a row-form iterate, and the reference's
// stabilized() test on two device CSR matrices.
//
// The cap keeps, in every column j of M_s, the diagonal and the cap_j - 1
// largest-|v| off-diagonals (ties: the smaller row), after the threshold,
// every step (DESIGN.md §8 decision 3; the oracle applies it through the
// reference's DropRule hook).  The column-form recursion applies it inside
// the SpGEMM epilogue, where a column of M is a row of M^T.  A whole-matrix
// build runs in row form instead (no transposes of tT and M), with a
// threshold-only epilogue, and then this pass: count the entries per column,
// flag the columns over their cap (few), gather the flagged columns' entries,
// rank them per column exactly as the epilogue would, and compact the rows
// that lost entries.  Same surviving set, hence the same matrix, bit for bit.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace sait {
namespace {

// entries are visited flat, 4 per thread (one 16-byte load of columns)
constexpr int kFlat = 4;
// entries per block of the flat compaction (cap_compact)
constexpr int kCompact = 1024;
// Column counts of a (sorted) CSR, added into cnt.  A block takes 1024
// consecutive rows; when their columns span at most kColBins (banded and
// near-diagonal matrices: the triangular factors, T, the SAIT iterates) it
// counts into a shared histogram and flushes only the touched bins -- one
// global atomic per (block, column) instead of one per entry -- else it
// falls back to one global atomic per entry.
constexpr int kColRows = 1024, kColBins = 8192;
__global__ void __launch_bounds__(256) col_counts_banded(int64_t nrows, const int32_t* __restrict__ rp,
                                                         const int32_t* __restrict__ ci, int32_t* __restrict__ cnt) {
  __shared__ int32_t h[kColBins];
  __shared__ int32_t lo_s, hi_s;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kColRows;
  const int64_t r1 = min(r0 + kColRows, nrows);
  if (threadIdx.x == 0) {
    lo_s = INT32_MAX;
    hi_s = -1;
  }
  __syncthreads();
  int32_t lo = INT32_MAX, hi = -1;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const int32_t b = rp[r], e = rp[r + 1];
    if (b < e) {
      lo = min(lo, ci[b]);
      hi = max(hi, ci[e - 1]);
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&lo_s, lo);
    atomicMax(&hi_s, hi);
  }
  __syncthreads();
  lo = lo_s;
  hi = hi_s;
  if (hi < lo) return;
  const int64_t e0 = rp[r0], e1 = rp[r1];
  if (static_cast<int64_t>(hi) - lo < kColBins) {
    const int range = hi - lo + 1;
    for (int b = threadIdx.x; b < range; b += blockDim.x) h[b] = 0;
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&h[ci[e] - lo], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < range; b += blockDim.x)
      if (h[b]) atomicAdd(&cnt[lo + b], h[b]);
  } else {
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&cnt[ci[e]], 1);
  }
}

// seglen[c] = number of c's entries when column c has more off-diagonals
// than its room (cap - 1, at least 0), else 0 (the diagonal is always
// present: +I, always kept by the threshold); flagged columns are listed
// and marked in a bitmap
__global__ void cap_flag(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ cap,
                         int32_t* __restrict__ seglen, uint32_t* __restrict__ bits, int32_t* __restrict__ list,
                         int32_t* __restrict__ nlist) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool f = false;
  if (c < n) {
    const int32_t room = max(cap[c] - 1, 0);
    f = cnt[c] - 1 > room;
    seglen[c] = f ? cnt[c] : 0;
  }
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (c < n && lane == 0) bits[c >> 5] = m;  // 32 consecutive columns per warp
  if (m) {
    int32_t base = 0;
    if (lane == 0) base = atomicAdd(nlist, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (f) list[base + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(c);
  }
}

// entries of flagged columns -> their column's segment (row, value,
// position); flat over the entries, the row of a (rare) match by binary search
__device__ __forceinline__ void cap_take(int64_t e, int32_t c, int64_t nrows, const int32_t* __restrict__ rp,
                                         const double* __restrict__ v, int32_t* __restrict__ cursor,
                                         int32_t* __restrict__ lrow, double* __restrict__ lval,
                                         int32_t* __restrict__ lpos) {
  int64_t lo = 0, hi = nrows;  // the row i with rp[i] <= e < rp[i + 1]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (rp[mid] <= e) lo = mid;
    else hi = mid;
  }
  const int32_t p = atomicAdd(&cursor[c], 1);
  lrow[p] = static_cast<int32_t>(lo);
  lval[p] = v[e];
  lpos[p] = static_cast<int32_t>(e);
}
__global__ void cap_gather(int64_t nnz, int64_t nrows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, const uint32_t* __restrict__ bits,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ lrow, double* __restrict__ lval,
                           int32_t* __restrict__ lpos) {
  const int64_t e0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kFlat;
  auto flagged = [&](int32_t c) { return (bits[c >> 5] >> (c & 31)) & 1u; };
  if (e0 + kFlat <= nnz) {
    const int4 c = *reinterpret_cast<const int4*>(ci + e0);
    if (flagged(c.x)) cap_take(e0, c.x, nrows, rp, v, cursor, lrow, lval, lpos);
    if (flagged(c.y)) cap_take(e0 + 1, c.y, nrows, rp, v, cursor, lrow, lval, lpos);
    if (flagged(c.z)) cap_take(e0 + 2, c.z, nrows, rp, v, cursor, lrow, lval, lpos);
    if (flagged(c.w)) cap_take(e0 + 3, c.w, nrows, rp, v, cursor, lrow, lval, lpos);
  } else {
    for (int64_t e = e0; e < nnz; ++e)
      if (flagged(ci[e])) cap_take(e, ci[e], nrows, rp, v, cursor, lrow, lval, lpos);
  }
}

// one warp per column: rank every off-diagonal by (|v| desc, row asc) among
// the column's off-diagonals; ranks >= room are dropped (column index -1)
__global__ void cap_rank(int32_t nflag, const int32_t* __restrict__ flagged, const int32_t* __restrict__ seglen,
                         const int32_t* __restrict__ segstart, const int32_t* __restrict__ cap,
                         const int32_t* __restrict__ lrow, const double* __restrict__ lval,
                         const int32_t* __restrict__ lpos, int32_t* __restrict__ ci, int32_t* __restrict__ rowdel,
                         int32_t* __restrict__ blkdel, unsigned long long* __restrict__ ndel) {
  const int64_t f = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= nflag) return;
  const int32_t c = flagged[f];
  const int32_t b = segstart[c], len = seglen[c];
  const int32_t room = max(cap[c] - 1, 0);
  const int32_t col = c;
  int killed = 0;
  for (int32_t t = lane; t < len; t += 32) {
    const int32_t row = lrow[b + t];
    if (row == col) continue;
    const double mv = fabs(lval[b + t]);
    int32_t rank = 0;
    for (int32_t q = 0; q < len; ++q) {
      const int32_t rq = lrow[b + q];
      if (rq == col || rq == row) continue;
      const double vq = fabs(lval[b + q]);
      rank += (vq > mv) || (vq == mv && rq < row);
    }
    if (rank >= room) {
      const int32_t p = lpos[b + t];
      ci[p] = -1;
      atomicAdd(&rowdel[row], 1);
      atomicAdd(&blkdel[p / kCompact], 1);
      ++killed;
    }
  }
  killed = __reduce_add_sync(0xffffffffu, killed);
  if (lane == 0 && killed) atomicAdd(ndel, static_cast<unsigned long long>(killed));
}

__global__ void cap_row_counts(int64_t nrows, const int32_t* __restrict__ rp, const int32_t* __restrict__ rowdel,
                               int32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nrows) cnt[i] = rp[i + 1] - rp[i] - rowdel[i];
}

// The compaction is flat over the entries, kCompact per block (4 per
// thread, warp-contiguous): an entry's new position is its old one minus the
// deletions before it -- those of earlier blocks (a scan of the per-block
// counts cap_rank keeps) plus those earlier in its block (ballots) -- so the
// reads and writes stay coalesced whatever the row lengths (the 8-lanes-per-
// row copy it replaces ran at ~2/3 of the copy bandwidth on C4's rows).
__global__ void __launch_bounds__(256) cap_compact(int64_t nnz, const int32_t* __restrict__ ci,
                                                   const double* __restrict__ v, const int32_t* __restrict__ blkshift,
                                                   const double* __restrict__ scale, int32_t* __restrict__ nci,
                                                   double* __restrict__ nv) {
  constexpr int kPer = kCompact / 256;
  __shared__ int32_t wdel[kPer * 8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kCompact;
  int32_t c[kPer];
  double x[kPer];
  unsigned del[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int64_t e = b0 + u * 256 + threadIdx.x;
    const bool in = e < nnz;
    c[u] = in ? ci[e] : 0;
    x[u] = in ? v[e] : 0.0;
    del[u] = __ballot_sync(0xffffffffu, c[u] < 0);
    if (lane == 0) wdel[u * 8 + w] = __popc(del[u]);
  }
  __syncthreads();
  int32_t before = blkshift[blockIdx.x];
  const unsigned below = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    for (int q = 0; q < 8; ++q)
      if (q < w) before += wdel[u * 8 + q];
    const int64_t e = b0 + u * 256 + threadIdx.x;
    if (e < nnz && c[u] >= 0) {
      const int64_t p = e - before - __popc(del[u] & below);
      nci[p] = c[u];
      nv[p] = scale ? __dmul_rn(x[u], scale[c[u]]) : x[u];  // scale_columns (kernels.cpp:236-246), fused
    }
    for (int q = w; q < 8; ++q) before += wdel[u * 8 + q];
  }
}

// the reference's stabilized(prev, cur) (sait.cpp:14-28), shapes already equal
__global__ void stable_rows(int64_t nrows, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                            const double* __restrict__ av, const int32_t* __restrict__ brp,
                            const int32_t* __restrict__ bci, const double* __restrict__ bv, int* __restrict__ differs) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 3;
  if (i >= nrows) return;
  bool diff = arp[i] != brp[i] || arp[i + 1] != brp[i + 1];
  if (!diff)
    for (int32_t q = arp[i] + (threadIdx.x & 7); q < arp[i + 1]; q += 8) {
      const double a = av[q], b = bv[q];
      const double fa = fabs(a), fb = fabs(b);
      const double mx = fa < fb ? fb : fa;
      if (aci[q] != bci[q] || fabs(__dsub_rn(b, a)) > __dmul_rn(1e-15, mx)) diff = true;
    }
  if (diff && *reinterpret_cast<volatile int*>(differs) == 0) atomicOr(differs, 1);
}

}  // namespace

void column_counts_add(const DevCsr& m, int32_t* cnt, cudaStream_t s) {
  if (m.nrows == 0 || m.nnz == 0) return;
  col_counts_banded<<<grid_for(m.nrows, kColRows), 256, 0, s>>>(m.nrows, m.rp, m.ci, cnt);
  SAIT_LAUNCHED();
}

// Applies the cap to m in place; returns the number of entries dropped.
// With out_scale (the last step), a compaction also scales the columns and
// *scaled is set.
int64_t cap_rowform(DevCsr& m, const int32_t* cap, cudaStream_t s, const double* out_scale, bool* scaled) {
  if (scaled) *scaled = false;
  const int64_t n = m.nrows;
  if (n == 0 || m.nnz == 0) return 0;
  int32_t* cnt = dalloc<int32_t>(n + 1, s);
  int32_t* seglen = dalloc<int32_t>(n + 1, s);
  int32_t* segstart = dalloc<int32_t>(n + 1, s);
  int32_t* flagged = dalloc<int32_t>(n + 1, s);
  uint32_t* bits = reinterpret_cast<uint32_t*>(dalloc<int32_t>((n + 31) / 32 + 1, s));
  int32_t* nflag_d = dalloc<int32_t>(1, s);
  SAIT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * n, s));
  SAIT_CUDA(cudaMemsetAsync(nflag_d, 0, sizeof(int32_t), s));
  col_counts_banded<<<grid_for(n, kColRows), 256, 0, s>>>(n, m.rp, m.ci, cnt);
  SAIT_LAUNCHED();
  cap_flag<<<grid_for(n, 256), 256, 0, s>>>(n, cnt, cap, seglen, bits, flagged, nflag_d);
  SAIT_LAUNCHED();
  const int64_t listed = scan_counts(seglen, segstart, n, s);
  int64_t deleted = 0;
  if (listed > 0) {
    int32_t nflag = 0;
    read_back(s, {{&nflag, nflag_d, sizeof nflag}});
    int32_t* lrow = dalloc<int32_t>(listed, s);
    double* lval = dalloc<double>(listed, s);
    int32_t* lpos = dalloc<int32_t>(listed, s);
    int32_t* rowdel = cnt;  // reused: deletions per row
    unsigned long long* ndel = reinterpret_cast<unsigned long long*>(dalloc<int64_t>(1, s));
    SAIT_CUDA(cudaMemsetAsync(rowdel, 0, sizeof(int32_t) * n, s));
    SAIT_CUDA(cudaMemsetAsync(ndel, 0, sizeof(unsigned long long), s));
    const int64_t nblk = (m.nnz + kCompact - 1) / kCompact;
    int32_t* blkdel = dalloc<int32_t>(nblk + 1, s);
    SAIT_CUDA(cudaMemsetAsync(blkdel, 0, sizeof(int32_t) * nblk, s));
    int32_t* cursor = dalloc<int32_t>(n, s);
    SAIT_CUDA(cudaMemcpyAsync(cursor, segstart, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    cap_gather<<<grid_for((m.nnz + kFlat - 1) / kFlat, 256), 256, 0, s>>>(m.nnz, n, m.rp, m.ci, m.v, bits, cursor,
                                                                          lrow, lval, lpos);
    SAIT_LAUNCHED();
    dfree(cursor, s);
    cap_rank<<<grid_for(int64_t{nflag} * 32, 256), 256, 0, s>>>(nflag, flagged, seglen, segstart, cap, lrow, lval,
                                                                 lpos, m.ci, rowdel, blkdel, ndel);
    SAIT_LAUNCHED();
    unsigned long long hd = 0;
    read_back(s, {{&hd, ndel, sizeof hd}});
    deleted = static_cast<int64_t>(hd);
    if (deleted > 0) {
      int32_t* ncnt = seglen;  // reused
      cap_row_counts<<<grid_for(n, 256), 256, 0, s>>>(n, m.rp, rowdel, ncnt);
      SAIT_LAUNCHED();
      DevCsr c;
      c.nrows = m.nrows;
      c.ncols = m.ncols;
      c.rp = dalloc<int32_t>(n + 1, s);
      c.nnz = scan_counts(ncnt, c.rp, n, s);
      c.ci = dalloc<int32_t>(c.nnz > 0 ? c.nnz : 1, s);
      c.v = dalloc<double>(c.nnz > 0 ? c.nnz : 1, s);
      int32_t* blkshift = dalloc<int32_t>(nblk + 1, s);
      scan_counts(blkdel, blkshift, nblk, s);
      cap_compact<<<static_cast<unsigned>(nblk), 256, 0, s>>>(m.nnz, m.ci, m.v, blkshift, out_scale, c.ci, c.v);
      SAIT_LAUNCHED();
      dfree(blkshift, s);
      free_csr(m, s);
      m = c;
      if (scaled) *scaled = out_scale != nullptr;
    }
    dfree(blkdel, s);
    dfree(lrow, s);
    dfree(lval, s);
    dfree(lpos, s);
    dfree(reinterpret_cast<int64_t*>(ndel), s);
  }
  dfree(cnt, s);
  dfree(seglen, s);
  dfree(segstart, s);
  dfree(flagged, s);
  dfree(reinterpret_cast<int32_t*>(bits), s);
  dfree(nflag_d, s);
  static const bool dbg = std::getenv("SAIT_DEBUG_CAP") != nullptr;
  if (dbg)
    std::fprintf(stderr, "cap_rowform: n %lld nnz %lld listed %lld deleted %lld\n", static_cast<long long>(n),
                 static_cast<long long>(m.nnz), static_cast<long long>(listed), static_cast<long long>(deleted));
  return deleted;
}

bool csr_stabilized(const DevCsr& prev, const DevCsr& cur, cudaStream_t s) {
  if (prev.nrows != cur.nrows || prev.nnz != cur.nnz) return false;
  if (cur.nrows == 0) return true;
  int* differs = dalloc<int>(1, s);
  SAIT_CUDA(cudaMemsetAsync(differs, 0, sizeof(int), s));
  stable_rows<<<grid_for(cur.nrows * 8, 256), 256, 0, s>>>(cur.nrows, prev.rp, prev.ci, prev.v, cur.rp, cur.ci,
                                                            cur.v, differs);
  SAIT_LAUNCHED();
  int h = 1;
  read_back(s, {{&h, differs, sizeof h}});
  dfree(differs, s);
  return h == 0;
}

}  // namespace sait
