// csr_ops.cu — device CSR plumbing: row-pointer scan, identity, transpose
// (csr.cpp:72-92), column scaling (kernels.cpp:236-246), copies.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace sait {

std::atomic<int64_t> g_launches{0};

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[kScanThreads / 32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = w;
  }
  __syncthreads();
  int64_t before = (wid > 0 ? warp_sums[wid - 1] : 0) + x - v;
  if (total) *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void scan_tile_sums(const int32_t* __restrict__ counts, int64_t n, int64_t* __restrict__ sums) {
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += counts[base + k];
  int64_t tot;
  block_exclusive_scan(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// Single block: exclusive scan of the tile sums in place; writes the grand total.
__global__ void scan_sums(int64_t* sums, int64_t ntiles, int64_t* total) {
  int64_t carry = 0;
  for (int64_t base = 0; base < ntiles; base += kScanThreads) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < ntiles ? sums[i] : 0;
    int64_t tot;
    int64_t ex = block_exclusive_scan(v, &tot);
    if (i < ntiles) sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_tiles(const int32_t* __restrict__ counts, int64_t n, const int64_t* __restrict__ sums,
                           int32_t* __restrict__ row_ptr, const int64_t* __restrict__ total) {
  int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  int32_t c[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    c[k] = base + k < n ? counts[base + k] : 0;
    s += c[k];
  }
  int64_t run = sums[blockIdx.x] + block_exclusive_scan(s, nullptr);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) row_ptr[base + k] = static_cast<int32_t>(run);
    run += c[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) row_ptr[n] = static_cast<int32_t>(*total);
}

__global__ void identity_kernel(int64_t n, int32_t* rp, int32_t* ci, double* v) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    rp[i] = static_cast<int32_t>(i);
    ci[i] = static_cast<int32_t>(i);
    v[i] = 1.0;
  }
  if (i == 0) rp[n] = static_cast<int32_t>(n);
}

__global__ void identity_rows_kernel(int64_t rows, int64_t col0, int32_t* rp, int32_t* ci, double* v) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < rows) {
    rp[i] = static_cast<int32_t>(i);
    ci[i] = static_cast<int32_t>(col0 + i);
    v[i] = 1.0;
  }
  if (i == 0) rp[rows] = static_cast<int32_t>(rows);
}

__global__ void count_cols(int64_t nrows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           int32_t* __restrict__ cnt) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) atomicAdd(&cnt[ci[e]], 1);
}

// Scatter entry (i, j, v) of A to row j of A^T at an atomically claimed slot;
// rows of the result are sorted afterwards.  Scaled value = v * scale[i]
// (scale_columns order, kernels.cpp:243).
// L lanes per source row: with long rows (>= 12 entries on average) 8 lanes
// keep independent claims in flight (a thread walking its row serialised
// them); short stencil rows stay one thread per row (neighbouring rows hit
// neighbouring columns, and 8 lanes per row only add contention).
template <int L>
__global__ void scatter_transpose(int64_t nrows, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ v, const double* __restrict__ scale,
                                  int32_t* __restrict__ cursor, int32_t* __restrict__ oci, double* __restrict__ ov) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  if (i >= nrows) return;
  const int lane = threadIdx.x & (L - 1);
  const double s = scale ? scale[i] : 1.0;
  for (int32_t e = rp[i] + lane; e < rp[i + 1]; e += L) {
    const int32_t pos = atomicAdd(&cursor[ci[e]], 1);
    SAIT_DCHECK(pos >= 0 && pos < rp[nrows], "transpose scatter position", pos, rp[nrows]);
    oci[pos] = static_cast<int32_t>(i);
    if (v) ov[pos] = scale ? __dmul_rn(v[e], s) : v[e];
  }
}

// Rows of <= G*K entries: G lanes per row (32/G rows per warp), K keys per
// lane (entries b + t*G + lane, coalesced), rank by counting smaller keys
// (keys within a row are distinct); longer rows are listed for the next
// sorter with one atomic per warp (a per-row atomic on one counter had
// serialised millions of rows).  (G, K) = (8, 2) for stencil-like rows,
// (16, 2) when rows average >= 12 entries.
template <int G, int K>
__global__ void sort_rows_warp(int64_t nrows, const int32_t* __restrict__ rp, int32_t* __restrict__ ci,
                               double* __restrict__ v, int32_t* __restrict__ long_rows, int32_t* __restrict__ nlong) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const int lane = threadIdx.x & (G - 1), wl = threadIdx.x & 31;
  const bool live = row < nrows;
  int32_t b = 0, len = 0;
  if (live) {
    b = rp[row];
    len = rp[row + 1] - b;
  }
  const bool lng = live && len > G * K && lane == 0;
  const unsigned lb = __ballot_sync(0xffffffffu, lng);
  if (lb) {
    int32_t base = 0;
    if (wl == 0) base = atomicAdd(nlong, __popc(lb));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lng) long_rows[base + __popc(lb & ((1u << wl) - 1u))] = static_cast<int32_t>(row);
  }
  const bool sortme = live && len > 1 && len <= G * K;
  int32_t key[K];
  double val[K];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    const int e = t * G + lane;
    const bool mine = sortme && e < len;
    key[t] = mine ? ci[b + e] : kKeyPad;
    val[t] = (mine && v) ? v[b + e] : 0.0;
  }
  int rank[K] = {};
#pragma unroll
  for (int o = 0; o < G; ++o)
#pragma unroll
    for (int t2 = 0; t2 < K; ++t2) {
      const int32_t other = __shfl_sync(0xffffffffu, key[t2], o, G);
#pragma unroll
      for (int t = 0; t < K; ++t) rank[t] += other < key[t];
    }
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (sortme && t * G + lane < len) {
      ci[b + rank[t]] = key[t];
      if (v) v[b + rank[t]] = val[t];
    }
}

// Rows listed by sort_rows_warp<8, 2> with 16 < len <= 32.  A warp takes two listed
// rows: both <= 16 entries (the common case for SAIT factors) -> one half-warp
// each; otherwise one after the other with the whole warp.  Rank by counting
// smaller keys (keys within a row are distinct).
__device__ __forceinline__ void rank_place(int32_t b, int32_t len, int lane, int width, int32_t* __restrict__ ci,
                                           double* __restrict__ v) {
  const bool mine = lane < len;
  const int32_t key = mine ? ci[b + lane] : kKeyPad;
  const double val = (mine && v) ? v[b + lane] : 0.0;
  int rank = 0;
  for (int o = 0; o < width; ++o) rank += __shfl_sync(0xffffffffu, key, o, width) < key;
  __syncwarp();
  if (mine) {
    ci[b + rank] = key;
    if (v) v[b + rank] = val;
  }
}

__global__ void sort_rows_mid(const int32_t* __restrict__ rows, int32_t nlist, const int32_t* __restrict__ rp,
                              int32_t* __restrict__ ci, double* __restrict__ v, int32_t* __restrict__ long_rows,
                              int32_t* __restrict__ nlong) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t r0 = 2 * w;
  if (r0 >= nlist) return;
  const int half = lane >> 4;
  const bool has = r0 + half < nlist;
  int32_t row = 0, b = 0, len = 0;
  if (has) {
    row = rows[r0 + half];
    b = rp[row];
    len = rp[row + 1] - b;
  }
  if (has && len > 32 && (lane & 15) == 0) long_rows[atomicAdd(nlong, 1)] = row;
  if (len > 32) len = 0;  // left to the block sorter
  const int32_t l0 = __shfl_sync(0xffffffffu, len, 0), l1 = __shfl_sync(0xffffffffu, len, 16);
  if (l0 <= 16 && l1 <= 16) {
    rank_place(b, len, lane & 15, 16, ci, v);
    return;
  }
  for (int h = 0; h < 2; ++h) {
    const int32_t bh = __shfl_sync(0xffffffffu, b, 16 * h), lh = h ? l1 : l0;
    if (lh > 1) rank_place(bh, lh, lane, 32, ci, v);
  }
}

constexpr int kSortBlock = 256;
constexpr int kSortSmem = 2048;  // entries sorted in shared memory per block

__global__ void sort_rows_block(const int32_t* __restrict__ rows, int32_t nrows_list, const int32_t* __restrict__ rp,
                                int32_t* __restrict__ ci, double* __restrict__ v, int32_t* __restrict__ huge_rows,
                                int32_t* __restrict__ nhuge) {
  __shared__ int32_t sk[kSortSmem];
  __shared__ double sv[kSortSmem];
  for (int32_t r = blockIdx.x; r < nrows_list; r += gridDim.x) {
    int32_t row = rows[r];
    int32_t b = rp[row], len = rp[row + 1] - b;
    if (len > kSortSmem) {
      if (threadIdx.x == 0) huge_rows[atomicAdd(nhuge, 1)] = row;
      continue;
    }
    int n2 = next_pow2(len);
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
      sk[i] = i < len ? ci[b + i] : kKeyPad;
      sv[i] = (i < len && v) ? v[b + i] : 0.0;
    }
    __syncthreads();
    bitonic_sort(sk, sv, n2, threadIdx.x, blockDim.x, BlockSync{});
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      ci[b + i] = sk[i];
      if (v) v[b + i] = sv[i];
    }
    __syncthreads();
  }
}

// One very long row at a time, sorted in a padded global scratch.
__global__ void sort_row_global(int32_t row, const int32_t* __restrict__ rp, int32_t* __restrict__ ci,
                                double* __restrict__ v, int32_t* __restrict__ sk, double* __restrict__ sv) {
  int32_t b = rp[row], len = rp[row + 1] - b;
  int n2 = next_pow2(len);
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    sk[i] = i < len ? ci[b + i] : kKeyPad;
    sv[i] = (i < len && v) ? v[b + i] : 0.0;
  }
  __syncthreads();
  bitonic_sort(sk, sv, n2, threadIdx.x, blockDim.x, BlockSync{});
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    ci[b + i] = sk[i];
    if (v) v[b + i] = sv[i];
  }
}

__global__ void scale_rows_kernel(int64_t nrows, const int32_t* __restrict__ rp, double* __restrict__ v,
                                  const double* __restrict__ d) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const double di = d[i];
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e) v[e] = __dmul_rn(v[e], di);
}

__global__ void scale_cols_kernel(int64_t nnz, const int32_t* __restrict__ ci, const double* __restrict__ v,
                                  const double* __restrict__ d, double* __restrict__ out) {
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < nnz) out[e] = __dmul_rn(v[e], d[ci[e]]);
}

}  // namespace

// row_ptr = exclusive scan of counts, the total also written to *total_dev
// (device); no host synchronisation.
void scan_counts_async(const int32_t* counts, int32_t* row_ptr, int64_t n, int64_t* total_dev, cudaStream_t s) {
  int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles < 1) ntiles = 1;
  int64_t* sums = dalloc<int64_t>(ntiles, s);
  scan_tile_sums<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(counts, n, sums);
  SAIT_LAUNCHED();
  scan_sums<<<1, kScanThreads, 0, s>>>(sums, ntiles, total_dev);
  SAIT_LAUNCHED();
  scan_tiles<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(counts, n, sums, row_ptr, total_dev);
  SAIT_LAUNCHED();
  dfree(sums, s);
}

int64_t scan_counts(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s) {
  int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles < 1) ntiles = 1;
  int64_t* sums = dalloc<int64_t>(ntiles + 1, s);
  int64_t* total = sums + ntiles;
  scan_tile_sums<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(counts, n, sums);
  SAIT_LAUNCHED();
  scan_sums<<<1, kScanThreads, 0, s>>>(sums, ntiles, total);
  SAIT_LAUNCHED();
  scan_tiles<<<static_cast<unsigned>(ntiles), kScanThreads, 0, s>>>(counts, n, sums, row_ptr, total);
  SAIT_LAUNCHED();
  int64_t h = 0;
  read_back(s, {{&h, total, sizeof h}});
  dfree(sums, s);
  if (h > INT32_MAX)
    throw Error(SAIT_ERR_NOMEM, "result has " + std::to_string(h) +
                                    " stored entries; the device CSR uses int32 indices (max 2^31-1)");
  return h;
}

void exclusive_scan_rows(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s) {
  scan_counts(counts, row_ptr, n, s);
}

int64_t read_last(const int32_t* row_ptr, int64_t n, cudaStream_t s) {
  int32_t h = 0;
  read_back(s, {{&h, row_ptr + n, sizeof h}});
  return h;
}

DevCsr make_identity(int64_t n, cudaStream_t s) {
  DevCsr m;
  m.nrows = m.ncols = m.nnz = n;
  m.rp = dalloc<int32_t>(n + 1, s);
  m.ci = dalloc<int32_t>(n, s);
  m.v = dalloc<double>(n, s);
  identity_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(n, m.rp, m.ci, m.v);
  SAIT_LAUNCHED();
  return m;
}

DevCsr make_identity_rows(int64_t rows, int64_t col0, int64_t ncols, cudaStream_t s) {
  DevCsr m;
  m.nrows = rows;
  m.ncols = ncols;
  m.nnz = rows;
  m.rp = dalloc<int32_t>(rows + 1, s);
  m.ci = dalloc<int32_t>(rows, s);
  m.v = dalloc<double>(rows, s);
  identity_rows_kernel<<<grid_for(rows + 1, 256), 256, 0, s>>>(rows, col0, m.rp, m.ci, m.v);
  SAIT_LAUNCHED();
  return m;
}

// Sort every row of (rp, ci, v) by column index.
void sort_rows(int64_t nrows, const int32_t* rp, int32_t* ci, double* v, cudaStream_t s, int64_t nnz) {
  if (nrows == 0) return;
  int32_t* lists = dalloc<int32_t>(3 * nrows + 3, s);
  int32_t* mid_rows = lists + 2 * nrows;
  int32_t* long_rows = lists;
  int32_t* huge_rows = lists + nrows;
  int32_t* counters = lists + 3 * nrows;  // [nlong, nhuge, nmid]
  SAIT_CUDA(cudaMemsetAsync(counters, 0, 3 * sizeof(int32_t), s));
  const bool wide = nnz >= 12 * nrows;
  if (wide)  // rows > 32 go straight to the block sorter
    sort_rows_warp<16, 2><<<grid_for(nrows * 16, 256), 256, 0, s>>>(nrows, rp, ci, v, long_rows, counters);
  else
    sort_rows_warp<8, 2><<<grid_for(nrows * 8, 256), 256, 0, s>>>(nrows, rp, ci, v, mid_rows, counters + 2);
  SAIT_LAUNCHED();
  int32_t hc[3];
  read_back(s, {{hc, counters, sizeof hc}});
  if (!wide && hc[2] > 0) {
    sort_rows_mid<<<grid_for(int64_t{hc[2]} * 16, 256), 256, 0, s>>>(mid_rows, hc[2], rp, ci, v, long_rows, counters);
    SAIT_LAUNCHED();
    read_back(s, {{hc, counters, sizeof hc}});
  }
  if (hc[0] > 0) {
    unsigned g = static_cast<unsigned>(std::min<int64_t>(hc[0], 4 * num_sms()));
    sort_rows_block<<<g, kSortBlock, 0, s>>>(long_rows, hc[0], rp, ci, v, huge_rows, counters + 1);
    SAIT_LAUNCHED();
    read_back(s, {{hc, counters, sizeof hc}});
    if (hc[1] > 0) {
      std::vector<int32_t> huge(hc[1]);
      SAIT_CUDA(cudaMemcpyAsync(huge.data(), huge_rows, hc[1] * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      std::vector<int32_t> hrp(nrows + 1);
      SAIT_CUDA(cudaMemcpyAsync(hrp.data(), rp, (nrows + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      SAIT_CUDA(cudaStreamSynchronize(s));
      int maxlen = 0;
      for (int32_t r : huge) maxlen = std::max(maxlen, hrp[r + 1] - hrp[r]);
      int n2 = next_pow2(maxlen);
      int32_t* sk = dalloc<int32_t>(n2, s);
      double* sv = dalloc<double>(n2, s);
      for (int32_t r : huge) {
        sort_row_global<<<1, 1024, 0, s>>>(r, rp, ci, v, sk, sv);
        SAIT_LAUNCHED();
      }
      dfree(sk, s);
      dfree(sv, s);
    }
  }
  dfree(lists, s);
}

DevCsr transpose(const DevCsr& a, const double* row_scale, cudaStream_t s) {
  DevCsr t;
  t.nrows = a.ncols;
  t.ncols = a.nrows;
  t.nnz = a.nnz;
  t.rp = dalloc<int32_t>(t.nrows + 1, s);
  t.ci = dalloc<int32_t>(t.nnz, s);
  t.v = a.v ? dalloc<double>(t.nnz, s) : nullptr;
  int32_t* cnt = dalloc<int32_t>(t.nrows + 1, s);
  SAIT_CUDA(cudaMemsetAsync(cnt, 0, (t.nrows + 1) * sizeof(int32_t), s));
  if (a.nrows > 0) {
    count_cols<<<grid_for(a.nrows, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, cnt);
    SAIT_LAUNCHED();
  }
  scan_counts(cnt, t.rp, t.nrows, s);
  SAIT_CUDA(cudaMemcpyAsync(cnt, t.rp, t.nrows * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (a.nrows > 0) {
    if (a.nnz >= 12 * a.nrows)
      scatter_transpose<8><<<grid_for(a.nrows * 8, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, a.v, row_scale, cnt, t.ci, t.v);
    else
      scatter_transpose<1><<<grid_for(a.nrows, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, a.v, row_scale, cnt, t.ci, t.v);
    SAIT_LAUNCHED();
  }
  dfree(cnt, s);
  sort_rows(t.nrows, t.rp, t.ci, t.v, s, t.nnz);
  return t;
}

void scale_columns(const DevCsr& a, const double* d, DevCsr& out, cudaStream_t s) {
  if (a.nnz == 0) return;
  scale_cols_kernel<<<grid_for(a.nnz, 256), 256, 0, s>>>(a.nnz, a.ci, a.v, d, out.v);
  SAIT_LAUNCHED();
}

void scale_rows(DevCsr& a, const double* d, cudaStream_t s) {
  if (a.nrows == 0) return;
  scale_rows_kernel<<<grid_for(a.nrows, 256), 256, 0, s>>>(a.nrows, a.rp, a.v, d);
  SAIT_LAUNCHED();
}

DevCsr copy_csr(const DevCsr& a, cudaStream_t s) {
  DevCsr c = a;
  c.rp = dalloc<int32_t>(a.nrows + 1, s);
  c.ci = dalloc<int32_t>(a.nnz, s);
  c.v = a.v ? dalloc<double>(a.nnz, s) : nullptr;
  SAIT_CUDA(cudaMemcpyAsync(c.rp, a.rp, (a.nrows + 1) * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (a.nnz) {
    SAIT_CUDA(cudaMemcpyAsync(c.ci, a.ci, a.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    if (a.v) SAIT_CUDA(cudaMemcpyAsync(c.v, a.v, a.nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  return c;
}

}  // namespace sait

// ---------------------------------------------------------------------------
// Column-block -> row-block redistribution (multi-GPU, SURVEY.md §8e "K4"):
// the distributed form of csr.cpp:72-92.  Each rank's column-sharded build
// yields M[:, C_r:C_{r+1}] (all n rows); rank q receives, from every rank r in
// ascending r, the rows [R_q, R_{q+1}) of that block and assembles its row
// block of M.  Column blocks are disjoint and ascending in r, so row i of the
// result is the concatenation of the pieces' rows i in part order (columns
// shifted by the part's col_offset): sorted, bitwise the global matrix's row.
namespace sait {
namespace {

__global__ void assemble_count(int64_t nrows, int nparts, const sait_row_piece* __restrict__ parts,
                               int32_t* __restrict__ len) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int32_t c = 0;
  for (int p = 0; p < nparts; ++p) c += parts[p].row_ptr[i + 1] - parts[p].row_ptr[i];
  len[i] = c;
}

// 8 lanes per row (rows hold ~7-30 entries), parts in order
__global__ void assemble_copy(int64_t nrows, int nparts, const sait_row_piece* __restrict__ parts,
                              const int32_t* __restrict__ rp, int32_t* __restrict__ ci, double* __restrict__ v) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = t >> 3;
  const int lane = static_cast<int>(t & 7);
  if (i >= nrows) return;
  int32_t o = rp[i];
  for (int p = 0; p < nparts; ++p) {
    const sait_row_piece q = parts[p];
    const int32_t b = q.row_ptr[i] - q.row_ptr[0], e = q.row_ptr[i + 1] - q.row_ptr[0];
    const int32_t off = static_cast<int32_t>(q.col_offset);
    for (int32_t k = b + lane; k < e; k += 8) {
      ci[o + (k - b)] = q.col_idx[k] + off;
      if (v) v[o + (k - b)] = q.values[k];
    }
    o += e - b;
  }
  SAIT_DCHECK(o == rp[i + 1], "assembled row length", o, rp[i + 1]);
}

__global__ void col_minmax(int64_t nnz, const int32_t* __restrict__ ci, int* __restrict__ mm) {
  int lo = INT32_MAX, hi = -1;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    lo = min(lo, ci[e]);
    hi = max(hi, ci[e]);
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void shift_cols(int64_t nnz, int32_t* __restrict__ ci, int32_t off) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < nnz) ci[e] += off;
}

__global__ void read_row_ptr(const int32_t* __restrict__ rp, int k, const int64_t* __restrict__ rows,
                             int64_t* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < k) out[j] = rp[rows[j]];
}

// Column-form work of column j of M at step 2 (the first step with products):
// sum over the entries (k, j) of tT of the number of entries of column k --
// the products the column's recursion forms.  Lower and upper T alike.
__global__ void column_counts(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              int64_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
    if (ci[e] != i) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + ci[e]), 1ull);
}
__global__ void column_work(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int64_t* __restrict__ cnt, int64_t* __restrict__ work) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
    if (ci[e] != i) atomicAdd(reinterpret_cast<unsigned long long*>(work + ci[e]),
                              static_cast<unsigned long long>(cnt[i] + 1));
}

}  // namespace

DevCsr assemble_rows(int nparts, const sait_row_piece* parts_host, int64_t nrows, int64_t ncols, cudaStream_t s) {
  DevCsr c;
  c.nrows = nrows;
  c.ncols = ncols;
  bool values = true;
  for (int p = 0; p < nparts; ++p) values = values && parts_host[p].values != nullptr;
  sait_row_piece* parts = dalloc<sait_row_piece>(nparts > 0 ? nparts : 1, s);
  if (nparts)
    SAIT_CUDA(cudaMemcpyAsync(parts, parts_host, sizeof(sait_row_piece) * nparts, cudaMemcpyHostToDevice, s));
  c.rp = dalloc<int32_t>(nrows + 1, s);
  int32_t* len = dalloc<int32_t>(nrows > 0 ? nrows : 1, s);
  if (nrows > 0) {
    assemble_count<<<grid_for(nrows, 256), 256, 0, s>>>(nrows, nparts, parts, len);
    SAIT_LAUNCHED();
  }
  c.nnz = scan_counts(len, c.rp, nrows, s);
  dfree(len, s);
  c.ci = dalloc<int32_t>(c.nnz > 0 ? c.nnz : 1, s);
  c.v = values ? dalloc<double>(c.nnz > 0 ? c.nnz : 1, s) : nullptr;
  if (nrows > 0) {
    assemble_copy<<<grid_for(nrows * 8, 256), 256, 0, s>>>(nrows, nparts, parts, c.rp, c.ci, c.v);
    SAIT_LAUNCHED();
  }
  dfree(parts, s);
  SAIT_CUDA(cudaStreamSynchronize(s));  // parts_host may be a caller temporary
  return c;
}

void col_span(const DevCsr& a, int64_t* lo, int64_t* hi, cudaStream_t s) {
  int* mm = dalloc<int>(2, s);
  const int init[2] = {INT32_MAX, -1};
  SAIT_CUDA(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s));
  if (a.nnz > 0) {
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(grid_for(a.nnz, 256), int64_t{num_sms()} * 8));
    col_minmax<<<grid, 256, 0, s>>>(a.nnz, a.ci, mm);
    SAIT_LAUNCHED();
  }
  int h[2];
  SAIT_CUDA(cudaMemcpyAsync(h, mm, sizeof h, cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  dfree(mm, s);
  *lo = h[1] < 0 ? 0 : h[0];
  *hi = h[1] < 0 ? 0 : int64_t{h[1]} + 1;
}

void shift_columns(DevCsr& a, int64_t off, int64_t ncols, cudaStream_t s) {
  if (a.nnz > 0 && off != 0) {
    shift_cols<<<grid_for(a.nnz, 256), 256, 0, s>>>(a.nnz, a.ci, static_cast<int32_t>(off));
    SAIT_LAUNCHED();
  }
  a.ncols = ncols;
}

void row_ptr_at(const DevCsr& a, const int64_t* rows_host, int k, int64_t* out_host, cudaStream_t s) {
  int64_t* d = dalloc<int64_t>(2 * (k > 0 ? k : 1), s);
  if (k > 0) {
    SAIT_CUDA(cudaMemcpyAsync(d, rows_host, sizeof(int64_t) * k, cudaMemcpyHostToDevice, s));
    read_row_ptr<<<grid_for(k, 128), 128, 0, s>>>(a.rp, k, d, d + k);
    SAIT_LAUNCHED();
    SAIT_CUDA(cudaMemcpyAsync(out_host, d + k, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
  }
  SAIT_CUDA(cudaStreamSynchronize(s));
  dfree(d, s);
}

void column_work_of(const DevCsr& t, int64_t* work, cudaStream_t s) {
  const int64_t n = t.nrows;
  int64_t* cnt = dalloc<int64_t>(n > 0 ? n : 1, s);
  SAIT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * n, s));
  SAIT_CUDA(cudaMemsetAsync(work, 0, sizeof(int64_t) * n, s));
  if (n > 0) {
    column_counts<<<grid_for(n, 256), 256, 0, s>>>(n, t.rp, t.ci, cnt);
    SAIT_LAUNCHED();
    column_work<<<grid_for(n, 256), 256, 0, s>>>(n, t.rp, t.ci, cnt, work);
    SAIT_LAUNCHED();
  }
  dfree(cnt, s);
}

}  // namespace sait
