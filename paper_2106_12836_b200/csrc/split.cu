// split.cu — K1: Jacobi splitting of a triangular T (sait.cpp:32-73).
//   inv_diag[i] = 1.0 / T[i,i]          (IEEE division, sait.cpp:63)
//   tT[i,j]     = (-T[i,j]) * inv_diag[i] for j != i (sait.cpp:64-69)
// Validation keeps the reference's precedence: non-square, then any entry
// outside the triangle (check_triangular, csr.cpp:124-139, first in row-major
// order), then the first row with a missing/zero diagonal (sait.cpp:59-62).
#include "common.cuh"

namespace sait {
namespace {

struct SplitErrors {
  unsigned long long tri;   // (row << 32) | local entry index, min over offenders
  unsigned long long diag;  // first singular row
};

__global__ void split_validate(int64_t n, bool lower, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const double* __restrict__ v,
                               SplitErrors* err) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t b = rp[i], e1 = rp[i + 1];
  bool have = false;
  double d = 0.0;
  for (int32_t e = b; e < e1; ++e) {
    int32_t j = ci[e];
    bool off = lower ? (j > i) : (j < i);
    if (off) {
      atomicMin(&err->tri, (static_cast<unsigned long long>(i) << 32) | static_cast<unsigned>(e - b));
      break;
    }
    if (j == i && !have) {
      have = true;
      d = v[e];
    }
  }
  if (!have || d == 0.0) atomicMin(&err->diag, static_cast<unsigned long long>(i));
}

// L lanes per row: 8 for long rows (coalesced reads and writes; a thread per
// row walked them with strided accesses), 1 for short stencil rows.  Every
// row holds exactly one diagonal (validated); entries after it shift down by
// one.
template <int kSplitLanes>
__global__ void split_write(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, double* __restrict__ inv_diag,
                            int32_t* __restrict__ trp, int32_t* __restrict__ tci, double* __restrict__ tv) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kSplitLanes;
  const int lane = threadIdx.x & (kSplitLanes - 1);
  const int base = (threadIdx.x & 31) & ~(kSplitLanes - 1);
  int32_t b = 0, e1 = 0;
  if (i <= n) {
    b = rp[i];
    if (lane == 0) trp[i] = b - static_cast<int32_t>(i);
    if (i < n) e1 = rp[i + 1];
  }
  double dl = 0.0;
  int32_t el = -1;
  for (int32_t e = b + lane; e < e1; e += kSplitLanes)
    if (ci[e] == i) {
      dl = v[e];
      el = e;
    }
  const unsigned found = (__ballot_sync(0xffffffffu, el >= 0) >> base) & ((1u << kSplitLanes) - 1u);
  const int src = base + (found ? __ffs(found) - 1 : 0);
  const double d = __shfl_sync(0xffffffffu, dl, src);
  const int32_t ed = __shfl_sync(0xffffffffu, el, src);
  if (i >= n) return;
  const double inv = 1.0 / d;
  if (lane == 0) inv_diag[i] = inv;
  const int32_t shift = static_cast<int32_t>(i);
  for (int32_t e = b + lane; e < e1; e += kSplitLanes) {
    if (e == ed) continue;
    const int32_t pos = e - shift - (e > ed ? 1 : 0);
    tci[pos] = ci[e];
    tv[pos] = __dmul_rn(-v[e], inv);
  }
}

}  // namespace

DevCsr jacobi_split(const DevCsr& t, bool lower, double* inv_diag, cudaStream_t s) {
  if (t.nrows != t.ncols) throw_invalid("jacobi_split: matrix is not square");
  int64_t n = t.nrows;
  SplitErrors h{~0ull, ~0ull};
  SplitErrors* d = dalloc<SplitErrors>(1, s);
  SAIT_CUDA(cudaMemsetAsync(d, 0xff, sizeof h, s));  // both fields ~0
  if (n > 0) {
    split_validate<<<grid_for(n, 256), 256, 0, s>>>(n, lower, t.rp, t.ci, t.v, d);
    SAIT_LAUNCHED();
  }
  read_back(s, {{&h, d, sizeof h}});
  dfree(d, s);
  if (h.tri != ~0ull) {
    int64_t row = static_cast<int64_t>(h.tri >> 32);
    int32_t local = static_cast<int32_t>(h.tri & 0xffffffffu), b = 0, col = 0;
    SAIT_CUDA(cudaMemcpyAsync(&b, t.rp + row, sizeof b, cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    SAIT_CUDA(cudaMemcpyAsync(&col, t.ci + b + local, sizeof col, cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    throw_invalid("check_triangular: entry (" + std::to_string(row) + ", " + std::to_string(col) +
                  ") outside stated triangle");
  }
  if (h.diag != ~0ull)
    throw_runtime("jacobi_split: singular matrix, zero diagonal at row " + std::to_string(h.diag));
  DevCsr tt;
  tt.nrows = tt.ncols = n;
  tt.nnz = t.nnz - n;
  tt.rp = dalloc<int32_t>(n + 1, s);
  tt.ci = dalloc<int32_t>(tt.nnz, s);
  tt.v = dalloc<double>(tt.nnz, s);
  if (t.nnz >= 12 * n)
    split_write<8><<<grid_for((n + 1) * 8, 256), 256, 0, s>>>(n, t.rp, t.ci, t.v, inv_diag, tt.rp, tt.ci, tt.v);
  else
    split_write<1><<<grid_for(n + 1, 256), 256, 0, s>>>(n, t.rp, t.ci, t.v, inv_diag, tt.rp, tt.ci, tt.v);
  SAIT_LAUNCHED();
  return tt;
}

}  // namespace sait
