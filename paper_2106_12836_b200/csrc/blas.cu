// blas.cu — K7: BLAS-1 / tall-skinny kernels of the device solver loops.
//
// Reductions use ONE canonical order (shared with oracle/solvers.c): blocks of
// 2048 elements; thread t of a 256-thread block sums x[i]*y[i] for
// i = 2048 b + t + 256 k, k = 0..7, sequentially from 0.0; the 256 sums are
// folded by a 32-lane xor butterfly (offsets 16..1) per warp and an 8-way
// butterfly (4,2,1) across warps; block partials are folded the same way by
// one block whose thread t first sums partials t, t+256, ... in order.  With
// every product rounded before its add, dots are bitwise reproducible and
// equal to the CPU restatement, so solver iteration counts match exactly.
#include "common.cuh"

namespace sait {
namespace {

constexpr int kT = 256, kK = 8, kB = kT * kK;
constexpr int kMaxM = 32;

__device__ __forceinline__ double warp_butterfly(double s) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
  return s;
}

// ((w0+w4)+(w2+w6)) + ((w1+w5)+(w3+w7)) : the 8-lane butterfly at lane 0
__device__ __forceinline__ double tree8(const double* w) {
  const double a0 = __dadd_rn(w[0], w[4]), a1 = __dadd_rn(w[1], w[5]);
  const double a2 = __dadd_rn(w[2], w[6]), a3 = __dadd_rn(w[3], w[7]);
  return __dadd_rn(__dadd_rn(a0, a2), __dadd_rn(a1, a3));
}

// part[j * nb + b] = canonical block partial of x . V_j
__global__ void __launch_bounds__(kT) mdot_partials(int64_t n, const double* __restrict__ x,
                                                     const double* __restrict__ V, int64_t ld, int m,
                                                     double* __restrict__ part, int64_t nb) {
  __shared__ double ws[kMaxM][8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kB + t;
  double xv[kK];
#pragma unroll
  for (int k = 0; k < kK; ++k) {
    const int64_t i = base + static_cast<int64_t>(kT) * k;
    xv[k] = i < n ? x[i] : 0.0;
  }
  for (int j = 0; j < m; ++j) {
    const double* v = V + ld * j;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const int64_t i = base + static_cast<int64_t>(kT) * k;
      if (i < n) s = __dadd_rn(s, __dmul_rn(xv[k], v[i]));
    }
    s = warp_butterfly(s);
    if (lane == 0) ws[j][warp] = s;
  }
  __syncthreads();
  if (t < m) part[static_cast<int64_t>(t) * nb + blockIdx.x] = tree8(ws[t]);
}

// out[j] = canonical fold of the nb partials of dot j (one block per j)
__global__ void __launch_bounds__(kT) mdot_final(const double* __restrict__ part, int64_t nb,
                                                  double* __restrict__ out, int sqrt_out) {
  __shared__ double ws[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* p = part + nb * blockIdx.x;
  double s = 0.0;
  for (int64_t q = t; q < nb; q += kT) s = __dadd_rn(s, p[q]);
  s = warp_butterfly(s);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (t == 0) {
    const double d = tree8(ws);
    out[blockIdx.x] = sqrt_out ? __dsqrt_rn(d) : d;
  }
}

// w[e] = (((w - h0 v0) - h1 v1) - ...)   (sequential in j)
__global__ void cgs_update(int64_t n, double* __restrict__ w, const double* __restrict__ V, int64_t ld, int m,
                           const double* __restrict__ h) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double t = w[e];
  for (int j = 0; j < m; ++j) t = __dsub_rn(t, __dmul_rn(h[j], V[ld * j + e]));
  w[e] = t;
}

// out = w / d[0]
__global__ void div_by(int64_t n, const double* __restrict__ w, const double* __restrict__ d, double* __restrict__ out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) out[e] = __ddiv_rn(w[e], d[0]);
}

// u = y0 v0 + y1 v1 + ...   (sequential in j, first term a product)
__global__ void lincomb(int64_t n, const double* __restrict__ V, int64_t ld, int k, const double* __restrict__ y,
                        double* __restrict__ u) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double t = __dmul_rn(y[0], V[e]);
  for (int j = 1; j < k; ++j) t = __dadd_rn(t, __dmul_rn(y[j], V[ld * j + e]));
  u[e] = t;
}

// y = y + a x  /  y = x + a y  /  y = x - y
__global__ void axpy_k(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __dadd_rn(y[e], __dmul_rn(a, x[e]));
}
__global__ void xpay_k(int64_t n, const double* __restrict__ x, double a, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __dadd_rn(x[e], __dmul_rn(a, y[e]));
}
__global__ void sub_k(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __dsub_rn(x[e], y[e]);
}
__global__ void add_k(int64_t n, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __dadd_rn(y[e], x[e]);
}

// out[:, j] = sum_q in[:, q] C[q][j]  (column-major blocks, C row-major kin x kout)
__global__ void block_lincomb_k(int64_t n, const double* __restrict__ in, int kin, const double* __restrict__ C,
                                int kout, double* __restrict__ out) {
  __shared__ double cs[48 * 16];
  for (int e = threadIdx.x; e < kin * kout; e += blockDim.x) cs[e] = C[e];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // each input element read once; output j accumulates q = 0, 1, ... in order
  double acc[16];
  const double x0 = in[i];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < kout) acc[j] = __dmul_rn(x0, cs[j]);
  for (int q = 1; q < kin; ++q) {
    const double xq = in[n * q + i];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < kout) acc[j] = __dadd_rn(acc[j], __dmul_rn(xq, cs[q * kout + j]));
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < kout) out[n * j + i] = acc[j];
}

// W[:, j] = (((W_j - X_0 G[0][j]) - X_1 G[1][j]) - ...)
__global__ void block_sub_lincomb_k(int64_t n, const double* __restrict__ X, int k, const double* __restrict__ G,
                                    double* __restrict__ W) {
  __shared__ double gs[16 * 16];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) gs[e] = G[e];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < k) w[j] = W[n * j + i];
  for (int q = 0; q < k; ++q) {
    const double xq = X[n * q + i];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < k) w[j] = __dsub_rn(w[j], __dmul_rn(xq, gs[q * k + j]));
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < k) W[n * j + i] = w[j];
}

// R[:, j] = AX[:, j] - lam[j] X[:, j]
__global__ void block_residual_k(int64_t n, int k, const double* __restrict__ AX, const double* __restrict__ X,
                                 const double* __restrict__ lam, double* __restrict__ R) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < k; ++j) R[n * j + i] = __dsub_rn(AX[n * j + i], __dmul_rn(lam[j], X[n * j + i]));
}

// Tall-skinny Gram tile: part[(a * kb + b) * nb + blk] = canonical block
// partial of A_a . B_b for a < ka <= 8, b < kb <= 8 (column-major blocks,
// leading dimension n).  Each thread keeps the 64 running sums of its 8
// strided elements in registers, so the tile's 16 columns are read once.
template <int TT>
__global__ void __launch_bounds__(kT) gram_tile_partials(int64_t n, const double* __restrict__ A, int ka,
                                                          const double* __restrict__ B, int kb,
                                                          double* __restrict__ part, int64_t nb) {
  __shared__ double ws[TT * TT][8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kB + t;
  double acc[TT][TT];
#pragma unroll
  for (int a = 0; a < TT; ++a)
#pragma unroll
    for (int b = 0; b < TT; ++b) acc[a][b] = 0.0;
#pragma unroll 2
  for (int k = 0; k < kK; ++k) {
    const int64_t i = base + static_cast<int64_t>(kT) * k;
    if (i < n) {
      double xa[TT], yb[TT];
#pragma unroll
      for (int a = 0; a < TT; ++a) xa[a] = a < ka ? A[n * a + i] : 0.0;
#pragma unroll
      for (int b = 0; b < TT; ++b) yb[b] = b < kb ? B[n * b + i] : 0.0;
#pragma unroll
      for (int a = 0; a < TT; ++a)
#pragma unroll
        for (int b = 0; b < TT; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(xa[a], yb[b]));
    }
  }
#pragma unroll
  for (int a = 0; a < TT; ++a)
#pragma unroll
    for (int b = 0; b < TT; ++b) {
      const double v = warp_butterfly(acc[a][b]);
      if (lane == 0) ws[a * TT + b][warp] = v;
    }
  __syncthreads();
  if (t < TT * TT) {
    const int a = t / TT, b = t % TT;
    if (a < ka && b < kb) part[static_cast<int64_t>(a * kb + b) * nb + blockIdx.x] = tree8(ws[t]);
  }
}

__global__ void hadamard_k(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dmul_rn(a[i], b[i]);
}
__global__ void add_into_k(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __dadd_rn(a[i], b[i]);
}

}  // namespace

void hadamard(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
  if (n <= 0) return;
  hadamard_k<<<grid_for(n, 256), 256, 0, s>>>(n, a, b, out);
  SAIT_LAUNCHED();
}
void add_into(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
  if (n <= 0) return;
  add_into_k<<<grid_for(n, 256), 256, 0, s>>>(n, a, b, out);
  SAIT_LAUNCHED();
}

void block_lincomb(int64_t n, const double* in, int kin, const double* C, int kout, double* out, cudaStream_t s) {
  block_lincomb_k<<<grid_for(n, 256), 256, 0, s>>>(n, in, kin, C, kout, out);
  SAIT_LAUNCHED();
}
void block_sub_lincomb(int64_t n, const double* X, int k, const double* G, double* W, cudaStream_t s) {
  block_sub_lincomb_k<<<grid_for(n, 256), 256, 0, s>>>(n, X, k, G, W);
  SAIT_LAUNCHED();
}
void block_residual(int64_t n, int k, const double* AX, const double* X, const double* lam, double* R,
                    cudaStream_t s) {
  block_residual_k<<<grid_for(n, 256), 256, 0, s>>>(n, k, AX, X, lam, R);
  SAIT_LAUNCHED();
}

int64_t dot_blocks(int64_t n) { return n > 0 ? (n + kB - 1) / kB : 1; }

// G[a * ldg + b] (device, a < ka, b < kb) = canonical dot of A_a and B_b,
// computed tile by tile (8 x 8); identical bits to multi_dot per entry.
void gram(int64_t n, const double* A, int ka, const double* B, int kb, double* G, int ldg, double* scratch,
          cudaStream_t s, bool upper_only) {
  const int64_t nb = dot_blocks(n);
  constexpr int TT = 8;
  for (int a0 = 0; a0 < ka; a0 += TT)
    for (int b0 = 0; b0 < kb; b0 += TT) {
      if (upper_only && b0 + TT <= a0) continue;
      const int ta = ka - a0 < TT ? ka - a0 : TT, tb = kb - b0 < TT ? kb - b0 : TT;
      gram_tile_partials<TT><<<static_cast<unsigned>(nb), kT, 0, s>>>(n, A + n * a0, ta, B + n * b0, tb, scratch, nb);
      SAIT_LAUNCHED();
      for (int a = 0; a < ta; ++a) {  // one final fold per tile row: tb blocks
        mdot_final<<<tb, kT, 0, s>>>(scratch + static_cast<int64_t>(a * tb) * nb, nb, G + (a0 + a) * ldg + b0, 0);
        SAIT_LAUNCHED();
      }
    }
}

void multi_dot(int64_t n, const double* x, const double* V, int64_t ld, int m, double* out, double* scratch,
               cudaStream_t s, bool sqrt_out) {
  const int64_t nb = dot_blocks(n);
  for (int j0 = 0; j0 < m; j0 += kMaxM) {
    const int mm = m - j0 < kMaxM ? m - j0 : kMaxM;
    mdot_partials<<<static_cast<unsigned>(nb), kT, 0, s>>>(n, x, V + ld * j0, ld, mm, scratch, nb);
    SAIT_LAUNCHED();
    mdot_final<<<mm, kT, 0, s>>>(scratch, nb, out + j0, sqrt_out ? 1 : 0);
    SAIT_LAUNCHED();
  }
}

void cgs_subtract(int64_t n, double* w, const double* V, int64_t ld, int m, const double* h, cudaStream_t s) {
  cgs_update<<<grid_for(n, 256), 256, 0, s>>>(n, w, V, ld, m, h);
  SAIT_LAUNCHED();
}
void divide_by(int64_t n, const double* w, const double* d, double* out, cudaStream_t s) {
  div_by<<<grid_for(n, 256), 256, 0, s>>>(n, w, d, out);
  SAIT_LAUNCHED();
}
void linear_combination(int64_t n, const double* V, int64_t ld, int k, const double* y, double* u, cudaStream_t s) {
  lincomb<<<grid_for(n, 256), 256, 0, s>>>(n, V, ld, k, y, u);
  SAIT_LAUNCHED();
}
void axpy(int64_t n, double a, const double* x, double* y, cudaStream_t s) {
  axpy_k<<<grid_for(n, 256), 256, 0, s>>>(n, a, x, y);
  SAIT_LAUNCHED();
}
void xpay(int64_t n, const double* x, double a, double* y, cudaStream_t s) {
  xpay_k<<<grid_for(n, 256), 256, 0, s>>>(n, x, a, y);
  SAIT_LAUNCHED();
}
void x_minus_y(int64_t n, const double* x, double* y, cudaStream_t s) {
  sub_k<<<grid_for(n, 256), 256, 0, s>>>(n, x, y);
  SAIT_LAUNCHED();
}
void y_plus_x(int64_t n, const double* x, double* y, cudaStream_t s) {
  add_k<<<grid_for(n, 256), 256, 0, s>>>(n, x, y);
  SAIT_LAUNCHED();
}

}  // namespace sait
