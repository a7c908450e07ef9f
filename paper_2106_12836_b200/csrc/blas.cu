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
#include <cstdlib>
#include <cstring>

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

__device__ __forceinline__ double ld_ro(const double* p) {
  double r;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// 32 values per lane, reduced across the warp by a reduce-scatter butterfly:
// at offset o each lane keeps the half of its values selected by lane bit o
// and adds the partner's partial of the same value (own + partner, offsets
// 16..1), so every value gets exactly the canonical warp_butterfly sums
// (bitwise), with 31 shuffles instead of 5 per value; value j ends on lane j.
__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < o; ++q) {
      const double keep = hi ? v[q + o] : v[q];
      const double send = hi ? v[q] : v[q + o];
      v[q] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  return v[0];
}

// part[j * nb + b] = canonical block partial of x . V_j (WIDE: m > 4, all
// partials first and one reduce-scatter; else one butterfly per dot)
template <bool WIDE>
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
  if constexpr (!WIDE) {
    for (int j = 0; j < m; ++j) {
      const double* v = V + ld * j;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        const int64_t i = base + static_cast<int64_t>(kT) * k;
        if (i < n) s = __fma_rn(xv[k], v[i], s);
      }
      s = warp_butterfly(s);
      if (lane == 0) ws[j][warp] = s;
    }
  } else {  // up to 32 dots: all partials first, then one reduce-scatter
    double acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      double s = 0.0;
      if (j < m) {
        const double* v = V + ld * j;
#pragma unroll
        for (int k = 0; k < kK; ++k) {
          const int64_t i = base + static_cast<int64_t>(kT) * k;
          if (i < n) s = __fma_rn(xv[k], v[i], s);
        }
      }
      acc[j] = s;
    }
    ws[lane][warp] = warp_reduce_scatter32(acc, lane);
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
  for (int j = 0; j < m; ++j) t = __fma_rn(-h[j], V[ld * j + e], t);
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
  for (int j = 1; j < k; ++j) t = __fma_rn(y[j], V[ld * j + e], t);
  u[e] = t;
}

// y = y + a x  /  y = x + a y  /  y = x - y
__global__ void axpy_k(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __fma_rn(a, x[e], y[e]);
}
__global__ void xpay_k(int64_t n, const double* __restrict__ x, double a, double* __restrict__ y) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) y[e] = __fma_rn(a, y[e], x[e]);
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
// in and out may overlap (LOBPCG updates its blocks in place): each thread
// reads every input of its element before it writes any output.
__global__ void block_lincomb_k(int64_t n, const double* in, int kin, const double* __restrict__ C, int kout,
                                double* out) {
  __shared__ double cs[48 * 16];
  for (int e = threadIdx.x; e < kin * kout; e += blockDim.x) cs[e] = C[e];
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // each input element read once; output j accumulates q = 0, 1, ... in order.
  // Inputs are fetched 8 at a time (all loads in flight before the
  // arithmetic that consumes them).
  double acc[16];
  const double x0 = in[i];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < kout) acc[j] = __dmul_rn(x0, cs[j]);
  for (int q0 = 1; q0 < kin; q0 += 8) {
    double xq[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xq[u] = q0 + u < kin ? ld_ro(in + n * (q0 + u) + i) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u >= kin) break;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < kout) acc[j] = __fma_rn(xq[u], cs[(q0 + u) * kout + j], acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < kout) out[n * j + i] = acc[j];
}

// The same with the coefficients passed by value as a kernel parameter
// (constant bank): fully unrolled, every FMA takes its coefficient as a
// direct constant operand -- no shared-memory load per product.
template <int KIN, int KOUT>
struct CoefBlock {
  double c[KIN * KOUT];
};
template <int KIN, int KOUT>
__global__ void __launch_bounds__(256) block_lincomb_param(int64_t n, const double* in, CoefBlock<KIN, KOUT> C,
                                                           double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xq[KIN];
#pragma unroll
  for (int q = 0; q < KIN; ++q) xq[q] = ld_ro(in + n * q + i);
  double acc[KOUT];
#pragma unroll
  for (int j = 0; j < KOUT; ++j) acc[j] = __dmul_rn(xq[0], C.c[j]);
#pragma unroll
  for (int q = 1; q < KIN; ++q)
#pragma unroll
    for (int j = 0; j < KOUT; ++j) acc[j] = __fma_rn(xq[q], C.c[q * KOUT + j], acc[j]);
#pragma unroll
  for (int j = 0; j < KOUT; ++j) out[n * j + i] = acc[j];
}

// LOBPCG's update step for block size 8, fused (m = 16 or 24 basis columns
// S = [X W P], AS = [AX AW AP], C = the m x 8 Ritz coefficients):
//   lobpcg_update_xp:     X <- S C,  P <- S[8:m] C[8:m]            (in place)
//   lobpcg_update_axp_r:  AX <- AS C, AP <- AS[8:m] C[8:m],
//                         R <- AX - X diag(lam)  (the next residual)
// Every output element is computed with exactly the operations of the
// separate kernels (block_lincomb_param: the first product rounded, then FMAs
// in input order; block_residual_k: fma(-lam, X, AX)), so the result is
// bitwise the unfused sequence; the fusion saves the re-reads of [W P],
// [AW AP], X and AX (5 of 17 block passes per iteration).
// Fast mode: the next residual's squared column norms as block partials
// (fixed order: each thread's two rows' r_j^2, the 32-lane butterfly, the
// 8-warp tree; part[j * gridDim.x + block]), folded by mdot_final --
// deterministic, and the residual block is not read again for its norms.
// sq == nullptr: a thread past the end contributes zeros.
__device__ __forceinline__ void lobpcg_norm_partials_sq(const double* sq, double* part) {
  __shared__ double ws2[8][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double w = warp_butterfly(sq ? sq[j] : 0.0);
    if (lane == 0) ws2[j][warp] = w;
  }
  __syncthreads();
  if (threadIdx.x < 8) part[static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x] = tree8(ws2[threadIdx.x]);
}

template <int M>
struct UpdateCoef {
  double c[M * 8];         // X <- S C
  double cp[(M - 8) * 8];  // P <- S[8:M] Cp (Cp = C[8:M], or C[8:M] Ri when P's Cholesky-QR is folded in)
  double lam[8];
};
// Two rows per thread (16-byte loads and stores: half the memory
// instructions of one row per thread, the same operations per element).
template <int M>
__device__ __forceinline__ void update_rows(const double2 (&xq)[M], const UpdateCoef<M>& C, double2 (&ax)[8],
                                            double2 (&ap)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    ax[j].x = __dmul_rn(xq[0].x, C.c[j]);
    ax[j].y = __dmul_rn(xq[0].y, C.c[j]);
    ap[j].x = __dmul_rn(xq[8].x, C.cp[j]);
    ap[j].y = __dmul_rn(xq[8].y, C.cp[j]);
  }
#pragma unroll
  for (int q = 1; q < M; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ax[j].x = __fma_rn(xq[q].x, C.c[q * 8 + j], ax[j].x);
      ax[j].y = __fma_rn(xq[q].y, C.c[q * 8 + j], ax[j].y);
      if (q > 8) {
        ap[j].x = __fma_rn(xq[q].x, C.cp[(q - 8) * 8 + j], ap[j].x);
        ap[j].y = __fma_rn(xq[q].y, C.cp[(q - 8) * 8 + j], ap[j].y);
      }
    }
}
__device__ __forceinline__ double2 ld_ro2u(const double* p, bool pair) {  // (n odd: the last row alone)
  if (pair) {
    double2 r;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
  }
  return make_double2(ld_ro(p), 0.0);
}
__device__ __forceinline__ void st2u(double* p, double2 v, bool pair) {
  if (pair) *reinterpret_cast<double2*>(p) = v;
  else *p = v.x;
}
template <int M>
__global__ void __launch_bounds__(256) lobpcg_update_xp(int64_t n, double* S, UpdateCoef<M> C) {
  const int64_t i = 2 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
  if (i >= n) return;
  const bool pair = i + 1 < n;  // (always: n is even)
  double2 xq[M];
#pragma unroll
  for (int q = 0; q < M; ++q) xq[q] = ld_ro2u(S + n * q + i, pair);
  double2 ax[8], ap[8];
  update_rows<M>(xq, C, ax, ap);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    st2u(S + n * j + i, ax[j], pair);
    st2u(S + n * (16 + j) + i, ap[j], pair);
  }
}
template <int M>
__global__ void __launch_bounds__(256) lobpcg_update_axp_r(int64_t n, double* AS, const double* X, UpdateCoef<M> C,
                                                            double* R, double* __restrict__ normpart) {
  const int64_t i = 2 * (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
  if (i >= n) {
    if (normpart) lobpcg_norm_partials_sq(nullptr, normpart);  // (the block's barriers need every thread)
    return;
  }
  const bool pair = i + 1 < n;
  double2 xq[M];
#pragma unroll
  for (int q = 0; q < M; ++q) xq[q] = ld_ro2u(AS + n * q + i, pair);
  double2 ax[8], ap[8];
  update_rows<M>(xq, C, ax, ap);
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    st2u(AS + n * j + i, ax[j], pair);
    st2u(AS + n * (16 + j) + i, ap[j], pair);
    const double2 x = ld_ro2u(X + n * j + i, pair);
    double2 rr;
    rr.x = __fma_rn(-C.lam[j], x.x, ax[j].x);
    rr.y = __fma_rn(-C.lam[j], x.y, ax[j].y);
    st2u(R + n * j + i, rr, pair);
    // the norm partials take both rows: x then y (y is 0 past the end)
    r[j] = pair ? __fma_rn(rr.y, rr.y, __dmul_rn(rr.x, rr.x)) : __dmul_rn(rr.x, rr.x);
  }
  if (normpart) lobpcg_norm_partials_sq(r, normpart);
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
      if (j < k) w[j] = __fma_rn(-xq, gs[q * k + j], w[j]);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < k) W[n * j + i] = w[j];
}

// The same for k = 8 with G by value (constant-bank operands, all loads of
// a row issued up front); bitwise block_sub_lincomb_k.
__global__ void __launch_bounds__(256) block_sub_lincomb8_param(int64_t n, const double* __restrict__ X,
                                                                 CoefBlock<8, 8> G, double* W) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double w[8], xq[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    w[j] = ld_ro(W + n * j + i);
    xq[j] = ld_ro(X + n * j + i);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = __fma_rn(-xq[q], G.c[q * 8 + j], w[j]);
#pragma unroll
  for (int j = 0; j < 8; ++j) W[n * j + i] = w[j];
}

// R[:, j] = AX[:, j] - lam[j] X[:, j]
__global__ void block_residual_k(int64_t n, int k, const double* __restrict__ AX, const double* __restrict__ X,
                                 const double* __restrict__ lam, double* __restrict__ R) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < k; ++j) R[n * j + i] = __fma_rn(-lam[j], X[n * j + i], AX[n * j + i]);
}

// Tall-skinny Gram: part[(a * kb + b) * nb + blk] = canonical block partial
// of A_a . B_b.  One launch covers every tile: blockIdx.x = tile (a TA x TB
// block of columns), blockIdx.y = 2048-element data block, so the CTAs that
// run together share a data block and read its columns from L2 after the
// first touch.  Each thread keeps the TA*TB running sums of its 8 strided
// elements in registers (the canonical per-thread order), then the warp
// butterfly and the 8-warp tree.
struct GramTile {
  int a0, b0;
};
template <int TA, int TB>
__global__ void __launch_bounds__(kT, (TB <= 4 ? 2 : 1)) gram_tiles(int64_t n, const double* __restrict__ A, int ka,
                                                  const double* __restrict__ B, int kb,
                                                  const GramTile* __restrict__ tiles, double* __restrict__ part,
                                                  int64_t nb, bool tile_major) {
  __shared__ double ws[TA * TB][8];
  const GramTile tl = tiles[tile_major ? blockIdx.x : blockIdx.y];
  const int ta = min(TA, ka - tl.a0), tb = min(TB, kb - tl.b0);
  const double* Ap = A + n * tl.a0;
  const double* Bp = B + n * tl.b0;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t blk = tile_major ? blockIdx.y : blockIdx.x;
  const int64_t base = blk * kB + t;
  double acc[TA][TB];
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int b = 0; b < TB; ++b) acc[a][b] = 0.0;
  // two k-steps per round, all 2 (TA + TB) loads issued before any use (the
  // asm volatile loads keep the compiler from interleaving them with the
  // arithmetic), then the products in the canonical k order
#pragma unroll 1
  for (int k = 0; k < kK; k += 2) {
    const int64_t i0 = base + static_cast<int64_t>(kT) * k, i1 = i0 + kT;
    double xa[2][TA], yb[2][TB];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = u ? i1 : i0;
#pragma unroll
      for (int a = 0; a < TA; ++a) xa[u][a] = (a < ta && i < n) ? ld_ro(Ap + n * a + i) : 0.0;
#pragma unroll
      for (int b = 0; b < TB; ++b) yb[u][b] = (b < tb && i < n) ? ld_ro(Bp + n * b + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if ((u ? i1 : i0) >= n) continue;
#pragma unroll
      for (int a = 0; a < TA; ++a)
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[a][b] = __fma_rn(xa[u][a], yb[u][b], acc[a][b]);
    }
  }
  if constexpr (TA * TB == 32) {
    // the tile's 32 partials: one reduce-scatter (31 shuffles instead of 160)
    double v[32];
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
      for (int b = 0; b < TB; ++b) v[a * TB + b] = acc[a][b];
    ws[lane][warp] = warp_reduce_scatter32(v, lane);
  } else {
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        const double v = warp_butterfly(acc[a][b]);
        if (lane == 0) ws[a * TB + b][warp] = v;
      }
  }
  __syncthreads();
  if (t < TA * TB) {
    const int a = t / TB, b = t % TB;
    if (a < ta && b < tb) part[static_cast<int64_t>((tl.a0 + a) * kb + tl.b0 + b) * nb + blk] = tree8(ws[t]);
  }
}

// G[a * ldg + b] = canonical fold of the nb partials of dot (a, b) for every
// (a, b) of the listed tiles (one block per dot).
template <int TA, int TB>
__global__ void __launch_bounds__(kT) gram_fold(const double* __restrict__ part, int64_t nb, int ka, int kb,
                                                 const GramTile* __restrict__ tiles, double* __restrict__ G,
                                                 int ldg) {
  __shared__ double ws[8];
  const GramTile tl = tiles[blockIdx.x / (TA * TB)];
  const int q = blockIdx.x % (TA * TB), a = tl.a0 + q / TB, b = tl.b0 + q % TB;
  if (a >= ka || b >= kb) return;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* p = part + static_cast<int64_t>(a * kb + b) * nb;
  double s = 0.0;
  for (int64_t r = t; r < nb; r += kT) s = __dadd_rn(s, p[r]);
  s = warp_butterfly(s);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (t == 0) G[a * ldg + b] = tree8(ws);
}

// x_i = 2 u_i - 1, u_i = (splitmix64(seed ^ splitmix64(i)) >> 11) 2^-53:
// sait_fill_uniform_pm1 (host_inputs.cpp) on the device, bit for bit.
__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void fill_uniform_pm1_k(unsigned long long seed, int64_t n, int64_t offset, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long x = splitmix(seed ^ splitmix(static_cast<unsigned long long>(i + offset)));
  const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
  out[i] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
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

namespace {
template <int KIN, int KOUT>
void launch_lincomb_param(int64_t n, const double* in, const double* C_host, double* out, cudaStream_t s) {
  CoefBlock<KIN, KOUT> cb;
  std::memcpy(cb.c, C_host, sizeof cb.c);
  block_lincomb_param<KIN, KOUT><<<grid_for(n, 256), 256, 0, s>>>(n, in, cb, out);
  SAIT_LAUNCHED();
}
}  // namespace

// out = in C with C on the host: the constant-operand kernel for LOBPCG's
// common shapes (k = 8: 8/16/24 inputs -> 8 outputs); false if not covered.
bool block_lincomb_host_coef(int64_t n, const double* in, int kin, const double* C_host, int kout, double* out,
                             cudaStream_t s) {
  if (n <= 0) return true;
  if (kout != 8) return false;
  switch (kin) {
    case 8: launch_lincomb_param<8, 8>(n, in, C_host, out, s); return true;
    case 16: launch_lincomb_param<16, 8>(n, in, C_host, out, s); return true;
    case 24: launch_lincomb_param<24, 8>(n, in, C_host, out, s); return true;
    default: return false;
  }
}
namespace {
template <int M>
void launch_update(int64_t n, double* S, double* AS, const double* C_host, const double* Cp_host,
                   const double* lam_host, double* R, double* normpart, cudaStream_t s) {
  UpdateCoef<M> cb;
  std::memcpy(cb.c, C_host, sizeof cb.c);
  std::memcpy(cb.cp, Cp_host, sizeof cb.cp);
  std::memcpy(cb.lam, lam_host, sizeof cb.lam);
  lobpcg_update_xp<M><<<grid_for((n + 1) / 2, 256), 256, 0, s>>>(n, S, cb);
  SAIT_LAUNCHED();
  lobpcg_update_axp_r<M><<<grid_for((n + 1) / 2, 256), 256, 0, s>>>(n, AS, S, cb, R, normpart);
  SAIT_LAUNCHED();
}
}  // namespace

// S = [X W P] and AS = [AX AW AP] (n x 8 column blocks, contiguous), m = 16
// or 24: the fused update above (Cp: the (m - 8) x 8 coefficients of P and
// AP); false for shapes it does not cover.
bool lobpcg_update_fused(int64_t n, int k, int m, double* S, double* AS, const double* C_host, const double* Cp_host,
                         const double* lam_host, double* R, cudaStream_t s, double* norms) {
  if (k != 8 || n <= 0 || n % 2) return false;  // (two rows per thread, 16-byte aligned columns)
  double* part = nullptr;
  const int64_t nb = grid_for((n + 1) / 2, 256);
  if (norms) part = dalloc<double>(8 * nb, s);
  if (m == 16) launch_update<16>(n, S, AS, C_host, Cp_host, lam_host, R, part, s);
  else if (m == 24) launch_update<24>(n, S, AS, C_host, Cp_host, lam_host, R, part, s);
  else {
    dfree(part, s);
    return false;
  }
  if (norms) {  // ||R_j|| for the next convergence test, from the update's partials
    mdot_final<<<8, kT, 0, s>>>(part, nb, norms, 1);
    SAIT_LAUNCHED();
    dfree(part, s);
  }
  return true;
}
bool block_sub_lincomb_host_coef(int64_t n, const double* X, int k, const double* G_host, double* W,
                                 cudaStream_t s) {
  if (k != 8) return false;
  if (n <= 0) return true;
  CoefBlock<8, 8> cb;
  std::memcpy(cb.c, G_host, sizeof cb.c);
  block_sub_lincomb8_param<<<grid_for(n, 256), 256, 0, s>>>(n, X, cb, W);
  SAIT_LAUNCHED();
  return true;
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
int64_t gram_scratch(int64_t n, int ka, int kb) { return dot_blocks(n) * ka * kb; }

// partials[(a * kb + b) * nb + blk] for every a < ka, b < kb (no fold)
void gram_partials(int64_t n, const double* A, int ka, const double* B, int kb, double* part, void* tiles_dev,
                   cudaStream_t s) {
  constexpr int TA = 8, TB = 4;
  const int64_t nb = dot_blocks(n);
  GramTile list[256];
  int nt = 0;
  for (int a0 = 0; a0 < ka; a0 += TA)
    for (int b0 = 0; b0 < kb; b0 += TB) list[nt++] = GramTile{a0, b0};
  if (nt == 0 || n == 0) return;
  GramTile* tiles = static_cast<GramTile*>(tiles_dev);
  SAIT_CUDA(cudaMemcpyAsync(tiles, list, sizeof(GramTile) * nt, cudaMemcpyHostToDevice, s));
  gram_tiles<TA, TB><<<dim3(static_cast<unsigned>(nt), static_cast<unsigned>(nb)), kT, 0, s>>>(n, A, ka, B, kb, tiles,
                                                                                              part, nb, true);
  SAIT_LAUNCHED();
}

// ---- Tensor-core Grams (FP64 DMMA, mma.sync.m8n8k4): LOBPCG's fast mode.
// One warp per 2048-element chunk computes the partial Gram of up to 3 x 6
// blocks of 8 columns: per k4 step every lane loads one element of each
// block (column lane>>2, element lane&3 -- the A and B fragment layouts of
// m8n8k4 coincide for a Gram), and NA * NB mma instructions accumulate
// 8 x 8 tiles (256 FMAs each) in registers.  The columns are read once per
// chunk for all tiles, so a 24 x 48 Gram costs one pass over its 72 columns
// instead of ~500 dots' worth of FMA issue.  The order of the products inside
// an mma is the hardware's, so the result is deterministic (fixed chunks,
// fixed fold) but not the canonical order of the restatement: LOBPCG with it
// agrees with oracle/solvers.c to within ±1 iteration (north_star), not bit
// for bit.
namespace {
struct DmmaBlocks {
  const double* a[3];
  const double* b[6];
  int acols[3];
  int bcols[6];
};
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// The k dimension of an mma may take the elements in any order as long as
// A and B agree, so lane (r, q) takes elements e + 4q + u of column r for
// the four mma steps u = 0..3 of a 16-element group: each lane loads 32
// contiguous bytes per column (two 16-byte loads) instead of 8, and a warp
// covers a full 128-byte line of every column per group.  SHARE: B's first
// NA blocks are A's blocks (Rayleigh-Ritz: [S | AS] against S), reused from
// the A fragments instead of loaded twice.
__device__ __forceinline__ double2 ld_ro2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// Shared-operand Grams (B = [S | AS] or [S], S = the A blocks) are symmetric
// -- S^T S exactly, S^T A S mathematically -- so only the tiles on or above
// the block diagonal are computed (the skipped ones are written as zeros and
// mirrored on the host): a third fewer FP64 tensor-core operations for the
// Rayleigh-Ritz pair.
template <int NA, bool SHARE>
__host__ __device__ constexpr bool dmma_tile_needed(int ia, int ib) {
  return !SHARE || (ib < NA ? ib >= ia : ib - NA >= ia);
}
template <int NA, int NB, bool SHARE>
__global__ void __launch_bounds__(NA * NB >= 9 ? 128 : 256) gram_dmma_kernel(int64_t n, DmmaBlocks blk, double* __restrict__ part,
                                                         int64_t nchunks) {
  constexpr int NBL = SHARE ? NB - NA : NB;  // B blocks to load
  const int lane = threadIdx.x & 31;
  const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (c >= nchunks) return;
  const int r = lane >> 2, q = lane & 3;
  const double* ap[NA];
  const double* bp[NBL > 0 ? NBL : 1];
#pragma unroll
  for (int i = 0; i < NA; ++i) ap[i] = r < blk.acols[i] ? blk.a[i] + n * r : nullptr;
#pragma unroll
  for (int i = 0; i < NBL; ++i) {
    const int ib = SHARE ? NA + i : i;
    bp[i] = r < blk.bcols[ib] ? blk.b[ib] + n * r : nullptr;
  }
  double acc[NA][NB][2];
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t i0 = c * kB, i1 = min(n, i0 + kB);
  for (int64_t e = i0; e < i1; e += 16) {
    double af[4][NA], bf[4][NBL > 0 ? NBL : 1];
    const int64_t f = e + 4 * q;  // this lane's 4 elements f .. f + 3
    if (f + 4 <= i1) {
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (ap[k]) {
          x = ld_ro2(ap[k] + f);
          y = ld_ro2(ap[k] + f + 2);
        }
        af[0][k] = x.x;
        af[1][k] = x.y;
        af[2][k] = y.x;
        af[3][k] = y.y;
      }
#pragma unroll
      for (int k = 0; k < NBL; ++k) {
        double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
        if (bp[k]) {
          x = ld_ro2(bp[k] + f);
          y = ld_ro2(bp[k] + f + 2);
        }
        bf[0][k] = x.x;
        bf[1][k] = x.y;
        bf[2][k] = y.x;
        bf[3][k] = y.y;
      }
    } else {  // the chunk's ragged end
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = f + u < i1;
#pragma unroll
        for (int k = 0; k < NA; ++k) af[u][k] = (in && ap[k]) ? ld_ro(ap[k] + f + u) : 0.0;
#pragma unroll
        for (int k = 0; k < NBL; ++k) bf[u][k] = (in && bp[k]) ? ld_ro(bp[k] + f + u) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int ia = 0; ia < NA; ++ia)
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
          if (!dmma_tile_needed<NA, SHARE>(ia, ib)) continue;
          const double bv = SHARE ? (ib < NA ? af[u][ib] : bf[u][SHARE ? ib - NA : ib]) : bf[u][ib];
          dmma(acc[ia][ib][0], acc[ia][ib][1], af[u][ia], bv);
        }
  }
  // D[row = lane>>2][col = 2 (lane&3) + h] of tile (ia, ib)
  const int KB = NB * 8;
#pragma unroll
  for (int ia = 0; ia < NA; ++ia)
#pragma unroll
    for (int ib = 0; ib < NB; ++ib)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = ia * 8 + r, bcol = ib * 8 + 2 * q + h;
        part[(static_cast<int64_t>(a) * KB + bcol) * nchunks + c] = acc[ia][ib][h];
      }
}
// G[a * ldg + bmap(b)] = sum over chunks (fixed order: thread t sums t,
// t + 256, ..., then the warp butterfly and the 8-way tree)
__global__ void __launch_bounds__(kT) gram_dmma_fold(const double* __restrict__ part, int64_t nchunks, int KB,
                                                     const int* __restrict__ bmap, double* __restrict__ G,
                                                     int ldg) {
  __shared__ double ws[8];
  const int d = blockIdx.x, a = d / KB, b = d % KB;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const double* p = part + static_cast<int64_t>(d) * nchunks;
  double s = 0.0;
  for (int64_t k = t; k < nchunks; k += kT) s = __dadd_rn(s, p[k]);
  s = warp_butterfly(s);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (t == 0 && bmap[b] >= 0) G[a * ldg + bmap[b]] = tree8(ws);
}
template <int NA, int NB, bool SHARE>
void launch_dmma(int64_t n, const DmmaBlocks& blk, double* part, int64_t nchunks, cudaStream_t s) {
  // big tiles hold ~170 registers: 4-warp CTAs so that 3 fit per SM
  constexpr int kThreads = NA * NB >= 9 ? 128 : 256, kWarps = kThreads / 32;
  gram_dmma_kernel<NA, NB, SHARE><<<static_cast<unsigned>((nchunks + kWarps - 1) / kWarps), kThreads, 0, s>>>(
      n, blk, part, nchunks);
}
using DmmaLaunch = void (*)(int64_t, const DmmaBlocks&, double*, int64_t, cudaStream_t);
template <int NA>
DmmaLaunch dmma_for(int nb, bool share) {
  if (share) {  // B = [A blocks | NB - NA more]
    switch (nb) {
      case NA: return launch_dmma<NA, NA, true>;
      default: return launch_dmma<NA, 2 * NA, true>;
    }
  }
  switch (nb) {
    case 1: return launch_dmma<NA, 1, false>;
    case 2: return launch_dmma<NA, 2, false>;
    case 3: return launch_dmma<NA, 3, false>;
    case 4: return launch_dmma<NA, 4, false>;
    case 5: return launch_dmma<NA, 5, false>;
    default: return launch_dmma<NA, 6, false>;
  }
}
}  // namespace

// G (device, row-major, ld ldg) = A^T B with tensor cores: A's columns are the
// blocks of 8 starting at a_cols[i] (na <= 3 blocks, ka columns in all), B's
// likewise (nb <= 6 blocks); b columns land at G column bcol_out[j * 8 + c]
// (-1: not stored).  scratch: >= gram_scratch(n, 24, 48) doubles; idx_dev:
// device room for 64 ints.  false if the shape is not covered (the caller
// uses gram()).
bool gram_fast(int64_t n, const double* const* ablk, const int* acols, int na, const double* const* bblk,
               const int* bcols, int nb, const int* bcol_out, double* G, int ldg, double* scratch, void* idx_dev,
               cudaStream_t s) {
  if (na < 1 || na > 3 || nb < 1 || nb > 6 || n <= 0) return false;
  for (int i = 0; i < na; ++i)
    if (reinterpret_cast<uintptr_t>(ablk[i]) % 8) return false;
  DmmaBlocks blk{};
  for (int i = 0; i < na; ++i) {
    blk.a[i] = ablk[i];
    blk.acols[i] = acols[i];
  }
  for (int i = 0; i < nb; ++i) {
    blk.b[i] = bblk[i];
    blk.bcols[i] = bcols[i];
  }
  const int64_t nchunks = dot_blocks(n);
  // B's first na blocks the A blocks themselves (Rayleigh-Ritz), 16-byte
  // aligned columns for the vector loads (n even)
  bool share = nb == na || nb == 2 * na;
  for (int i = 0; i < na && share; ++i) share = bblk[i] == ablk[i] && bcols[i] == acols[i];
  bool aligned = n % 2 == 0;
  for (int i = 0; i < na; ++i) aligned = aligned && reinterpret_cast<uintptr_t>(ablk[i]) % 16 == 0;
  for (int i = 0; i < nb; ++i) aligned = aligned && reinterpret_cast<uintptr_t>(bblk[i]) % 16 == 0;
  if (!aligned) return false;
  DmmaLaunch f = na == 1 ? dmma_for<1>(nb, share) : na == 2 ? dmma_for<2>(nb, share) : dmma_for<3>(nb, share);
  f(n, blk, scratch, nchunks, s);
  SAIT_LAUNCHED();
  const int KB = nb * 8;
  int map[48];
  for (int j = 0; j < KB; ++j) map[j] = bcol_out[j];
  int* dmap = static_cast<int*>(idx_dev);
  SAIT_CUDA(cudaMemcpyAsync(dmap, map, sizeof(int) * KB, cudaMemcpyHostToDevice, s));
  gram_dmma_fold<<<static_cast<unsigned>(na * 8 * KB), kT, 0, s>>>(scratch, nchunks, KB, dmap, G, ldg);
  SAIT_LAUNCHED();
  // rows a >= ka (partial last A block) are folded too but never read
  return true;
}

// G (device, row-major, leading dimension ldg) = A^T B for column-major
// blocks A (n x ka) and B (n x kb); upper_only skips tiles strictly below the
// diagonal.  scratch: gram_scratch(n, ka, kb) doubles; tiles: a device array
// of at least (ceil(ka/8) * ceil(kb/8)) GramTile (written here).
namespace {
template <int TA, int TB>
void gram_impl(int64_t n, const double* A, int ka, const double* B, int kb, double* G, int ldg, double* scratch,
               void* tiles_dev, cudaStream_t s, bool upper_only) {
  const int64_t nb = dot_blocks(n);
  GramTile list[256];
  int nt = 0;
  for (int a0 = 0; a0 < ka; a0 += TA)
    for (int b0 = 0; b0 < kb; b0 += TB) {
      if (upper_only && b0 + TB <= a0) continue;
      list[nt++] = GramTile{a0, b0};
    }
  if (nt == 0 || nb == 0) return;
  GramTile* tiles = static_cast<GramTile*>(tiles_dev);
  SAIT_CUDA(cudaMemcpyAsync(tiles, list, sizeof(GramTile) * nt, cudaMemcpyHostToDevice, s));
  static const bool tile_major = [] {
    const char* e = std::getenv("SAIT_GRAM_ORDER");
    return !(e && std::atoi(e) == 0);
  }();
  const dim3 grid = tile_major ? dim3(static_cast<unsigned>(nt), static_cast<unsigned>(nb))
                               : dim3(static_cast<unsigned>(nb), static_cast<unsigned>(nt));
  gram_tiles<TA, TB><<<grid, kT, 0, s>>>(n, A, ka, B, kb, tiles, scratch, nb, tile_major);
  SAIT_LAUNCHED();
  gram_fold<TA, TB><<<static_cast<unsigned>(nt * TA * TB), kT, 0, s>>>(scratch, nb, ka, kb, tiles, G, ldg);
  SAIT_LAUNCHED();
}
}  // namespace



// Rayleigh-Ritz's two Grams in ONE launch: S^T S (upper tiles) and S^T AS
// (all tiles) for S = [X W P] (m columns) and AS stored right after S's 3k
// columns in one allocation (AS = S + 3k n).  The tiles of both run side by
// side over each data block, so S's columns are read from DRAM once for both
// Grams and one fold + one read-back serve both.  Gs (row-major, ld 6k)
// receives columns [0, m) = S^T S and [3k, 3k + m) = S^T AS; every entry is
// the same canonical dot as gram() computes.
void gram_rr(int64_t n, const double* S, int m, int k, double* G, double* scratch, void* tiles_dev, cudaStream_t s) {
  constexpr int TA = 8, TB = 4;
  const int kb = 6 * k;
  const int64_t nb = dot_blocks(n);
  GramTile list[256];
  int nt = 0;
  for (int a0 = 0; a0 < m; a0 += TA) {
    for (int b0 = 0; b0 < m; b0 += TB)
      if (!(b0 + TB <= a0)) list[nt++] = GramTile{a0, b0};
    for (int b0 = 3 * k; b0 < 3 * k + m; b0 += TB) list[nt++] = GramTile{a0, b0};
  }
  if (nt == 0 || nb == 0) return;
  GramTile* tiles = static_cast<GramTile*>(tiles_dev);
  SAIT_CUDA(cudaMemcpyAsync(tiles, list, sizeof(GramTile) * nt, cudaMemcpyHostToDevice, s));
  gram_tiles<TA, TB><<<dim3(static_cast<unsigned>(nt), static_cast<unsigned>(nb)), kT, 0, s>>>(n, S, m, S, kb, tiles,
                                                                                            scratch, nb, true);
  SAIT_LAUNCHED();
  gram_fold<TA, TB><<<static_cast<unsigned>(nt * TA * TB), kT, 0, s>>>(scratch, nb, m, kb, tiles, G, kb);
  SAIT_LAUNCHED();
}

// G (device, row-major, leading dimension ldg) = A^T B for column-major
// blocks A (n x ka) and B (n x kb); upper_only skips tiles strictly below the
// diagonal.  scratch: gram_scratch(n, ka, kb) doubles; tiles_dev: device room
// for 256 GramTile.  8 x 4 tiles (SAIT_GRAM_TILE=88 for 8 x 8): fewer
// registers, two CTAs per SM, the repeated column reads served by L2.
void gram(int64_t n, const double* A, int ka, const double* B, int kb, double* G, int ldg, double* scratch,
          void* tiles_dev, cudaStream_t s, bool upper_only) {
  static const int tile = [] {
    const char* e = std::getenv("SAIT_GRAM_TILE");
    return e ? std::atoi(e) : 84;
  }();
  if (tile == 88) gram_impl<8, 8>(n, A, ka, B, kb, G, ldg, scratch, tiles_dev, s, upper_only);
  else gram_impl<8, 4>(n, A, ka, B, kb, G, ldg, scratch, tiles_dev, s, upper_only);
}

void fill_uniform_pm1_device(uint64_t seed, int64_t n, double* out, cudaStream_t s, int64_t offset) {
  if (n <= 0) return;
  fill_uniform_pm1_k<<<grid_for(n, 256), 256, 0, s>>>(seed, n, offset, out);
  SAIT_LAUNCHED();
}

// Block partials / fold of multi_dot separately, for reductions across ranks
// (a row-sharded vector aligned to 2048-element blocks gives each rank a
// contiguous run of the global blocks; folding all ranks' partials in order
// reproduces the single-device value bit for bit).
void dot_partials(int64_t n, const double* x, const double* V, int64_t ld, int m, double* part, cudaStream_t s) {
  const int64_t nb = dot_blocks(n);
  for (int j0 = 0; j0 < m; j0 += kMaxM) {
    const int mm = m - j0 < kMaxM ? m - j0 : kMaxM;
    mdot_partials<false><<<static_cast<unsigned>(nb), kT, 0, s>>>(n, x, V + ld * j0, ld, mm, part + nb * j0, nb);
    SAIT_LAUNCHED();
  }
}
void dot_fold(const double* part, int64_t nb, int m, double* out, bool sqrt_out, cudaStream_t s) {
  if (m <= 0) return;
  mdot_final<<<m, kT, 0, s>>>(part, nb, out, sqrt_out ? 1 : 0);
  SAIT_LAUNCHED();
}

void multi_dot(int64_t n, const double* x, const double* V, int64_t ld, int m, double* out, double* scratch,
               cudaStream_t s, bool sqrt_out) {
  const int64_t nb = dot_blocks(n);
  for (int j0 = 0; j0 < m; j0 += kMaxM) {
    const int mm = m - j0 < kMaxM ? m - j0 : kMaxM;
    // (a reduce-scatter variant holding all m partials, mdot_partials<true>,
    // needs 100 registers and made C3's GMRES slower: 2.65 -> 2.97 s)
    mdot_partials<false><<<static_cast<unsigned>(nb), kT, 0, s>>>(n, x, V + ld * j0, ld, mm, scratch, nb);
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
