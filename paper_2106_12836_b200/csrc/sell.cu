// sell.cu — sliced-ELL (SELL-32) apply format for the SAIT factors.
//
// The apply reads each factor once per vector, so its speed is set by how the
// CSR stream maps onto HBM.  For the stencil-derived SAIT factors rows are
// almost uniform (C2: 97.7% of rows have exactly 7 entries; a 32-row slice
// pads by 0.34%), so the pair keeps a SELL-32 copy built once at pair
// creation: slice s stores its 32 rows column-major, width = the slice's
// longest row, so lane j of a warp owns row 32 s + j and every load of the
// slice is a coalesced 128 B (indices) / 256 B (values) warp transaction
// straight into registers — no shared-memory staging, no block barriers.
// x gathers of neighbouring rows are neighbouring too (stencil), hence
// coalesced.  Each thread still sums its row in stored order without FMA, so
// results stay bitwise equal to the reference's spmv (kernels.cpp:18-24);
// padded slots carry col = -1 and are skipped (never multiplied), so a
// non-finite x cannot leak into a row through padding.
//
// Rows too irregular for slicing (padding > kMaxPad) keep the CSR kernels.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <unordered_map>

#include "common.cuh"

namespace sait {
namespace {

constexpr int kSlice = 32;
constexpr int64_t kPfMinSlices = 1 << 18;  // factors with at least this many slices prefetch
constexpr int kPfDistance = 8192;
constexpr double kMaxPad = 1.25;
constexpr double kSortPad = 1.10;

__device__ __forceinline__ int32_t ld_na(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_na(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ int16_t ld_na(const int16_t* p) {
  int16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.s16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

// Column storage of a SELL slice slot: absolute int32 columns (-1 = padding)
// or int16 deltas col - row (INT16_MIN = padding) when every |col - row| of
// the matrix fits, which saves 2 of the 12 bytes streamed per entry.
// slice_base(s, base) = where slice s's slot-0 indices start in the policy's
// array (the element offset base for per-entry storage).
struct Idx32 {
  const int32_t* p;
  __device__ __forceinline__ int64_t slice_base(int64_t /*s*/, int64_t base) const { return base; }
  __device__ __forceinline__ int32_t col(int64_t e, int32_t /*row*/) const { return ld_na(p + e); }
};
struct Idx16 {
  const int16_t* p;
  __device__ __forceinline__ int64_t slice_base(int64_t /*s*/, int64_t base) const { return base; }
  __device__ __forceinline__ int32_t col(int64_t e, int32_t row) const {
    const int16_t d = ld_na(p + e);
    return d == INT16_MIN ? -1 : row + d;
  }
};
// Shared slice patterns: a few KB of deltas serve every slice, so they stay
// in L1 and only the values stream from HBM (8 instead of 10 B per entry).
struct IdxDict {
  const int32_t* pat;
  const int32_t* dict;  // col - row deltas, INT32_MIN = padding
  __device__ __forceinline__ int64_t slice_base(int64_t s, int64_t /*base*/) const { return __ldg(pat + s); }
  __device__ __forceinline__ int32_t col(int64_t e, int32_t row) const {
    const int32_t d = __ldg(dict + e);
    return d == INT32_MIN ? -1 : row + d;
  }
};

// A plain (weak, coherent) load.  The x of a programmatic dependent SpMV is
// written by the prerequisite grid while this grid is already resident, so
// it must not go through the non-coherent read-only path (ld.global.nc
// requires the data to be unchanged for the kernel's lifetime); after
// griddepcontrol.wait the prerequisite's writes are visible to weak loads.
__device__ __forceinline__ double ld_weak(const double* p) {
  double r;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(r) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

__global__ void slice_widths(int64_t n, const int32_t* __restrict__ rp, int64_t nslices, int64_t* __restrict__ width) {
  int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int64_t r0 = s * kSlice, r1 = r0 + kSlice < n ? r0 + kSlice : n;
  int32_t w = 0;
  for (int64_t r = r0; r < r1; ++r) w = max(w, rp[r + 1] - rp[r]);
  width[s] = static_cast<int64_t>(w) * kSlice;
}

__global__ void scan_i64_inplace(int64_t* a, int64_t n) {  // single block, exclusive, a[n] = total
  __shared__ int64_t carry_s;
  __shared__ int64_t warp_tot[32];
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < n ? a[i] : 0, x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    int64_t before = 0, tot = 0;
    for (int q = 0; q < nw; ++q) {
      if (q < wid) before += warp_tot[q];
      tot += warp_tot[q];
    }
    if (i < n) a[i] = carry_s + before + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) a[n] = carry_s;
}

__global__ void max_col_delta(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              int* __restrict__ out) {
  int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int m = 0;
  if (r < n)
    for (int32_t e = rp[r]; e < rp[r + 1]; ++e) m = max(m, abs(static_cast<int>(ci[e] - r)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void fill_sell16(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const int64_t* __restrict__ soff,
                            int16_t* __restrict__ scol, double* __restrict__ sval,
                            const int32_t* __restrict__ perm) {
  const int64_t pos = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t s = pos / kSlice;
  int lane = static_cast<int>(pos % kSlice);
  const int64_t r = perm ? (pos < (n + kSlice - 1) / kSlice * kSlice ? perm[pos] : n) : pos;  // the slot's row
  int64_t nslices = (n + kSlice - 1) / kSlice;
  if (s >= nslices) return;
  int64_t base = soff[s];
  int32_t w = static_cast<int32_t>((soff[s + 1] - base) / kSlice);
  int32_t b = 0, len = 0;
  if (r < n) {
    b = rp[r];
    len = rp[r + 1] - b;
  }
  for (int32_t k = 0; k < w; ++k) {
    int64_t dst = base + static_cast<int64_t>(k) * kSlice + lane;
    if (k < len) {
      scol[dst] = static_cast<int16_t>(ci[b + k] - r);
      sval[dst] = v[b + k];
    } else {
      scol[dst] = INT16_MIN;
      sval[dst] = 0.0;
    }
  }
}

__global__ void fill_sell(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const int64_t* __restrict__ soff,
                          int32_t* __restrict__ scol, double* __restrict__ sval,
                            const int32_t* __restrict__ perm) {
  const int64_t pos = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t s = pos / kSlice;
  int lane = static_cast<int>(pos % kSlice);
  const int64_t r = perm ? (pos < (n + kSlice - 1) / kSlice * kSlice ? perm[pos] : n) : pos;  // the slot's row
  int64_t nslices = (n + kSlice - 1) / kSlice;
  if (s >= nslices) return;
  int64_t base = soff[s];
  int32_t w = static_cast<int32_t>((soff[s + 1] - base) / kSlice);
  int32_t b = 0, len = 0;
  if (r < n) {
    b = rp[r];
    len = rp[r + 1] - b;
  }
  for (int32_t k = 0; k < w; ++k) {
    int64_t dst = base + static_cast<int64_t>(k) * kSlice + lane;
    if (k < len) {
      scol[dst] = ci[b + k];
      sval[dst] = v[b + k];
    } else {
      scol[dst] = -1;
      sval[dst] = 0.0;
    }
  }
}

// One warp per slice (grid-stride), lane = row.  Loads are batched 8 slots at
// a time so each thread has 16 independent streaming loads and 8 gathers in
// flight.  PDL: when launched as a programmatic dependent (the M_U half of a
// pair), the first batch of indices/values is loaded before waiting for the
// producer of x (the M_L half), overlapping that grid's tail.
template <class IDX, bool PDL_WAIT>
__global__ void __launch_bounds__(256) sell_spmv_kernel(int64_t n, int64_t s_begin, int64_t nslices,
                                                         const int64_t* __restrict__ soff, IDX idx,
                                                         const double* __restrict__ sval,
                                                         const double* __restrict__ x, double* __restrict__ y,
                                                         int pf, const int32_t* __restrict__ perm) {
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t s = s_begin + static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;  // grid = one slice per warp
  const int64_t base = soff[s];
  const int32_t w = static_cast<int32_t>((soff[s + 1] - base) >> 5);
  // L2 prefetch of the values of the slice one wave ahead (pf slices; 0 =
  // off): one bulk prefetch by lane 0, fire and forget, so HBM reads run
  // ahead of the warps' dependent load chains (C5: 223 -> 212 us per launch;
  // at C2 size it does not pay, 25.4 -> 26.5 us)
  if (pf > 0 && lane == 0 && s + pf < nslices) {
    const int64_t pb = soff[s + pf], pe = soff[s + pf + 1];
    if (pe > pb)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sval + pb),
                   "r"(static_cast<uint32_t>((pe - pb) * 8))
                   : "memory");
  }
  const int32_t row = perm ? perm[s * kSlice + lane] : static_cast<int32_t>(s * kSlice) + lane;
  const int64_t e0 = base + lane;
  const int64_t i0 = idx.slice_base(s, base) + lane;
  double acc = 0.0;
  for (int32_t k0 = 0; k0 < w; k0 += 8) {
    int32_t c[8];
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = -1;
      v[j] = 0.0;
      if (k0 + j < w) {
        c[j] = idx.col(i0 + static_cast<int64_t>(k0 + j) * kSlice, row);
        v[j] = ld_na(sval + e0 + static_cast<int64_t>(k0 + j) * kSlice);
        SAIT_DCHECK(c[j] >= -1, "sell column", c[j], -1);
      }
    }
    if (PDL_WAIT && k0 == 0) pdl_wait();  // x is the previous grid's output
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double xv = c[j] >= 0 ? (PDL_WAIT ? ld_weak(x + c[j]) : __ldg(x + c[j])) : 0.0;
      if (c[j] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[j], xv));
    }
  }
  if (row < n) y[row] = acc;
}

// Row-major block of NV vectors: lane = row, NV accumulators per thread; the
// slice's indices/values are read once for all NV vectors.
template <int NV, class IDX>
__global__ void __launch_bounds__(256) sell_spmm_kernel(int64_t n, int64_t nslices, const int64_t* __restrict__ soff,
                                                         IDX idx, const double* __restrict__ sval,
                                                         const double* __restrict__ x, double* __restrict__ y,
                                                         const int32_t* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); s < nslices;
       s += warps) {
    const int64_t base = soff[s];
    const int64_t ib = idx.slice_base(s, base);
    const int32_t w = static_cast<int32_t>((soff[s + 1] - base) >> 5);
    const int64_t row = perm ? perm[s * kSlice + lane] : s * kSlice + lane;
    double acc[NV];
#pragma unroll
    for (int c = 0; c < NV; ++c) acc[c] = 0.0;
    for (int32_t k0 = 0; k0 < w; k0 += 4) {
      int32_t col[4];
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        col[j] = -1;
        v[j] = 0.0;
        if (k0 + j < w) {
          col[j] = idx.col(ib + (k0 + j) * kSlice + lane, static_cast<int32_t>(row));
          v[j] = ld_na(sval + base + (k0 + j) * kSlice + lane);
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (col[j] < 0) continue;
        const double2* xr = reinterpret_cast<const double2*>(x + static_cast<int64_t>(col[j]) * NV);
#pragma unroll
        for (int c = 0; c < NV / 2; ++c) {
          const double2 xx = __ldg(xr + c);
          acc[2 * c] = __dadd_rn(acc[2 * c], __dmul_rn(v[j], xx.x));
          acc[2 * c + 1] = __dadd_rn(acc[2 * c + 1], __dmul_rn(v[j], xx.y));
        }
      }
    }
    if (row < n) {
      double2* yr = reinterpret_cast<double2*>(y + row * NV);
#pragma unroll
      for (int c = 0; c < NV / 2; ++c) yr[c] = make_double2(acc[2 * c], acc[2 * c + 1]);
    }
  }
}

// Column-major block (n x NV, leading dimension ld): lane = row, NV
// accumulators; each index/value read once for all NV vectors, x gathered
// per column (neighbouring rows -> neighbouring x: coalesced).  The kernel is
// bound by loads in flight per SM = resident warps x gathers per warp
// (BATCH slots x NV columns); the shapes per index format are the measured
// best (tools/block_time.py, C5 block-8 pair: 1.93 -> 1.31 ms for the
// dictionary format, the int16/int32 formats spill at 40 registers).
template <class IDX>
struct CmShape {
  static constexpr int kThreads = 256, kMinBlocks = 1, kBatch = 2;
};
template <>
struct CmShape<IdxDict> {
  static constexpr int kThreads = 128, kMinBlocks = 12, kBatch = 3;
};
template <int NV, class IDX>
__global__ void __launch_bounds__(CmShape<IDX>::kThreads, CmShape<IDX>::kMinBlocks) sell_spmm_cm_kernel(int64_t n, int64_t nslices,
                                                                             const int64_t* __restrict__ soff, IDX idx,
                                                                             const double* __restrict__ sval,
                                                                             const double* __restrict__ x, int64_t ldx,
                                                                             double* __restrict__ y, int64_t ldy,
                                                                             int nv, const int32_t* __restrict__ perm) {
  const int lane = threadIdx.x & 31;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int64_t base = soff[s];
  const int64_t ib = idx.slice_base(s, base) + lane;
  const double* __restrict__ vp = sval + base + lane;
  const int32_t w = static_cast<int32_t>((soff[s + 1] - base) >> 5);
  const int32_t row = perm ? perm[s * kSlice + lane] : static_cast<int32_t>(s * kSlice) + lane;
  double acc[NV];
#pragma unroll
  for (int c = 0; c < NV; ++c) acc[c] = 0.0;
  constexpr int kBatch = CmShape<IDX>::kBatch;
  for (int32_t k0 = 0; k0 < w; k0 += kBatch) {
    int32_t col[kBatch];
    double v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      col[j] = -1;
      v[j] = 0.0;
      if (k0 + j < w) {
        col[j] = idx.col(ib + (k0 + j) * kSlice, row);
        v[j] = ld_na(vp + (k0 + j) * kSlice);
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (col[j] < 0) continue;
      // one running pointer down the block's columns (no per-column 64-bit
      // offsets held in registers: occupancy is what bounds this kernel)
      const double* p = x + col[j];
#pragma unroll
      for (int c = 0; c < NV; ++c) {
        if (c < nv) acc[c] = __dadd_rn(acc[c], __dmul_rn(v[j], __ldg(p)));
        p += ldx;
      }
    }
  }
  if (row < n) {
    double* q = y + row;
#pragma unroll
    for (int c = 0; c < NV; ++c) {
      if (c < nv) *q = acc[c];
      q += ldy;
    }
  }
}

// ---------------------------------------------------------------- peer halo
// y = A x_ext on a row block of a sharded factor, where the extended vector
// is [halo below | own | halo above] and the halo entries are read straight
// from the neighbouring ranks' buffers (peer memory over NVLink) instead of
// being exchanged first: the transfer overlaps the math slice by slice.  A
// warp whose slice touches a halo column first waits (acquire, system scope)
// until the owner has published this epoch's values; warps of interior slices
// never wait.  A wait longer than 20 s traps (a peer that died) instead of
// hanging.
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// No "memory" clobber: a clobber would pin every surrounding gather in
// program order (one x load in flight instead of eight); the acquire of the
// owner's flag (wait_epoch_sys, which does clobber) already orders these
// loads after it.
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double r;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void wait_epoch_sys(const int* flag, int epoch) {
  if (ld_acquire_sys(flag) - epoch >= 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  unsigned ns = 64;
  while (ld_acquire_sys(flag) - epoch < 0) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      printf("sait: halo wait timed out (flag %p = %d, waiting for epoch %d, block %d)\n", flag,
             ld_acquire_sys(flag), epoch, blockIdx.x);
      __trap();
    }
  }
}

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The last CTA of the grid to finish publishes *flag = epoch: every CTA
// fences its stores device-wide and counts itself; the one that completes the
// count fences system-wide (peers over NVLink read the data) and releases the
// flag, then rearms the counter for the next launch (stream-ordered).
__device__ __forceinline__ void publish_when_grid_done(int* flag, unsigned* count, int epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      __threadfence_system();
      st_release_sys(flag, epoch);
      *count = 0;
    }
  }
}

template <class IDX, bool PDL>
__global__ void __launch_bounds__(256) sell_spmv_halo_kernel(int64_t n, int64_t s_begin, int64_t s_end,
                                                              const int64_t* __restrict__ soff, IDX idx,
                                                              const double* __restrict__ sval,
                                                              const double* __restrict__ x, double* __restrict__ y,
                                                              HaloArgs h) {
  if (PDL) pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int64_t s = s_begin + static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s < s_end) {
    const int64_t base = soff[s];
    const int32_t w = static_cast<int32_t>((soff[s + 1] - base) >> 5);
    const int32_t row = static_cast<int32_t>(s * kSlice) + lane;
    const int64_t e0 = base + lane;
    const int64_t i0 = idx.slice_base(s, base) + lane;
    bool lo_ready = false, hi_ready = false;
    double acc = 0.0;
    for (int32_t k0 = 0; k0 < w; k0 += 8) {
      int32_t c[8];
      double v[8];
      bool lo = false, hi = false;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = -1;
        v[j] = 0.0;
        if (k0 + j < w) {
          c[j] = idx.col(i0 + static_cast<int64_t>(k0 + j) * kSlice, row);
          v[j] = ld_na(sval + e0 + static_cast<int64_t>(k0 + j) * kSlice);
          lo |= c[j] >= 0 && c[j] < h.own_lo;
          hi |= c[j] >= h.own_hi;
          SAIT_DCHECK(c[j] < 0 || c[j] >= h.own_hi || c[j] >= h.own_lo || c[j] + h.lo_shift >= 0, "halo lo index",
                      c[j] + h.lo_shift, 0);
        }
      }
      if (PDL && k0 == 0) pdl_wait();  // the own x is the previous grid's output
      if (__any_sync(0xffffffffu, lo || hi)) {  // a boundary batch: wait for the owners, read over NVLink
        if (!lo_ready && __any_sync(0xffffffffu, lo)) {
          wait_epoch_sys(h.lo_flag, h.epoch);
          lo_ready = true;
        }
        if (!hi_ready && __any_sync(0xffffffffu, hi)) {
          wait_epoch_sys(h.hi_flag, h.epoch);
          hi_ready = true;
        }
        double xv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          xv[j] = c[j] < 0           ? 0.0
                  : c[j] < h.own_lo  ? ld_relaxed_sys(h.lo_src + (c[j] + h.lo_shift))
                  : c[j] >= h.own_hi ? ld_relaxed_sys(h.hi_src + (c[j] + h.hi_shift))
                                     : (PDL ? ld_weak(x + c[j]) : __ldg(x + c[j]));
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c[j] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[j], xv[j]));
      } else {  // interior batch: the single-GPU kernel's loads
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double xv = c[j] >= 0 ? (PDL ? ld_weak(x + c[j]) : __ldg(x + c[j])) : 0.0;
          if (c[j] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[j], xv));
        }
      }
    }
    if (row < n) y[row] = acc;
  } else if (PDL) {
    pdl_wait();  // keep the grid's completion after the prerequisite's
  }
  if (h.pub_flag) publish_when_grid_done(h.pub_flag, h.pub_count, h.epoch);
}

__global__ void copy_slices_publish_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t a0,
                                           int64_t n0, int64_t a1, int64_t n1, int* flag, unsigned* count,
                                           int epoch) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n0 + n1;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = k < n0 ? a0 + k : a1 + (k - n0);
    dst[e] = src[e];
  }
  publish_when_grid_done(flag, count, epoch);
}

// flag = epoch, ordered after everything queued before it on the stream
__global__ void publish_epoch_kernel(int* flag, int epoch) {
  asm volatile("fence.sc.sys;" ::: "memory");
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
}

unsigned sell_grid(int64_t nslices) {  // one slice per warp, 8 warps per CTA
  return static_cast<unsigned>(std::max<int64_t>(1, (nslices + 7) / 8));
}

// rows per dependency group of the chunked host apply (column_group_deps)
constexpr int kGroupRows = 256;

}  // namespace

// lo/hi[g] = column-group range touched by the rows of group g (256 rows).
__global__ void pair_deps(int64_t nU, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          int64_t gU, int32_t* __restrict__ lo, int32_t* __restrict__ hi) {
  int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= gU) return;
  int64_t r0 = g * kGroupRows, r1 = r0 + kGroupRows < nU ? r0 + kGroupRows : nU;
  int32_t mn = INT32_MAX, mx = -1;
  for (int64_t r = r0; r < r1; ++r) {
    int32_t b = rp[r], e = rp[r + 1];
    if (b < e) {
      mn = min(mn, ci[b]);
      mx = max(mx, ci[e - 1]);
    }
  }
  lo[g] = mx < 0 ? 1 : mn / kGroupRows;
  hi[g] = mx < 0 ? 0 : mx / kGroupRows;
}

void column_group_deps(const DevCsr& m, int32_t* lo, int32_t* hi, cudaStream_t s) {
  const int64_t g = (m.nrows + kGroupRows - 1) / kGroupRows;
  if (g == 0) return;
  pair_deps<<<grid_for(g, 128), 128, 0, s>>>(m.nrows, m.rp, m.ci, g, lo, hi);
  SAIT_LAUNCHED();
}

namespace {

// ---- shared slice patterns (see IdxDict)
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// slot delta col - row of a SELL entry (INT32_MIN for padding), from either
// per-entry index form
template <class IDX>
__device__ __forceinline__ int32_t slot_delta(const IDX& idx, int64_t e, int32_t row) {
  const int32_t c = idx.col(e, row);
  return c < 0 ? INT32_MIN : c - row;
}

// one warp per slice: a hash of (width, every lane's deltas)
template <class IDX>
__global__ void slice_hash(int64_t nslices, const int64_t* __restrict__ soff, IDX idx,
                           unsigned long long* __restrict__ h) {
  const int lane = threadIdx.x & 31;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int64_t base = soff[s];
  const int32_t w = static_cast<int32_t>((soff[s + 1] - base) >> 5);
  const int32_t row = static_cast<int32_t>(s * kSlice) + lane;
  unsigned long long x = static_cast<unsigned long long>(w) * 0x100000001B3ull + static_cast<unsigned long long>(lane);
  for (int32_t k = 0; k < w; ++k)
    x = mix64(x ^ static_cast<unsigned int>(slot_delta(idx, base + static_cast<int64_t>(k) * kSlice + lane, row)));
  x = mix64(x + static_cast<unsigned long long>(lane) * 0xD6E8FEB86659FD93ull);
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) h[s] = mix64(x ^ static_cast<unsigned long long>(w));
}

// any slice whose deltas differ from its representative's -> *bad
template <class IDX>
__global__ void slice_verify(int64_t nslices, const int64_t* __restrict__ soff, IDX idx,
                             const int32_t* __restrict__ rep, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int64_t r = rep[s];
  if (r == s) return;
  const int64_t b = soff[s], br = soff[r];
  const int64_t len = soff[s + 1] - b;
  if (len != soff[r + 1] - br) {
    if (lane == 0) atomicOr(bad, 1);
    return;
  }
  const int32_t row = static_cast<int32_t>(s * kSlice) + lane, rrow = static_cast<int32_t>(r * kSlice) + lane;
  bool diff = false;
  for (int64_t e = lane; e < len; e += kSlice) diff |= slot_delta(idx, b + e, row) != slot_delta(idx, br + e, rrow);
  if (__any_sync(0xffffffffu, diff) && lane == 0) atomicOr(bad, 1);
}

template <class IDX>
__global__ void slice_gather_dict(int64_t nslices, const int64_t* __restrict__ soff, IDX idx,
                                  const int32_t* __restrict__ rep, const int32_t* __restrict__ pat,
                                  int32_t* __restrict__ dict) {
  const int lane = threadIdx.x & 31;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices || rep[s] != s) return;
  const int64_t b = soff[s], len = soff[s + 1] - b;
  const int32_t row = static_cast<int32_t>(s * kSlice) + lane;
  for (int64_t e = lane; e < len; e += kSlice) dict[pat[s] + e] = slot_delta(idx, b + e, row);
}

// Replace the per-entry indices (int16 deltas or int32 columns) by a
// dictionary of the distinct slices' int32 delta blocks when it is small
// (<= 1M deltas) and actually saves bytes.
void try_slice_dictionary(SellMatrix& m, bool forced, cudaStream_t s) {
  static const bool off = [] {
    const char* e = std::getenv("SAIT_SELL_DICT");
    return e && std::atoi(e) == 0;
  }();
  if ((off && !forced) || (!m.dcol && !m.col) || m.nslices == 0) return;
  const int64_t ns = m.nslices;
  unsigned long long* dh = dalloc<unsigned long long>(ns, s);
  if (m.dcol) slice_hash<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx16{m.dcol}, dh);
  else slice_hash<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx32{m.col}, dh);
  SAIT_LAUNCHED();
  std::vector<unsigned long long> hh(ns);
  std::vector<int64_t> so(ns + 1);
  SAIT_CUDA(cudaMemcpyAsync(hh.data(), dh, sizeof(unsigned long long) * ns, cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaMemcpyAsync(so.data(), m.soff, sizeof(int64_t) * (ns + 1), cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  dfree(dh, s);
  std::unordered_map<unsigned long long, int32_t> first;
  first.reserve(64);
  std::vector<int32_t> rep(ns), pat(ns);
  int64_t elems = 0;
  constexpr int64_t kMaxDict = int64_t{1} << 20;
  for (int64_t q = 0; q < ns; ++q) {
    auto it = first.find(hh[q]);
    if (it == first.end()) {
      const int64_t len = so[q + 1] - so[q];
      if (elems + len > kMaxDict) return;  // too many distinct blocks: keep per-entry deltas
      it = first.emplace(hh[q], static_cast<int32_t>(q)).first;
      pat[q] = static_cast<int32_t>(elems);
      elems += len;
    } else {
      pat[q] = pat[it->second];
    }
    rep[q] = it->second;
  }
  if (elems * 4 > m.padded) return;  // little repetition: no saving
  int32_t* d = dalloc<int32_t>(2 * ns, s);
  int* bad = dalloc<int>(1, s);
  SAIT_CUDA(cudaMemcpyAsync(d, rep.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
  SAIT_CUDA(cudaMemcpyAsync(d + ns, pat.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, s));
  SAIT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  if (m.dcol) slice_verify<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx16{m.dcol}, d, bad);
  else slice_verify<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx32{m.col}, d, bad);
  SAIT_LAUNCHED();
  int hb = 0;
  SAIT_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  dfree(bad, s);
  if (hb) {  // a hash collision: keep the per-entry deltas
    dfree(d, s);
    return;
  }
  m.dict = dalloc<int32_t>(elems, s);
  m.dict_elems = elems;
  if (m.dcol)
    slice_gather_dict<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx16{m.dcol}, d, d + ns, m.dict);
  else
    slice_gather_dict<<<grid_for(ns * kSlice, 256), 256, 0, s>>>(ns, m.soff, Idx32{m.col}, d, d + ns, m.dict);
  SAIT_LAUNCHED();
  m.pat = dalloc<int32_t>(ns, s);
  SAIT_CUDA(cudaMemcpyAsync(m.pat, d + ns, sizeof(int32_t) * ns, cudaMemcpyDeviceToDevice, s));
  dfree(d, s);
  dfree(m.dcol, s);
  dfree(m.col, s);
  m.dcol = nullptr;
  m.col = nullptr;
  SAIT_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

// Rows of a ragged factor sorted by length (longest first, ties by row)
// within windows of kSigmaRows rows -- SELL-C-sigma: slices then hold rows
// of similar length, and no row moves further than the window, so the x
// gathers and y stores keep their locality.  Host side, once per pair;
// returns false (m unchanged) if the sorted slices would not pad less.
constexpr int64_t kSigmaRows = 1024;
bool sort_rows_in_windows(const DevCsr& a, SellMatrix& m, cudaStream_t s) {
  static const bool on = [] {  // SAIT_SELL_SIGMA=0: ragged factors keep the CSR kernels
    const char* e = std::getenv("SAIT_SELL_SIGMA");
    return !(e && std::atoi(e) == 0);
  }();
  if (!on) return false;
  const int64_t n = a.nrows, slots = m.nslices * kSlice;
  std::vector<int32_t> rp(n + 1);
  SAIT_CUDA(cudaMemcpyAsync(rp.data(), a.rp, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> perm(slots, static_cast<int32_t>(n));
  std::vector<int64_t> soff(m.nslices + 1, 0);
  const int64_t nwin = (n + kSigmaRows - 1) / kSigmaRows;
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nwin; ++w) {
    const int64_t r0 = w * kSigmaRows, r1 = std::min(n, r0 + kSigmaRows);
    int32_t* pw = perm.data() + r0;
    for (int64_t r = r0; r < r1; ++r) pw[r - r0] = static_cast<int32_t>(r);
    std::stable_sort(pw, pw + (r1 - r0),
                     [&](int32_t x, int32_t y) { return rp[x + 1] - rp[x] > rp[y + 1] - rp[y]; });
    for (int64_t q = r0 / kSlice; q < (r1 + kSlice - 1) / kSlice; ++q) {  // slice widths: its first (longest) row
      const int32_t r = perm[q * kSlice];
      soff[q + 1] = static_cast<int64_t>(rp[r + 1] - rp[r]) * kSlice;
    }
  }
  for (int64_t q = 0; q < m.nslices; ++q) soff[q + 1] += soff[q];
  if (soff[m.nslices] >= m.padded) return false;  // no better than the natural order
  m.padded = soff[m.nslices];
  m.perm = dalloc<int32_t>(slots, s);
  SAIT_CUDA(cudaMemcpyAsync(m.perm, perm.data(), sizeof(int32_t) * slots, cudaMemcpyHostToDevice, s));
  SAIT_CUDA(cudaMemcpyAsync(m.soff, soff.data(), sizeof(int64_t) * (m.nslices + 1), cudaMemcpyHostToDevice, s));
  SAIT_CUDA(cudaStreamSynchronize(s));  // (host vectors go out of scope)
  return true;
}

SellMatrix make_sell(const DevCsr& a, int format, cudaStream_t s, bool allow_perm) {
  SellMatrix m;
  m.n = a.nrows;
  if (a.nrows == 0 || !a.v) return m;
  m.nslices = (a.nrows + kSlice - 1) / kSlice;
  m.soff = dalloc<int64_t>(m.nslices + 1, s);
  slice_widths<<<grid_for(m.nslices, 256), 256, 0, s>>>(a.nrows, a.rp, m.nslices, m.soff);
  SAIT_LAUNCHED();
  scan_i64_inplace<<<1, 1024, 0, s>>>(m.soff, m.nslices);
  SAIT_LAUNCHED();
  SAIT_CUDA(cudaMemcpyAsync(&m.padded, m.soff + m.nslices, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  // ragged rows (padding > kSortPad): sort them by length within windows
  // when that pads markedly less (C4's factors: 24 % -> 5 %); beyond kMaxPad
  // unsorted and sorted alike: the CSR kernels
  const double nnz_d = static_cast<double>(std::max<int64_t>(a.nnz, 1));
  if (allow_perm && static_cast<double>(m.padded) > kSortPad * nnz_d + 64.0) {
    const int64_t natural = m.padded;
    std::vector<int64_t> soff_nat(m.nslices + 1);
    SAIT_CUDA(cudaMemcpyAsync(soff_nat.data(), m.soff, sizeof(int64_t) * (m.nslices + 1), cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (sort_rows_in_windows(a, m, s) && static_cast<double>(m.padded) > 0.95 * static_cast<double>(natural)) {
      dfree(m.perm, s);  // not worth the permutation: back to the natural order
      m.perm = nullptr;
      m.padded = natural;
      SAIT_CUDA(cudaMemcpyAsync(m.soff, soff_nat.data(), sizeof(int64_t) * (m.nslices + 1), cudaMemcpyHostToDevice, s));
      SAIT_CUDA(cudaStreamSynchronize(s));
    }
  }
  if (static_cast<double>(m.padded) > kMaxPad * nnz_d + 64.0) {
    dfree(m.soff, s);
    dfree(m.perm, s);
    return SellMatrix{};  // too irregular even row-sorted: keep the CSR kernels
  }
  // int16 column deltas when every |col - row| fits (and INT16_MIN is free as
  // the padding marker); SAIT_SELL_INDEX=32 forces absolute int32 columns
  int maxd = 0;
  {
    int* d = dalloc<int>(1, s);
    SAIT_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
    max_col_delta<<<grid_for(a.nrows, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, d);
    SAIT_LAUNCHED();
    SAIT_CUDA(cudaMemcpyAsync(&maxd, d, sizeof(int), cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    dfree(d, s);
  }
  static const bool force32 = [] {
    const char* e = std::getenv("SAIT_SELL_INDEX");
    return e && std::atoi(e) == 32;
  }();
  const bool want32 = format == SAIT_FMT_SELL_I32 || (format == SAIT_FMT_AUTO && force32);
  m.val = dalloc<double>(m.padded, s);
  if (maxd <= 32767 && !want32) {
    m.dcol = dalloc<int16_t>(m.padded, s);
    fill_sell16<<<grid_for(m.nslices * kSlice, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, a.v, m.soff, m.dcol, m.val,
                                                                  m.perm);
  } else {
    m.col = dalloc<int32_t>(m.padded, s);
    fill_sell<<<grid_for(m.nslices * kSlice, 256), 256, 0, s>>>(a.nrows, a.rp, a.ci, a.v, m.soff, m.col, m.val,
                                                                m.perm);
  }
  SAIT_LAUNCHED();
  SAIT_CUDA(cudaStreamSynchronize(s));
  if (!m.perm && (format == SAIT_FMT_AUTO || format == SAIT_FMT_SELL_DICT))
    try_slice_dictionary(m, format == SAIT_FMT_SELL_DICT, s);
  return m;
}

void free_sell(SellMatrix& m, cudaStream_t s) {
  dfree(m.soff, s);
  dfree(m.col, s);
  dfree(m.dcol, s);
  dfree(m.pat, s);
  dfree(m.dict, s);
  dfree(m.val, s);
  dfree(m.perm, s);
  m = SellMatrix{};
}

void sell_spmv(const SellMatrix& m, const double* x, double* y, cudaStream_t s) {
  sell_spmv_rows(m, 0, m.n, x, y, s, false);
}

void sell_spmv_rows(const SellMatrix& m, int64_t row0, int64_t row1, const double* x, double* y, cudaStream_t s,
                    bool pdl) {
  const int64_t s0 = row0 / kSlice, s1 = std::min<int64_t>((row1 + kSlice - 1) / kSlice, m.nslices);
  if (s1 <= s0) return;
  if (m.perm && (row0 != 0 || row1 < m.n))  // slots of a row-sorted copy are not row ranges
    throw std::runtime_error("sell_spmv_rows: a row range of a row-sorted SELL copy");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sell_grid(s1 - s0));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  const int pf = m.nslices >= kPfMinSlices ? kPfDistance : 0;
  if (m.dict) {
    IdxDict ix{m.pat, m.dict};
    if (pdl) SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<IdxDict, true>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
    else SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<IdxDict, false>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
  } else if (m.dcol) {
    Idx16 ix{m.dcol};
    if (pdl) SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<Idx16, true>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
    else SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<Idx16, false>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
  } else {
    Idx32 ix{m.col};
    if (pdl) SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<Idx32, true>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
    else SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_kernel<Idx32, false>, m.n, s0, s1, m.soff, ix, m.val, x, y, pf, m.perm));
  }
  SAIT_LAUNCHED();
}

template <class IDX>
void launch_halo(const SellMatrix& m, IDX ix, int64_t s0, int64_t s1, const double* x_ext, const HaloArgs& h,
                 double* y, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sell_grid(s1 - s0));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (pdl) SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_halo_kernel<IDX, true>, m.n, s0, s1, m.soff, ix, m.val, x_ext, y, h));
  else SAIT_CUDA(cudaLaunchKernelEx(&cfg, sell_spmv_halo_kernel<IDX, false>, m.n, s0, s1, m.soff, ix, m.val, x_ext, y, h));
  SAIT_LAUNCHED();
}

void sell_spmv_halo_slices(const SellMatrix& m, int64_t s0, int64_t s1, const double* x_ext, const HaloArgs& h,
                           double* y, cudaStream_t s, bool pdl) {
  s1 = std::min(s1, m.nslices);
  if (s1 <= s0) {
    if (h.pub_flag) publish_epoch(h.pub_flag, h.epoch, s);
    return;
  }
  if (m.dict) launch_halo(m, IdxDict{m.pat, m.dict}, s0, s1, x_ext, h, y, s, pdl);
  else if (m.dcol) launch_halo(m, Idx16{m.dcol}, s0, s1, x_ext, h, y, s, pdl);
  else launch_halo(m, Idx32{m.col}, s0, s1, x_ext, h, y, s, pdl);
}

void sell_spmv_halo(const SellMatrix& m, const double* x_ext, const HaloArgs& h, double* y, cudaStream_t s, bool pdl) {
  sell_spmv_halo_slices(m, 0, m.nslices, x_ext, h, y, s, pdl);
}

// Under lazy module loading (the CUDA 12 default) a kernel's first launch
// loads it, and loading synchronises the context: if a peer-halo kernel of
// another rank in this process is already spinning on a flag that this launch
// would eventually publish, that never returns.  Load every kernel of the
// peer data path up front (cudaFuncGetAttributes forces the load).
void preload_peer_kernels() {
  cudaFuncAttributes a;
  const void* fns[] = {
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<IdxDict, true>),
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<IdxDict, false>),
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<Idx16, true>),
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<Idx16, false>),
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<Idx32, true>),
      reinterpret_cast<const void*>(sell_spmv_halo_kernel<Idx32, false>),
      reinterpret_cast<const void*>(sell_spmv_kernel<IdxDict, true>),
      reinterpret_cast<const void*>(sell_spmv_kernel<IdxDict, false>),
      reinterpret_cast<const void*>(sell_spmv_kernel<Idx16, true>),
      reinterpret_cast<const void*>(sell_spmv_kernel<Idx16, false>),
      reinterpret_cast<const void*>(sell_spmv_kernel<Idx32, true>),
      reinterpret_cast<const void*>(sell_spmv_kernel<Idx32, false>),
      reinterpret_cast<const void*>(copy_slices_publish_kernel),
      reinterpret_cast<const void*>(publish_epoch_kernel),
  };
  for (const void* f : fns) SAIT_CUDA(cudaFuncGetAttributes(&a, f));
}

namespace {
// boundary slices of a row block: lo_end = 1 + the last slice with a column
// below own_lo, hi_begin = the first slice with a column >= own_hi
__global__ void halo_slice_bounds_kernel(int64_t nslices, const int64_t* __restrict__ soff, const int32_t* col,
                                         const int16_t* dcol, const int32_t* pat, const int32_t* dict,
                                         int64_t own_lo, int64_t own_hi, unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const int64_t s = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= nslices) return;
  const int64_t base = soff[s], len = soff[s + 1] - base;
  const int32_t row = static_cast<int32_t>(s * kSlice) + lane;
  bool lo = false, hi = false;
  for (int64_t e = lane; e < len; e += kSlice) {
    int32_t c;
    if (dict) {
      const int32_t d = dict[pat[s] + e];
      c = d == INT32_MIN ? -1 : row + d;
    } else if (dcol) {
      const int16_t d = dcol[base + e];
      c = d == INT16_MIN ? -1 : row + d;
    } else {
      c = col[base + e];
    }
    lo |= c >= 0 && c < own_lo;
    hi |= c >= own_hi;
  }
  const bool any_lo = __any_sync(0xffffffffu, lo), any_hi = __any_sync(0xffffffffu, hi);
  if (lane == 0) {
    if (any_lo) atomicMax(out, static_cast<unsigned long long>(s + 1));
    if (any_hi) atomicMin(out + 1, static_cast<unsigned long long>(s));
  }
}
}  // namespace

void halo_slice_bounds(const SellMatrix& m, int64_t own_lo, int64_t own_hi, int64_t* lo_end, int64_t* hi_begin,
                       cudaStream_t s) {
  unsigned long long h[2] = {0ull, static_cast<unsigned long long>(m.nslices)};
  unsigned long long* d = dalloc<unsigned long long>(2, s);
  SAIT_CUDA(cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, s));
  if (m.nslices) {
    halo_slice_bounds_kernel<<<sell_grid(m.nslices), 256, 0, s>>>(m.nslices, m.soff, m.col, m.dcol, m.pat, m.dict,
                                                                  own_lo, own_hi, d);
    SAIT_LAUNCHED();
  }
  SAIT_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, s));
  SAIT_CUDA(cudaStreamSynchronize(s));
  dfree(d, s);
  *lo_end = static_cast<int64_t>(h[0]);
  *hi_begin = static_cast<int64_t>(h[1]);
}

void copy_slices_publish(const double* src, double* dst, int64_t a0, int64_t n0, int64_t a1, int64_t n1, int* flag,
                         unsigned* count, int epoch, cudaStream_t s) {
  const int64_t tot = n0 + n1;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((tot + 1023) / 1024, 296)));
  copy_slices_publish_kernel<<<grid, 256, 0, s>>>(src, dst, a0, n0, a1, n1, flag, count, epoch);
  SAIT_LAUNCHED();
}

void publish_epoch(int* flag, int epoch, cudaStream_t s) {
  publish_epoch_kernel<<<1, 1, 0, s>>>(flag, epoch);
  SAIT_LAUNCHED();
}

namespace {
template <class IDX>
void launch_cm(const SellMatrix& m, IDX ix, const double* x, int64_t ldx, double* y, int64_t ldy, int nv,
               cudaStream_t s) {
  constexpr int wpb = CmShape<IDX>::kThreads / 32;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, (m.nslices + wpb - 1) / wpb));
  sell_spmm_cm_kernel<8, IDX><<<grid, CmShape<IDX>::kThreads, 0, s>>>(m.n, m.nslices, m.soff, ix, m.val, x, ldx, y,
                                                                      ldy, nv, m.perm);
}
}  // namespace

void sell_spmm_colmajor(const SellMatrix& m, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                        cudaStream_t s) {
  if (m.nslices == 0) return;
  for (int c0 = 0; c0 < nvec; c0 += 8) {
    const int nv = nvec - c0 < 8 ? nvec - c0 : 8;
    if (m.dict)
      launch_cm(m, IdxDict{m.pat, m.dict}, x + ldx * c0, ldx, y + ldy * c0, ldy, nv, s);
    else if (m.dcol)
      launch_cm(m, Idx16{m.dcol}, x + ldx * c0, ldx, y + ldy * c0, ldy, nv, s);
    else
      launch_cm(m, Idx32{m.col}, x + ldx * c0, ldx, y + ldy * c0, ldy, nv, s);
    SAIT_LAUNCHED();
  }
}

template <int NV, class IDX>
void launch_spmm(const SellMatrix& m, IDX ix, const double* x, double* y, cudaStream_t s) {
  sell_spmm_kernel<NV, IDX><<<sell_grid(m.nslices), 256, 0, s>>>(m.n, m.nslices, m.soff, ix, m.val, x, y, m.perm);
}

bool sell_spmm(const SellMatrix& m, const double* x, double* y, int nvec, cudaStream_t s) {
  if (m.nslices == 0) return true;
  switch (nvec) {
    case 1:
      sell_spmv(m, x, y, s);
      return true;
    case 2:
      if (m.dict) launch_spmm<2>(m, IdxDict{m.pat, m.dict}, x, y, s);
      else if (m.dcol) launch_spmm<2>(m, Idx16{m.dcol}, x, y, s);
      else launch_spmm<2>(m, Idx32{m.col}, x, y, s);
      break;
    case 4:
      if (m.dict) launch_spmm<4>(m, IdxDict{m.pat, m.dict}, x, y, s);
      else if (m.dcol) launch_spmm<4>(m, Idx16{m.dcol}, x, y, s);
      else launch_spmm<4>(m, Idx32{m.col}, x, y, s);
      break;
    case 8:
      if (m.dict) launch_spmm<8>(m, IdxDict{m.pat, m.dict}, x, y, s);
      else if (m.dcol) launch_spmm<8>(m, Idx16{m.dcol}, x, y, s);
      else launch_spmm<8>(m, Idx32{m.col}, x, y, s);
      break;
    default:
      return false;
  }
  SAIT_LAUNCHED();
  return true;
}

}  // namespace sait
