// trisolve.cu — F2: exact triangular solve on the device (the sequential
// baseline that the SAIT pair replaces; kernels.cpp:196-234,
// ExactIluPreconditioner preconditioner.cpp:28-32).
//
// Analysis (once per factor): the dependency level of every row
// (level = 1 + max level of the rows it reads), then the rows sorted by level.
// Levels come from a synchronization-free pass in solve order: a warp claims
// 32 consecutive rows, waits (acquire) for the levels of the rows outside its
// block, then resolves the dependencies inside its block with a 32-step
// shared-memory scan, and publishes the 32 levels (release).
//
// Solve: warps claim 32 rows at a time in level order from an atomic counter,
// so every row a lane waits for was claimed earlier by a running warp (no
// deadlock) and the lanes of a warp rarely wait on each other.  One lane per
// row gathers its dependencies as their epoch-tagged completion flags appear,
// then performs the reference's sequential update acc = b_i;
// acc -= t_ij * x_j (stored order, j != i); x_i = acc / t_ii — bitwise the
// reference's result.  Entries on the wrong side of the diagonal read x as 0,
// as the reference's zero-initialised vector does.
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace sait {
namespace {

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_cg(const double* p) {
  double r;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
// spin until *p satisfies pred, backing off so that the polling warps leave
// issue slots and L2 bandwidth to the warps doing work
__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <class P>
__device__ __forceinline__ int wait_for(const int* p, P pred, unsigned max_ns) {
  int v = ld_acq(p);
  if (pred(v)) return v;
  unsigned ns = 64;
  do {
    __nanosleep(ns);
    if (ns < max_ns) ns <<= 1;
    v = ld_rlx(p);
  } while (!pred(v));
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  return v;
}

constexpr int kRowRegs = 8;

__device__ __forceinline__ bool depends(bool lower, int64_t i, int64_t j) { return lower ? j < i : j > i; }

// lev[i] = 1 + max lev[j] over the rows i reads (0 = not yet known).
__global__ void __launch_bounds__(256) levels_kernel(int64_t n, bool lower, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci, int* __restrict__ lev,
                                                      int* __restrict__ count, int* __restrict__ maxlev,
                                                      unsigned long long* __restrict__ counter, unsigned max_ns) {
  __shared__ int sl[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  while (true) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(counter, 32ull);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= static_cast<unsigned long long>(n)) return;
    const int64_t k = static_cast<int64_t>(c0) + lane;
    const bool active = k < n;
    const int64_t i = lower ? k : n - 1 - k;
    int ext = 0;
    unsigned inner = 0;  // lanes of this block that row i reads
    if (active) {
      for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = ci[e];
        if (!depends(lower, i, j)) continue;
        const int64_t kj = lower ? j : n - 1 - j;  // solve position of j (< k)
        if (kj >= static_cast<int64_t>(c0)) {
          inner |= 1u << static_cast<int>(kj - static_cast<int64_t>(c0));
        } else {
          ext = max(ext, wait_for(lev + j, [](int v) { return v != 0; }, max_ns));
        }
      }
    }
    // resolve in-block dependencies in solve order
    int mine = 0;
    for (int t = 0; t < 32; ++t) {
      if (lane == t) {
        int m = ext;
        for (unsigned bits = inner; bits; bits &= bits - 1) m = max(m, sl[w][__ffs(bits) - 1]);
        mine = m + 1;
        sl[w][t] = mine;
      }
      __syncwarp();
    }
    if (active) {
      st_rel(lev + i, mine);
      atomicAdd(count + (mine - 1), 1);
      atomicMax(maxlev, mine);
    }
    __syncwarp();
  }
}

__global__ void scatter_by_level(int64_t n, const int* __restrict__ lev, int32_t* __restrict__ cursor,
                                 int32_t* __restrict__ perm) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) perm[atomicAdd(cursor + (lev[i] - 1), 1)] = static_cast<int32_t>(i);
}

__global__ void __launch_bounds__(256) sptrsv_levels(int64_t n, bool lower, const int32_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci, const double* __restrict__ v,
                                                      const int32_t* __restrict__ perm,
                                                      const double* __restrict__ b, double* __restrict__ x,
                                                      int* __restrict__ done, int epoch,
                                                      unsigned long long* __restrict__ counter,
                                                      int* __restrict__ bad_pos, unsigned max_ns) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(counter, 32ull);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= static_cast<unsigned long long>(n)) return;
    const int64_t k = static_cast<int64_t>(c0) + lane;
    if (k < n) {
      const int64_t i = perm[k];
      const int32_t e0 = rp[i], e1 = rp[i + 1];
      double acc = b[i], diag = 0.0;
      bool have = false;
      if (e1 - e0 <= kRowRegs) {
        // short row: entries in registers, all dependency flags polled together,
        // all x loads in flight together, then the ordered update
        int32_t cj[kRowRegs];
        double cv[kRowRegs], xv[kRowRegs];
#pragma unroll
        for (int q = 0; q < kRowRegs; ++q) {
          cj[q] = e0 + q < e1 ? ci[e0 + q] : static_cast<int32_t>(i);
          cv[q] = e0 + q < e1 ? v[e0 + q] : 0.0;
        }
        unsigned ns = 32;
        while (true) {
          bool ready = true;
#pragma unroll
          for (int q = 0; q < kRowRegs; ++q)
            if (depends(lower, i, cj[q]) && ld_rlx(done + cj[q]) != epoch) ready = false;
          if (ready) break;
          __nanosleep(ns);
          if (ns < max_ns) ns <<= 1;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
        for (int q = 0; q < kRowRegs; ++q) xv[q] = depends(lower, i, cj[q]) ? ld_cg(x + cj[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < kRowRegs; ++q) {
          if (e0 + q >= e1) break;
          if (cj[q] == i) {
            diag = cv[q];
            have = true;
          } else {
            acc = __dsub_rn(acc, __dmul_rn(cv[q], xv[q]));
          }
        }
      } else {
        for (int32_t e = e0; e < e1; ++e) {
          const int32_t j = ci[e];
          if (j == i) {
            diag = v[e];
            have = true;
            continue;
          }
          double xj = 0.0;
          if (depends(lower, i, j)) {
            wait_for(done + j, [epoch](int f) { return f == epoch; }, max_ns);
            xj = ld_cg(x + j);
          }
          acc = __dsub_rn(acc, __dmul_rn(v[e], xj));
        }
      }
      if (!have || diag == 0.0) {
        atomicMin(bad_pos, static_cast<int>(lower ? i : n - 1 - i));  // first failing row in solve order
        x[i] = 0.0;
      } else {
        x[i] = __ddiv_rn(acc, diag);
      }
      st_rel(done + i, epoch);
    }
  }
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Resident warps poll while they wait: more warps than a few levels' worth of
// rows only adds polling traffic to L2, so the grid is capped
// (SAIT_TRSV_BLOCKS_PER_SM for the solve, SAIT_TRSV_ANALYSIS_BLOCKS_PER_SM
// for the level pass; 0 = occupancy limit).
unsigned resident_grid(const void* kernel, int64_t n, const char* env, int dflt) {
  int per_sm = 0;
  SAIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
  const int cap = env_int(env, dflt);
  if (cap > 0) per_sm = std::min(per_sm, cap);
  const int64_t blocks_needed = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(
      1, std::min<int64_t>(int64_t{std::max(per_sm, 1)} * num_sms(), blocks_needed)));
}

}  // namespace

TrisolvePlan analyse_triangular(const DevCsr& t, bool lower, cudaStream_t s) {
  TrisolvePlan p;
  const int64_t n = t.nrows;
  if (n == 0) return p;
  int* lev = dalloc<int>(n, s);
  int* count = dalloc<int>(n + 1, s);
  int* maxlev = dalloc<int>(1, s);
  unsigned long long* counter = dalloc<unsigned long long>(1, s);
  SAIT_CUDA(cudaMemsetAsync(lev, 0, sizeof(int) * n, s));
  SAIT_CUDA(cudaMemsetAsync(count, 0, sizeof(int) * (n + 1), s));
  SAIT_CUDA(cudaMemsetAsync(maxlev, 0, sizeof(int), s));
  SAIT_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
  levels_kernel<<<resident_grid(reinterpret_cast<const void*>(levels_kernel), n, "SAIT_TRSV_ANALYSIS_BLOCKS_PER_SM", 0), 256, 0, s>>>(
      n, lower, t.rp, t.ci, lev, count, maxlev, counter, static_cast<unsigned>(env_int("SAIT_TRSV_ANALYSIS_SLEEP_NS", 1024)));
  SAIT_LAUNCHED();
  int32_t* start = dalloc<int32_t>(n + 1, s);
  scan_counts(count, start, n, s);  // level l's rows go to [start[l-1], start[l])
  p.perm = dalloc<int32_t>(n, s);
  scatter_by_level<<<grid_for(n, 256), 256, 0, s>>>(n, lev, start, p.perm);
  SAIT_LAUNCHED();
  int h = 0;
  read_back(s, {{&h, maxlev, sizeof(int)}});
  p.nlevels = h;
  dfree(lev, s);
  dfree(count, s);
  dfree(maxlev, s);
  dfree(counter, s);
  dfree(start, s);
  return p;
}

void free_trisolve_plan(TrisolvePlan& p, cudaStream_t s) {
  dfree(p.perm, s);
  p = TrisolvePlan{};
}

// x = T^-1 b (lower or upper); throws like trisolve on a zero/missing diagonal.
void trisolve(const DevCsr& t, bool lower, const TrisolvePlan& plan, const double* b, double* x,
              TrisolveState& st, cudaStream_t s) {
  const int64_t n = t.nrows;
  if (n == 0) return;
  if (!st.done) {
    st.done = dalloc<int>(n, s);
    st.counter = dalloc<unsigned long long>(1, s);
    st.bad = dalloc<int>(1, s);
    SAIT_CUDA(cudaMemsetAsync(st.done, 0, sizeof(int) * n, s));
  }
  SAIT_CUDA(cudaMemsetAsync(st.counter, 0, sizeof(unsigned long long), s));
  SAIT_CUDA(cudaMemsetAsync(st.bad, 0x7f, sizeof(int), s));
  const int epoch = ++st.epoch;
  sptrsv_levels<<<resident_grid(reinterpret_cast<const void*>(sptrsv_levels), n, "SAIT_TRSV_BLOCKS_PER_SM", 1), 256, 0, s>>>(
      n, lower, t.rp, t.ci, t.v, plan.perm, b, x, st.done, epoch, st.counter, st.bad,
      static_cast<unsigned>(env_int("SAIT_TRSV_SLEEP_NS", 2048)));
  SAIT_LAUNCHED();
  int hb = 0;
  read_back(s, {{&hb, st.bad, sizeof(int)}});
  if (hb != 0x7f7f7f7f) {
    const int64_t row = lower ? hb : n - 1 - hb;
    throw_runtime("trisolve: singular matrix, zero diagonal at row " + std::to_string(row));
  }
}

void free_trisolve_state(TrisolveState& st, cudaStream_t s) {
  dfree(st.done, s);
  dfree(st.counter, s);
  dfree(st.bad, s);
  st = TrisolveState{};
}

}  // namespace sait
