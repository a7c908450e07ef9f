// ilu.cu — F1: ILU(0) on the device, bitwise the reference's factors
// (ilu.hpp:27, ilu.cpp:98-173 with level 0: the factors keep A's pattern).
//
// Row i of the IKJ elimination reads the finished U rows k of the columns k
// in its strictly lower part and nothing else, so the rows form the same
// dependency DAG as a lower triangular solve on A's pattern.  The rows are
// processed in level order (trisolve.cu's analysis) by one lane each, which
// waits for the completion flags of its rows k and then performs exactly the
// reference's operation sequence on its own row (in place, in A's layout):
//   for k in L(i) ascending:  f = w_k / u_kk;  w_k = f;
//                              for j in U(k), j != k, j in row i:  w_j -= f * u_kj
// so every value is rounded as in the reference.  A final pass splits the
// rows into L (strict part + explicit unit diagonal) and U (diagonal and up).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"

namespace sait {
namespace {

__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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

// diag[i] = position of (i, i) in row i, or -1; first missing row -> *bad
__global__ void find_diagonal(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                              int32_t* __restrict__ diag, int* __restrict__ bad) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t lo = rp[i], hi = rp[i + 1];
  while (lo < hi) {  // first column >= i (columns strictly increase)
    const int32_t mid = (lo + hi) >> 1;
    if (ci[mid] < i) lo = mid + 1;
    else hi = mid;
  }
  const bool ok = lo < rp[i + 1] && ci[lo] == i;
  diag[i] = ok ? lo : -1;
  if (!ok) atomicMin(bad, static_cast<int>(i));
}

// max |a_ij| over the stored values; NaN is skipped like std::max(max, NaN)
__global__ void max_abs_kernel(int64_t nnz, const double* __restrict__ v, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double a = fabs(v[e]);
    if (m < a) m = a;  // std::max(m, a) = (m < a) ? a : m
  }
  for (int o = 16; o; o >>= 1) {
    const double b = __shfl_xor_sync(0xffffffffu, m, o);
    if (m < b) m = b;
  }
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

constexpr int kRowSmem = 32;  // rows up to this length work in shared memory
constexpr int kIluSmem = 256 * kRowSmem * (sizeof(double) + sizeof(int32_t));

__global__ void __launch_bounds__(256) ilu0_rows(int64_t n, const int32_t* __restrict__ rp,
                                                  const int32_t* __restrict__ ci, const int32_t* __restrict__ diag,
                                                  const int32_t* __restrict__ perm, double* __restrict__ w,
                                                  double* __restrict__ pivot, int* __restrict__ done,
                                                  unsigned long long* __restrict__ counter, double tol,
                                                  int* __restrict__ bad, unsigned max_ns) {
  extern __shared__ __align__(16) unsigned char ilu_smem[];  // kIluSmem bytes
  double (*sw)[kRowSmem] = reinterpret_cast<double (*)[kRowSmem]>(ilu_smem);
  int32_t (*sc)[kRowSmem] = reinterpret_cast<int32_t (*)[kRowSmem]>(ilu_smem + 256 * kRowSmem * sizeof(double));
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long c0 = 0;
    if (lane == 0) c0 = atomicAdd(counter, 32ull);
    c0 = __shfl_sync(0xffffffffu, c0, 0);
    if (c0 >= static_cast<unsigned long long>(n)) return;
    const int64_t kk = static_cast<int64_t>(c0) + lane;
    if (kk >= n) continue;
    const int32_t i = perm[kk];
    const int32_t e0 = rp[i], e1 = rp[i + 1], d = diag[i];
    // wait for every pivot row this row eliminates against
    unsigned ns = 32;
    while (true) {
      int pending = 0;
#pragma unroll 4
      for (int32_t p = e0; p < d; ++p) pending += ld_rlx(done + ci[p]) == 0;
      if (!pending) break;
      __nanosleep(ns);
      if (ns < max_ns) ns <<= 1;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const int32_t len = e1 - e0;
    if (len <= kRowSmem) {
      // the row's columns and values in this lane's shared-memory slots; each
      // U(k) row is fetched 8 entries at a time with all loads in flight, then
      // merged -- the same operations in the same order as below
      int32_t* rc = sc[threadIdx.x];
      double* rw = sw[threadIdx.x];
      for (int32_t q = 0; q < len; ++q) {
        rc[q] = ci[e0 + q];
        rw[q] = w[e0 + q];
      }
      for (int32_t p = 0; p < d - e0; ++p) {
        const int32_t k = rc[p];
        const int32_t q0 = diag[k] + 1, q1 = rp[k + 1];
        const double f = __ddiv_rn(rw[p], ld_cg(pivot + k));
        rw[p] = f;
        int32_t at = p + 1;
        for (int32_t qb = q0; qb < q1 && at < len; qb += 8) {
          int32_t cj[8];
          double uv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            cj[u] = qb + u < q1 ? ci[qb + u] : INT32_MAX;
            uv[u] = qb + u < q1 ? ld_cg(w + qb + u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int32_t j = cj[u];
            while (at < len && rc[at] < j) ++at;
            if (at < len && rc[at] == j) rw[at] = __dsub_rn(rw[at], __dmul_rn(f, uv[u]));
          }
        }
      }
      for (int32_t q = 0; q < len; ++q) w[e0 + q] = rw[q];
    } else {
      for (int32_t p = e0; p < d; ++p) {
        const int32_t k = ci[p];
        const double f = __ddiv_rn(w[p], ld_cg(pivot + k));
        w[p] = f;
        // U(k) = entries after k's diagonal (ascending); merge into row i's tail
        const int32_t q1 = rp[k + 1];
        int32_t at = p + 1;
        for (int32_t q = diag[k] + 1; q < q1 && at < e1; ++q) {
          const int32_t j = ci[q];
          while (at < e1 && ci[at] < j) ++at;
          if (at < e1 && ci[at] == j) w[at] = __dsub_rn(w[at], __dmul_rn(f, ld_cg(w + q)));
        }
      }
    }
    const double piv = w[d];
    if (piv == 0.0 || fabs(piv) < tol) atomicMin(bad, i);
    pivot[i] = piv;
    st_rel(done + i, 1);
  }
}

// L row i = strict lower part + unit diagonal; U row i = diagonal onward
__global__ void split_counts(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ diag,
                             int32_t* __restrict__ lc, int32_t* __restrict__ uc) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  lc[i] = diag[i] - rp[i] + 1;
  uc[i] = rp[i + 1] - diag[i];
}

__global__ void split_fill(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ w, const int32_t* __restrict__ diag,
                           const int32_t* __restrict__ lrp, int32_t* __restrict__ lci, double* __restrict__ lv,
                           const int32_t* __restrict__ urp, int32_t* __restrict__ uci, double* __restrict__ uv) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t e0 = rp[i], d = diag[i], e1 = rp[i + 1];
  int32_t o = lrp[i];
  for (int32_t e = e0; e < d; ++e, ++o) {
    lci[o] = ci[e];
    lv[o] = w[e];
  }
  lci[o] = static_cast<int32_t>(i);
  lv[o] = 1.0;
  o = urp[i];
  for (int32_t e = d; e < e1; ++e, ++o) {
    uci[o] = ci[e];
    uv[o] = w[e];
  }
}

// ILU(1) pattern helpers: Lp = tril(A, -1) + I, Up = triu(A, 1) + I (values
// 1.0) so that pattern(Lp Up) = pattern(A) U {(i, j): a_ik != 0, a_kj != 0,
// k < i, k < j}, the level <= 1 fill of ilu.cpp:27-91 (fill through level-1
// entries would have level 2).
__global__ void tri_plus_identity_counts(int64_t n, const int32_t* __restrict__ rp,
                                         const int32_t* __restrict__ diag, int32_t* __restrict__ lc,
                                         int32_t* __restrict__ uc) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  lc[i] = diag[i] - rp[i] + 1;
  uc[i] = rp[i + 1] - diag[i];
}
__global__ void tri_plus_identity_fill(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                       const int32_t* __restrict__ diag, const int32_t* __restrict__ lrp,
                                       int32_t* __restrict__ lci, double* __restrict__ lv,
                                       const int32_t* __restrict__ urp, int32_t* __restrict__ uci,
                                       double* __restrict__ uv) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t o = lrp[i];
  for (int32_t e = rp[i]; e < diag[i]; ++e, ++o) {
    lci[o] = ci[e];
    lv[o] = 1.0;
  }
  lci[o] = static_cast<int32_t>(i);
  lv[o] = 1.0;
  o = urp[i];
  for (int32_t e = diag[i]; e < rp[i + 1]; ++e, ++o) {  // the diagonal first, then j > i
    uci[o] = ci[e];
    uv[o] = 1.0;
  }
}
// w = 0 on the fill pattern P, then A's values at their positions (both rows sorted)
__global__ void scatter_into_pattern(int64_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                     const double* __restrict__ av, const int32_t* __restrict__ prp,
                                     const int32_t* __restrict__ pci, double* __restrict__ w) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t q = prp[i];
  const int32_t q1 = prp[i + 1];
  for (int32_t e = q; e < q1; ++e) w[e] = 0.0;
  for (int32_t e = arp[i]; e < arp[i + 1]; ++e) {
    while (q < q1 && pci[q] < aci[e]) ++q;
    w[q] = av[e];  // A's pattern is contained in P
  }
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

}  // namespace

void ilu_device(const DevCsr& a, int level, DevCsr& L, DevCsr& U, cudaStream_t s) {
  if (a.nrows != a.ncols) throw_invalid("ilu_k: matrix is not square");
  if (level < 0) throw_invalid("ilu_k: negative fill level");
  if (level > 1) throw_invalid("ilu_k: the device factorization supports fill levels 0 and 1 (use the host ilu_k)");
  const int64_t n = a.nrows;
  L = DevCsr{};
  U = DevCsr{};
  L.nrows = L.ncols = U.nrows = U.ncols = n;
  if (n == 0) {
    L.rp = dalloc<int32_t>(1, s);
    U.rp = dalloc<int32_t>(1, s);
    SAIT_CUDA(cudaMemsetAsync(L.rp, 0, sizeof(int32_t), s));
    SAIT_CUDA(cudaMemsetAsync(U.rp, 0, sizeof(int32_t), s));
    L.ci = dalloc<int32_t>(1, s);
    U.ci = dalloc<int32_t>(1, s);
    L.v = dalloc<double>(1, s);
    U.v = dalloc<double>(1, s);
    return;
  }
  int32_t* diag = dalloc<int32_t>(n, s);
  int* flags = dalloc<int>(n + 2, s);  // done[0..n), bad diagonal, bad pivot
  unsigned long long* scratch = dalloc<unsigned long long>(2, s);  // max |a| bits, claim counter
  double* w = nullptr;
  double* pivot = nullptr;
  TrisolvePlan plan;
  int32_t *lc = nullptr, *uc = nullptr;
  DevCsr owned_pattern;  // level 1: the fill pattern (level 0 borrows A's)
  auto cleanup = [&] {
    free_csr(owned_pattern, s);
    dfree(diag, s);
    dfree(flags, s);
    dfree(scratch, s);
    dfree(w, s);
    dfree(pivot, s);
    dfree(lc, s);
    dfree(uc, s);
    free_trisolve_plan(plan, s);
  };
  try {
    int* done = flags;
    int* bad = flags + n;
    SAIT_CUDA(cudaMemsetAsync(done, 0, sizeof(int) * n, s));
    SAIT_CUDA(cudaMemsetAsync(bad, 0x7f, sizeof(int) * 2, s));
    SAIT_CUDA(cudaMemsetAsync(scratch, 0, sizeof(unsigned long long) * 2, s));
    find_diagonal<<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, a.ci, diag, bad);
    SAIT_LAUNCHED();
    if (a.nnz) {
      max_abs_kernel<<<grid_for(a.nnz, 256, int64_t{4} * num_sms() * 8), 256, 0, s>>>(a.nnz, a.v, scratch);
      SAIT_LAUNCHED();
    }
    int hb[2];
    unsigned long long amax_bits = 0;
    read_back(s, {{hb, bad, sizeof hb}, {&amax_bits, scratch, sizeof amax_bits}});
    if (hb[0] != 0x7f7f7f7f)
      throw_invalid("ilu_k: structurally zero diagonal at row " + std::to_string(hb[0]));
    double amax;
    std::memcpy(&amax, &amax_bits, sizeof amax);
    const double tol = 1e-14 * amax;  // kPivotBreakdownFactor * max_abs (ilu.cpp:107-108)

    // the factorization pattern P: A's (level 0) or A's plus level-1 fill
    DevCsr P = a;  // borrowed for level 0
    if (level == 1) {
      lc = dalloc<int32_t>(n, s);
      uc = dalloc<int32_t>(n, s);
      tri_plus_identity_counts<<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, diag, lc, uc);
      SAIT_LAUNCHED();
      DevCsr lp, up;
      lp.nrows = lp.ncols = up.nrows = up.ncols = n;
      lp.rp = dalloc<int32_t>(n + 1, s);
      up.rp = dalloc<int32_t>(n + 1, s);
      lp.nnz = scan_counts(lc, lp.rp, n, s);
      up.nnz = scan_counts(uc, up.rp, n, s);
      lp.ci = dalloc<int32_t>(lp.nnz, s);
      lp.v = dalloc<double>(lp.nnz, s);
      up.ci = dalloc<int32_t>(up.nnz, s);
      up.v = dalloc<double>(up.nnz, s);
      tri_plus_identity_fill<<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, a.ci, diag, lp.rp, lp.ci, lp.v, up.rp, up.ci,
                                                               up.v);
      SAIT_LAUNCHED();
      SpgemmResult pr = spgemm_fused(lp, up, Epilogue{}, s);  // all-positive values: no cancellation
      free_csr(lp, s);
      free_csr(up, s);
      dfree(lc, s);
      dfree(uc, s);
      lc = uc = nullptr;
      P = pr.c;
      owned_pattern = P;
      find_diagonal<<<grid_for(n, 256), 256, 0, s>>>(n, P.rp, P.ci, diag, bad);  // diagonal positions in P
      SAIT_LAUNCHED();
    }
    w = dalloc<double>(P.nnz, s);
    pivot = dalloc<double>(n, s);
    if (level == 0) {
      SAIT_CUDA(cudaMemcpyAsync(w, a.v, sizeof(double) * a.nnz, cudaMemcpyDeviceToDevice, s));
    } else {
      scatter_into_pattern<<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, a.ci, a.v, P.rp, P.ci, w);
      SAIT_LAUNCHED();
    }
    plan = analyse_triangular(P, true, s);
    int per_sm = 0;
    SAIT_CUDA(cudaFuncSetAttribute(ilu0_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, kIluSmem));
    SAIT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ilu0_rows, 256, kIluSmem));
    per_sm = std::max(1, std::min(per_sm, env_int("SAIT_ILU_BLOCKS_PER_SM", 1)));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(int64_t{per_sm} * num_sms(), (n + 255) / 256));
    ilu0_rows<<<grid, 256, kIluSmem, s>>>(n, P.rp, P.ci, diag, plan.perm, w, pivot, done, scratch + 1, tol, bad + 1,
                                   static_cast<unsigned>(env_int("SAIT_ILU_SLEEP_NS", 2048)));
    SAIT_LAUNCHED();
    read_back(s, {{hb, bad, sizeof hb}});
    if (hb[1] != 0x7f7f7f7f) {
      double piv = 0.0;
      SAIT_CUDA(cudaMemcpyAsync(&piv, pivot + hb[1], sizeof piv, cudaMemcpyDeviceToHost, s));
      SAIT_CUDA(cudaStreamSynchronize(s));
      char buf[64];
      std::snprintf(buf, sizeof buf, "%f", std::fabs(piv));
      throw_runtime("ilu_k: pivot breakdown at row " + std::to_string(hb[1]) + " (|pivot| = " + buf + ")");
    }
    lc = dalloc<int32_t>(n, s);
    uc = dalloc<int32_t>(n, s);
    split_counts<<<grid_for(n, 256), 256, 0, s>>>(n, P.rp, diag, lc, uc);
    SAIT_LAUNCHED();
    L.rp = dalloc<int32_t>(n + 1, s);
    U.rp = dalloc<int32_t>(n + 1, s);
    L.nnz = scan_counts(lc, L.rp, n, s);
    U.nnz = scan_counts(uc, U.rp, n, s);
    L.ci = dalloc<int32_t>(L.nnz, s);
    L.v = dalloc<double>(L.nnz, s);
    U.ci = dalloc<int32_t>(U.nnz, s);
    U.v = dalloc<double>(U.nnz, s);
    split_fill<<<grid_for(n, 256), 256, 0, s>>>(n, P.rp, P.ci, w, diag, L.rp, L.ci, L.v, U.rp, U.ci, U.v);
    SAIT_LAUNCHED();
  } catch (...) {
    cleanup();
    free_csr(L, s);
    free_csr(U, s);
    throw;
  }
  cleanup();
}

}  // namespace sait
