// sort.cuh — small in-memory sorts of (int key, double value) pairs used to
// emit CSR rows with strictly increasing column indices (the CSR invariant of
// csr.hpp:20-22).  Keys within one row are distinct, so no stability issue.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sait {

constexpr int32_t kKeyPad = 0x7fffffff;  // padding key, sorts last

// Bitonic sort of keys[0..n2) ascending (n2 a power of two), values follow.
// Executed by `nthreads` cooperating threads with index `tid`; `sync` is the
// matching barrier (__syncwarp for one warp, __syncthreads for a block).
template <class Sync>
__device__ __forceinline__ void bitonic_sort(int32_t* keys, double* vals, int n2, int tid,
                                             int nthreads, Sync sync) {
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += nthreads) {
        int p = i ^ j;
        if (p > i) {
          bool up = (i & k) == 0;
          int32_t a = keys[i], b = keys[p];
          if ((a > b) == up) {
            keys[i] = b;
            keys[p] = a;
            double t = vals[i];
            vals[i] = vals[p];
            vals[p] = t;
          }
        }
      }
      sync();
    }
  }
}

struct WarpSync {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

__host__ __device__ __forceinline__ int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

}  // namespace sait
