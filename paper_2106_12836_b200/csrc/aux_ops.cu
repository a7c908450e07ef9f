// aux_ops.cu — boundary helpers: index narrowing/widening at upload/download,
// CSR validation (csr.cpp:94-122), fill-cap sizes (A15), host-vector apply.
#include <cmath>

#include "common.cuh"

namespace sait {
namespace {

__global__ void narrow_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<int32_t>(in[i]);
}

__global__ void widen_kernel(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// First failing row in row order, with the reference's per-row check order:
// row_ptr decrease (1), column out of range (2), columns not increasing (3).
__global__ void validate_kernel(int64_t nrows, int64_t ncols, int64_t nnz, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ ci, unsigned long long* first) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int32_t b = rp[i], e = rp[i + 1];
  unsigned code = 0;
  if (e < b || b < 0 || e > nnz) {
    code = 1;
  } else {
    int64_t prev = -1;
    for (int32_t q = b; q < e; ++q) {
      int32_t j = ci[q];
      if (j < 0 || j >= ncols) {
        code = 2;
        break;
      }
      if (j <= prev) {
        code = 3;
        break;
      }
      prev = j;
    }
  }
  if (code) atomicMin(first, (static_cast<unsigned long long>(i) << 2) | code);
}

__global__ void cap_kernel(int64_t n, double f, int32_t* __restrict__ cnt) {
  int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) {
    double c = floor(__dmul_rn(f, static_cast<double>(cnt[j])));
    cnt[j] = c > 2147483647.0 ? 2147483647 : static_cast<int32_t>(c);
  }
}

__global__ void zc_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t n, int vec) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vec == 2) {
    if (2 * i + 1 < n) reinterpret_cast<double2*>(dst)[i] = reinterpret_cast<const double2*>(src)[i];
  } else if (i < n) {
    dst[i] = src[i];
  }
}

}  // namespace

// Diagnostics: milliseconds for device->host-mapped (dir 0) or
// host-mapped->device (dir 1) copies done by SM stores/loads.
extern "C" double sait_debug_zero_copy_ms(double* host_mapped, int64_t n, int dir, int vec) {
  double* d = nullptr;
  cudaMalloc(&d, n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t work = vec == 2 ? n / 2 : n;
  auto run = [&] {
    if (dir == 0) zc_copy_kernel<<<grid_for(work, 256), 256>>>(d, host_mapped, n, vec);
    else zc_copy_kernel<<<grid_for(work, 256), 256>>>(host_mapped, d, n, vec);
  };
  run();
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) run();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(d);
  return ms / 10.0;
}

void narrow_indices(const int64_t* in, int32_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  narrow_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  SAIT_LAUNCHED();
}

void widen_indices(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  widen_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  SAIT_LAUNCHED();
}

void validate_device_csr(const DevCsr& m, cudaStream_t s) {
  if (m.nrows == 0) return;
  unsigned long long h = ~0ull;
  unsigned long long* d = dalloc<unsigned long long>(1, s);
  SAIT_CUDA(cudaMemsetAsync(d, 0xff, sizeof h, s));  // ~0
  validate_kernel<<<grid_for(m.nrows, 256), 256, 0, s>>>(m.nrows, m.ncols, m.nnz, m.rp, m.ci, d);
  SAIT_LAUNCHED();
  read_back(s, {{&h, d, sizeof h}});
  dfree(d, s);
  if (h == ~0ull) return;
  std::string row = std::to_string(h >> 2);
  switch (h & 3) {
    case 1: throw_invalid("validate: row_ptr decreasing at row " + row);
    case 2: throw_invalid("validate: column out of range in row " + row);
    default: throw_invalid("validate: columns not strictly increasing in row " + row);
  }
}

void column_counts_add(const DevCsr& m, int32_t* cnt, cudaStream_t s);  // cap.cu

void column_caps(const DevCsr& t, double factor, int32_t* cap, cudaStream_t s) {
  SAIT_CUDA(cudaMemsetAsync(cap, 0, sizeof(int32_t) * (t.ncols ? t.ncols : 1), s));
  column_counts_add(t, cap, s);
  if (t.ncols) {
    cap_kernel<<<grid_for(t.ncols, 256), 256, 0, s>>>(t.ncols, factor, cap);
    SAIT_LAUNCHED();
  }
}

// z = M_U (M_L r) with host r / z: H2D, the pair, D2H on one stream.
void pair_apply_host_pipelined(const DevCsr& ml, const DevCsr& mu, const double* h_r, double* h_z,
                               cudaStream_t s) {
  const int64_t n = ml.ncols, m = ml.nrows;
  double* r = dalloc<double>(n, s);
  double* y = dalloc<double>(m, s);
  double* z = dalloc<double>(mu.nrows, s);
  SAIT_CUDA(cudaMemcpyAsync(r, h_r, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  spmv(ml, r, y, s);
  spmv(mu, y, z, s);
  SAIT_CUDA(cudaMemcpyAsync(h_z, z, sizeof(double) * mu.nrows, cudaMemcpyDeviceToHost, s));
  dfree(r, s);
  dfree(y, s);
  dfree(z, s);
  SAIT_CUDA(cudaStreamSynchronize(s));
}

}  // namespace sait
