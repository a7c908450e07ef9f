// common.cuh — shared device-side types and helpers of libsait_b200.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "sait_c.h"

namespace sait {

constexpr int kWarp = 32;

// Error carrying a sait_status; the C ABI turns it into a status + message.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(SAIT_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Error(SAIT_ERR_RUNTIME, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(SAIT_ERR_CUDA, std::string("cuda: ") + cudaGetErrorString(e) + " in " + what + " at " +
                                   file + ":" + std::to_string(line));
}
#define SAIT_CUDA(x) ::sait::cuda_check((x), #x, __FILE__, __LINE__)

extern std::atomic<int64_t> g_launches;
// Every kernel launch goes through this: counts it and checks the launch error.
#define SAIT_LAUNCHED()                                                   \
  do {                                                                    \
    ::sait::g_launches.fetch_add(1, std::memory_order_relaxed);          \
    ::sait::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
  } while (0)

inline cudaStream_t as_stream(sait_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Device-side range checks of derived indices, compiled in by `make checked`
// (-DSAIT_DEVICE_CHECKS): a failed check prints where and traps.  No-ops in
// the production build.
#ifdef SAIT_DEVICE_CHECKS
#define SAIT_DCHECK(cond, what, v, lim)                                                                   \
  do {                                                                                                    \
    if (!(cond)) {                                                                                        \
      printf("SAIT_DCHECK failed: %s (%lld vs %lld) at %s:%d block %d thread %d\n", what,                 \
             static_cast<long long>(v), static_cast<long long>(lim), __FILE__, __LINE__, blockIdx.x, threadIdx.x); \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
#else
#define SAIT_DCHECK(cond, what, v, lim) \
  do {                                  \
  } while (0)
#endif

// Device CSR: int32 indices, fp64 values (values may be null for a pattern).
struct DevCsr {
  int64_t nrows = 0, ncols = 0, nnz = 0;
  int32_t* rp = nullptr;
  int32_t* ci = nullptr;
  double* v = nullptr;
};

// Stream-ordered allocation from the device pool.
void debug_alloc_time(size_t bytes, double ms);  // capi.cu (SAIT_DEBUG_ALLOC)
bool debug_alloc_enabled();
template <class T>
T* dalloc(size_t count, cudaStream_t s) {
  void* p = nullptr;
  // +256 bytes: bulk copies round transfers up to whole 16-byte granules and
  // may read up to 15 bytes past the last element.
  if (debug_alloc_enabled()) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaMallocAsync(&p, count * sizeof(T) + 256, s);
    debug_alloc_time(count * sizeof(T), std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    if (e == cudaErrorMemoryAllocation) throw Error(SAIT_ERR_NOMEM, "out of device memory");
    SAIT_CUDA(e);
    return static_cast<T*>(p);
  }
  cudaError_t e = cudaMallocAsync(&p, count * sizeof(T) + 256, s);
  if (e == cudaErrorMemoryAllocation) throw Error(SAIT_ERR_NOMEM, "out of device memory");
  SAIT_CUDA(e);
  return static_cast<T*>(p);
}
inline void dfree(void* p, cudaStream_t s) {
  if (p) SAIT_CUDA(cudaFreeAsync(p, s));
}
inline void free_csr(DevCsr& m, cudaStream_t s) {
  dfree(m.rp, s);
  dfree(m.ci, s);
  dfree(m.v, s);
  m.rp = m.ci = nullptr;
  m.v = nullptr;
}

// Function attributes (dynamic shared memory limits, carve-outs) belong to a
// device context: true the first time `key` is seen on the current device
// (thread-safe; the pair build runs two host threads).
inline bool first_on_device(const void* key) {
  static std::mutex m;
  static std::vector<std::pair<int, const void*>> seen;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(m);
  for (const auto& e : seen)
    if (e.first == dev && e.second == key) return false;
  seen.emplace_back(dev, key);
  return true;
}

inline int num_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return sms;
}

// Small device -> host reads (sizes, counters, flags) through pinned
// buffers: a pageable destination makes the copy stage through the driver.
// All listed reads share one stream synchronisation.  The 4 KB pinned
// buffers live in a process-wide free list (the pair build's worker thread
// is short-lived; pinning per thread would cost more than it saves).
struct ReadItem {
  void* host;
  const void* dev;
  size_t bytes;
};
inline std::mutex& readback_mutex() {
  static std::mutex m;
  return m;
}
inline std::vector<char*>& readback_pool() {
  static std::vector<char*> v;
  return v;
}
constexpr size_t kReadbackBytes = 4096;
inline void read_back(cudaStream_t s, std::initializer_list<ReadItem> items) {
  size_t total = 0;
  for (const ReadItem& it : items) total += (it.bytes + 15) / 16 * 16;
  if (total > kReadbackBytes) throw std::runtime_error("read_back: more than 4 KB requested");
  char* buf = nullptr;
  {
    std::lock_guard<std::mutex> lk(readback_mutex());
    if (!readback_pool().empty()) {
      buf = readback_pool().back();
      readback_pool().pop_back();
    }
  }
  if (!buf && cudaMallocHost(&buf, kReadbackBytes) != cudaSuccess)
    throw std::runtime_error("read_back: cudaMallocHost failed");
  struct Return {
    char* b;
    ~Return() {
      std::lock_guard<std::mutex> lk(readback_mutex());
      readback_pool().push_back(b);
    }
  } ret{buf};
  size_t off = 0;
  for (const ReadItem& it : items) {
    cuda_check(cudaMemcpyAsync(buf + off, it.dev, it.bytes, cudaMemcpyDeviceToHost, s), "readback", __FILE__,
               __LINE__);
    off += (it.bytes + 15) / 16 * 16;
  }
  cuda_check(cudaStreamSynchronize(s), "readback sync", __FILE__, __LINE__);
  off = 0;
  for (const ReadItem& it : items) {
    std::memcpy(it.host, buf + off, it.bytes);
    off += (it.bytes + 15) / 16 * 16;
  }
}

inline unsigned grid_for(int64_t work, int per_block, int64_t cap = 1 << 30) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------- kernels API
// (implemented in the .cu files; all enqueue on `s`)

// csr_ops.cu
// exclusive scan of per-row counts into row_ptr[0..n]; returns the total
// (synchronises; throws if it exceeds the int32 index range)
int64_t scan_counts(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s);
void sort_rows(int64_t nrows, const int32_t* rp, int32_t* ci, double* v, cudaStream_t s, int64_t nnz = -1);
void exclusive_scan_rows(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s);
int64_t read_last(const int32_t* row_ptr, int64_t n, cudaStream_t s);  // syncs
DevCsr make_identity(int64_t n, cudaStream_t s);
// rows [0, rows) with a single 1.0 at column row + col0 (a block of I of order ncols)
DevCsr make_identity_rows(int64_t rows, int64_t col0, int64_t ncols, cudaStream_t s);
DevCsr transpose(const DevCsr& a, const double* row_scale, cudaStream_t s);
void scale_columns(const DevCsr& a, const double* d, DevCsr& out, cudaStream_t s);
void scale_rows(DevCsr& a, const double* d, cudaStream_t s);  // v *= d[row]
DevCsr copy_csr(const DevCsr& a, cudaStream_t s);

// split.cu
// Validates triangularity / diagonal with the reference's precedence, then
// fills inv_diag and tT (no stored diagonal).  Throws like jacobi_split.
DevCsr jacobi_split(const DevCsr& t, bool lower, double* inv_diag, cudaStream_t s);

// spgemm.cu
struct Epilogue {
  bool add_identity = false;   // insert 1.0 / add 1.0 at col == row
  int drop = 0;                // 0 none, 1 threshold, 2 pattern, 3 threshold+cap
  double tau = 0.0;
  const int32_t* prp = nullptr;  // pattern row_ptr (drop == 2)
  const int32_t* pci = nullptr;
  const int32_t* cap = nullptr;  // per-column max entries incl. diagonal (drop == 3), global index
  int64_t diag_offset = 0;       // row i's diagonal sits at column i + diag_offset (column blocks)
  // stabilization check against a previous iterate with identical shape
  const int32_t* qrp = nullptr;
  const int32_t* qci = nullptr;
  const double* qv = nullptr;
  int64_t qnnz = -1;  // its stored entries, if known: a result of another size is not stable
  // final step of a row-form build: written values are v * out_scale[col]
  // (scale_columns, kernels.cpp:236-246, fused); staging and the
  // stabilization compare see the unscaled values
  const double* out_scale = nullptr;
};
struct SpgemmResult {
  DevCsr c;
  bool changed = true;   // vs the comparison iterate (true if no comparison)
  int64_t products = 0;
};
SpgemmResult spgemm_fused(const DevCsr& a, const DevCsr& b, const Epilogue& epi, cudaStream_t s);
// drop(a I + I) for a strictly triangular square a with a threshold / no-drop
// epilogue (diag_offset 0; a cap epilogue is treated as threshold -- the
// caller guarantees it cannot bind): the first recursion step
SpgemmResult first_step_identity(const DevCsr& a, const Epilogue& epi, cudaStream_t s);

// spmv.cu
// csr_ops.cu: column-block -> row-block redistribution helpers
DevCsr assemble_rows(int nparts, const sait_row_piece* parts_host, int64_t nrows, int64_t ncols, cudaStream_t s);
void col_span(const DevCsr& a, int64_t* lo, int64_t* hi, cudaStream_t s);
void shift_columns(DevCsr& a, int64_t off, int64_t ncols, cudaStream_t s);
void row_ptr_at(const DevCsr& a, const int64_t* rows_host, int k, int64_t* out_host, cudaStream_t s);
void column_work_of(const DevCsr& t, int64_t* work, cudaStream_t s);
// sell.cu
struct SellMatrix {
  int64_t n = 0, nslices = 0, padded = 0;
  int64_t* soff = nullptr;  // nslices + 1 element offsets (multiples of 32)
  int32_t* col = nullptr;   // absolute columns, -1 marks padding ...
  int16_t* dcol = nullptr;  // ... or col - row deltas, INT16_MIN marks padding
  // ... or shared slice patterns: slice s reads its col - row deltas from
  // dict[pat[s] + k*32 + lane] (regular matrices repeat a few patterns)
  int32_t* pat = nullptr;
  int32_t* dict = nullptr;
  int64_t dict_elems = 0;
  double* val = nullptr;
  // rows too ragged for 32-row slices in their natural order: sorted by
  // length within windows of kSigmaRows rows; slot position p holds row
  // perm[p] (n: padding).  Only the whole-vector kernels take such a copy.
  int32_t* perm = nullptr;
  bool ok() const { return soff != nullptr; }
  int index_kind() const { return dict ? 2 : dcol ? 1 : 0; }  // 2 dict, 1 int16, 0 int32
};
// format: SAIT_FMT_AUTO (dictionary > int16 deltas > int32 columns, whichever
// applies; SAIT_SELL_DICT=0 / SAIT_SELL_INDEX=32 steer it) or one forced
// SAIT_FMT_SELL_* (falling back down that list when the matrix does not allow
// it).  Empty if too irregular for slicing (padding > 25%): CSR kernels.
SellMatrix make_sell(const DevCsr& a, int format, cudaStream_t s, bool allow_perm = false);
void free_sell(SellMatrix& m, cudaStream_t s);
// per 256-row group g of m: [lo[g], hi[g]] = 256-column groups its entries touch
void column_group_deps(const DevCsr& m, int32_t* lo, int32_t* hi, cudaStream_t s);
constexpr int64_t kDepGroupRows = 256;
void sell_spmv(const SellMatrix& m, const double* x, double* y, cudaStream_t s);
// row block of a sharded factor reading its halo from peer buffers (sell.cu)
struct HaloArgs {
  int64_t own_lo = 0, own_hi = 0;  // ext columns [own_lo, own_hi) are local
  const double* lo_src = nullptr;  // x[c] = lo_src[c + lo_shift] for c < own_lo
  int64_t lo_shift = 0;
  const double* hi_src = nullptr;  // x[c] = hi_src[c + hi_shift] for c >= own_hi
  int64_t hi_shift = 0;
  const int* lo_flag = nullptr;    // the owners' published epochs
  const int* hi_flag = nullptr;
  int epoch = 0;
  // optional: once every CTA's y stores are done, the last CTA publishes
  // *pub_flag = epoch (system-scope release; pub_count: a zeroed counter)
  int* pub_flag = nullptr;
  unsigned* pub_count = nullptr;
};
// x_ext: own columns read x_ext[c] (c in [own_lo, own_hi)); pdl: launched as
// a programmatic dependent of the preceding kernel (x read after its end)
void sell_spmv_halo(const SellMatrix& m, const double* x_ext, const HaloArgs& h, double* y, cudaStream_t s,
                    bool pdl = false);
// the same over slices [s0, s1) only (publishes through h.pub_flag even when empty)
void sell_spmv_halo_slices(const SellMatrix& m, int64_t s0, int64_t s1, const double* x_ext, const HaloArgs& h,
                           double* y, cudaStream_t s, bool pdl);
// force-load the peer data path's kernels (lazy module loading would
// synchronise the context at a first launch, see sell.cu)
void preload_peer_kernels();
// [0, lo_end) and [hi_begin, nslices): the slices that read halo columns
void halo_slice_bounds(const SellMatrix& m, int64_t own_lo, int64_t own_hi, int64_t* lo_end, int64_t* hi_begin,
                       cudaStream_t s);
void publish_epoch(int* flag, int epoch, cudaStream_t s);
// dst[k] = src[k] for the two boundary slices [a0, a0 + n0), [a1, a1 + n1),
// then *flag = epoch (system-scope release) once all CTAs are done
void copy_slices_publish(const double* src, double* dst, int64_t a0, int64_t n0, int64_t a1, int64_t n1, int* flag,
                         unsigned* count, int epoch, cudaStream_t s);
// rows [row0, row1) only (row0 a multiple of 32)
void sell_spmv_rows(const SellMatrix& m, int64_t row0, int64_t row1, const double* x, double* y, cudaStream_t s,
                    bool pdl = false);  // pdl: programmatic dependent of the previous kernel on s
// column-major blocks (leading dimensions ldx / ldy), any nvec
void sell_spmm_colmajor(const SellMatrix& m, const double* x, int64_t ldx, double* y, int64_t ldy, int nvec,
                        cudaStream_t s);
bool sell_spmm(const SellMatrix& m, const double* x, double* y, int nvec, cudaStream_t s);  // row-major block
void spmv(const DevCsr& a, const double* x, double* y, cudaStream_t s);
void spmm_rowmajor(const DevCsr& a, const double* x, double* y, int nvec, cudaStream_t s);
void transpose_block(const double* in, double* out, int64_t n, int nvec, bool to_rowmajor,
                     cudaStream_t s);

// trisolve.cu: synchronization-free exact triangular solve (kernels.cpp:196-234)
struct TrisolvePlan {  // per factor: rows sorted by dependency level
  int32_t* perm = nullptr;
  int64_t nlevels = 0;
};
TrisolvePlan analyse_triangular(const DevCsr& t, bool lower, cudaStream_t s);
void free_trisolve_plan(TrisolvePlan& p, cudaStream_t s);
struct TrisolveState {  // completion flags (epoch-tagged) + claim counter, per stream
  int* done = nullptr;
  unsigned long long* counter = nullptr;
  int* bad = nullptr;
  int epoch = 0;
};
void trisolve(const DevCsr& t, bool lower, const TrisolvePlan& plan, const double* b, double* x,
              TrisolveState& st, cudaStream_t s);
void free_trisolve_state(TrisolveState& st, cudaStream_t s);

// ilu.cu: ILU(k) for k = 0, 1 on the device, bitwise ilu_k(a, k) (ilu.cpp:27-173)
void ilu_device(const DevCsr& a, int level, DevCsr& L, DevCsr& U, cudaStream_t s);

// blas.cu (elementwise helpers)
void hadamard(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);  // out = a * b
void add_into(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);  // out = a + b

}  // namespace sait
