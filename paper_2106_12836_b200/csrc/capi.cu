// capi.cu — the C ABI of include/sait_c.h over the device kernels.
// Each entry point cites the reference interface it replaces (paths relative
// to /root/reference/proj/core/).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <omp.h>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <thread>
#include <unordered_map>
#include <utility>
#include <string>
#include <vector>

#include "common.cuh"

namespace sait {
bool debug_alloc_enabled() {
  static const bool on = std::getenv("SAIT_DEBUG_ALLOC") != nullptr;
  return on;
}
void debug_alloc_time(size_t bytes, double ms) {
  if (ms > 1.0) std::fprintf(stderr, "[alloc] %.1f MB took %.2f ms\n", bytes / 1e6, ms);
}
}  // namespace sait


struct sait_dcsr_s {
  int dev = 0;
  sait::DevCsr m;
};

struct sait_op_s {
  int dev = 0;
  sait_dcsr_s* a = nullptr;
  bool owns = false;
  sait::SellMatrix sell;
};

struct sait_exact_s {
  int dev = 0;
  sait_dcsr_s* l = nullptr;
  sait_dcsr_s* u = nullptr;
  bool owns = false;
  sait::TrisolvePlan pl, pu;  // level order of each factor (analysed at create)
  struct Work {
    double* y = nullptr;
    sait::TrisolveState sl, su;
    // applies on one stream from several threads take turns (each apply
    // reuses this stream's buffers and flags)
    std::shared_ptr<std::mutex> mu = std::make_shared<std::mutex>();
  };
  std::mutex mu;
  std::unordered_map<cudaStream_t, Work> ws;  // per-stream flags + y
};

namespace {
class Recursion;
}  // namespace
namespace sait {
void exact_apply_internal(sait_exact_t p, const double* r, double* z, cudaStream_t s);
}
struct sait_build_session_s {
  int dev = 0;
  cudaStream_t s = nullptr;
  int64_t c0 = 0, c1 = 0, n = 0;
  double* inv = nullptr;
  sait::DevCsr ttT;  // the recursion's fixed operand: tT^T, or tT in row form
  bool row_form = false;
  int32_t* cap = nullptr;
  Recursion* rec = nullptr;
  cudaEvent_t e0 = nullptr;
};

struct sait_pair_s {
  int dev = 0;
  sait_dcsr_s* ml = nullptr;
  sait_dcsr_s* mu = nullptr;
  bool owns = false;
  sait::SellMatrix sl, su;  // SELL-32 copies used by the apply (empty: CSR kernels)
  // per-stream scratch (y = M_L r): applies on one stream are ordered, so one
  // buffer per stream honours the concurrent-apply contract
  struct Work {
    // applies on one stream from several threads take turns (they share
    // this stream's y, staging buffers and flags)
    std::shared_ptr<std::mutex> mu = std::make_shared<std::mutex>();
    double* y = nullptr;
    // host-vector pipeline (lazily created)
    cudaStream_t s_in = nullptr, s_out = nullptr;
    double *r_dev = nullptr, *z_dev = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_u;
    cudaEvent_t ev_entry = nullptr, ev_out_done = nullptr;
    // column-major host block apply: kBlkSlots device slots per side
    double *blk_r = nullptr, *blk_z = nullptr;
    double *pin_r = nullptr, *pin_z = nullptr;  // pinned staging of pageable caller blocks
    size_t pin_r_elems = 0, pin_z_elems = 0;
    cudaEvent_t ev_blk_in[4] = {}, ev_blk_done[4] = {}, ev_blk_out[4] = {};
  };
  // chunking of the host-vector apply: row boundaries (multiples of 256) and,
  // per chunk, the last r-chunk M_L needs and the last y-chunk M_U needs
  std::vector<int64_t> chunk_rows, u_rows;
  std::vector<int32_t> needL_hi;
  std::mutex mu_ws;
  std::unordered_map<cudaStream_t, Work> ws;
};

namespace sait {
int64_t scan_counts(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s);
void validate_device_csr(const DevCsr& m, cudaStream_t s);
void narrow_indices(const int64_t* in, int32_t* out, int64_t n, cudaStream_t s);
void widen_indices(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s);
void column_caps(const DevCsr& t, double factor, int32_t* cap, cudaStream_t s);
int64_t cap_rowform(DevCsr& m, const int32_t* cap, cudaStream_t s, const double* out_scale, bool* scaled);
bool csr_stabilized(const DevCsr& prev, const DevCsr& cur, cudaStream_t s);
void pair_apply_host_pipelined(const DevCsr& ml, const DevCsr& mu, const double* h_r, double* h_z,
                               cudaStream_t s);
}  // namespace sait

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SAIT_OK;
  } catch (const sait::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return SAIT_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SAIT_ERR_RUNTIME;
  }
}

// Grow the stream-ordered pool once by `bytes` (one allocation, freed back
// into the pool and kept, the release threshold being unlimited), so later
// builds carve their buffers out of existing mappings instead of paying for
// new ones allocation by allocation (the first builds of a process).
void reserve_pool(cudaMemPool_t pool, size_t bytes) {
  void* p = nullptr;
  if (bytes && cudaMallocFromPoolAsync(&p, bytes, pool, nullptr) == cudaSuccess) {
    cudaFreeAsync(p, nullptr);
    cudaStreamSynchronize(nullptr);
  }
  cudaGetLastError();
}

// Grows the pool to `bytes` in one bulk mapping when it holds less: a fresh
// process's first build otherwise maps its working set allocation by
// allocation (~6.5 GB/s; the first config-4 build took 0.27 s against
// 0.14 s warm, one bulk 12 GiB mapping 0.07 s).  Capped at 80 % of the free
// device memory; the pool keeps what it maps (release threshold unlimited),
// as it would after the incremental growth.
void ensure_pool(size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t have = 0;
  cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &have);
  if (have >= bytes) return;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return;
  const size_t want = std::min(bytes, have + free_b / 10 * 8);
  if (want > have) reserve_pool(pool, want);
}

void init_device_pool() {
  static std::once_flag once[64];
  int dev = 0;
  SAIT_CUDA(cudaGetDevice(&dev));
  std::call_once(once[dev & 63], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      if (const char* e = std::getenv("SAIT_POOL_RESERVE_MB"))
        reserve_pool(pool, static_cast<size_t>(std::max(0LL, std::atoll(e))) << 20);
    }
  });
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    SAIT_CUDA(cudaGetDevice(&prev));
    if (prev != dev) SAIT_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

sait_dcsr_s* wrap(const sait::DevCsr& m) {
  auto* h = new sait_dcsr_s;
  SAIT_CUDA(cudaGetDevice(&h->dev));
  h->m = m;
  return h;
}

void need(const void* p, const char* what) {
  if (!p) sait::throw_invalid(std::string(what) + ": null handle or pointer");
}

std::string fmt_double(double v) {  // std::to_string(double) == "%f"
  char b[64];
  std::snprintf(b, sizeof b, "%f", v);
  return b;
}

void host_csr_alloc(sait_host_csr* out, int64_t nrows, int64_t ncols, int64_t nnz, bool values) {
  out->nrows = nrows;
  out->ncols = ncols;
  out->row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (nrows + 1)));
  out->col_idx = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (nnz ? nnz : 1)));
  out->values = values ? static_cast<double*>(std::malloc(sizeof(double) * (nnz ? nnz : 1))) : nullptr;
  if (!out->row_ptr || !out->col_idx || (values && !out->values)) throw std::bad_alloc();
}

// Host <-> device CSR transfers (the drop-in API takes and returns int64 /
// fp64 host matrices, csr.hpp:24-43): chunked through two pinned staging
// buffers per device, so the PCIe copy of one chunk overlaps the host-side
// narrowing (int64 -> int32, out-of-range indices -> -1, which validation
// then reports) / widening / copying of the next, which runs on all host
// cores (OpenMP).  Pageable copies go through the driver's own staging at a
// few GB/s and fault in fresh pages one by one; this moves 4 of the 12 bytes
// of an index as int32 across the bus and touches the user's pages in
// parallel.
namespace {
constexpr size_t kStageBytes = size_t{32} << 20;
struct Staging {
  std::mutex mu;
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
};
Staging& staging() {
  static Staging st[64];
  int dev = 0;
  SAIT_CUDA(cudaGetDevice(&dev));
  Staging& x = st[dev & 63];
  if (!x.buf[0]) {
    for (int b = 0; b < 2; ++b) {
      SAIT_CUDA(cudaMallocHost(&x.buf[b], kStageBytes));
      SAIT_CUDA(cudaEventCreateWithFlags(&x.done[b], cudaEventDisableTiming));
    }
  }
  return x;
}
// dev_dst[0, count) <- fill(pinned, first, n) chunk by chunk
template <class Fill>
void staged_h2d(Staging& st, char* dev_dst, int64_t count, size_t elem, Fill fill, cudaStream_t s) {
  const int64_t per = static_cast<int64_t>(kStageBytes / elem);
  int k = 0;
  for (int64_t c = 0; c < count; c += per, ++k) {
    const int b = k & 1;
    const int64_t n = std::min(per, count - c);
    SAIT_CUDA(cudaEventSynchronize(st.done[b]));  // the copy that last read this buffer
    fill(st.buf[b], c, n);
    SAIT_CUDA(cudaMemcpyAsync(dev_dst + c * elem, st.buf[b], n * elem, cudaMemcpyHostToDevice, s));
    SAIT_CUDA(cudaEventRecord(st.done[b], s));
  }
}
// drain(pinned, first, n) <- dev_src[0, count) chunk by chunk (the D2H of the
// next chunk is in flight while the host drains this one)
template <class Drain>
void staged_d2h(Staging& st, const char* dev_src, int64_t count, size_t elem, Drain drain, cudaStream_t s) {
  const int64_t per = static_cast<int64_t>(kStageBytes / elem);
  const int64_t chunks = (count + per - 1) / per;
  auto issue = [&](int64_t k) {
    const int b = static_cast<int>(k & 1);
    const int64_t c = k * per, n = std::min(per, count - c);
    SAIT_CUDA(cudaMemcpyAsync(st.buf[b], dev_src + c * elem, n * elem, cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaEventRecord(st.done[b], s));
  };
  if (chunks > 0) issue(0);
  for (int64_t k = 0; k < chunks; ++k) {
    if (k + 1 < chunks) issue(k + 1);  // its buffer was drained two iterations ago
    const int b = static_cast<int>(k & 1);
    SAIT_CUDA(cudaEventSynchronize(st.done[b]));
    const int64_t c = k * per, n = std::min(per, count - c);
    drain(st.buf[b], c, n);
  }
}
void narrow_host(const int64_t* in, char* out, int64_t n) {
  int32_t* o = reinterpret_cast<int32_t*>(out);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) o[i] = (in[i] < 0 || in[i] > INT32_MAX) ? -1 : static_cast<int32_t>(in[i]);
}
void widen_host(const char* in, int64_t* out, int64_t n) {
  const int32_t* x = reinterpret_cast<const int32_t*>(in);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = x[i];
}
void copy_host(const char* in, char* out, int64_t bytes) {
  const int64_t nb = (bytes + (1 << 20) - 1) >> 20;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t o = b << 20;
    std::memcpy(out + o, in + o, static_cast<size_t>(std::min<int64_t>(int64_t{1} << 20, bytes - o)));
  }
}
}  // namespace

sait::DevCsr upload(const sait_host_csr* m, cudaStream_t s) {
  need(m, "sait_csr_upload");
  if (m->nrows < 0 || m->ncols < 0) sait::throw_invalid("validate: negative dimension");
  need(m->row_ptr, "sait_csr_upload(row_ptr)");
  if (m->row_ptr[0] != 0) sait::throw_invalid("validate: bad row_ptr head");
  const int64_t nnz = m->row_ptr[m->nrows];
  if (nnz < 0) sait::throw_invalid("validate: bad row_ptr tail");
  if (nnz > INT32_MAX || m->nrows >= INT32_MAX || m->ncols >= INT32_MAX)
    sait::throw_invalid("sait_csr_upload: " + std::to_string(nnz) +
                        " entries / dimensions exceed the int32 device index range");
  if (nnz && !m->col_idx) sait::throw_invalid("sait_csr_upload: null col_idx");
  sait::DevCsr d;
  d.nrows = m->nrows;
  d.ncols = m->ncols;
  d.nnz = nnz;
  d.rp = sait::dalloc<int32_t>(d.nrows + 1, s);
  d.ci = sait::dalloc<int32_t>(nnz, s);
  d.v = m->values ? sait::dalloc<double>(nnz, s) : nullptr;
  {
    Staging& st = staging();
    std::lock_guard<std::mutex> lk(st.mu);
    staged_h2d(st, reinterpret_cast<char*>(d.rp), d.nrows + 1, 4,
               [&](char* p, int64_t c, int64_t n) { narrow_host(m->row_ptr + c, p, n); }, s);
    if (nnz) {
      staged_h2d(st, reinterpret_cast<char*>(d.ci), nnz, 4,
                 [&](char* p, int64_t c, int64_t n) { narrow_host(m->col_idx + c, p, n); }, s);
      if (m->values)
        staged_h2d(st, reinterpret_cast<char*>(d.v), nnz, 8, [&](char* p, int64_t c, int64_t n) {
          copy_host(reinterpret_cast<const char*>(m->values + c), p, n * 8);
        }, s);
    }
    for (int b = 0; b < 2; ++b) SAIT_CUDA(cudaEventSynchronize(st.done[b]));  // staging free for the next caller
  }
  try {
    sait::validate_device_csr(d, s);
  } catch (...) {
    sait::free_csr(d, s);
    throw;
  }
  return d;
}

void to_host(const sait::DevCsr& m, cudaStream_t s, int64_t* rp, int64_t* ci, double* v) {
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mu);
  staged_d2h(st, reinterpret_cast<const char*>(m.rp), m.nrows + 1, 4,
             [&](const char* p, int64_t c, int64_t n) { widen_host(p, rp + c, n); }, s);
  if (m.nnz) {
    staged_d2h(st, reinterpret_cast<const char*>(m.ci), m.nnz, 4,
               [&](const char* p, int64_t c, int64_t n) { widen_host(p, ci + c, n); }, s);
    if (v && m.v)
      staged_d2h(st, reinterpret_cast<const char*>(m.v), m.nnz, 8, [&](const char* p, int64_t c, int64_t n) {
        copy_host(p, reinterpret_cast<char*>(v + c), n * 8);
      }, s);
  }
}

// Identity of order n used as the right factor for the elementwise kernels.
sait::Epilogue no_epilogue() { return sait::Epilogue{}; }

struct BuildOut {
  sait::DevCsr mt;  // final unit-diagonal iterate: M^T (column form) or M (row form)
  int steps_run = 0;
  bool stabilized = false;
  bool scaled = false;  // row form: the last step already applied scale_columns
  int64_t products = 0;
};

// The recursion of sait.cpp:75-136.  Column form: row j of M_s^T is
//   drop( sum_{k in M_{s-1}^T[j,:]} M_{s-1}^T[j,k] * tT^T[k,:] + e_j ),
// bitwise equal to the reference's row form (same products, same
// ascending-k order, commutative products).  Rows [c0, c0 + rows) of M^T
// (= a block of columns of M) evolve independently; only the early-stop
// decision is global, so the caller supplies it between steps.  Column-sharded
// blocks need the column form (the fill cap, per column of M, is then part of
// the SpGEMM epilogue).
// Row form (row_form = true, whole matrix, threshold/pattern/none): the
// reference's own orientation, row i of M_s = drop(sum_k tT[i,k] M_{s-1}[k,:]
// + e_i) with op = tT -- the same products in the same order, and neither
// tT nor the result needs a transpose; a fill cap runs as a per-column pass
// after each step (cap_rowform).
class Recursion {
 public:
  // op_from_split: op is the iteration matrix of jacobi_split (no stored
  // diagonal), which the first-step filter pass relies on; the generic
  // sait_polynomial accepts any square iteration matrix and keeps the
  // generic product (add_identity adds 1.0 to a stored diagonal there).
  Recursion(const sait::DevCsr& op, const sait_drop_spec& spec, const int32_t* cap, int64_t c0, int64_t rows,
            cudaStream_t s, bool row_form = false, const double* out_scale = nullptr, bool op_from_split = true)
      : ttT_(op), spec_(spec), s_(s), row_form_(row_form), out_scale_(row_form ? out_scale : nullptr),
        op_from_split_(op_from_split) {
    // row form with the fill cap: the product keeps the threshold only and
    // cap_rowform applies the per-column cap after it; the column scaling is
    // left to finish (the cap ranks unscaled values)
    row_cap_ = row_form && spec.kind == SAIT_DROP_THRESHOLD_CAP ? cap : nullptr;
    if (row_cap_) {  // the last step's compaction (if any) scales instead
      cap_scale_ = out_scale_;
      out_scale_ = nullptr;
    }
    a_ = sait::make_identity_rows(rows, c0, op.nrows, s);
    epi_.add_identity = true;
    epi_.diag_offset = c0;
    if (spec.kind == SAIT_DROP_THRESHOLD) {
      epi_.drop = 1;
      epi_.tau = spec.tau;
    } else if (spec.kind == SAIT_DROP_THRESHOLD_CAP) {
      epi_.drop = row_cap_ ? 1 : 3;
      epi_.tau = spec.tau;
      epi_.cap = row_cap_ ? nullptr : cap;
    }
    pattern_left_ = spec.kind == SAIT_DROP_PATTERN ? spec.pattern_steps : 0;
    main_left_ = spec.kind == SAIT_DROP_PATTERN ? spec.refine_steps : spec.steps;
    if (spec.kind == SAIT_DROP_PATTERN && pattern_left_ == 0) capture_pattern();
  }
  ~Recursion() {
    sait::free_csr(a_, s_);
    if (pattern_.rp) sait::free_csr(pattern_, s_);
  }
  int remaining() const { return pattern_left_ + main_left_; }
  // One step; returns whether this block changed (pattern-growth steps of
  // sait_pat have no early-stop check, sait.cpp:122-125: they report true).
  bool step() {
    if (pattern_left_ > 0) {
      sait::Epilogue e0;
      e0.add_identity = true;
      e0.diag_offset = epi_.diag_offset;
      advance(product(e0));
      if (--pattern_left_ == 0) capture_pattern();
      return true;
    }
    epi_.qrp = a_.rp;
    epi_.qci = a_.ci;
    epi_.qv = a_.v;
    epi_.qnnz = a_.nnz;
    // the last allowed step writes M D^-1 directly (an earlier early stop
    // leaves the scaling to finish)
    const bool last = out_scale_ && main_left_ == 1;
    epi_.out_scale = last ? out_scale_ : nullptr;
    const bool first = steps_run_ == 0;
    sait::SpgemmResult r = product(epi_);
    epi_.out_scale = nullptr;
    scaled_ = last;
    // the cap cannot bind at the first step (see product); after it, a step
    // that dropped entries for the cap is compared again, capped
    if (row_cap_ && !first) {
      const bool last_cap = cap_scale_ && main_left_ == 1;
      bool sc = false;
      if (sait::cap_rowform(r.c, row_cap_, s_, last_cap ? cap_scale_ : nullptr, &sc) > 0)
        r.changed = !sait::csr_stabilized(a_, r.c, s_);  // (no kernel when the sizes differ)
      scaled_ = sc;
    }
    const bool changed = r.changed;
    advance(std::move(r));
    --main_left_;
    return changed;
  }
  void stop_stabilized() {
    stabilized_ = true;
    main_left_ = 0;
  }
  BuildOut take() {
    BuildOut o;
    o.mt = a_;
    a_ = sait::DevCsr{};
    o.steps_run = steps_run_;
    o.stabilized = stabilized_;
    o.scaled = scaled_;
    o.products = products_;
    return o;
  }

 private:
  sait::SpgemmResult product(const sait::Epilogue& e) {
    // M_0 = I (whole matrix): the first step is tT + I (row form) or tT^T + I
    // (column form) filtered -- no products to accumulate.  The A15 cap cannot
    // bind there: column j keeps at most nnz(T[:, j]) entries and the cap is
    // floor(f nnz(T[:, j])) with f >= 1.
    if (op_from_split_ && steps_run_ == 0 && e.diag_offset == 0 && a_.nrows == ttT_.nrows &&
        (e.drop == 0 || e.drop == 1 || e.drop == 3))
      return sait::first_step_identity(ttT_, e, s_);
    return row_form_ ? sait::spgemm_fused(ttT_, a_, e, s_) : sait::spgemm_fused(a_, ttT_, e, s_);
  }
  void advance(sait::SpgemmResult&& r) {
    products_ += r.products;
    sait::free_csr(a_, s_);
    a_ = r.c;
    ++steps_run_;
  }
  void capture_pattern() {  // S = pattern(M_p) (sait.cpp:126)
    pattern_ = sait::copy_csr(a_, s_);
    epi_.drop = 2;
    epi_.prp = pattern_.rp;
    epi_.pci = pattern_.ci;
  }
  const sait::DevCsr& ttT_;  // tT^T (column form) or tT (row form)
  sait_drop_spec spec_;
  cudaStream_t s_;
  bool row_form_ = false;
  const double* out_scale_ = nullptr;
  const int32_t* row_cap_ = nullptr;  // row form with the fill cap
  const double* cap_scale_ = nullptr;
  bool op_from_split_ = true;
  bool scaled_ = false;
  sait::DevCsr a_, pattern_;
  sait::Epilogue epi_;
  int pattern_left_ = 0, main_left_ = 0, steps_run_ = 0;
  bool stabilized_ = false;
  int64_t products_ = 0;
};

BuildOut run_recursion(const sait::DevCsr& ttT, const sait_drop_spec& spec, const int32_t* cap, cudaStream_t s,
                       bool op_from_split = true) {
  Recursion r(ttT, spec, cap, 0, ttT.nrows, s, false, nullptr, op_from_split);
  while (r.remaining() > 0)
    if (!r.step()) r.stop_stabilized();
  return r.take();
}

void check_spec(const sait_drop_spec* spec) {
  need(spec, "sait_build(spec)");
  switch (spec->kind) {
    case SAIT_DROP_THRESHOLD:
      if (!(spec->tau >= 0.0 && spec->tau < 1.0))
        sait::throw_invalid("sait_thr: threshold must be in [0, 1), got " + fmt_double(spec->tau));
      break;
    case SAIT_DROP_THRESHOLD_CAP:
      if (!(spec->tau >= 0.0 && spec->tau < 1.0))
        sait::throw_invalid("sait_thr: threshold must be in [0, 1), got " + fmt_double(spec->tau));
      if (!(spec->cap_factor >= 1.0))
        sait::throw_invalid("sait_thr_cap: cap factor must be >= 1, got " + fmt_double(spec->cap_factor));
      break;
    case SAIT_DROP_PATTERN:
      if (spec->pattern_steps < 0) sait::throw_invalid("sait_pat: pattern_steps must be >= 0");
      if (spec->refine_steps < 1) sait::throw_invalid("sait_pat: refine_steps must be >= 1");
      break;
    case SAIT_DROP_NONE:
      break;
    default:
      sait::throw_invalid("sait_build: unknown drop kind " + std::to_string(spec->kind));
  }
}

// Chunking of the host-vector apply (see pair_apply_host_chunked).
void plan_host_chunks(sait_pair_t p) {
  const sait::DevCsr& L = p->ml->m;
  const sait::DevCsr& U = p->mu->m;
  p->chunk_rows.clear();
  p->u_rows.clear();
  const int64_t n = L.nrows;
  if (!(L.ncols == n && U.nrows == n && U.ncols == n) || n < (int64_t{1} << 17) || !p->sl.ok() || !p->su.ok() ||
      p->sl.perm || p->su.perm)
    return;  // small, non-square or row-sorted pairs: one-shot path
  const int64_t G = sait::kDepGroupRows;
  const int64_t ng = (n + G - 1) / G;
  // Copy sizes (MB of r / z per chunk): short head chunks start the z stream
  // early, short tail chunks keep the drain (z still leaving after the last r
  // chunk landed) short, ~4 MB in between (on PCIe5, async copies much
  // smaller than that lose H2D/D2H concurrency).  SAIT_PIPE_MB =
  // "head,...;mid;tail,..." (or the older "first,mid,last").
  std::vector<double> head{3.0}, tail;
  double mb_mid = 4.0;
  if (const char* e = std::getenv("SAIT_PIPE_MB")) {
    auto parse = [](const std::string& t) {
      std::vector<double> v;
      size_t a = 0;
      while (a < t.size()) {
        size_t b2 = t.find(',', a);
        if (b2 == std::string::npos) b2 = t.size();
        if (b2 > a) v.push_back(std::atof(t.substr(a, b2 - a).c_str()));
        a = b2 + 1;
      }
      return v;
    };
    const std::string spec(e);
    const size_t s1 = spec.find(';');
    if (s1 == std::string::npos) {
      const std::vector<double> v = parse(spec);
      head.assign(1, v.size() > 0 ? v[0] : 2.0);
      mb_mid = v.size() > 1 ? v[1] : 4.0;
      tail.assign(1, v.size() > 2 ? v[2] : 1.0);
    } else {
      const size_t s2 = spec.find(';', s1 + 1);
      head = parse(spec.substr(0, s1));
      mb_mid = std::atof(spec.substr(s1 + 1, s2 == std::string::npos ? std::string::npos : s2 - s1 - 1).c_str());
      tail = s2 == std::string::npos ? std::vector<double>{} : parse(spec.substr(s2 + 1));
    }
  }
  if (!(mb_mid > 0.0)) mb_mid = 1e9;  // "head;;tail": the middle as one chunk
  auto rows_of = [&](double mb) {
    return std::max<int64_t>(G, static_cast<int64_t>(mb * (1 << 20) / 8.0) / G * G);
  };
  std::vector<int32_t> lhi(ng), uhi(ng);
  int32_t* d = sait::dalloc<int32_t>(4 * ng, nullptr);
  sait::column_group_deps(L, d, d + ng, nullptr);
  sait::column_group_deps(U, d + 2 * ng, d + 3 * ng, nullptr);
  SAIT_CUDA(cudaMemcpy(lhi.data(), d + ng, sizeof(int32_t) * ng, cudaMemcpyDeviceToHost));
  SAIT_CUDA(cudaMemcpy(uhi.data(), d + 3 * ng, sizeof(int32_t) * ng, cudaMemcpyDeviceToHost));
  sait::dfree(d, nullptr);
  SAIT_CUDA(cudaDeviceSynchronize());
  {
    std::vector<int64_t> hr, tr;
    int64_t used = 0;
    for (double mb : head) hr.push_back(rows_of(mb)), used += hr.back();
    for (double mb : tail) tr.push_back(rows_of(mb)), used += tr.back();
    const int64_t rm = rows_of(mb_mid);
    std::vector<int64_t>& b = p->chunk_rows;
    b.push_back(0);
    if (n > used + rm / 2) {
      int64_t at = 0;
      for (int64_t r : hr) b.push_back(at += r);
      const int64_t mid = n - used;
      const int64_t km = std::max<int64_t>(1, (mid + rm / 2) / rm);
      const int64_t step = (mid / km + G - 1) / G * G;
      for (int64_t c = 1; c < km; ++c) b.push_back(at + c * step);
      at = n - used + at;  // start of the tail chunks
      if (!tr.empty()) b.push_back(at);
      for (size_t t = 0; t + 1 < tr.size(); ++t) b.push_back(at += tr[t]);
    }
    if (b.back() != n) b.push_back(n);
  }
  const int64_t nk = static_cast<int64_t>(p->chunk_rows.size()) - 1;
  std::vector<int32_t> chunk_of_group(ng + 1);
  for (int64_t c = 0, g2 = 0; c < nk; ++c)
    for (; g2 < ng && g2 * G < p->chunk_rows[c + 1]; ++g2) chunk_of_group[g2] = static_cast<int32_t>(c);
  p->needL_hi.assign(nk, 0);
  for (int64_t g2 = 0; g2 < ng; ++g2)
    if (lhi[g2] >= 0)
      p->needL_hi[chunk_of_group[g2]] =
          std::max<int32_t>(p->needL_hi[chunk_of_group[g2]], chunk_of_group[std::min<int64_t>(lhi[g2], ng - 1)]);
  for (int64_t c = 1; c < nk; ++c) p->needL_hi[c] = std::max(p->needL_hi[c], p->needL_hi[c - 1]);
  // M_U chunk c = the rows whose y reads end below chunk boundary c+1, so it
  // can run (and its z leave) as soon as M_L chunk c is done.
  p->u_rows.assign(nk + 1, n);
  p->u_rows[0] = 0;
  int64_t g = 0, run = -1;
  for (int64_t c = 0; c + 1 < nk; ++c) {
    const int64_t bound_group = p->chunk_rows[c + 1] / G;  // y groups < bound are complete
    while (g < ng && std::max<int64_t>(run, uhi[g]) < bound_group) run = std::max<int64_t>(run, uhi[g++]);
    p->u_rows[c + 1] = std::max(p->u_rows[c], std::min(n, g * G));
  }
}

}  // namespace

namespace sait {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace sait

extern "C" {

const char* sait_last_error(void) { return g_err.c_str(); }
int sait_abi_version(void) { return SAIT_ABI_VERSION; }

void sait_host_csr_free(sait_host_csr* m) {
  if (!m) return;
  std::free(m->row_ptr);
  std::free(m->col_idx);
  std::free(m->values);
  m->row_ptr = m->col_idx = nullptr;
  m->values = nullptr;
}

int64_t sait_kernel_launch_count(void) { return sait::g_launches.load(); }

int sait_device_pool_reserve(int device, int64_t bytes) {
  return guarded([&] {
    if (bytes < 0) sait::throw_invalid("sait_device_pool_reserve: bytes must be >= 0");
    DeviceGuard g(device);
    init_device_pool();
    cudaMemPool_t pool;
    SAIT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    void* p = nullptr;
    SAIT_CUDA(cudaMallocFromPoolAsync(&p, static_cast<size_t>(bytes), pool, nullptr));
    SAIT_CUDA(cudaFreeAsync(p, nullptr));
    SAIT_CUDA(cudaStreamSynchronize(nullptr));
  });
}

// Diagnostics: seconds for H2D alone / D2H alone / both on two streams.
void sait_debug_copy_probe(const double* h_src, double* h_dst, int64_t n, int chunks, double* out3) {
  double *a = nullptr, *b = nullptr;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  auto run = [&](bool up, bool down) {
    cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    int64_t step = (n + std::abs(chunks) - 1) / std::abs(chunks);
    if (chunks > 0) {
      for (int64_t o = 0; o < n; o += step) {
        int64_t m = std::min(step, n - o);
        if (up) cudaMemcpyAsync(a + o, h_src + o, m * 8, cudaMemcpyHostToDevice, s1);
        if (down) cudaMemcpyAsync(h_dst + o, b + o, m * 8, cudaMemcpyDeviceToHost, s2);
      }
    } else {
      for (int64_t o = 0; up && o < n; o += step)
        cudaMemcpyAsync(a + o, h_src + o, std::min(step, n - o) * 8, cudaMemcpyHostToDevice, s1);
      for (int64_t o = 0; down && o < n; o += step)
        cudaMemcpyAsync(h_dst + o, b + o, std::min(step, n - o) * 8, cudaMemcpyDeviceToHost, s2);
    }
    cudaDeviceSynchronize();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  run(true, true);
  out3[0] = run(true, false);
  out3[1] = run(false, true);
  out3[2] = run(true, true);
  cudaStreamDestroy(s1);
  cudaStreamDestroy(s2);
  cudaFree(a);
  cudaFree(b);
}

// Diagnostics (not part of sait_c.h): memory type of a pointer as this
// library's runtime sees it (0 unregistered, 1 host/pinned, 2 device, 3 managed).
// Index storage of a pair factor's SELL copy (which: 0 = M_L, 1 = M_U):
// 2 shared slice patterns, 1 int16 deltas, 0 int32 columns, -1 no SELL copy.
int sait_debug_pair_index_kind(sait_pair_t p, int which) {
  if (!p) return -1;
  const sait::SellMatrix& m = which == 0 ? p->sl : p->su;
  return m.ok() ? m.index_kind() : -1;
}

int sait_debug_pointer_type(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return static_cast<int>(a.type);
}

int sait_device_synchronize(void) {
  return guarded([] { SAIT_CUDA(cudaDeviceSynchronize()); });
}

int sait_device_alloc(size_t bytes, void** ptr) {
  return guarded([&] {
    need(ptr, "sait_device_alloc");
    init_device_pool();
    cudaError_t e = cudaMalloc(ptr, (bytes ? bytes : 1) + 256);
    if (e == cudaErrorMemoryAllocation) throw sait::Error(SAIT_ERR_NOMEM, "out of device memory");
    SAIT_CUDA(e);
  });
}
void sait_device_free(void* ptr) {
  if (ptr) cudaFree(ptr);
}
int sait_memcpy(void* dst, const void* src, size_t bytes, int kind) {
  return guarded([&] {
    if (bytes == 0) return;
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                             : kind == 2 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    SAIT_CUDA(cudaMemcpy(dst, src, bytes, k));
  });
}
int sait_stream_create(sait_stream_t* stream) {
  return guarded([&] {
    cudaStream_t s;
    SAIT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
  });
}
void sait_stream_destroy(sait_stream_t stream) {
  if (stream) cudaStreamDestroy(sait::as_stream(stream));
}

int sait_host_alloc(size_t bytes, void** ptr) {
  return guarded([&] { SAIT_CUDA(cudaMallocHost(ptr, bytes ? bytes : 1)); });
}
void sait_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

// ---------------------------------------------------------------- device CSR

int sait_csr_upload(const sait_host_csr* m, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(out, "sait_csr_upload(out)");
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr d = upload(m, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(d);
  });
}

int sait_csr_info(sait_dcsr_t m, int64_t* nrows, int64_t* ncols, int64_t* nnz) {
  return guarded([&] {
    need(m, "sait_csr_info");
    if (nrows) *nrows = m->m.nrows;
    if (ncols) *ncols = m->m.ncols;
    if (nnz) *nnz = m->m.nnz;
  });
}

int sait_csr_download(sait_dcsr_t m, int64_t* row_ptr, int64_t* col_idx, double* values, sait_stream_t stream) {
  return guarded([&] {
    need(m, "sait_csr_download");
    DeviceGuard g(m->dev);
    to_host(m->m, sait::as_stream(stream), row_ptr, col_idx, values);
  });
}

int sait_csr_to_host(sait_dcsr_t m, sait_stream_t stream, sait_host_csr* out) {
  return guarded([&] {
    need(m, "sait_csr_to_host");
    need(out, "sait_csr_to_host(out)");
    DeviceGuard g(m->dev);
    host_csr_alloc(out, m->m.nrows, m->m.ncols, m->m.nnz, m->m.v != nullptr);
    to_host(m->m, sait::as_stream(stream), out->row_ptr, out->col_idx, out->values);
  });
}

int sait_csr_device_arrays(sait_dcsr_t m, const int32_t** row_ptr, const int32_t** col_idx, const double** values) {
  return guarded([&] {
    need(m, "sait_csr_device_arrays");
    if (row_ptr) *row_ptr = m->m.rp;
    if (col_idx) *col_idx = m->m.ci;
    if (values) *values = m->m.v;
  });
}

int sait_csr_assemble_rows(int nparts, const sait_row_piece* parts, int64_t nrows, int64_t ncols,
                           sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(out, "sait_csr_assemble_rows(out)");
    if (nparts < 0 || (nparts > 0 && !parts)) sait::throw_invalid("sait_csr_assemble_rows: bad parts");
    if (nrows < 0 || ncols < 0 || nrows > INT32_MAX || ncols > INT32_MAX)
      sait::throw_invalid("sait_csr_assemble_rows: dimensions out of range");
    for (int p = 0; p < nparts; ++p)
      if (!parts[p].row_ptr || !parts[p].col_idx) sait::throw_invalid("sait_csr_assemble_rows: null piece");
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr c = sait::assemble_rows(nparts, parts, nrows, ncols, s);
    if (c.nnz > INT32_MAX) {
      sait::free_csr(c, s);
      sait::throw_invalid("sait_csr_assemble_rows: more than 2^31-1 entries");
    }
    *out = wrap(c);
  });
}

int sait_csr_col_span(sait_dcsr_t m, int64_t* lo, int64_t* hi, sait_stream_t stream) {
  return guarded([&] {
    need(m, "sait_csr_col_span");
    DeviceGuard g(m->dev);
    int64_t a = 0, b = 0;
    sait::col_span(m->m, &a, &b, sait::as_stream(stream));
    if (lo) *lo = a;
    if (hi) *hi = b;
  });
}

int sait_csr_shift_cols(sait_dcsr_t m, int64_t offset, int64_t new_ncols, sait_stream_t stream) {
  return guarded([&] {
    need(m, "sait_csr_shift_cols");
    if (new_ncols < 0 || new_ncols > INT32_MAX || offset > INT32_MAX || offset < -int64_t{INT32_MAX})
      sait::throw_invalid("sait_csr_shift_cols: out of range");
    DeviceGuard g(m->dev);
    sait::shift_columns(m->m, offset, new_ncols, sait::as_stream(stream));
  });
}

int sait_csr_row_ptr_at(sait_dcsr_t m, const int64_t* rows, int k, int64_t* out, sait_stream_t stream) {
  return guarded([&] {
    need(m, "sait_csr_row_ptr_at");
    if (k < 0 || (k > 0 && (!rows || !out))) sait::throw_invalid("sait_csr_row_ptr_at: bad arguments");
    for (int j = 0; j < k; ++j)
      if (rows[j] < 0 || rows[j] > m->m.nrows) sait::throw_invalid("sait_csr_row_ptr_at: row out of range");
    DeviceGuard g(m->dev);
    init_device_pool();
    sait::row_ptr_at(m->m, rows, k, out, sait::as_stream(stream));
  });
}

int sait_column_work(sait_dcsr_t t, int64_t* d_work, sait_stream_t stream) {
  return guarded([&] {
    need(t, "sait_column_work");
    need(d_work, "sait_column_work(work)");
    if (t->m.nrows != t->m.ncols) sait::throw_invalid("sait_column_work: matrix is not square");
    DeviceGuard g(t->dev);
    init_device_pool();
    sait::column_work_of(t->m, d_work, sait::as_stream(stream));
  });
}

void sait_csr_free(sait_dcsr_t m) {
  if (!m) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->dev);
  cudaFree(m->m.rp);
  cudaFree(m->m.ci);
  if (m->m.v) cudaFree(m->m.v);
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

// ------------------------------------------------------------------- kernels

int sait_spmv(sait_dcsr_t a, const double* d_x, int64_t xlen, double* d_y, int64_t ylen, sait_stream_t stream) {
  return guarded([&] {
    need(a, "spmv");
    if (xlen != a->m.ncols)
      sait::throw_invalid("spmv: vector length " + std::to_string(xlen) + " does not match ncols " +
                          std::to_string(a->m.ncols));
    if (ylen != a->m.nrows) sait::throw_invalid("spmv: output length mismatch");
    DeviceGuard g(a->dev);
    sait::spmv(a->m, d_x, d_y, sait::as_stream(stream));
  });
}

int sait_spmm(sait_dcsr_t a, const double* d_x, double* d_y, int64_t nvec, sait_stream_t stream) {
  return guarded([&] {
    need(a, "spmm");
    if (nvec < 0) sait::throw_invalid("spmm: negative block width");
    if (nvec == 0 || a->m.nrows == 0) return;
    if (!d_x || !d_y) sait::throw_invalid("spmm: null block");
    DeviceGuard g(a->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    const sait::DevCsr& m = a->m;
    // column-major blocks in slabs of 8/4/2/1 vectors: transposed to
    // row-major, one CSR block product per slab (the matrix read once per
    // slab instead of once per column), transposed back
    const int64_t slab = std::min<int64_t>(nvec, 8);
    double* xt = sait::dalloc<double>(m.ncols * slab, s);
    double* yt = sait::dalloc<double>(m.nrows * slab, s);
    for (int64_t c = 0; c < nvec;) {
      const int w = nvec - c >= 8 ? 8 : nvec - c >= 4 ? 4 : nvec - c >= 2 ? 2 : 1;
      const double* x = d_x + c * m.ncols;
      double* y = d_y + c * m.nrows;
      if (w == 1) {
        sait::spmv(m, x, y, s);
      } else {
        sait::transpose_block(x, xt, m.ncols, w, true, s);
        sait::spmm_rowmajor(m, xt, yt, w, s);
        sait::transpose_block(yt, y, m.nrows, w, false, s);
      }
      c += w;
    }
    sait::dfree(xt, s);
    sait::dfree(yt, s);
  });
}

int sait_spgemm(sait_dcsr_t a, sait_dcsr_t b, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(a, "spgemm");
    need(b, "spgemm");
    need(out, "spgemm(out)");
    DeviceGuard g(a->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::SpgemmResult r = sait::spgemm_fused(a->m, b->m, no_epilogue(), s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r.c);
  });
}

namespace {
// elementwise row filters run as the fused SpGEMM M * I (m * 1.0 == m exactly)
sait::DevCsr through_identity(const sait::DevCsr& m, const sait::Epilogue& epi, cudaStream_t s) {
  sait::DevCsr eye = sait::make_identity(m.ncols, s);
  sait::SpgemmResult r = sait::spgemm_fused(m, eye, epi, s);
  sait::free_csr(eye, s);
  return r.c;
}
}  // namespace

int sait_add_identity(sait_dcsr_t m, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(m, "add_identity");
    need(out, "add_identity(out)");
    if (m->m.nrows != m->m.ncols) sait::throw_invalid("add_identity: matrix is not square");
    DeviceGuard g(m->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::Epilogue e;
    e.add_identity = true;
    sait::DevCsr r = through_identity(m->m, e, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r);
  });
}

int sait_drop_by_threshold(sait_dcsr_t m, double tau, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(m, "drop_by_threshold");
    need(out, "drop_by_threshold(out)");
    if (!(tau >= 0.0 && tau < 1.0))
      sait::throw_invalid("drop_by_threshold: tau must be in [0, 1), got " + fmt_double(tau));
    DeviceGuard g(m->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr r;
    if (tau == 0.0) {
      r = sait::copy_csr(m->m, s);
    } else {
      sait::Epilogue e;
      e.drop = 1;
      e.tau = tau;
      r = through_identity(m->m, e, s);
    }
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r);
  });
}

int sait_drop_by_pattern(sait_dcsr_t m, sait_dcsr_t pattern, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(m, "drop_by_pattern");
    need(pattern, "drop_by_pattern");
    need(out, "drop_by_pattern(out)");
    if (m->m.nrows != pattern->m.nrows || m->m.ncols != pattern->m.ncols)
      sait::throw_invalid("drop_by_pattern: shape mismatch");
    DeviceGuard g(m->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::Epilogue e;
    e.drop = 2;
    e.prp = pattern->m.rp;
    e.pci = pattern->m.ci;
    sait::DevCsr r = through_identity(m->m, e, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r);
  });
}

int sait_scale_columns(sait_dcsr_t m, const double* d_d, int64_t dlen, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(m, "scale_columns");
    need(out, "scale_columns(out)");
    if (dlen != m->m.ncols) sait::throw_invalid("scale_columns: scale vector length mismatch");
    DeviceGuard g(m->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr r = sait::copy_csr(m->m, s);
    sait::scale_columns(m->m, d_d, r, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r);
  });
}

int sait_transpose(sait_dcsr_t m, sait_stream_t stream, sait_dcsr_t* out) {
  return guarded([&] {
    need(m, "transpose");
    need(out, "transpose(out)");
    DeviceGuard g(m->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr r = sait::transpose(m->m, nullptr, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *out = wrap(r);
  });
}

// ---------------------------------------------------------------------- SAIT

int sait_jacobi_split(sait_dcsr_t t, int lower, double* d_inv_diag, sait_stream_t stream, sait_dcsr_t* tt) {
  return guarded([&] {
    need(t, "jacobi_split");
    need(tt, "jacobi_split(out)");
    DeviceGuard g(t->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr r = sait::jacobi_split(t->m, lower != 0, d_inv_diag, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *tt = wrap(r);
  });
}

int sait_build_session_create(sait_dcsr_t t, int lower, const sait_drop_spec* spec, int64_t col0, int64_t col1,
                              sait_stream_t stream, sait_build_session_t* out) {
  return guarded([&] {
    need(t, "sait_build");
    need(out, "sait_build(out)");
    check_spec(spec);
    DeviceGuard g(t->dev);
    init_device_pool();
    const int64_t n = t->m.nrows;
    if (col0 < 0 || col1 < col0 || col1 > n) sait::throw_invalid("sait_build: bad column block");
    auto* ss = new sait_build_session_s;
    ss->dev = t->dev;
    ss->s = sait::as_stream(stream);
    ss->c0 = col0;
    ss->c1 = col1;
    ss->n = n;
    cudaStream_t s = ss->s;
    SAIT_CUDA(cudaEventCreate(&ss->e0));
    SAIT_CUDA(cudaEventRecord(ss->e0, s));
    ss->inv = sait::dalloc<double>(n, s);
    sait::DevCsr tt;
    try {
      tt = sait::jacobi_split(t->m, lower != 0, ss->inv, s);
      if (spec->kind != SAIT_DROP_PATTERN && spec->steps < 1) {
        sait::free_csr(tt, s);
        sait::throw_invalid("sait_polynomial: steps must be >= 1");
      }
    } catch (...) {
      sait::dfree(ss->inv, s);
      cudaEventDestroy(ss->e0);
      delete ss;
      throw;
    }
    // whole-matrix builds run in row form (no transposes; the fill cap is a
    // pass after each step, cap.cu); column blocks need the column form;
    // SAIT_BUILD_COLUMN_FORM=1 forces it (tests)
    static const bool force_column = [] {
      const char* e = std::getenv("SAIT_BUILD_COLUMN_FORM");
      return e && std::atoi(e) != 0;
    }();
    ss->row_form = !force_column && col0 == 0 && col1 == n;
    if (ss->row_form) {
      ss->ttT = tt;
    } else {
      ss->ttT = sait::transpose(tt, nullptr, s);
      sait::free_csr(tt, s);
    }
    if (spec->kind == SAIT_DROP_THRESHOLD_CAP) {
      ss->cap = sait::dalloc<int32_t>(n, s);
      sait::column_caps(t->m, spec->cap_factor, ss->cap, s);
    }
    ss->rec = new Recursion(ss->ttT, *spec, ss->cap, col0, col1 - col0, s, ss->row_form, ss->inv);
    // the build's working set (two iterates, the staging area, tT, the
    // plan): ~64 B per entry of T plus ~40 B per row, mapped up front
    if (!std::getenv("SAIT_NO_POOL_ESTIMATE"))
      ensure_pool(static_cast<size_t>(64 * t->m.nnz * (col1 - col0) / std::max<int64_t>(n, 1) + 40 * n));
    *out = ss;
  });
}

int sait_build_session_remaining(sait_build_session_t ss) { return ss && ss->rec ? ss->rec->remaining() : 0; }

int sait_build_session_step(sait_build_session_t ss, int* changed) {
  return guarded([&] {
    need(ss, "sait_build_session_step");
    DeviceGuard g(ss->dev);
    if (!ss->rec || ss->rec->remaining() == 0) sait::throw_invalid("sait_build_session_step: no steps left");
    const bool ch = ss->rec->step();
    if (changed) *changed = ch ? 1 : 0;
  });
}

int sait_build_session_stop(sait_build_session_t ss) {
  return guarded([&] {
    need(ss, "sait_build_session_stop");
    ss->rec->stop_stabilized();
  });
}

int sait_build_session_finish(sait_build_session_t ss, int transposed, sait_dcsr_t* out, sait_build_stats* stats) {
  return guarded([&] {
    need(ss, "sait_build_session_finish");
    need(out, "sait_build_session_finish(out)");
    DeviceGuard g(ss->dev);
    cudaStream_t s = ss->s;
    BuildOut bo = ss->rec->take();
    sait::DevCsr m;
    // column j of M is scaled by inv_diag[j] (kernels.cpp:236-246); rows of the
    // M^T block are the global columns c0 + i
    if (ss->row_form) {  // bo.mt is M itself (whole matrix): scale its columns in place
      if (!bo.scaled) sait::scale_columns(bo.mt, ss->inv, bo.mt, s);
      if (transposed) {
        m = sait::transpose(bo.mt, nullptr, s);
        sait::free_csr(bo.mt, s);
      } else {
        m = bo.mt;
      }
    } else {
      if (transposed) {
        m = sait::copy_csr(bo.mt, s);
        sait::scale_rows(m, ss->inv + ss->c0, s);
      } else {
        m = sait::transpose(bo.mt, ss->inv + ss->c0, s);
      }
      sait::free_csr(bo.mt, s);
    }
    cudaEvent_t e1;
    SAIT_CUDA(cudaEventCreate(&e1));
    SAIT_CUDA(cudaEventRecord(e1, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    SAIT_CUDA(cudaEventElapsedTime(&ms, ss->e0, e1));
    cudaEventDestroy(e1);
    if (stats) {
      stats->steps_run = bo.steps_run;
      stats->stabilized = bo.stabilized ? 1 : 0;
      stats->nnz_out = m.nnz;
      stats->products = bo.products;
      stats->seconds = ms * 1e-3;
    }
    *out = wrap(m);
  });
}

void sait_build_session_destroy(sait_build_session_t ss) {
  if (!ss) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ss->dev);
  delete ss->rec;
  sait::free_csr(ss->ttT, ss->s);
  sait::dfree(ss->inv, ss->s);
  sait::dfree(ss->cap, ss->s);
  cudaStreamSynchronize(ss->s);
  cudaEventDestroy(ss->e0);
  if (prev >= 0) cudaSetDevice(prev);
  delete ss;
}

int sait_build(sait_dcsr_t t, int lower, const sait_drop_spec* spec, sait_stream_t stream, sait_dcsr_t* m_out,
               sait_build_stats* stats) {
  sait_build_session_t ss = nullptr;
  int rc = sait_build_session_create(t, lower, spec, 0, t ? t->m.nrows : 0, stream, &ss);
  if (rc) return rc;
  while (rc == SAIT_OK && sait_build_session_remaining(ss) > 0) {
    int changed = 1;
    rc = sait_build_session_step(ss, &changed);
    if (rc == SAIT_OK && !changed) rc = sait_build_session_stop(ss);  // single block: local == global
  }
  if (rc == SAIT_OK) rc = sait_build_session_finish(ss, 0, m_out, stats);
  sait_build_session_destroy(ss);
  return rc;
}

int sait_build_pair(sait_dcsr_t lower, sait_dcsr_t upper, const sait_drop_spec* spec, sait_stream_t stream,
                    sait_dcsr_t* ml_out, sait_dcsr_t* mu_out, sait_build_stats* stats2) {
  if (!lower || !upper || !ml_out || !mu_out) {
    sait::set_last_error("sait_build_pair: null argument");
    return SAIT_ERR_INVALID_ARGUMENT;
  }
  // The two recursions are independent: M_U builds on its own stream from a
  // second host thread while M_L builds on `stream`, so each one's kernels
  // fill the other's host-synchronisation gaps.
  int rc_u = SAIT_OK;
  std::string err_u;
  sait_dcsr_t mu = nullptr;
  std::thread tu([&] {
    cudaSetDevice(upper->dev);
    cudaStream_t su = nullptr;
    if (cudaStreamCreateWithFlags(&su, cudaStreamNonBlocking) != cudaSuccess) {
      rc_u = SAIT_ERR_CUDA;
      err_u = "sait_build_pair: cannot create a stream";
      return;
    }
    rc_u = sait_build(upper, 0, spec, su, &mu, stats2 ? stats2 + 1 : nullptr);
    if (rc_u) err_u = sait_last_error();
    cudaStreamSynchronize(su);
    cudaStreamDestroy(su);
  });
  sait_dcsr_t ml = nullptr;
  const int rc_l = sait_build(lower, 1, spec, stream, &ml, stats2);
  tu.join();
  if (rc_l || rc_u) {
    if (ml) sait_csr_free(ml);
    if (mu) sait_csr_free(mu);
    if (!rc_l) sait::set_last_error(err_u);
    return rc_l ? rc_l : rc_u;
  }
  *ml_out = ml;
  *mu_out = mu;
  return SAIT_OK;
}

int sait_polynomial(sait_dcsr_t tt, int steps, sait_stream_t stream, sait_dcsr_t* m_out, sait_build_stats* stats) {
  return guarded([&] {
    need(tt, "sait_polynomial");
    need(m_out, "sait_polynomial(out)");
    if (steps < 1) sait::throw_invalid("sait_polynomial: steps must be >= 1");
    if (tt->m.nrows != tt->m.ncols) sait::throw_invalid("add_identity: matrix is not square");
    DeviceGuard g(tt->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr ttT = sait::transpose(tt->m, nullptr, s);
    sait_drop_spec sp{SAIT_DROP_NONE, 0.0, steps, 0, 0, 0.0};
    BuildOut bo = run_recursion(ttT, sp, nullptr, s, /*op_from_split=*/false);
    sait::free_csr(ttT, s);
    sait::DevCsr m = sait::transpose(bo.mt, nullptr, s);
    sait::free_csr(bo.mt, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    if (stats) {
      stats->steps_run = bo.steps_run;
      stats->stabilized = bo.stabilized ? 1 : 0;
      stats->nnz_out = m.nnz;
      stats->products = bo.products;
      stats->seconds = 0.0;
    }
    *m_out = wrap(m);
  });
}

int sait_pat_capture_pattern(sait_dcsr_t t, int lower, int pattern_steps, sait_stream_t stream,
                             sait_dcsr_t* pattern_out) {
  return guarded([&] {
    need(t, "sait_pat_capture_pattern");
    need(pattern_out, "sait_pat_capture_pattern(out)");
    if (pattern_steps < 0) sait::throw_invalid("sait_pat_capture_pattern: pattern_steps must be >= 0");
    DeviceGuard g(t->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    const int64_t n = t->m.nrows;
    double* inv = sait::dalloc<double>(n, s);
    sait::DevCsr tt;
    try {
      tt = sait::jacobi_split(t->m, lower != 0, inv, s);
    } catch (...) {
      sait::dfree(inv, s);
      throw;
    }
    sait::dfree(inv, s);
    sait::DevCsr pat;
    if (pattern_steps == 0) {
      pat = sait::make_identity(n, s);
      sait::free_csr(tt, s);
    } else {
      sait::DevCsr ttT = sait::transpose(tt, nullptr, s);
      sait::free_csr(tt, s);
      sait_drop_spec sp{SAIT_DROP_NONE, 0.0, pattern_steps, 0, 0, 0.0};
      BuildOut bo = run_recursion(ttT, sp, nullptr, s);  // sait_polynomial(split, p, {})
      sait::free_csr(ttT, s);
      pat = sait::transpose(bo.mt, nullptr, s);
      sait::free_csr(bo.mt, s);
    }
    sait::dfree(pat.v, s);
    pat.v = nullptr;
    SAIT_CUDA(cudaStreamSynchronize(s));
    *pattern_out = wrap(pat);
  });
}

int sait_jacobi_sweeps_apply(sait_dcsr_t t, int lower, const double* d_b, int sweeps, double* d_x,
                             sait_stream_t stream) {
  return guarded([&] {
    need(t, "jacobi_sweeps_apply");
    if (sweeps < 1) sait::throw_invalid("jacobi_sweeps_apply: sweeps must be >= 1");
    DeviceGuard g(t->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    const int64_t n = t->m.nrows;
    double* inv = sait::dalloc<double>(n, s);
    sait::DevCsr tt;
    try {
      tt = sait::jacobi_split(t->m, lower != 0, inv, s);
    } catch (...) {
      sait::dfree(inv, s);
      throw;
    }
    double* scaled = sait::dalloc<double>(n, s);
    double* tmp = sait::dalloc<double>(n, s);
    sait::hadamard(n, inv, d_b, scaled, s);  // D^-1 b  (inv * b)
    SAIT_CUDA(cudaMemcpyAsync(d_x, scaled, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    for (int k = 1; k < sweeps; ++k) {
      sait::spmv(tt, d_x, tmp, s);
      sait::add_into(n, tmp, scaled, d_x, s);  // x = tmp + scaled
    }
    sait::free_csr(tt, s);
    sait::dfree(inv, s);
    sait::dfree(scaled, s);
    sait::dfree(tmp, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
  });
}

// ------------------------------------------------------------ SpMV operator

int sait_operator_create(sait_dcsr_t a, int take_ownership, sait_op_t* out) {
  return guarded([&] {
    need(a, "sait_operator_create");
    need(out, "sait_operator_create(out)");
    DeviceGuard g(a->dev);
    init_device_pool();
    auto* op = new sait_op_s;
    op->dev = a->dev;
    op->a = a;
    op->owns = take_ownership != 0;
    op->sell = sait::make_sell(a->m, SAIT_FMT_AUTO, nullptr);
    *out = op;
  });
}

int sait_operator_apply(sait_op_t op, const double* d_x, int64_t xlen, double* d_y, int64_t ylen,
                        sait_stream_t stream) {
  return guarded([&] {
    need(op, "spmv");
    const sait::DevCsr& m = op->a->m;
    if (xlen != m.ncols)
      sait::throw_invalid("spmv: vector length " + std::to_string(xlen) + " does not match ncols " +
                          std::to_string(m.ncols));
    if (ylen != m.nrows) sait::throw_invalid("spmv: output length mismatch");
    DeviceGuard g(op->dev);
    cudaStream_t s = sait::as_stream(stream);
    if (op->sell.ok()) sait::sell_spmv(op->sell, d_x, d_y, s);
    else sait::spmv(m, d_x, d_y, s);
  });
}

int sait_operator_apply_halo(sait_op_t op, const double* d_x_ext, int64_t ext_len, const sait_halo_t* halo,
                             double* d_y, int64_t ylen, sait_stream_t stream) {
  return guarded([&] {
    need(op, "spmv_halo");
    need(halo, "spmv_halo(halo)");
    const sait::DevCsr& m = op->a->m;
    if (ext_len != m.ncols)
      sait::throw_invalid("spmv: vector length " + std::to_string(ext_len) + " does not match ncols " +
                          std::to_string(m.ncols));
    if (ylen != m.nrows) sait::throw_invalid("spmv: output length mismatch");
    if (!op->sell.ok()) sait::throw_invalid("spmv_halo: the operator has no SELL copy");
    if (halo->own_lo < 0 || halo->own_hi > ext_len || halo->own_lo > halo->own_hi)
      sait::throw_invalid("spmv_halo: own segment outside the extended vector");
    if ((halo->own_lo > 0 && (!halo->lo_src || !halo->lo_flag)) ||
        (halo->own_hi < ext_len && (!halo->hi_src || !halo->hi_flag)))
      sait::throw_invalid("spmv_halo: halo source missing");
    DeviceGuard g(op->dev);
    sait::HaloArgs h;
    h.own_lo = halo->own_lo;
    h.own_hi = halo->own_hi;
    h.lo_src = halo->lo_src;
    h.lo_shift = halo->lo_shift;
    h.hi_src = halo->hi_src;
    h.hi_shift = halo->hi_shift;
    h.lo_flag = halo->lo_flag;
    h.hi_flag = halo->hi_flag;
    h.epoch = halo->epoch;
    sait::sell_spmv_halo(op->sell, d_x_ext, h, d_y, sait::as_stream(stream));
  });
}

}  // extern "C"

namespace {
sait::HaloArgs to_halo(const sait_halo_t& x, int epoch) {
  sait::HaloArgs h;
  h.own_lo = x.own_lo;
  h.own_hi = x.own_hi;
  h.lo_src = x.lo_src;
  h.lo_shift = x.lo_shift;
  h.hi_src = x.hi_src;
  h.hi_shift = x.hi_shift;
  h.lo_flag = x.lo_flag;
  h.hi_flag = x.hi_flag;
  h.epoch = epoch;
  return h;
}
}  // namespace

struct sait_peer_pair_s {
  int dev = 0;
  sait_op_t op[2] = {nullptr, nullptr};
  sait_peer_factor_desc d[2];
  // per factor: slices [0, lo_end) and [hi_begin, nslices) read halo
  // columns; [lo_end, hi_begin) is interior and runs the single-GPU kernel
  int64_t lo_end[2] = {0, 0}, hi_begin[2] = {0, 0};
  unsigned* count = nullptr;  // grid-done counters of the two publishing kernels
  int epoch = 0;
  std::mutex mu;  // one apply at a time (the epochs and buffers are shared)
};

namespace {
// One factor of a peer pair: interior slices (single-GPU kernel, PDL), then the
// boundary slice ranges (halo kernel).  The launch that carries h.pub_flag is
// the last one and is not a programmatic dependent, so when its last CTA
// publishes, every y store of the factor has completed.
void run_factor(sait_peer_pair_t p, int f, const double* x_ext, sait::HaloArgs h, double* y, cudaStream_t s) {
  const sait::SellMatrix& m = p->op[f]->sell;
  const int64_t ns = m.nslices, lo_end = std::min(p->lo_end[f], ns), hi_begin = std::max(p->hi_begin[f], lo_end);
  const bool publish = h.pub_flag != nullptr;
  sait::HaloArgs hq = h;
  hq.pub_flag = nullptr;
  hq.pub_count = nullptr;
  // interior rows [lo_end * 32, hi_begin * 32): no halo columns
  if (hi_begin > lo_end) {
    const int64_t r0 = lo_end * 32 - 0, r1 = std::min<int64_t>(hi_begin * 32, m.n);
    sait::sell_spmv_rows(m, r0, r1, x_ext, y, s, true);
  }
  const bool has_lo = lo_end > 0, has_hi = hi_begin < ns;
  if (has_lo) sait::sell_spmv_halo_slices(m, 0, lo_end, x_ext, (publish && !has_hi) ? h : hq, y, s, !publish || has_hi);
  if (has_hi) sait::sell_spmv_halo_slices(m, hi_begin, ns, x_ext, publish ? h : hq, y, s, !publish);
  if (publish && !has_lo && !has_hi) sait::publish_epoch(h.pub_flag, h.epoch, s);
}
}  // namespace

extern "C" {

int sait_peer_pair_create(sait_op_t ml, sait_op_t mu, const sait_peer_factor_desc* desc, sait_peer_pair_t* out) {
  return guarded([&] {
    need(ml, "peer_pair");
    need(mu, "peer_pair");
    need(desc, "peer_pair(desc)");
    need(out, "peer_pair(out)");
    sait_op_t ops[2] = {ml, mu};
    for (int f = 0; f < 2; ++f) {
      const sait_peer_factor_desc& x = desc[f];
      const sait::DevCsr& m = ops[f]->a->m;
      if (!ops[f]->sell.ok()) sait::throw_invalid("peer_pair: the operator has no SELL copy");
      if (!x.ext[0] || !x.ext[1] || !x.flag) sait::throw_invalid("peer_pair: null buffer");
      if (x.ext_len != m.ncols || x.own_offset < 0 || x.own_offset + x.own_len > x.ext_len)
        sait::throw_invalid("peer_pair: extended vector layout does not match the operator");
      for (int par = 0; par < 2; ++par) {
        const sait_halo_t& h = x.halo[par];
        if ((h.own_lo > 0 && (!h.lo_src || !h.lo_flag)) || (h.own_hi < x.ext_len && (!h.hi_src || !h.hi_flag)))
          sait::throw_invalid("peer_pair: halo source missing");
      }
    }
    if (ops[0]->a->m.nrows != desc[1].own_len || ops[1]->a->m.nrows != desc[1].own_len ||
        desc[0].own_len != desc[1].own_len)
      sait::throw_invalid("peer_pair: row blocks do not chain");
    for (int f = 0; f < 2; ++f) {
      const sait_peer_factor_desc& x = desc[f];
      if (x.send_n0 < 0 || x.send_n1 < 0 || x.send_a0 < 0 || x.send_a1 < 0 || x.send_a0 + x.send_n0 > x.own_len ||
          x.send_a1 + x.send_n1 > x.own_len)
        sait::throw_invalid("peer_pair: send range outside the own segment");
    }
    DeviceGuard g(ml->dev);
    auto* p = new sait_peer_pair_s;
    p->dev = ml->dev;
    p->op[0] = ml;
    p->op[1] = mu;
    p->d[0] = desc[0];
    p->d[1] = desc[1];
    SAIT_CUDA(cudaMalloc(&p->count, 2 * sizeof(unsigned)));
    SAIT_CUDA(cudaMemset(p->count, 0, 2 * sizeof(unsigned)));
    sait::preload_peer_kernels();
    for (int f = 0; f < 2; ++f) {
      sait::halo_slice_bounds(ops[f]->sell, desc[f].halo[0].own_lo, desc[f].halo[0].own_hi, &p->lo_end[f],
                              &p->hi_begin[f], nullptr);
      if (std::getenv("SAIT_DEBUG_PEER"))
        std::fprintf(stderr, "peer_pair f=%d own=[%lld,%lld) ext=%lld slices=%lld lo_end=%lld hi_begin=%lld send=(%lld,%lld)(%lld,%lld)\n", f,
                     (long long)desc[f].halo[0].own_lo, (long long)desc[f].halo[0].own_hi, (long long)desc[f].ext_len,
                     (long long)ops[f]->sell.nslices, (long long)p->lo_end[f], (long long)p->hi_begin[f],
                     (long long)desc[f].send_a0, (long long)desc[f].send_n0, (long long)desc[f].send_a1,
                     (long long)desc[f].send_n1);
    }
    *out = p;
  });
}

int sait_peer_pair_apply(sait_peer_pair_t p, const double* d_r, double* d_z, sait_stream_t stream) {
  return guarded([&] {
    need(p, "peer_pair_apply");
    DeviceGuard g(p->dev);
    std::lock_guard<std::mutex> lk(p->mu);
    cudaStream_t s = sait::as_stream(stream);
    const int e = ++p->epoch;
    const int par = e & 1;
    const sait_peer_factor_desc &L = p->d[0], &U = p->d[1];
    // 1. the slices of r the neighbours read -> M_L's extended vector, publish
    if (L.send_n0 + L.send_n1 > 0)
      sait::copy_slices_publish(d_r, L.ext[par] + L.own_offset, L.send_a0, L.send_n0, L.send_a1, L.send_n1, L.flag,
                                p->count, e, s);
    // 2. M_L: own x straight from r (ext column c = r[c - own_offset]), y into
    //    M_U's own segment.  Interior slices first with the single-GPU kernel
    //    (no waiting: the halo transfer overlaps them), then the boundary
    //    slices, which read the halo over NVLink after the owners' flags; the
    //    last launch's last CTA publishes flag_U.
    sait::HaloArgs hl = to_halo(L.halo[par], e);
    if (U.send_n0 + U.send_n1 > 0) {
      hl.pub_flag = U.flag;
      hl.pub_count = p->count + 1;
    }
    run_factor(p, 0, d_r - L.own_offset, hl, U.ext[par] + U.own_offset, s);
    // 3. M_U, the same way (programmatic dependent of M_L's last launch)
    run_factor(p, 1, U.ext[par], to_halo(U.halo[par], e), d_z, s);
  });
}

void sait_peer_pair_destroy(sait_peer_pair_t p) {
  if (!p) return;
  if (p->count) {
    cudaSetDevice(p->dev);
    cudaDeviceSynchronize();
    cudaFree(p->count);
  }
  delete p;
}

int sait_publish_epoch(int* d_flag, int epoch, sait_stream_t stream) {
  return guarded([&] {
    need(d_flag, "publish_epoch");
    sait::publish_epoch(d_flag, epoch, sait::as_stream(stream));
  });
}

int sait_ipc_handle(const void* d_ptr, void* handle64) {
  return guarded([&] {
    need(d_ptr, "ipc_handle");
    need(handle64, "ipc_handle(out)");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    SAIT_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    std::memcpy(handle64, &h, sizeof h);
  });
}

int sait_ipc_open(const void* handle64, void** d_ptr) {
  return guarded([&] {
    need(handle64, "ipc_open");
    need(d_ptr, "ipc_open(out)");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    SAIT_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int sait_ipc_close(void* d_ptr) {
  return guarded([&] {
    need(d_ptr, "ipc_close");
    SAIT_CUDA(cudaIpcCloseMemHandle(d_ptr));
  });
}

void sait_operator_destroy(sait_op_t op) {
  if (!op) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(op->dev);
  cudaDeviceSynchronize();
  sait::free_sell(op->sell, nullptr);
  cudaDeviceSynchronize();
  if (op->owns) sait_csr_free(op->a);
  if (prev >= 0) cudaSetDevice(prev);
  delete op;
}

// ------------------------------------------------------------ device ILU(0)

int sait_ilu0(sait_dcsr_t a, sait_stream_t stream, sait_dcsr_t* lower, sait_dcsr_t* upper) {
  return sait_ilu_device(a, 0, stream, lower, upper);
}

int sait_ilu_device(sait_dcsr_t a, int level, sait_stream_t stream, sait_dcsr_t* lower, sait_dcsr_t* upper) {
  return guarded([&] {
    need(a, "ilu_k");
    need(lower, "ilu_k(lower)");
    need(upper, "ilu_k(upper)");
    if (!a->m.v) sait::throw_invalid("ilu_k: matrix has no values");
    DeviceGuard g(a->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::DevCsr L, U;
    sait::ilu_device(a->m, level, L, U, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
    *lower = wrap(L);
    *upper = wrap(U);
  });
}

// --------------------------------------------------------- exact triangular

int sait_trisolve(sait_dcsr_t t, int lower, const double* d_b, int64_t blen, double* d_x,
                  sait_stream_t stream) {
  return guarded([&] {
    need(t, "trisolve");
    if (t->m.nrows != t->m.ncols) sait::throw_invalid("trisolve: matrix is not square");
    if (blen != t->m.nrows) sait::throw_invalid("trisolve: right-hand side length mismatch");
    DeviceGuard g(t->dev);
    init_device_pool();
    cudaStream_t s = sait::as_stream(stream);
    sait::TrisolveState st;
    sait::TrisolvePlan plan;
    try {
      plan = sait::analyse_triangular(t->m, lower != 0, s);
      sait::trisolve(t->m, lower != 0, plan, d_b, d_x, st, s);
    } catch (...) {
      sait::free_trisolve_state(st, s);
      sait::free_trisolve_plan(plan, s);
      throw;
    }
    sait::free_trisolve_state(st, s);
    sait::free_trisolve_plan(plan, s);
  });
}

int sait_exact_ilu_create(sait_dcsr_t lower, sait_dcsr_t upper, int take_ownership, sait_exact_t* out) {
  return guarded([&] {
    need(lower, "ExactIluPreconditioner");
    need(upper, "ExactIluPreconditioner");
    need(out, "ExactIluPreconditioner(out)");
    DeviceGuard g(lower->dev);
    init_device_pool();
    auto* p = new sait_exact_s;
    p->dev = lower->dev;
    p->l = lower;
    p->u = upper;
    try {
      p->pl = sait::analyse_triangular(lower->m, true, nullptr);
      p->pu = sait::analyse_triangular(upper->m, false, nullptr);
    } catch (...) {
      sait::free_trisolve_plan(p->pl, nullptr);
      delete p;
      throw;
    }
    p->owns = take_ownership != 0;
    *out = p;
  });
}

int sait_exact_ilu_info(sait_exact_t p, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    need(p, "ExactIluPreconditioner");
    if (n) *n = p->l->m.nrows;
    if (nnz) *nnz = p->l->m.nnz + p->u->m.nnz;
  });
}

int sait_exact_ilu_apply(sait_exact_t p, const double* d_r, int64_t rlen, double* d_z, int64_t zlen,
                         sait_stream_t stream) {
  return guarded([&] {
    need(p, "ExactIluPreconditioner::apply");
    const sait::DevCsr& L = p->l->m;
    const sait::DevCsr& U = p->u->m;
    if (L.nrows != L.ncols || U.nrows != U.ncols) sait::throw_invalid("trisolve: matrix is not square");
    if (rlen != L.nrows || U.nrows != L.nrows) sait::throw_invalid("trisolve: right-hand side length mismatch");
    if (zlen != U.nrows) sait::throw_invalid("ExactIluPreconditioner: output length mismatch");
    DeviceGuard g(p->dev);
    init_device_pool();
    sait::exact_apply_internal(p, d_r, d_z, sait::as_stream(stream));
  });
}

void sait_exact_ilu_destroy(sait_exact_t p) {
  if (!p) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(p->dev);
  cudaDeviceSynchronize();
  for (auto& kv : p->ws) {
    sait::dfree(kv.second.y, nullptr);
    sait::free_trisolve_state(kv.second.sl, nullptr);
    sait::free_trisolve_state(kv.second.su, nullptr);
  }
  sait::free_trisolve_plan(p->pl, nullptr);
  sait::free_trisolve_plan(p->pu, nullptr);
  cudaDeviceSynchronize();
  if (p->owns) {
    sait_csr_free(p->l);
    sait_csr_free(p->u);
  }
  if (prev >= 0) cudaSetDevice(prev);
  delete p;
}

// -------------------------------------------------------- pair preconditioner

int sait_pair_create(sait_dcsr_t ml, sait_dcsr_t mu, int take_ownership, sait_pair_t* out) {
  return sait_pair_create_ex(ml, mu, take_ownership, SAIT_FMT_AUTO, out);
}

int sait_pair_create_ex(sait_dcsr_t ml, sait_dcsr_t mu, int take_ownership, int format, sait_pair_t* out) {
  return guarded([&] {
    if (format < SAIT_FMT_AUTO || format > SAIT_FMT_SELL_DICT)
      sait::throw_invalid("sait_pair_create_ex: unknown format " + std::to_string(format));
    need(ml, "SaitPairPreconditioner");
    need(mu, "SaitPairPreconditioner");
    need(out, "SaitPairPreconditioner(out)");
    if (ml->m.nrows != mu->m.ncols) sait::throw_invalid("SaitPairPreconditioner: factor shapes do not chain");
    if (ml->dev != mu->dev) sait::throw_invalid("SaitPairPreconditioner: factors live on different devices");
    if (!ml->m.v || !mu->m.v) sait::throw_invalid("SaitPairPreconditioner: factors have no values");
    DeviceGuard g(ml->dev);
    init_device_pool();
    auto* p = new sait_pair_s;
    p->dev = ml->dev;
    p->ml = ml;
    p->mu = mu;
    p->owns = take_ownership != 0;
    if (format != SAIT_FMT_CSR) {
      p->sl = sait::make_sell(ml->m, format, nullptr, /*allow_perm=*/true);
      p->su = sait::make_sell(mu->m, format, nullptr, /*allow_perm=*/true);
    }
    plan_host_chunks(p);
    *out = p;
  });
}

int sait_pair_info(sait_pair_t p, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    need(p, "sait_pair_info");
    if (n) *n = p->ml->m.ncols;
    if (nnz) *nnz = p->ml->m.nnz + p->mu->m.nnz;
  });
}

int sait_pair_format(sait_pair_t p, int which, sait_factor_format* out) {
  return guarded([&] {
    need(p, "sait_pair_format");
    need(out, "sait_pair_format(out)");
    const sait::DevCsr& m = which == 0 ? p->ml->m : p->mu->m;
    const sait::SellMatrix& sm = which == 0 ? p->sl : p->su;
    sait_factor_format f{};
    f.nrows = m.nrows;
    f.nnz = m.nnz;
    // x read once (banded factors: neighbouring slices share x lines in L2),
    // y written once
    const int64_t vec = 8 * m.ncols + 8 * m.nrows;
    if (!sm.ok()) {
      f.format = SAIT_FMT_CSR;
      f.stored_slots = m.nnz;
      f.stream_bytes = 12 * m.nnz + 4 * (m.nrows + 1) + vec;
    } else {
      f.stored_slots = sm.padded;
      f.nslices = sm.nslices;
      f.dict_elems = sm.dict_elems;
      f.row_sorted = sm.perm ? 1 : 0;
      // (+ the row permutation of a row-sorted copy: one int32 per slot position)
      const int64_t soff = 8 * (sm.nslices + 1) + (sm.perm ? 4 * sm.nslices * 32 : 0);
      switch (sm.index_kind()) {
        case 2:  // values stream; one int32 pattern offset per slice; the dictionary once
          f.format = SAIT_FMT_SELL_DICT;
          f.stream_bytes = 8 * sm.padded + soff + 4 * sm.nslices + 4 * sm.dict_elems + vec;
          break;
        case 1:
          f.format = SAIT_FMT_SELL_I16;
          f.stream_bytes = 10 * sm.padded + soff + vec;
          break;
        default:
          f.format = SAIT_FMT_SELL_I32;
          f.stream_bytes = 12 * sm.padded + soff + vec;
      }
    }
    *out = f;
  });
}

int sait_pair_factors(sait_pair_t p, sait_dcsr_t* ml, sait_dcsr_t* mu) {
  return guarded([&] {
    need(p, "sait_pair_factors");
    if (ml) *ml = p->ml;
    if (mu) *mu = p->mu;
  });
}

}  // extern "C"

namespace {
// M_U's SpMV is launched as a programmatic dependent of M_L's (PDL): its
// CTAs start and load their matrix slices while M_L's tail runs, then wait
// (griddepcontrol.wait) before touching y.  SAIT_PDL=0 disables.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SAIT_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// One factor's SpMV with the fastest kernel available for it.
void factor_spmv(sait_pair_t p, int which, const double* x, double* y, cudaStream_t s) {
  const sait::DevCsr& m = which == 0 ? p->ml->m : p->mu->m;
  const sait::SellMatrix& sm = which == 0 ? p->sl : p->su;
  // both halves are programmatic dependents of whatever precedes them on s:
  // M_U of M_L, and M_L of the previous kernel (e.g. the last apply's M_U),
  // each loading its first index/value batch before griddepcontrol.wait
  if (sm.ok()) sait::sell_spmv_rows(sm, 0, sm.n, x, y, s, pdl_enabled());
  else sait::spmv(m, x, y, s);
}

sait_pair_s::Work& pair_work(sait_pair_t p, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(p->mu_ws);
  auto it = p->ws.find(s);
  if (it != p->ws.end()) return it->second;
  sait_pair_s::Work w;
  const int64_t n = p->ml->m.nrows;
  SAIT_CUDA(cudaMalloc(&w.y, sizeof(double) * (n > 0 ? n : 1) + 256));
  SAIT_CUDA(cudaDeviceSynchronize());
  return p->ws.emplace(s, w).first->second;
}
// z = M_U (M_L r) for HOST r/z, overlapping the PCIe copies with the two
// SpMVs chunk by chunk: r chunks stream in on s_in; M_L chunk c runs as soon as
// the r chunks its columns reach have landed; M_U chunk c runs once the y
// chunks it reads exist (bounded bandwidth of the triangular factors), and its
// z chunk streams out on s_out while later r chunks are still arriving.
bool device_mapped(const void* p);

// Host-vector applies are synchronous, so the stream is an implementation
// detail when the caller passes none: each calling thread gets its own, and
// concurrent host applies from several threads run side by side.
cudaStream_t host_call_stream(sait_stream_t stream) {
  if (stream) return sait::as_stream(stream);
  struct Holder {
    cudaStream_t s = nullptr;
    ~Holder() {
      if (s) cudaStreamDestroy(s);
    }
  };
  thread_local Holder h;
  if (!h.s) SAIT_CUDA(cudaStreamCreateWithFlags(&h.s, cudaStreamNonBlocking));
  return h.s;
}

void ensure_side_streams(sait_pair_s::Work& w) {
  if (w.s_in) return;
  SAIT_CUDA(cudaStreamCreateWithFlags(&w.s_in, cudaStreamNonBlocking));
  SAIT_CUDA(cudaStreamCreateWithFlags(&w.s_out, cudaStreamNonBlocking));
  SAIT_CUDA(cudaEventCreateWithFlags(&w.ev_entry, cudaEventDisableTiming));
  SAIT_CUDA(cudaEventCreateWithFlags(&w.ev_out_done, cudaEventDisableTiming));
}

bool block_host_pipeline_enabled() {
  const char* e = std::getenv("SAIT_BLOCK_HOST_PIPELINE");
  return !(e && std::atoi(e) == 0);
}

bool host_zc_out_enabled() {
  const char* e = std::getenv("SAIT_HOST_ZC_OUT");
  return !(e && std::atoi(e) == 0);
}

void pair_apply_host_chunked(sait_pair_t p, const double* h_r, double* h_z, cudaStream_t s) {
  sait_pair_s::Work& w = pair_work(p, s);
  std::lock_guard<std::mutex> lk(*w.mu);
  const int64_t k = static_cast<int64_t>(p->chunk_rows.size()) - 1;
  const int64_t n = p->ml->m.nrows;
  // each resource on its own: the dataflow and block paths share this Work
  // and create only what they use
  ensure_side_streams(w);
  if (!w.r_dev) {
    SAIT_CUDA(cudaMalloc(&w.r_dev, sizeof(double) * n + 256));
    SAIT_CUDA(cudaMalloc(&w.z_dev, sizeof(double) * n + 256));
  }
  if (w.ev_in.size() != static_cast<size_t>(k)) {
    w.ev_in.resize(k);
    w.ev_u.resize(k);
    for (auto& e : w.ev_in) SAIT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : w.ev_u) SAIT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  static const bool dbg = std::getenv("SAIT_DEBUG_PIPE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  auto mark = [&](const std::string& nm, cudaStream_t st) {
    if (!dbg) return;
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, st);
    marks.emplace_back(nm, e);
  };
  const auto t_enq = std::chrono::steady_clock::now();
  mark("start", s);
  // order the side streams after whatever the caller queued on s
  SAIT_CUDA(cudaEventRecord(w.ev_entry, s));
  SAIT_CUDA(cudaStreamWaitEvent(w.s_in, w.ev_entry, 0));
  SAIT_CUDA(cudaStreamWaitEvent(w.s_out, w.ev_entry, 0));
  const auto& b = p->chunk_rows;
  for (int64_t c = 0; c < k; ++c) {
    SAIT_CUDA(cudaMemcpyAsync(w.r_dev + b[c], h_r + b[c], sizeof(double) * (b[c + 1] - b[c]), cudaMemcpyHostToDevice,
                              w.s_in));
    SAIT_CUDA(cudaEventRecord(w.ev_in[c], w.s_in));
    mark("h2d" + std::to_string(c), w.s_in);
  }
  const auto& ub = p->u_rows;
  // z straight into the caller's (pinned, device-mapped) host buffer: the M_U
  // chunks' stores cross PCIe as they are produced, so no D2H stage trails the
  // last input chunk (SAIT_HOST_ZC_OUT=0 keeps the copy-engine D2H chunks).
  const bool zc_out = host_zc_out_enabled() && device_mapped(h_z);
  for (int64_t c = 0; c < k; ++c) {
    SAIT_CUDA(cudaStreamWaitEvent(s, w.ev_in[p->needL_hi[c]], 0));
    sait::sell_spmv_rows(p->sl, b[c], b[c + 1], w.r_dev, w.y, s);
    mark("L" + std::to_string(c), s);
    if (ub[c + 1] > ub[c]) {
      if (zc_out) {
        sait::sell_spmv_rows(p->su, ub[c], ub[c + 1], w.y, h_z, s);
        mark("U" + std::to_string(c), s);
        continue;
      }
      sait::sell_spmv_rows(p->su, ub[c], ub[c + 1], w.y, w.z_dev, s);
      SAIT_CUDA(cudaEventRecord(w.ev_u[c], s));
      mark("U" + std::to_string(c), s);
      SAIT_CUDA(cudaStreamWaitEvent(w.s_out, w.ev_u[c], 0));
      SAIT_CUDA(cudaMemcpyAsync(h_z + ub[c], w.z_dev + ub[c], sizeof(double) * (ub[c + 1] - ub[c]),
                                cudaMemcpyDeviceToHost, w.s_out));
      mark("d2h" + std::to_string(c), w.s_out);
    }
  }
  SAIT_CUDA(cudaEventRecord(w.ev_out_done, w.s_out));
  SAIT_CUDA(cudaStreamWaitEvent(s, w.ev_out_done, 0));
  mark("end", s);
  if (dbg) {  // host-side timeline: poll the marks, microseconds since enqueue start
    const auto t_done = std::chrono::steady_clock::now();
    std::vector<double> at(marks.size(), -1.0);
    size_t left = marks.size();
    while (left) {
      for (size_t i = 0; i < marks.size(); ++i)
        if (at[i] < 0 && cudaEventQuery(marks[i].second) == cudaSuccess) {
          at[i] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_enq).count();
          --left;
        }
    }
    std::fprintf(stderr, "enqueue=%.1f ", std::chrono::duration<double, std::micro>(t_done - t_enq).count());
    for (size_t i = 0; i < marks.size(); ++i) {
      std::fprintf(stderr, "%s=%.1f ", marks[i].first.c_str(), at[i]);
      cudaEventDestroy(marks[i].second);
    }
    std::fprintf(stderr, "\n");
  }
  SAIT_CUDA(cudaStreamSynchronize(s));
}

// Host memory the GPU can address directly (pinned / registered under UVA).
bool device_mapped(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

// Column-major block of HOST vectors (apply_block, preconditioner.cpp:47-49):
// a three-stage pipeline over groups of vectors.  Group g's r columns are
// copied in on s_in (one copy), the SpMV pair runs per vector on s, and the
// group's z columns are copied out on s_out, so the H2D of g+1 and the D2H of
// g-1 share the full-duplex PCIe link with the pairs of g; kBlkSlots device
// slots per side bound how far the input runs ahead.  Throughput is
// max(H2D, D2H) per vector instead of their sum.  Each cross-stream hand-off
// costs the copy engines a few tens of microseconds, so the middle groups
// hold several vectors, while single-vector head and tail groups keep the
// pipeline fill and drain short (SAIT_BLK_GROUPS = "head,..;mid;tail,..").
constexpr int kBlkSlotsMax = 4;
int blk_slots() {
  static const int v = [] {
    const char* e = std::getenv("SAIT_BLK_SLOTS");
    const int k = e ? std::atoi(e) : 3;
    return std::min(std::max(k, 1), kBlkSlotsMax);
  }();
  return v;
}
struct BlkGroups {
  std::vector<int> head, tail;
  int mid = 4;
  int max() const {
    int m = mid;
    for (int g : head) m = std::max(m, g);
    for (int g : tail) m = std::max(m, g);
    return m;
  }
};
const BlkGroups& blk_groups() {
  static const BlkGroups v = [] {
    BlkGroups b;
    b.head = {1};
    b.tail = {1};
    const char* e = std::getenv("SAIT_BLK_GROUPS");
    if (!e) return b;
    auto parse = [](const std::string& t) {
      std::vector<int> out;
      size_t a = 0;
      while (a < t.size()) {
        size_t c = t.find(',', a);
        if (c == std::string::npos) c = t.size();
        if (c > a) out.push_back(std::max(1, std::atoi(t.substr(a, c - a).c_str())));
        a = c + 1;
      }
      return out;
    };
    const std::string spec(e);
    const size_t s1 = spec.find(';');
    const size_t s2 = s1 == std::string::npos ? std::string::npos : spec.find(';', s1 + 1);
    if (s1 == std::string::npos || s2 == std::string::npos) {
      b.head.clear();
      b.tail.clear();
      b.mid = std::max(1, std::atoi(spec.c_str()));
      return b;
    }
    b.head = parse(spec.substr(0, s1));
    b.mid = std::max(1, std::atoi(spec.substr(s1 + 1, s2 - s1 - 1).c_str()));
    b.tail = parse(spec.substr(s2 + 1));
    return b;
  }();
  return v;
}
// group sizes covering nvec vectors: head groups, middle groups, tail groups
std::vector<int64_t> blk_group_sizes(int64_t nvec) {
  const BlkGroups& b = blk_groups();
  std::vector<int64_t> head, tail, out;
  int64_t left = nvec;
  for (int g : b.head)
    if (left > 0) {
      head.push_back(std::min<int64_t>(g, left));
      left -= head.back();
    }
  for (auto it = b.tail.rbegin(); it != b.tail.rend(); ++it)
    if (left > 0) {
      tail.insert(tail.begin(), std::min<int64_t>(*it, left));
      left -= tail.front();
    }
  out = head;
  while (left > 0) {
    out.push_back(std::min<int64_t>(b.mid, left));
    left -= out.back();
  }
  out.insert(out.end(), tail.begin(), tail.end());
  return out;
}

// Pageable caller blocks (the reference's callers hold std::vector storage):
// a cudaMemcpyAsync from or to pageable memory is staged by the driver on
// the calling thread at ~13 GB/s, H2D and D2H taking turns.  Instead each
// group is copied by the host cores (OpenMP, 1 MB pieces) into a pinned slot
// of its own and DMA'd from there, and z groups come back through pinned
// slots the same way, so the DMA of one group overlaps the host copies of its
// neighbours.  SAIT_STAGE_THREADS bounds the copying threads (default: the
// OpenMP maximum, at most 16); SAIT_HOST_STAGING=0 leaves it to the driver.
bool host_staging_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SAIT_HOST_STAGING");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}
int stage_threads() {
  static const int v = [] {
    const char* e = std::getenv("SAIT_STAGE_THREADS");
    const int k = e ? std::atoi(e) : std::min(omp_get_max_threads(), 16);
    return std::max(k, 1);
  }();
  return v;
}
// SAIT_STAGE_COPY: 0 = memcpy in 1 MB pieces, 1 = one contiguous memcpy per
// thread, 2 (default on x86-64) = streaming (non-temporal) 16-byte stores,
// which skip the read-for-ownership of the destination lines.
int stage_copy_mode() {
  static const int v = [] {
    const char* e = std::getenv("SAIT_STAGE_COPY");
#if defined(__x86_64__)
    return e ? std::atoi(e) : 2;
#else
    return e ? std::min(std::atoi(e), 1) : 1;
#endif
  }();
  return v;
}
void copy_streaming(char* d, const char* s, size_t bytes) {
#if defined(__x86_64__)
  size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
  if (head > bytes) head = bytes;
  std::memcpy(d, s, head);
  d += head, s += head, bytes -= head;
  const size_t body = bytes & ~size_t{63};
  for (size_t o = 0; o < body; o += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + o));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + o + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + o + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + o + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + o), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + o + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + o + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + o + 48), e);
  }
  _mm_sfence();
  std::memcpy(d + body, s + body, bytes - body);
#else
  std::memcpy(d, s, bytes);
#endif
}
void host_copy_parallel(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = size_t{1} << 20;
  const int64_t pieces = static_cast<int64_t>((bytes + kPiece - 1) / kPiece);
  const int nt = static_cast<int>(std::min<int64_t>(stage_threads(), pieces));
  const int mode = stage_copy_mode();
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  if (mode == 0) {
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int64_t i = 0; i < pieces; ++i) {
      const size_t o = static_cast<size_t>(i) * kPiece;
      std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kPiece, bytes - o));
    }
    return;
  }
  // one contiguous, 4 KB-aligned range per thread
  const size_t per = ((bytes + nt - 1) / nt + 4095) & ~size_t{4095};
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int t = 0; t < nt; ++t) {
    const size_t o = static_cast<size_t>(t) * per;
    if (o >= bytes) continue;
    const size_t len = std::min(per, bytes - o);
    if (mode == 2) copy_streaming(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, len);
    else std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, len);
  }
}

void pair_apply_block_host_pipelined(sait_pair_t p, const double* h_r, double* h_z, int64_t n, int64_t nvec,
                                     cudaStream_t s) {
  const int kBlkSlots = blk_slots();
  const int64_t gmax = blk_groups().max();
  const bool stage_in = host_staging_enabled() && !device_mapped(h_r);
  const bool stage_out = host_staging_enabled() && !device_mapped(h_z);
  sait_pair_s::Work& w = pair_work(p, s);
  std::lock_guard<std::mutex> lk(*w.mu);
  ensure_side_streams(w);
  if (!w.blk_r) {
    SAIT_CUDA(cudaMalloc(&w.blk_r, sizeof(double) * n * gmax * kBlkSlots + 256));
    SAIT_CUDA(cudaMalloc(&w.blk_z, sizeof(double) * n * gmax * kBlkSlots + 256));
    for (int q = 0; q < kBlkSlots; ++q)
      for (cudaEvent_t* e : {&w.ev_blk_in[q], &w.ev_blk_done[q], &w.ev_blk_out[q]})
        SAIT_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  SAIT_CUDA(cudaEventRecord(w.ev_entry, s));
  SAIT_CUDA(cudaStreamWaitEvent(w.s_in, w.ev_entry, 0));
  SAIT_CUDA(cudaStreamWaitEvent(w.s_out, w.ev_entry, 0));
  // SAIT_DEBUG_BLK: per-group device timeline (H2D, pairs, D2H start/end) to stderr
  static const bool dbg = std::getenv("SAIT_DEBUG_BLK") != nullptr;
  std::vector<cudaEvent_t> tl;
  auto mark = [&](cudaStream_t st) {
    if (!dbg) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tl.push_back(e);
  };
  std::vector<int64_t> groups = blk_group_sizes(nvec);
  int64_t gstage = gmax;
  if (stage_in || stage_out) {
    // uniform groups of at most 64 MB bound the pinned slots
    gstage = std::max<int64_t>(1, std::min<int64_t>(gmax, (int64_t{64} << 20) / (8 * std::max<int64_t>(n, 1))));
    groups.clear();
    for (int64_t left = nvec; left > 0; left -= groups.back()) groups.push_back(std::min(gstage, left));
    const size_t need = static_cast<size_t>(n) * gstage * kBlkSlots;
    if (stage_in && w.pin_r_elems < need) {
      if (w.pin_r) SAIT_CUDA(cudaFreeHost(w.pin_r));
      w.pin_r = nullptr, w.pin_r_elems = 0;
      SAIT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.pin_r), sizeof(double) * need, cudaHostAllocDefault));
      w.pin_r_elems = need;
    }
    if (stage_out && w.pin_z_elems < need) {
      if (w.pin_z) SAIT_CUDA(cudaFreeHost(w.pin_z));
      w.pin_z = nullptr, w.pin_z_elems = 0;
      SAIT_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.pin_z), sizeof(double) * need, cudaHostAllocDefault));
      w.pin_z_elems = need;
    }
  }
  std::vector<int64_t> gstart(groups.size() + 1, 0);
  for (size_t gi = 0; gi < groups.size(); ++gi) gstart[gi + 1] = gstart[gi] + groups[gi];
  // z of group go leaves its pinned slot for the caller's pageable block
  auto drain = [&](size_t go) {
    const int qo = static_cast<int>(go % kBlkSlots);
    SAIT_CUDA(cudaEventSynchronize(w.ev_blk_out[qo]));
    host_copy_parallel(h_z + gstart[go] * n, w.pin_z + static_cast<size_t>(qo) * gstage * n,
                       sizeof(double) * n * groups[go]);
  };
  int64_t v0 = 0;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const int64_t g = groups[gi];
    const int q = static_cast<int>(gi % kBlkSlots);
    double* r = w.blk_r + q * gmax * n;
    double* z = w.blk_z + q * gmax * n;
    const double* src = h_r + v0 * n;
    if (stage_in) {
      double* pr = w.pin_r + static_cast<size_t>(q) * gstage * n;
      if (gi >= static_cast<size_t>(kBlkSlots)) SAIT_CUDA(cudaEventSynchronize(w.ev_blk_in[q]));  // slot's last H2D
      host_copy_parallel(pr, src, sizeof(double) * n * g);
      src = pr;
    }
    if (gi >= static_cast<size_t>(kBlkSlots))
      SAIT_CUDA(cudaStreamWaitEvent(w.s_in, w.ev_blk_done[q], 0));  // the pairs of gi-slots read r
    mark(w.s_in);
    SAIT_CUDA(cudaMemcpyAsync(r, src, sizeof(double) * n * g, cudaMemcpyHostToDevice, w.s_in));
    mark(w.s_in);
    SAIT_CUDA(cudaEventRecord(w.ev_blk_in[q], w.s_in));
    SAIT_CUDA(cudaStreamWaitEvent(s, w.ev_blk_in[q], 0));
    if (gi >= static_cast<size_t>(kBlkSlots))
      SAIT_CUDA(cudaStreamWaitEvent(s, w.ev_blk_out[q], 0));  // z of gi-slots copied out
    mark(s);
    for (int64_t c = 0; c < g; ++c) {
      factor_spmv(p, 0, r + c * n, w.y, s);
      factor_spmv(p, 1, w.y, z + c * n, s);
    }
    mark(s);
    SAIT_CUDA(cudaEventRecord(w.ev_blk_done[q], s));
    SAIT_CUDA(cudaStreamWaitEvent(w.s_out, w.ev_blk_done[q], 0));
    mark(w.s_out);
    // the pinned z slot q still holds group gi - slots until it is drained
    if (stage_out && gi >= static_cast<size_t>(kBlkSlots)) drain(gi - kBlkSlots);
    double* dst = stage_out ? w.pin_z + static_cast<size_t>(q) * gstage * n : h_z + v0 * n;
    SAIT_CUDA(cudaMemcpyAsync(dst, z, sizeof(double) * n * g, cudaMemcpyDeviceToHost, w.s_out));
    mark(w.s_out);
    SAIT_CUDA(cudaEventRecord(w.ev_blk_out[q], w.s_out));
    v0 += g;
  }
  if (stage_out)
    for (size_t go = groups.size() > static_cast<size_t>(kBlkSlots) ? groups.size() - kBlkSlots : 0; go < groups.size();
         ++go)
      drain(go);
  SAIT_CUDA(cudaEventRecord(w.ev_out_done, w.s_out));
  SAIT_CUDA(cudaStreamWaitEvent(s, w.ev_out_done, 0));
  SAIT_CUDA(cudaStreamSynchronize(s));
  if (dbg) {
    SAIT_CUDA(cudaDeviceSynchronize());
    auto at = [&](size_t i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tl[0], tl[i]);
      return 1e3 * ms;
    };
    const size_t ng = groups.size();
    for (size_t gi = 0; gi < ng; ++gi) {
      if (gi > 6 && gi + 3 < ng) continue;
      const size_t b = gi * 6;
      std::fprintf(stderr, "g%zu(%lld) h2d %.0f-%.0f pair %.0f-%.0f d2h %.0f-%.0f us\n", gi,
                   static_cast<long long>(groups[gi]), at(b), at(b + 1), at(b + 2), at(b + 3), at(b + 4), at(b + 5));
    }
    for (auto e : tl) cudaEventDestroy(e);
  }
}

}  // namespace

namespace sait {
// z = M_U (M_L r) on device vectors (used by the solver loops)
void pair_apply_internal(sait_pair_t p, const double* r, double* z, cudaStream_t s) {
  sait_pair_s::Work& w = pair_work(p, s);
  std::lock_guard<std::mutex> lk(*w.mu);  // the two launches of one apply stay adjacent on s
  factor_spmv(p, 0, r, w.y, s);
  factor_spmv(p, 1, w.y, z, s);
}
int64_t pair_dim(sait_pair_t p) { return p->ml->m.ncols; }
int pair_device(sait_pair_t p) { return p->dev; }

// z = U^-1 (L^-1 r) on device vectors (ExactIluPreconditioner::apply)
void exact_apply_internal(sait_exact_t p, const double* r, double* z, cudaStream_t s) {
  sait_exact_s::Work* w;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    w = &p->ws[s];
    if (!w->y && p->l->m.nrows) w->y = sait::dalloc<double>(p->l->m.nrows, s);
  }
  std::lock_guard<std::mutex> turn(*w->mu);
  sait::trisolve(p->l->m, true, p->pl, r, w->y, w->sl, s);   // y = L^-1 r (unit_lower_triangular)
  sait::trisolve(p->u->m, false, p->pu, w->y, z, w->su, s);  // z = U^-1 y (upper_triangular)
}
int64_t exact_dim(sait_exact_t p) { return p->l->m.nrows; }
}  // namespace sait

extern "C" {

int sait_pair_apply(sait_pair_t p, const double* d_r, int64_t rlen, double* d_z, int64_t zlen, sait_stream_t stream) {
  return guarded([&] {
    need(p, "apply");
    const sait::DevCsr& L = p->ml->m;
    const sait::DevCsr& U = p->mu->m;
    if (rlen != L.ncols)
      sait::throw_invalid("spmv: vector length " + std::to_string(rlen) + " does not match ncols " +
                          std::to_string(L.ncols));
    if (zlen != U.nrows) sait::throw_invalid("spmv: output length mismatch");
    DeviceGuard g(p->dev);
    cudaStream_t s = sait::as_stream(stream);
    sait::pair_apply_internal(p, d_r, d_z, s);
  });
}

int sait_pair_spmv_factor(sait_pair_t p, int which, const double* d_x, double* d_y, sait_stream_t stream) {
  return guarded([&] {
    need(p, "sait_pair_spmv_factor");
    DeviceGuard g(p->dev);
    cudaStream_t s = sait::as_stream(stream);
    factor_spmv(p, which != 0, d_x, d_y, s);
  });
}

int sait_pair_apply_host(sait_pair_t p, const double* h_r, int64_t rlen, double* h_z, int64_t zlen,
                         sait_stream_t stream) {
  return guarded([&] {
    need(p, "apply");
    const sait::DevCsr& L = p->ml->m;
    const sait::DevCsr& U = p->mu->m;
    if (rlen != L.ncols)
      sait::throw_invalid("spmv: vector length " + std::to_string(rlen) + " does not match ncols " +
                          std::to_string(L.ncols));
    if (zlen != U.nrows) sait::throw_invalid("spmv: output length mismatch");
    DeviceGuard g(p->dev);
    cudaStream_t s = host_call_stream(stream);
    if (p->chunk_rows.size() >= 3) pair_apply_host_chunked(p, h_r, h_z, s);
    else sait::pair_apply_host_pipelined(L, U, h_r, h_z, s);
  });
}

namespace {
// Row-major block product with one factor (fastest available kernel).
void factor_spmm(sait_pair_t p, int which, const double* x, double* y, int nvec, cudaStream_t s) {
  if (nvec == 1) {
    factor_spmv(p, which, x, y, s);
    return;
  }
  const sait::SellMatrix& sm = which == 0 ? p->sl : p->su;
  if (sm.ok() && sait::sell_spmm(sm, x, y, nvec, s)) return;
  sait::spmm_rowmajor(which == 0 ? p->ml->m : p->mu->m, x, y, nvec, s);
}

// Column-major slab of w (1, 2, 4 or 8) vectors: transpose to row-major, run
// the block SpMM pair (matrix read once per slab), transpose back.
void apply_slab(sait_pair_t p, const double* r_cm, double* z_cm, int64_t n, int w, double* rt, double* y,
                double* zt, cudaStream_t s) {
  if (w == 1) {
    factor_spmv(p, 0, r_cm, y, s);
    factor_spmv(p, 1, y, z_cm, s);
    return;
  }
  sait::transpose_block(r_cm, rt, n, w, true, s);
  factor_spmm(p, 0, rt, y, w, s);
  factor_spmm(p, 1, y, zt, w, s);
  sait::transpose_block(zt, z_cm, n, w, false, s);
}

void apply_block_device(sait_pair_t p, const double* d_r, double* d_z, int64_t n, int64_t nvec, int layout,
                        cudaStream_t s) {
  const sait::DevCsr& L = p->ml->m;
  const sait::DevCsr& U = p->mu->m;
  if (n != L.ncols || n != U.nrows) sait::throw_invalid("spmm: dimension mismatch");
  if (layout != 0 && layout != 1) sait::throw_invalid("apply_block: layout must be 0 or 1");
  if (nvec <= 0 || n == 0) return;
  if (layout == 1 && (nvec == 1 || nvec == 2 || nvec == 4 || nvec == 8)) {
    double* y = sait::dalloc<double>(L.nrows * nvec, s);
    factor_spmm(p, 0, d_r, y, static_cast<int>(nvec), s);
    factor_spmm(p, 1, y, d_z, static_cast<int>(nvec), s);
    sait::dfree(y, s);
    return;
  }
  if (layout == 0 && p->sl.ok() && p->su.ok()) {
    // column-major straight through the SELL block kernels (no transposes)
    double* y = sait::dalloc<double>(L.nrows * nvec, s);
    sait::sell_spmm_colmajor(p->sl, d_r, n, y, L.nrows, static_cast<int>(nvec), s);
    sait::sell_spmm_colmajor(p->su, y, L.nrows, d_z, n, static_cast<int>(nvec), s);
    sait::dfree(y, s);
    return;
  }
  const double* rcm = d_r;
  double* zcm = d_z;
  double* tmp_r = nullptr;
  double* tmp_z = nullptr;
  if (layout == 1) {  // row-major in: work column-major, convert at the ends
    tmp_r = sait::dalloc<double>(n * nvec, s);
    tmp_z = sait::dalloc<double>(n * nvec, s);
    sait::transpose_block(d_r, tmp_r, n, static_cast<int>(nvec), false, s);
    rcm = tmp_r;
    zcm = tmp_z;
  }
  double* y = sait::dalloc<double>(L.nrows * 8, s);
  double* rt = sait::dalloc<double>(n * 8, s);
  double* zt = sait::dalloc<double>(n * 8, s);
  for (int64_t c0 = 0; c0 < nvec;) {
    int64_t left = nvec - c0;
    int w = left >= 8 ? 8 : (left >= 4 ? 4 : (left >= 2 ? 2 : 1));
    apply_slab(p, rcm + c0 * n, zcm + c0 * n, n, w, rt, y, zt, s);
    c0 += w;
  }
  sait::dfree(y, s);
  sait::dfree(rt, s);
  sait::dfree(zt, s);
  if (layout == 1) {
    sait::transpose_block(tmp_z, d_z, n, static_cast<int>(nvec), true, s);
    sait::dfree(tmp_r, s);
    sait::dfree(tmp_z, s);
  }
}
}  // namespace

int sait_pair_apply_block(sait_pair_t p, const double* d_r, double* d_z, int64_t n, int64_t nvec, int layout,
                          sait_stream_t stream) {
  return guarded([&] {
    need(p, "apply_block");
    DeviceGuard g(p->dev);
    apply_block_device(p, d_r, d_z, n, nvec, layout, sait::as_stream(stream));
  });
}

int sait_pair_apply_block_host(sait_pair_t p, const double* h_r, double* h_z, int64_t n, int64_t nvec, int layout,
                               sait_stream_t stream) {
  return guarded([&] {
    need(p, "apply_block");
    DeviceGuard g(p->dev);
    if (layout == 0 && nvec > 1 && n == p->ml->m.nrows && n == p->mu->m.nrows && block_host_pipeline_enabled()) {
      pair_apply_block_host_pipelined(p, h_r, h_z, n, nvec, host_call_stream(stream));
      return;
    }
    cudaStream_t s = sait::as_stream(stream);
    double* r = sait::dalloc<double>(n * nvec, s);
    double* z = sait::dalloc<double>(n * nvec, s);
    SAIT_CUDA(cudaMemcpyAsync(r, h_r, sizeof(double) * n * nvec, cudaMemcpyHostToDevice, s));
    apply_block_device(p, r, z, n, nvec, layout, s);
    SAIT_CUDA(cudaMemcpyAsync(h_z, z, sizeof(double) * n * nvec, cudaMemcpyDeviceToHost, s));
    sait::dfree(r, s);
    sait::dfree(z, s);
    SAIT_CUDA(cudaStreamSynchronize(s));
  });
}

void sait_pair_destroy(sait_pair_t p) {
  if (!p) return;
  {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->dev);
    cudaDeviceSynchronize();
    sait::free_sell(p->sl, nullptr);
    sait::free_sell(p->su, nullptr);
    for (auto& kv : p->ws) {
      auto& w = kv.second;
      cudaFree(w.y);
      if (w.r_dev) cudaFree(w.r_dev);
      if (w.z_dev) cudaFree(w.z_dev);
      if (w.blk_r) cudaFree(w.blk_r);
      if (w.blk_z) cudaFree(w.blk_z);
      if (w.pin_r) cudaFreeHost(w.pin_r);
      if (w.pin_z) cudaFreeHost(w.pin_z);
      for (int q = 0; q < 4; ++q)
        for (cudaEvent_t e : {w.ev_blk_in[q], w.ev_blk_done[q], w.ev_blk_out[q]})
          if (e) cudaEventDestroy(e);
      for (auto e : w.ev_in) cudaEventDestroy(e);
      for (auto e : w.ev_u) cudaEventDestroy(e);
      if (w.ev_entry) cudaEventDestroy(w.ev_entry);
      if (w.ev_out_done) cudaEventDestroy(w.ev_out_done);
      if (w.s_in) cudaStreamDestroy(w.s_in);
      if (w.s_out) cudaStreamDestroy(w.s_out);
    }
    cudaDeviceSynchronize();
    if (prev >= 0) cudaSetDevice(prev);
  }
  if (p->owns) {
    sait_csr_free(p->ml);
    sait_csr_free(p->mu);
  }
  delete p;
}

}  // extern "C"

namespace sait {
void pair_apply_block_internal(sait_pair_t p, const double* r, double* z, int64_t n, int64_t nvec, int layout,
                               cudaStream_t s) {
  apply_block_device(p, r, z, n, nvec, layout, s);
}
}  // namespace sait
