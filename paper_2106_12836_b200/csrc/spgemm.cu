// spgemm.cu — K2/K3: row-wise Gustavson SpGEMM C = A B with a fused epilogue
// (+I, threshold / pattern / fill-cap drop, stabilization compare).
//
// Reference semantics (kernels.cpp:34-102): output (i, j) accumulates
//   acc = a(i,k1) * b(k1,j);  acc = acc + a(i,k) * b(k,j)  for later k
// in increasing order of k along A's row i; the product is rounded before
// the add (no FMA); columns are emitted sorted.  add_identity
// (kernels.cpp:104-134) then adds 1.0 to / inserts 1.0 at the diagonal, and
// the drop rule (kernels.cpp:136-194, or the A15 cap) filters the row.
//
// B200 design: one warp per output row, a per-warp open-addressing hash table
// in shared memory (global memory for very long rows).  Lanes take the row's
// products 32 at a time in (k, b-entry) order; lanes that hit the same output
// column in one round are grouped with __match_any_sync and their leader folds
// the group's products into the slot in lane order, i.e. in increasing k.
// Rounds are separated by __syncwarp, so every output entry sees its products
// in exactly the reference order: the result is bitwise identical while all
// 32 lanes stay busy.  The count pass computes each row's post-drop length
// (values are needed to know what survives a threshold), a scan sizes C, and
// the numeric pass recomputes, compacts, bitonic-sorts and writes the row.
#include <algorithm>
#include <vector>

#include <cstdlib>

#include "common.cuh"
#include "sort.cuh"

namespace sait {

int64_t scan_counts(const int32_t* counts, int32_t* row_ptr, int64_t n, cudaStream_t s);
void scan_counts_async(const int32_t* counts, int32_t* row_ptr, int64_t n, int64_t* total_dev, cudaStream_t s);

namespace {

constexpr int32_t kEmpty = -1;
constexpr int kFresh = 1 << 30;
// Row bins: 0/1/2 = tiny (< 8/16/32 products, <= 8/16/32 A entries: register
// path, 4/2/1 rows per warp), 3..9 = shared-memory tables of 64 .. 4096
// slots, 10 = global-memory tables.
constexpr int kTinyBins = 3;
#ifndef SAIT_WIN_PHASED
#define SAIT_WIN_PHASED 1
#endif
#ifndef SAIT_HASH_PHASED
#define SAIT_HASH_PHASED 0
#endif
constexpr int kFirstSmemBin = kTinyBins;
constexpr int kNumSmemBins = 7;
constexpr int kMinLogSlots = 6;
constexpr int kGlobalBin = kFirstSmemBin + kNumSmemBins;
// window bins: rows whose product columns all fall in [base, base + 128 Q)
// (Q = kWinQ[i]), accumulated by direct addressing instead of hashing
// (below); the smaller windows fit more rows in flight per SM.  Rows whose
// columns span 1024 or more stay in the hash-table bins: a 2048-slot window
// holds 16 KB per warp, and the 512-slot tables did those rows faster (C4:
// 8.2 vs 10.2 ms per build)
constexpr int kNumWinBins = 5;
constexpr int kWinQ[kNumWinBins] = {4, 5, 6, 7, 8};
__host__ __device__ constexpr int win_q(int i) { return 4 + i; }  // kWinQ[i] (device code)
constexpr int kWinBin0 = kGlobalBin + 1;
constexpr int kNumBins = kWinBin0 + kNumWinBins;
constexpr int kTinyG[kTinyBins] = {8, 16, 32};

struct Args {
  int64_t n;
  int64_t ncols;
  const int32_t* arp;
  const int32_t* aci;
  const double* av;
  const int32_t* brp;
  const int32_t* bci;
  const double* bv;
  Epilogue epi;
  int32_t* ccount;       // count pass
  const int32_t* crp;    // numeric pass
  int32_t* cci;
  double* cv;
  int* changed;
  // hash-table rows: the count pass stages each row's sorted survivors at a
  // bump-allocated position (stage_pos[j], -1 if the staging area overflowed)
  int32_t* stage_col;
  double* stage_val;
  int32_t* stage_pos;
  unsigned long long* stage_cursor;
  int64_t stage_cap;
};

// Per-warp staging for one chunk of <= 32 entries of A's row.
struct WarpStage {
  double aval[32];
  double prod[32];
  int32_t off[33];
  int32_t bstart[32];
};

__device__ __forceinline__ int hash_slot(int32_t col, int shift) {
  return static_cast<int>((static_cast<uint32_t>(col) * 0x9E3779B1u) >> shift);
}

// Returns the slot of `col`, inserting it if absent; bit 30 set = inserted.
__device__ __forceinline__ int find_or_insert(int32_t* key, int mask, int shift, int32_t col) {
  int s = hash_slot(col, shift) & mask;
  while (true) {
    int32_t k = *reinterpret_cast<volatile int32_t*>(&key[s]);
    if (k == col) return s;
    if (k == kEmpty) {
      int32_t old = atomicCAS(&key[s], kEmpty, col);
      if (old == kEmpty) return s | kFresh;
      if (old == col) return s;
    }
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ bool in_pattern(const int32_t* __restrict__ pci, int32_t b, int32_t e, int32_t col) {
  while (b < e) {
    int32_t m = (b + e) >> 1;
    int32_t c = pci[m];
    if (c == col) return true;
    if (c < col) b = m + 1;
    else e = m;
  }
  return false;
}

// Where a row's entries accumulate: an open-addressing hash table of 2^logs
// slots, or (window rows) a direct-addressed window of columns
// [base, base + 32 * words) with an occupancy bitmap.  insert returns the
// slot, | kFresh when the column was absent (the first product is assigned).
struct HashTable {
  static constexpr bool kPhased = SAIT_HASH_PHASED;
  int32_t* key;
  int logs;
  __device__ void clear(int lane) const {
    for (int s = lane; s < (1 << logs); s += 32) key[s] = kEmpty;
  }
  __device__ int insert(int32_t col) const { return find_or_insert(key, (1 << logs) - 1, 32 - logs, col); }
  __device__ void apply(int32_t col, double prod, double* val) const {
    const int hs = insert(col);
    const int s = hs & ~kFresh;
    val[s] = (hs & kFresh) ? prod : __dadd_rn(val[s], prod);
  }
};
struct WindowTable {
  static constexpr bool kPhased = SAIT_WIN_PHASED;
  uint32_t* bits;
  int32_t base;
  int words;
  __device__ void clear(int lane) const {
    for (int w = lane; w < words; w += 32) bits[w] = 0u;
  }
  __device__ int insert(int32_t col) const {
    const int s = col - base;
    SAIT_DCHECK(s >= 0 && s < 32 * words, "spgemm window slot", s, 32 * words);
    const uint32_t b = 1u << (s & 31);
    return (atomicOr(&bits[s >> 5], b) & b) ? s : (s | kFresh);
  }
  __device__ void apply(int32_t col, double prod, double* val) const {
    const int hs = insert(col);
    const int s = hs & ~kFresh;
    val[s] = (hs & kFresh) ? prod : __dadd_rn(val[s], prod);
  }
};
// Direct-addressed window for threshold builds (tau > 0, +I): empty slots
// hold -0.0, the additive identity of IEEE addition (-0.0 + x == x for
// every x, +0.0 and NaN included), so "assign the first product, add the
// later ones" is a plain add -- no occupancy test, no bitmap, no atomics --
// and an empty slot fails |v| >= tau like any dropped entry (the diagonal,
// always kept, is always occupied: +I).  The window is filled with -0.0 once
// per warp; the survivor scan restores every slot it drops and the write
// pass every slot it emits, so nothing is cleared per row.
constexpr int kStageChunk = 2048;  // staging entries a warp claims at once (window rows)
struct ZeroWindow {
  int32_t base;
  int slots;
  __device__ void apply(int32_t col, double prod, double* val) const {
    const int s = col - base;
    SAIT_DCHECK(s >= 0 && s < slots, "spgemm window slot", s, slots);
    val[s] = __dadd_rn(val[s], prod);
  }
};

// Accumulates row j of A*B (+I) into the table.
template <class TABLE>
__device__ void accumulate_row(const Args& g, int32_t j, const TABLE& tab, double* val, WarpStage* st, int lane) {
  tab.clear(lane);
  __syncwarp();
  const int32_t a0 = g.arp[j], a1 = g.arp[j + 1];
  for (int32_t ab = a0; ab < a1; ab += 32) {
    const int nt = min(32, a1 - ab);
    int32_t len = 0, bst = 0;
    double aval = 0.0;
    if (lane < nt) {
      int32_t k = g.aci[ab + lane];
      aval = g.av[ab + lane];
      bst = g.brp[k];
      len = g.brp[k + 1] - bst;
    }
    int32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    // the entries with products, compacted (their offsets strictly increase)
    const int32_t excl = incl - len;
    const bool has = len > 0;  // (lanes >= nt have len 0)
    const unsigned ne = __ballot_sync(0xffffffffu, has);
    if (has) {
      const int r = __popc(ne & ((1u << lane) - 1u));
      st->off[r] = excl;
      st->bstart[r] = bst;
      st->aval[r] = aval;
    }
    __syncwarp();
    // product pb + lane of this chunk -> (B column, a * b); the loads of
    // round r+1 are issued before round r's table updates (software
    // pipelining).  Owner of product pb = the last entry starting at or
    // before it (a ballot); lane l's owner is that entry advanced by the
    // entries starting in (pb, pb + l] (bits of a warp OR-reduction) — no
    // divergent search.
    auto fetch = [&](int32_t pb, int32_t& c, double& a, double& b, int& owner) {
      const int r0 = __popc(__ballot_sync(0xffffffffu, has && excl <= pb)) - 1;
      const int32_t d = excl - pb;
      const unsigned starts = __reduce_or_sync(0xffffffffu, (has && d > 0 && d < 32) ? (1u << d) : 0u);
      const int32_t p = pb + lane;
      c = -1 - lane;  // unique dummy for idle lanes
      a = 0.0;
      b = 0.0;
      owner = r0;
      if (p < total) {
        const int r = r0 + __popc(starts & ((2u << lane) - 1u));
        SAIT_DCHECK(r >= 0 && r < 32 && p >= st->off[r], "spgemm product owner", r, 32);
        const int32_t bi = st->bstart[r] + (p - st->off[r]);
        c = g.bci[bi];
        a = st->aval[r];
        b = g.bv[bi];
        owner = r;
      }
    };
    int32_t ncol;
    double na, nb;
    int nown;
    fetch(0, ncol, na, nb, nown);
    for (int32_t pb = 0; pb < total; pb += 32) {
      const bool act = pb + lane < total;
      const int32_t col = ncol;
      const int own = nown;
      const double prod = act ? __dmul_rn(na, nb) : 0.0;
      if (pb + 32 < total) fetch(pb + 32, ncol, na, nb, nown);
      if constexpr (TABLE::kPhased) {
        // direct-addressed table: the products of one B row have distinct
        // columns, so the round's B rows are applied one after the other
        // (phase = owner entry, i.e. increasing k) with all of a row's
        // lanes at once -- the same adds in the same order as the grouped
        // path below, without __match_any_sync
        const int rlo = __shfl_sync(0xffffffffu, own, 0);
        const int rhi = __reduce_max_sync(0xffffffffu, own);
        for (int ph = rlo; ph <= rhi; ++ph) {
          if (act && own == ph) tab.apply(col, prod, val);
          __syncwarp();
        }
      } else {
        st->prod[lane] = prod;
        const unsigned grp = __match_any_sync(0xffffffffu, col);
        __syncwarp();
        if (act && (__ffs(grp) - 1) == lane) {
          const int hs = tab.insert(col);
          const int s = hs & ~kFresh;
          double acc = (hs & kFresh) ? prod : __dadd_rn(val[s], prod);
          unsigned rest = grp & (grp - 1);  // later lanes = later k
          while (rest) {
            const int m = __ffs(rest) - 1;
            acc = __dadd_rn(acc, st->prod[m]);
            rest &= rest - 1;
          }
          val[s] = acc;
        }
        __syncwarp();
      }
    }
  }
  if (g.epi.add_identity && lane == 0) tab.apply(j + static_cast<int32_t>(g.epi.diag_offset), 1.0, val);
  __syncwarp();
}

// Applies the drop rule and compacts the survivors to [0, live) in one pass
// over the table (slot order; a chunk's destinations never pass the chunk
// being read).  Returns live (same value in all lanes).  The A15 fill cap
// then ranks the compacted survivors only.
__device__ int drop_compact(const Args& g, int32_t row, int32_t* key, double* val, int logs, int lane) {
  const int slots = 1 << logs;
  const int32_t j = row + static_cast<int32_t>(g.epi.diag_offset);  // the diagonal's column
  const int drop = g.epi.drop;
  const bool thr = (drop == 1 || drop == 3) && g.epi.tau != 0.0;
  int32_t pb = 0, pe = 0;
  if (drop == 2) {
    pb = g.epi.prp[row];
    pe = g.epi.prp[row + 1];
  }
  const unsigned below = (1u << lane) - 1u;
  int live = 0, offdiag = 0;
  for (int c = 0; c < slots; c += 32) {
    const int32_t k = key[c + lane];
    const double v = val[c + lane];
    bool keep = k >= 0;
    if (keep) {
      if (thr) keep = (k == j) || (fabs(v) >= g.epi.tau);
      else if (drop == 2) keep = in_pattern(g.epi.pci, pb, pe, k);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {
      const int d = live + __popc(bal & below);
      key[d] = k;
      val[d] = v;
      offdiag += (k != j);
    }
    live += __popc(bal);
  }
  __syncwarp();
  if (drop == 3) {
    offdiag = __reduce_add_sync(0xffffffffu, offdiag);
    int room = g.epi.cap[j] - 1;
    if (room < 0) room = 0;
    if (offdiag > room) {
      // rank of each surviving off-diagonal by (|v| desc, col asc); mark the
      // ones ranked >= room as "to kill" (-3 - col) without disturbing ranks.
      for (int s = lane; s < live; s += 32) {
        const int32_t k = key[s];
        if (k == j) continue;
        const double mv = fabs(val[s]);
        int rank = 0;
        for (int q = 0; q < live; ++q) {
          int32_t kq = key[q];
          if (kq <= -3) kq = -3 - kq;
          if (kq == j || kq == k) continue;
          const double mq = fabs(val[q]);
          rank += (mq > mv) || (mq == mv && kq < k);
        }
        if (rank >= room) key[s] = -3 - k;
      }
      __syncwarp();
      int kept = 0;
      for (int c = 0; c < live; c += 32) {
        const bool in = c + lane < live;
        const int32_t k = in ? key[c + lane] : -1;
        const double v = in ? val[c + lane] : 0.0;
        const bool keep = k >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
          const int d = kept + __popc(bal & below);
          key[d] = k;
          val[d] = v;
        }
        kept += __popc(bal);
      }
      __syncwarp();
      live = kept;
    }
  }
  return live;
}

// sorts the compacted survivors [0, live) by column: one register bitonic
// network over the warp for rows of <= 32 survivors (almost all), the shared
// memory network above that.
__device__ void sort_live(int32_t* key, double* val, int live, int lane, bool narrow) {
  if (live <= 32) {
    const int32_t k0 = lane < live ? key[lane] : INT32_MAX;
    int32_t col;
    int src;
    // a network over the first W = next_pow2(live) lanes only (lanes >= W
    // hold padding and never exchange with lanes < W)
    const int w = live <= 2 ? 2 : 1 << (32 - __clz(live - 1));
    if (narrow) {  // columns < 2^26: (column, lane) in 32 bits
      uint32_t kk = k0 == INT32_MAX ? 0xffffffffu : (static_cast<uint32_t>(k0) << 5) | static_cast<uint32_t>(lane);
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1) {
        if (k > w) break;
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          const uint32_t ok = __shfl_xor_sync(0xffffffffu, kk, jj);
          const bool keep_min = ((lane & jj) == 0) == ((lane & k) == 0);
          kk = keep_min ? min(kk, ok) : max(kk, ok);
        }
      }
      col = static_cast<int32_t>(kk >> 5);
      src = static_cast<int>(kk & 31u);
    } else {
      int64_t kk = k0 == INT32_MAX ? INT64_MAX : (static_cast<int64_t>(k0) << 5) | lane;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1) {
        if (k > w) break;
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
          const int64_t ok = __shfl_xor_sync(0xffffffffu, kk, jj);
          const bool keep_min = ((lane & jj) == 0) == ((lane & k) == 0);
          kk = keep_min ? min(kk, ok) : max(kk, ok);
        }
      }
      col = static_cast<int32_t>(kk >> 5);
      src = static_cast<int>(kk & 31);
    }
    const double v = lane < live ? val[src] : 0.0;
    __syncwarp();
    if (lane < live) {
      key[lane] = col;
      val[lane] = v;
    }
    __syncwarp();
    return;
  }
  const int n2 = next_pow2(live);
  for (int s = live + lane; s < n2; s += 32) key[s] = kKeyPad;
  __syncwarp();
  bitonic_sort(key, val, n2, lane, 32, WarpSync{});
}

// the early-stop comparison of row j (sorted cols/vals) with the previous iterate
__device__ __forceinline__ void compare_row(const Args& g, int32_t j, const int32_t* col, const double* v, int live,
                                            int lane) {
  const int32_t qb = g.epi.qrp[j], ql = g.epi.qrp[j + 1] - qb;
  bool diff = ql != live;
  if (!diff) {
    for (int s = lane; s < live; s += 32) {
      const double a = g.epi.qv[qb + s], b = v[s];
      const double fa = fabs(a), fb = fabs(b);
      const double mx = fa < fb ? fb : fa;  // std::max(fa, fb)
      if (g.epi.qci[qb + s] != col[s] || fabs(__dsub_rn(b, a)) > __dmul_rn(1e-15, mx)) diff = true;
    }
  }
  if (__any_sync(0xffffffffu, diff) && lane == 0 && *reinterpret_cast<volatile int*>(g.changed) == 0)
    atomicOr(g.changed, 1);
}

__device__ void process_row(const Args& g, int32_t j, int32_t* key, double* val, int logs, WarpStage* st,
                            int lane, bool numeric) {
  if (numeric && g.stage_pos && g.stage_pos[j] >= 0) return;  // staged: copied by spgemm_stage_emit
  accumulate_row(g, j, HashTable{key, logs}, val, st, lane);
  const int live = drop_compact(g, j, key, val, logs, lane);
  const bool narrow = g.ncols < (int64_t{1} << 26);
  if (!numeric) {
    if (lane == 0) g.ccount[j] = live;
    if (!g.stage_pos) return;
    sort_live(key, val, live, lane, narrow);
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(g.stage_cursor, static_cast<unsigned long long>(live));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const bool fits = pos + static_cast<unsigned long long>(live) <= static_cast<unsigned long long>(g.stage_cap);
    if (fits)
      for (int s = lane; s < live; s += 32) {
        g.stage_col[pos + s] = key[s];
        g.stage_val[pos + s] = val[s];
      }
    if (lane == 0) g.stage_pos[j] = fits ? static_cast<int32_t>(pos) : -1;
    __syncwarp();
    return;
  }
  sort_live(key, val, live, lane, narrow);
  const int32_t out = g.crp[j];
  for (int s = lane; s < live; s += 32) {
    g.cci[out + s] = key[s];
    g.cv[out + s] = g.epi.out_scale ? __dmul_rn(val[s], g.epi.out_scale[key[s]]) : val[s];
  }
  if (g.epi.qrp) compare_row(g, j, key, val, live, lane);
  __syncwarp();
}

// Window rows (the window bins): every product column of row j lies in
// [base, base + 1024 R), so the row accumulates by direct addressing -- one
// atomicOr on an occupancy bitmap per new column instead of hash probing and
// table clearing -- and its entries come out of the bitmap already in column
// order (no sort).  Lane l owns bitmap words l, l + 32, ... (R words): it
// tests its occupied slots against the drop rule, the survivors are counted
// per lane and placed by a warp exclusive scan in (word, bit) order = column
// order, and written straight to the staging area (count pass) or the final
// row (numeric pass, with the early-stop compare on the fly).  Same products,
// same order of adds per column: bitwise the hash path.
template <int R>
__device__ __forceinline__ void window_survivors(const Args& g, int32_t j, const uint32_t* bits, const double* val,
                                                 int32_t base, int lane, uint32_t (&keep)[R]) {
  const int32_t jd = j + static_cast<int32_t>(g.epi.diag_offset);
  const int drop = g.epi.drop;
  const bool thr = (drop == 1 || drop == 3) && g.epi.tau != 0.0;
  int32_t pb = 0, pe = 0;
  if (drop == 2) {
    pb = g.epi.prp[j];
    pe = g.epi.prp[j + 1];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int w = lane + 32 * r;
    uint32_t m = bits[w], k = 0u;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int32_t col = base + 32 * w + b;
      bool ok = true;
      if (thr) ok = (col == jd) || (fabs(val[32 * w + b]) >= g.epi.tau);
      else if (drop == 2) ok = in_pattern(g.epi.pci, pb, pe, col);
      if (ok) k |= 1u << b;
    }
    keep[r] = k;
  }
}

template <int R>
__device__ void process_row_window(const Args& g, int32_t j, int32_t base, uint32_t* bits, uint32_t* kbits,
                                   double* val, WarpStage* st, int lane, bool numeric) {
  if (numeric && g.stage_pos && g.stage_pos[j] >= 0) return;  // staged: copied by spgemm_stage_emit
  accumulate_row(g, j, WindowTable{bits, base, 32 * R}, val, st, lane);
  uint32_t keep[R];
  window_survivors<R>(g, j, bits, val, base, lane, keep);
  const int32_t jd = j + static_cast<int32_t>(g.epi.diag_offset);
  if (g.epi.drop == 3) {  // A15 fill cap: the diagonal + the (cap - 1) largest |v| off-diagonals
    int off = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w = lane + 32 * r;
      off += __popc(keep[r]);
      const int d = jd - base - 32 * w;
      if (d >= 0 && d < 32 && ((keep[r] >> d) & 1u)) --off;
      kbits[w] = keep[r];
    }
    off = __reduce_add_sync(0xffffffffu, off);
    int room = g.epi.cap[jd] - 1;
    if (room < 0) room = 0;
    __syncwarp();
    if (off > room) {  // rank by (|v| desc, column asc) among the kept off-diagonals
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int w = lane + 32 * r;
        uint32_t m = keep[r], kill = 0u;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          const int32_t col = base + 32 * w + b;
          if (col == jd) continue;
          const double mv = fabs(val[32 * w + b]);
          int rank = 0;
          for (int q = 0; q < 32 * R; ++q) {
            uint32_t mq = kbits[q];
            while (mq) {
              const int bq = __ffs(mq) - 1;
              mq &= mq - 1;
              const int32_t cq = base + 32 * q + bq;
              if (cq == jd || cq == col) continue;
              const double vq = fabs(val[32 * q + bq]);
              rank += (vq > mv) || (vq == mv && cq < col);
            }
          }
          if (rank >= room) kill |= 1u << b;
        }
        keep[r] &= ~kill;
      }
    }
    __syncwarp();
  }
  // survivors in column order: word-major (word w = lane + 32 r), bit order
  int cnt[R], pre[R], live = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    cnt[r] = __popc(keep[r]);
    int incl = cnt[r];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    pre[r] = live + incl - cnt[r];
    live += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (!numeric) {
    if (lane == 0) g.ccount[j] = live;
    if (!g.stage_pos) return;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(g.stage_cursor, static_cast<unsigned long long>(live));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const bool fits = pos + static_cast<unsigned long long>(live) <= static_cast<unsigned long long>(g.stage_cap);
    if (fits) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int w = lane + 32 * r;
        uint32_t m = keep[r];
        int o = pre[r];
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          g.stage_col[pos + o] = base + 32 * w + b;
          g.stage_val[pos + o] = val[32 * w + b];
          ++o;
        }
      }
    }
    if (lane == 0) g.stage_pos[j] = fits ? static_cast<int32_t>(pos) : -1;
    __syncwarp();
    return;
  }
  const int32_t out = g.crp[j];
  bool cmp = g.epi.qrp != nullptr, diff = false;
  int32_t qb = 0;
  if (cmp) {
    qb = g.epi.qrp[j];
    if (g.epi.qrp[j + 1] - qb != live) {
      diff = true;
      cmp = false;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int w = lane + 32 * r;
    uint32_t m = keep[r];
    int o = pre[r];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int32_t c = base + 32 * w + b;
      const double v = val[32 * w + b];
      g.cci[out + o] = c;
      g.cv[out + o] = g.epi.out_scale ? __dmul_rn(v, g.epi.out_scale[c]) : v;
      if (cmp) {  // the reference's stabilized() test (sait.cpp:14-28)
        const double a = g.epi.qv[qb + o];
        const double fa = fabs(a), fb = fabs(v);
        const double mx = fa < fb ? fb : fa;
        if (g.epi.qci[qb + o] != c || fabs(__dsub_rn(v, a)) > __dmul_rn(1e-15, mx)) diff = true;
      }
      ++o;
    }
  }
  if (__any_sync(0xffffffffu, diff) && lane == 0 && *reinterpret_cast<volatile int*>(g.changed) == 0)
    atomicOr(g.changed, 1);
  __syncwarp();
}

// The next window row's A data, loaded in stages while the current row runs
// (stage 1: its id; 2: its A extent and window base; 3: its first 32 A
// entries; 4: their B row extents), so a row starts with its first round's
// fetch instead of a chain of four dependent global loads.
struct RowAhead {
  int32_t j = -1, a0 = 0, a1 = 0, base = 0, bst = 0, len = 0;
  int32_t k = 0;
  double aval = 0.0;
  int stage = 0;  // loads issued so far
  __device__ __forceinline__ void step(const Args& g, const int32_t* __restrict__ rows, int32_t r,
                                       const int32_t* __restrict__ wbase, int lane) {
    switch (stage) {
      case 0:
        j = rows[r];
        break;
      case 1:
        a0 = g.arp[j];
        a1 = g.arp[j + 1];
        base = wbase[j];
        break;
      case 2:
        if (lane < a1 - a0) {
          k = g.aci[a0 + lane];
          aval = g.av[a0 + lane];
        }
        break;
      case 3:
        bst = 0;
        len = 0;
        if (lane < a1 - a0) {
          bst = g.brp[k];
          len = g.brp[k + 1] - bst;
        }
        break;
      default:
        return;
    }
    ++stage;
  }
};

// accumulate_zero's staging of one chunk of <= 32 A entries: entry r's value
// and its B row start minus its first product index, one 16-byte load
struct __align__(16) ZEnt {
  double aval;
  int32_t bbase;  // B entry of product p = bbase + p
  int32_t pad;
};
struct ZStage {
  ZEnt e[32];
};

// accumulate_row for a ZeroWindow with the row's first A chunk already
// loaded (cur) and the next row's loads advanced between rounds (nx).
__device__ __forceinline__ int32_t accumulate_zero(const Args& g, const RowAhead& cur, RowAhead& nx,
                                                   const int32_t* __restrict__ rows, int32_t rn,
                                                   const int32_t* __restrict__ wbase, const ZeroWindow& tab,
                                                   double* val, ZStage* st, int lane) {
  int32_t hi = -1;
  const int32_t j = cur.j, a0 = cur.a0, a1 = cur.a1;
  int rounds = 0;
  for (int32_t ab = a0; ab < a1; ab += 32) {
    const int nt = min(32, a1 - ab);
    int32_t len = 0, bst = 0;
    double aval = 0.0;
    if (ab == a0) {
      len = cur.len;
      bst = cur.bst;
      aval = cur.aval;
    } else if (lane < nt) {
      const int32_t k = g.aci[ab + lane];
      aval = g.av[ab + lane];
      bst = g.brp[k];
      len = g.brp[k + 1] - bst;
    }
    int32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const int32_t excl = incl - len;
    const bool has = len > 0;
    const unsigned ne = __ballot_sync(0xffffffffu, has);
    if (has) {
      const int r = __popc(ne & ((1u << lane) - 1u));
      st->e[r] = ZEnt{aval, bst - excl, 0};
    }
    __syncwarp();
    auto fetch = [&](int32_t pb, int32_t& c, double& a, double& b, int& owner) {
      const int r0 = __popc(__ballot_sync(0xffffffffu, has && excl <= pb)) - 1;
      const int32_t d = excl - pb;
      const unsigned starts = __reduce_or_sync(0xffffffffu, (has && d > 0 && d < 32) ? (1u << d) : 0u);
      const int32_t p = pb + lane;
      c = -1;
      a = 0.0;
      b = 0.0;
      owner = r0;
      if (p < total) {
        const int r = r0 + __popc(starts & ((2u << lane) - 1u));
        SAIT_DCHECK(r >= 0 && r < 32, "spgemm product owner", r, 32);
        const ZEnt z = st->e[r];
        const int32_t bi = z.bbase + p;
        c = g.bci[bi];
        a = z.aval;
        b = g.bv[bi];
        owner = r;
      }
    };
    int32_t ncol;
    double na, nb;
    int nown;
    fetch(0, ncol, na, nb, nown);
    for (int32_t pb = 0; pb < total; pb += 32) {
      const bool act = pb + lane < total;
      const int32_t col = ncol;
      const int own = nown;
      const double prod = act ? __dmul_rn(na, nb) : 0.0;
      if (pb + 32 < total) fetch(pb + 32, ncol, na, nb, nown);
      if (rounds < 4) nx.step(g, rows, rn, wbase, lane);  // one stage of the next row per round
      ++rounds;
      const int rlo = __shfl_sync(0xffffffffu, own, 0);
      const int rhi = __reduce_max_sync(0xffffffffu, own);
      if (act) hi = max(hi, col);
      for (int ph = rlo; ph <= rhi; ++ph) {  // one B row at a time: k order
        if (act && own == ph) tab.apply(col, prod, val);
        __syncwarp();
      }
    }
  }
  if (g.epi.add_identity && lane == 0) {
    const int32_t jd = j + static_cast<int32_t>(g.epi.diag_offset);
    tab.apply(jd, 1.0, val);
    hi = max(hi, jd);
  }
  hi = __reduce_max_sync(0xffffffffu, hi);
  __syncwarp();
  return hi;
}

// Window rows of threshold builds (tau > 0, +I; other epilogues keep the
// bitmap window above): a ZeroWindow.  The survivor scan walks the touched
// 64-slot groups [base, hi] with two slots per lane (one 16-byte load),
// keeps the diagonal and |v| >= tau, puts -0.0 back into the dropped slots
// and keeps the survivors' masks per group (lane q holds group q's even- and
// odd-slot ballots).  The write pass gives survivor i (column order) to lane
// i % 32, which finds its slot from the groups' prefix counts and writes it,
// putting -0.0 back.  Same products, same add order: bitwise the hash path.
template <int Q, bool numeric>
__device__ void process_row_window_z(const Args& g, const RowAhead& cur, RowAhead& nx,
                                     const int32_t* __restrict__ rows, int32_t rn, const int32_t* __restrict__ wbase,
                                     double* val, uint32_t* kbits, ZStage* st, int lane,
                                     unsigned long long& cpos, unsigned long long& cend) {
  const int32_t j = cur.j, base = cur.base;
  if (numeric && g.stage_pos && g.stage_pos[j] >= 0) return;  // staged: copied by spgemm_stage_emit
  const int32_t hi = accumulate_zero(g, cur, nx, rows, rn, wbase, ZeroWindow{base, 128 * Q}, val, st, lane);
  const int32_t jd = j + static_cast<int32_t>(g.epi.diag_offset);
  const int sd = jd - base;  // the diagonal's slot
  const double tau = g.epi.tau;
  const int ngroups = ((hi - base) >> 6) + 1;
  SAIT_DCHECK(ngroups >= 1 && ngroups <= 2 * Q, "spgemm window groups", ngroups, 2 * Q);
  uint32_t kE = 0u, kO = 0u;
  for (int q0 = 0; q0 < ngroups; q0 += 4) {  // four groups' loads in flight
    double2 v[4];  // (groups past ngroups: inside the window when 2 Q % 4 == 0, else guarded)
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if ((2 * Q) % 4 == 0 || q0 + u < 2 * Q) v[u] = *reinterpret_cast<const double2*>(&val[64 * (q0 + u) + 2 * lane]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u;
      if (q >= ngroups) continue;
      const int s0 = 64 * q + 2 * lane;
      const bool k0 = s0 == sd || fabs(v[u].x) >= tau;
      const bool k1 = s0 + 1 == sd || fabs(v[u].y) >= tau;
      // one 16-byte store per lane (4 wavefronts per group; two predicated
      // 8-byte stores cost 8): dropped slots back to -0.0, kept ones as they are
      *reinterpret_cast<double2*>(&val[s0]) = make_double2(k0 ? v[u].x : -0.0, k1 ? v[u].y : -0.0);
      const unsigned E = __ballot_sync(0xffffffffu, k0), O = __ballot_sync(0xffffffffu, k1);
      if (lane == q) {
        kE = E;
        kO = O;
      }
    }
  }
  int live = __reduce_add_sync(0xffffffffu, __popc(kE) + __popc(kO));
  if (g.epi.drop == 3) {  // A15 fill cap: the diagonal + the (cap - 1) largest |v| off-diagonals
    int room = g.epi.cap[jd] - 1;
    if (room < 0) room = 0;
    if (live - 1 > room) {  // rare: rank by (|v| desc, column asc) among the kept off-diagonals
      if (lane < ngroups) {
        kbits[2 * lane] = kE;
        kbits[2 * lane + 1] = kO;
      }
      __syncwarp();
      unsigned long long kill = 0ull;  // bit 2q + parity
      for (int q = 0; q < ngroups; ++q)
        for (int par = 0; par < 2; ++par) {
          if (!((kbits[2 * q + par] >> lane) & 1u)) continue;
          const int sl = 64 * q + 2 * lane + par;
          if (sl == sd) continue;
          const double mv = fabs(val[sl]);
          int rank = 0;
          for (int q2 = 0; q2 < ngroups; ++q2)
            for (int p2 = 0; p2 < 2; ++p2) {
              uint32_t m = kbits[2 * q2 + p2];
              while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int s2 = 64 * q2 + 2 * b + p2;
                if (s2 == sd || s2 == sl) continue;
                const double vq = fabs(val[s2]);
                rank += (vq > mv) || (vq == mv && s2 < sl);
              }
            }
          if (rank >= room) kill |= 1ull << (2 * q + par);
        }
      __syncwarp();
      while (kill) {
        const int bi = __ffsll(static_cast<long long>(kill)) - 1;
        kill &= kill - 1;
        atomicAnd(&kbits[bi], ~(1u << lane));
        val[64 * (bi >> 1) + 2 * lane + (bi & 1)] = -0.0;
      }
      __syncwarp();
      if (lane < ngroups) {
        kE = kbits[2 * lane];
        kO = kbits[2 * lane + 1];
      }
      live = __reduce_add_sync(0xffffffffu, __popc(kE) + __popc(kO));
    }
  }
  // write pass: the groups with survivors, in column order
  int32_t* ocol = nullptr;
  double* oval = nullptr;
  bool write = true, cmp = false, diff = false;
  int32_t qb = 0;
  if constexpr (!numeric) {
    if (lane == 0) g.ccount[j] = live;
    write = g.stage_pos != nullptr;
    if (write) {
      // staging space comes in per-warp chunks (one global atomic per
      // ~kStageChunk entries instead of one per row)
      if (cpos + static_cast<unsigned long long>(live) > cend) {
        const unsigned long long want = max(static_cast<unsigned long long>(kStageChunk),
                                            static_cast<unsigned long long>(live));
        unsigned long long p0 = 0;
        if (lane == 0) p0 = atomicAdd(g.stage_cursor, want);
        cpos = __shfl_sync(0xffffffffu, p0, 0);
        cend = cpos + want;
      }
      const unsigned long long pos = cpos;
      cpos += static_cast<unsigned long long>(live);
      write = pos + static_cast<unsigned long long>(live) <= static_cast<unsigned long long>(g.stage_cap);
      if (lane == 0) g.stage_pos[j] = write ? static_cast<int32_t>(pos) : -1;
      ocol = g.stage_col + pos;
      oval = g.stage_val + pos;
    }
  } else {
    const int32_t out = g.crp[j];
    ocol = g.cci + out;
    oval = g.cv + out;
    cmp = g.epi.qrp != nullptr;
    if (cmp) {
      qb = g.epi.qrp[j];
      if (g.epi.qrp[j + 1] - qb != live) {
        diff = true;
        cmp = false;
      }
    }
  }
  const bool scale = numeric && g.epi.out_scale;
  auto emit = [&](int p, int32_t c, double v) {
    ocol[p] = c;
    if constexpr (!numeric) {
      oval[p] = v;
      return;
    }
    oval[p] = scale ? __dmul_rn(v, g.epi.out_scale[c]) : v;
    if (cmp) {  // the reference's stabilized() test (sait.cpp:14-28)
      const double a = g.epi.qv[qb + p];
      const double fa = fabs(a), fb = fabs(v);
      const double mx = fa < fb ? fb : fa;
      if (g.epi.qci[qb + p] != c || fabs(__dsub_rn(v, a)) > __dmul_rn(1e-15, mx)) diff = true;
    }
  };
  // survivor i of the row goes to lane i % 32: its group is the last group
  // starting at or before i (start markers + a warp prefix max), its slot
  // the (i - group start)-th set bit in slot order (even slot 2b before odd
  // slot 2b + 1), found by a 5-step binary search on b
  const int cnt = __popc(kE) + __popc(kO);
  int excl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, excl, o);
    if (lane >= o) excl += y;
  }
  excl -= cnt;
  int32_t* mk = reinterpret_cast<int32_t*>(kbits);
  for (int c0 = 0; c0 < live; c0 += 32) {
    mk[lane] = -1;
    __syncwarp();
    if (cnt > 0 && excl < c0 + 32 && excl + cnt > c0) mk[excl > c0 ? excl - c0 : 0] = lane;
    __syncwarp();
    int gq = mk[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, gq, o);
      if (lane >= o) gq = max(gq, y);
    }
    const int i = c0 + lane;
    const int gs = gq < 0 ? 0 : gq;
    const int r = i - __shfl_sync(0xffffffffu, excl, gs);
    const unsigned E = __shfl_sync(0xffffffffu, kE, gs), O = __shfl_sync(0xffffffffu, kO, gs);
    __syncwarp();
    if (i < live) {
      int lo = 0;  // largest b with (survivors in slots < 2b) <= r
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int b = lo + step;
        const unsigned m = (1u << b) - 1u;
        if (__popc(E & m) + __popc(O & m) <= r) lo = b;
      }
      const unsigned m = (1u << lo) - 1u;
      const bool even = ((E >> lo) & 1u) && __popc(E & m) + __popc(O & m) == r;
      const int sl = 64 * gs + 2 * lo + (even ? 0 : 1);
      const double v = val[sl];
      if (write) emit(i, base + sl, v);
      val[sl] = -0.0;
    }
  }
  if (numeric && __any_sync(0xffffffffu, diff) && lane == 0 && *reinterpret_cast<volatile int*>(g.changed) == 0)
    atomicOr(g.changed, 1);
  __syncwarp();
}

// Numeric pass of staged rows: 8 lanes per row (4 rows per warp; the rows
// keep ~7-16 survivors, so a warp per row idled most lanes and a thread per
// row made uncoalesced strided reads) copy the sorted survivors to the final
// row and run the early-stop compare.  G = 0: hash-table rows staged at
// stage_pos[j]; G > 0: tiny rows staged in the G-entry slot of their bin
// position.
template <int G, int kLanes>
__device__ __forceinline__ void emit_rows(const Args& g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                          const int32_t* __restrict__ tcol, const double* __restrict__ tval,
                                          const int8_t* __restrict__ bin_of = nullptr) {
  __shared__ int blk_changed;
  if (threadIdx.x == 0) blk_changed = 0;
  __syncthreads();
  const int sl = threadIdx.x & (kLanes - 1);
  const int64_t t0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / kLanes;
  const int64_t nt = (static_cast<int64_t>(gridDim.x) * blockDim.x) / kLanes;
  bool diff = false;
  for (int64_t r = t0; r < nrows_bin; r += nt) {
    // staged rows in row order (bin_of: the hash / window rows) or a bin's list
    if (bin_of && bin_of[r] < kFirstSmemBin) continue;
    const int32_t j = bin_of ? static_cast<int32_t>(r) : rows[r];
    const int32_t* col;
    const double* v;
    if (G == 0) {
      const int32_t pos = g.stage_pos[j];
      if (pos < 0) continue;  // overflowed: recomputed by the hash kernel
      col = g.stage_col + pos;
      v = g.stage_val + pos;
    } else {
      col = tcol + r * G;
      v = tval + r * G;
    }
    const int32_t out = g.crp[j], live = g.crp[j + 1] - out;
    bool cmp = g.epi.qrp != nullptr && !diff;
    int32_t qb = 0;
    if (cmp) {
      qb = g.epi.qrp[j];
      if (g.epi.qrp[j + 1] - qb != live) {
        diff = true;
        cmp = false;
      }
    }
    for (int s = sl; s < live; s += kLanes) {
      const int32_t c = col[s];
      const double b = v[s];
      g.cci[out + s] = c;
      g.cv[out + s] = g.epi.out_scale ? __dmul_rn(b, g.epi.out_scale[c]) : b;
      if (cmp) {  // the reference's stabilized() test (sait.cpp:14-28)
        const double a = g.epi.qv[qb + s];
        const double fa = fabs(a), fb = fabs(b);
        const double mx = fa < fb ? fb : fa;  // std::max(fa, fb)
        if (g.epi.qci[qb + s] != c || fabs(__dsub_rn(b, a)) > __dmul_rn(1e-15, mx)) diff = true;
      }
    }
  }
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) blk_changed = 1;
  __syncthreads();
  if (threadIdx.x == 0 && blk_changed) atomicOr(g.changed, 1);
}

__global__ void __launch_bounds__(256) spgemm_stage_emit(Args g, const int8_t* __restrict__ bin_of) {
  // every staged row, in row order: the output is written front to back
  emit_rows<0, 8>(g, nullptr, static_cast<int32_t>(g.n), nullptr, nullptr, bin_of);
}

__host__ __device__ constexpr int smem_per_warp(int logs) {
  return ((1 << logs) * 12 + static_cast<int>(sizeof(WarpStage)) + 15) / 16 * 16;
}

template <int LOGS>
__global__ void __launch_bounds__(256) spgemm_smem(Args g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                                   bool numeric) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* mine = smem + w * smem_per_warp(LOGS);
  double* val = reinterpret_cast<double*>(mine);
  int32_t* key = reinterpret_cast<int32_t*>(mine + (1 << LOGS) * 8);
  WarpStage* st = reinterpret_cast<WarpStage*>(mine + (1 << LOGS) * 12);
  const int warps = blockDim.x >> 5;
  for (int32_t r = blockIdx.x * warps + w; r < nrows_bin; r += gridDim.x * warps)
    process_row(g, rows[r], key, val, LOGS, st, lane, numeric);
}

__host__ __device__ constexpr int window_smem_per_warp(int R) {
  return (1024 * R * 8 + 64 * R * 4 + static_cast<int>(sizeof(WarpStage)) + 15) / 16 * 16;
}
constexpr int window_warps(int R) { return R == 1 ? 8 : 4; }

template <int R>
__global__ void __launch_bounds__(256) spgemm_window(Args g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                                     const int32_t* __restrict__ wbase, bool numeric) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* mine = smem + w * window_smem_per_warp(R);
  double* val = reinterpret_cast<double*>(mine);
  uint32_t* bits = reinterpret_cast<uint32_t*>(mine + 1024 * R * 8);
  uint32_t* kbits = bits + 32 * R;
  WarpStage* st = reinterpret_cast<WarpStage*>(kbits + 32 * R);
  const int warps = blockDim.x >> 5;
  for (int32_t r = blockIdx.x * warps + w; r < nrows_bin; r += gridDim.x * warps) {
    const int32_t j = rows[r];
    process_row_window<R>(g, j, wbase[j], bits, kbits, val, st, lane, numeric);
  }
}

constexpr int kRun = 8;  // window rows: consecutive list rows per warp
__host__ __device__ constexpr int zwindow_smem_per_warp(int Q) {
  return (128 * Q * 8 + 64 * 4 + static_cast<int>(sizeof(ZStage)) + 15) / 16 * 16;
}
template <int Q>
__global__ void __launch_bounds__(256) spgemm_window_z(Args g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                                       const int32_t* __restrict__ wbase, bool numeric) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* mine = smem + w * zwindow_smem_per_warp(Q);
  double* val = reinterpret_cast<double*>(mine);
  uint32_t* kbits = reinterpret_cast<uint32_t*>(mine + 128 * Q * 8);
  ZStage* st = reinterpret_cast<ZStage*>(kbits + 64);
  for (int s = lane; s < 128 * Q; s += 32) val[s] = -0.0;
  __syncwarp();
  // warp w takes runs of kRun consecutive list rows, run w, w + W, ...
  // (W = all warps): rows processed side by side stay close (their B rows
  // share L2), and a warp's staging chunk holds whole runs, so the numeric
  // copy (list order) reads the staging area in runs too
  const int warps = blockDim.x >> 5;
  const int64_t jump = static_cast<int64_t>(gridDim.x) * warps * kRun;
  auto next_row = [&](int64_t r) { return (r + 1) % kRun ? r + 1 : r + 1 - kRun + jump; };
  unsigned long long cpos = 0, cend = 0;  // this warp's staging chunk
  int64_t r = (static_cast<int64_t>(blockIdx.x) * warps + w) * kRun;
  RowAhead nx;
  if (r < nrows_bin)
    while (nx.stage < 4) nx.step(g, rows, static_cast<int32_t>(r), wbase, lane);
  for (; r < nrows_bin; r = next_row(r)) {
    const RowAhead cur = nx;
    const int64_t rn64 = next_row(r);
    const int32_t rn = static_cast<int32_t>(min(rn64, static_cast<int64_t>(nrows_bin)));
    nx = RowAhead{};
    if (rn64 >= nrows_bin) nx.stage = 4;
    if (numeric)
      process_row_window_z<Q, true>(g, cur, nx, rows, rn, wbase, val, kbits, st, lane, cpos, cend);
    else
      process_row_window_z<Q, false>(g, cur, nx, rows, rn, wbase, val, kbits, st, lane, cpos, cend);
    while (nx.stage < 4) nx.step(g, rows, rn, wbase, lane);
  }
}

// Very long rows: table in global scratch (per-row offsets), one warp per row.
__global__ void spgemm_global(Args g, const int32_t* __restrict__ rows, const int64_t* __restrict__ offs,
                              const int8_t* __restrict__ logs_of, int32_t nrows_bin, int32_t* gkey, double* gval,
                              bool numeric) {
  __shared__ WarpStage stage[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  for (int32_t r = blockIdx.x * warps + w; r < nrows_bin; r += gridDim.x * warps)
    process_row(g, rows[r], gkey + offs[r], gval + offs[r], logs_of[r], &stage[w], lane, numeric);
}

// ---------------------------------------------------------------- tiny rows
// Rows with < G products and <= G entries in A's row (G = 8, 16, 32): a group
// of G lanes per row (32/G rows per warp), one product per lane (plus the +I
// pseudo-product at lane P), a bitonic sort inside the group by (column,
// lane) — lane order is product order, i.e. increasing k — and a sequential
// sum over each run of equal columns: exactly the reference order, no shared
// memory.  The count pass stages the sorted survivors in a G-entry slot per
// row; the numeric pass is a copy (+ stabilization compare).
// The row's operands up to B's row extents.
struct TinyFetch {
  int32_t j, m, len, bst;
  double aval;
  bool live;
};
__device__ __forceinline__ TinyFetch tiny_fetch(const Args& g, const int32_t* __restrict__ rows, int64_t r,
                                                int32_t nrows_bin, int lane) {
  TinyFetch f{0, 0, 0, 0, 0.0, r < nrows_bin};
  if (f.live) {
    f.j = rows[r];
    const int32_t a0 = g.arp[f.j];
    f.m = g.arp[f.j + 1] - a0;
    if (lane < f.m) {
      const int32_t k = g.aci[a0 + lane];
      f.aval = g.av[a0 + lane];
      f.bst = g.brp[k];
      f.len = g.brp[k + 1] - f.bst;
    }
  }
  return f;
}

template <int G>
__device__ __forceinline__ void tiny_row(const Args& g, const TinyFetch& f, int lane, int64_t slot,
                                         int32_t* __restrict__ tcol, double* __restrict__ tval) {
  constexpr unsigned kAll = 0xffffffffu;
  const int grp = (threadIdx.x & 31) / G;
  const int32_t j = f.j, m = f.m, len = f.len, bst = f.bst;
  const bool live_row = f.live;
  const double aval = f.aval;
  int32_t incl = len;
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    const int32_t y = __shfl_up_sync(kAll, incl, o, G);
    if (lane >= o) incl += y;
  }
  const int32_t excl = incl - len;
  const int P = __shfl_sync(kAll, incl, G - 1, G);
  // t(p) = largest t < m with excl_t <= p  (zero-length entries share offsets)
  int t = 0;
#pragma unroll
  for (int step = G / 2; step >= 1; step >>= 1) {
    const int cand = t + step;
    const int32_t e = __shfl_sync(kAll, excl, cand < G ? cand : G - 1, G);
    if (cand < m && e <= lane) t = cand;
  }
  const int32_t bs = __shfl_sync(kAll, bst, t, G);
  const int32_t ex = __shfl_sync(kAll, excl, t, G);
  const double at = __shfl_sync(kAll, aval, t, G);
  const int32_t jd = j + static_cast<int32_t>(g.epi.diag_offset);
  // sort key (column, lane): 32-bit while columns < 2^26, else 64-bit
  double val0 = 0.0;
  int32_t col0 = INT32_MAX;
  if (live_row) {
    if (lane < P) {
      const int32_t bi = bs + (lane - ex);
      col0 = g.bci[bi];
      val0 = __dmul_rn(at, g.bv[bi]);
    } else if (lane == P && g.epi.add_identity) {
      col0 = jd;  // +1.0 after the products (add_identity)
      val0 = 1.0;
    }
  }
  int32_t col;
  double val;
  if (g.ncols < (int64_t{1} << 26)) {
    uint32_t key = col0 == INT32_MAX ? 0xffffffffu : (static_cast<uint32_t>(col0) << 5) | static_cast<uint32_t>(lane);
#pragma unroll
    for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const uint32_t ok = __shfl_xor_sync(kAll, key, jj, G);
        const bool keep_min = ((lane & jj) == 0) == ((lane & k) == 0);
        key = keep_min ? min(key, ok) : max(key, ok);
      }
    }
    col = key == 0xffffffffu ? INT32_MAX : static_cast<int32_t>(key >> 5);
    val = __shfl_sync(kAll, val0, static_cast<int>(key & 31u) & (G - 1), G);
  } else {
    int64_t key = col0 == INT32_MAX ? INT64_MAX : (static_cast<int64_t>(col0) << 5) | lane;
#pragma unroll
    for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        const int64_t ok = __shfl_xor_sync(kAll, key, jj, G);
        const bool keep_min = ((lane & jj) == 0) == ((lane & k) == 0);
        key = keep_min ? min(key, ok) : max(key, ok);
      }
    }
    col = key == INT64_MAX ? INT32_MAX : static_cast<int32_t>(key >> 5);
    val = __shfl_sync(kAll, val0, static_cast<int>(key & 31) & (G - 1), G);
  }
  const bool valid = col != INT32_MAX;
  const int32_t prev = __shfl_up_sync(kAll, col, 1, G);
  const bool head = valid && (lane == 0 || prev != col);
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
  const int shift = grp * G;
  // each run of equal columns summed sequentially by its head, in product
  // order; run length = distance to the next head (valid keys form a prefix)
  const unsigned heads = (__ballot_sync(kAll, head) >> shift) & gmask;
  const int nvalid = __popc((__ballot_sync(kAll, valid) >> shift) & gmask);
  const unsigned later = heads & ~((2u << lane) - 1u);
  const int run = head ? (later ? __ffs(later) - 1 : nvalid) - lane : 0;
  const int maxrun = __reduce_max_sync(kAll, run);
  double acc = val;
  for (int d = 1; d < maxrun; ++d) {
    const double v = __shfl_down_sync(kAll, val, d, G);
    if (d < run) acc = __dadd_rn(acc, v);
  }
  bool keep = head;
  const int drop = g.epi.drop;
  if (head && (drop == 1 || drop == 3) && g.epi.tau != 0.0) keep = (col == jd) || (fabs(acc) >= g.epi.tau);
  else if (head && drop == 2) keep = in_pattern(g.epi.pci, g.epi.prp[j], g.epi.prp[j + 1], col);
  if (drop == 3) {
    const unsigned offm = (__ballot_sync(kAll, keep && col != jd) >> shift) & gmask;
    int room = live_row ? g.epi.cap[jd] - 1 : 0;
    if (room < 0) room = 0;
    if (__any_sync(kAll, live_row && __popc(offm) > room)) {
      const double mv = fabs(acc);
      int rank = 0;
      for (int q = 0; q < G; ++q) {
        const double mq = __shfl_sync(kAll, mv, q, G);
        const int32_t cq = __shfl_sync(kAll, col, q, G);
        if ((offm >> q) & 1u) rank += (mq > mv) || (mq == mv && cq < col);
      }
      if (__popc(offm) > room && keep && col != jd && rank >= room) keep = false;
    }
  }
  const unsigned km = (__ballot_sync(kAll, keep) >> shift) & gmask;
  if (live_row) {
    if (lane == 0) g.ccount[j] = __popc(km);
    if (keep) {
      const int pos = __popc(km & ((1u << lane) - 1u));
      SAIT_DCHECK(pos < G, "spgemm tiny staging slot", pos, G);
      tcol[slot * G + pos] = col;
      tval[slot * G + pos] = acc;
    }
  }
}

// 8 CTAs/SM (32 registers): the tiny rows are latency-bound on their
// dependent fetch chain, full occupancy hides it (-14 % vs 38 registers at 6
// CTAs/SM, despite an 8-byte spill in the G = 32 instance)
template <int G>
__global__ void __launch_bounds__(256, 8) spgemm_tiny(Args g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                                    int32_t* __restrict__ tcol, double* __restrict__ tval) {
  constexpr int kPerWarp = 32 / G;
  const int lane = threadIdx.x & (G - 1);
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int sub = (threadIdx.x & 31) / G;
  // (fetching the next row ahead was measured slower: the tiny rows are
  // bound by shuffle throughput, not by the load chain)
  for (int64_t w = warp0; w * kPerWarp < nrows_bin; w += nwarps) {
    const TinyFetch cur = tiny_fetch(g, rows, w * kPerWarp + sub, nrows_bin, lane);
    tiny_row<G>(g, cur, lane, w * kPerWarp + sub, tcol, tval);
  }
}

// numeric pass of the tiny rows: staged slot -> final row, + early-stop
// compare (emit_rows, L = 4 lanes per row when the output averages <= 8
// entries per row -- stencil factors -- else 8).
template <int G, int L>
__global__ void __launch_bounds__(256) spgemm_tiny_emit(Args g, const int32_t* __restrict__ rows, int32_t nrows_bin,
                                                         const int32_t* __restrict__ tcol,
                                                         const double* __restrict__ tval) {
  emit_rows<G, L>(g, rows, nrows_bin, tcol, tval);
}

// products per row (P_j) -> table bin; histogram of bins; total products
// (warp-aggregated: one shared atomic per warp and bin, one per warp for
// the total).
__global__ void plan_rows(Args g, int8_t* __restrict__ bin_of, int32_t* __restrict__ pcap,
                          int32_t* __restrict__ hist, unsigned long long* __restrict__ total, int slack_pct,
                          bool win) {
  __shared__ int32_t h[kNumBins];
  __shared__ unsigned long long tsum;
  if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
  if (threadIdx.x == 0) tsum = 0;
  __syncthreads();
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int64_t p = 0;
  int bin = -1;
  if (j < g.n) {
    const int32_t e0 = g.arp[j], e1 = g.arp[j + 1];
#pragma unroll 4
    for (int32_t e = e0; e < e1; ++e) {
      const int32_t k = g.aci[e];
      p += g.brp[k + 1] - g.brp[k];
    }
    int64_t distinct = (p < g.ncols ? p : g.ncols) + 1;  // +1: the identity entry
    int logs = kMinLogSlots;
    // slots >= slack * distinct (and > distinct: find_or_insert needs an empty slot)
    const int64_t need = (distinct * slack_pct + 99) / 100;
    while ((int64_t{1} << logs) < need || (int64_t{1} << logs) <= distinct) ++logs;
    bin = kFirstSmemBin + logs - kMinLogSlots;
    if (bin > kGlobalBin) bin = kGlobalBin;
    const int32_t m = e1 - e0;
    bool windowed = false;
    int32_t lo = INT32_MAX, hi = -1;
    if (win && logs >= 8) {  // big hash rows: the column span, from the first / last entry of each B row
      const int32_t jd = static_cast<int32_t>(j + g.epi.diag_offset);
      if (g.epi.add_identity) lo = hi = jd;
      for (int32_t e = e0; e < e1; ++e) {
        const int32_t k = g.aci[e];
        const int32_t b0 = g.brp[k], b1 = g.brp[k + 1];
        if (b1 > b0) {
          lo = min(lo, g.bci[b0]);
          hi = max(hi, g.bci[b1 - 1]);
        }
      }
    }
    if (win && logs >= 8 && hi >= lo) {  // ... whose columns span < 128 Q (at most 1024)
      const int32_t span = hi - lo;
#pragma unroll
      for (int q = kNumWinBins - 1; q >= 0; --q)
        if (span < 128 * win_q(q)) bin = kWinBin0 + q, windowed = true;
    }
    if (p < 32 && m <= 32) bin = (p < 8 && m <= 8) ? 0 : (p < 16 && m <= 16) ? 1 : 2;
    bin_of[j] = static_cast<int8_t>(bin);
    pcap[j] = windowed ? lo : logs;  // window rows: the window's first column; else the table log2 size
  }
  unsigned long long ps = static_cast<unsigned long long>(p);
  unsigned long long ph = bin >= kFirstSmemBin ? ps : 0ull;  // products of hash-table rows
  for (int o = 16; o; o >>= 1) {
    ps += __shfl_xor_sync(0xffffffffu, ps, o);
    ph += __shfl_xor_sync(0xffffffffu, ph, o);
  }
  if (lane == 0 && ps) atomicAdd(&tsum, ps);
  if (lane == 0 && ph) atomicAdd(total + 1, ph);
  const unsigned grp = __match_any_sync(0xffffffffu, bin);
  if (bin >= 0 && lane == __ffs(grp) - 1) atomicAdd(&h[bin], __popc(grp));
  __syncthreads();
  if (threadIdx.x < kNumBins && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
  if (threadIdx.x == 0 && tsum) atomicAdd(total, tsum);
}

__global__ void gather_logs(const int32_t* __restrict__ rows, int32_t count, const int32_t* __restrict__ logs_of,
                            int8_t* __restrict__ out) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < count) out[q] = static_cast<int8_t>(logs_of[rows[q]]);
}

// Rows -> per-bin lists.  Block-aggregated: a block takes 1024 consecutive
// rows, counts them per bin in shared memory (warp-aggregated shared
// atomics), claims one range per (block, bin) with a global atomic, then
// scatters.  (One global atomic per (warp, bin) serialised ~65 K warps on a
// handful of cursors: 46 us per 2 M-row launch.)
constexpr int kBinRowsPerThread = 4;
__global__ void __launch_bounds__(256) scatter_bins(int64_t n, const int8_t* __restrict__ bin_of,
                                                    int32_t* __restrict__ cursor, int32_t* __restrict__ lists) {
  __shared__ int32_t cnt[kNumBins];
  __shared__ int32_t base[kNumBins];
  if (threadIdx.x < kNumBins) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * kBinRowsPerThread +
                     static_cast<int64_t>(w) * 32 * kBinRowsPerThread;
  int b[kBinRowsPerThread], pos[kBinRowsPerThread];
#pragma unroll
  for (int q = 0; q < kBinRowsPerThread; ++q) {
    const int64_t j = j0 + q * 32 + lane;
    b[q] = j < n ? bin_of[j] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, b[q]);
    const int leader = __ffs(grp) - 1;
    int lb = 0;
    if (lane == leader && b[q] >= 0) lb = atomicAdd(&cnt[b[q]], __popc(grp));
    pos[q] = __shfl_sync(0xffffffffu, lb, leader) + __popc(grp & ((1u << lane) - 1u));
  }
  __syncthreads();
  if (threadIdx.x < kNumBins && cnt[threadIdx.x]) base[threadIdx.x] = atomicAdd(&cursor[threadIdx.x], cnt[threadIdx.x]);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kBinRowsPerThread; ++q)
    if (b[q] >= 0) lists[base[b[q]] + pos[q]] = static_cast<int32_t>(j0 + q * 32 + lane);
}

// Order-preserving variant: each bin's list holds its rows in ascending row
// order.  The hash-table rows gather B rows near their own row (banded and
// geometric patterns alike), so rows processed side by side share their B
// rows in L2 only if neighbouring list entries are neighbouring rows; the
// atomic cursors above interleave 1024-row chunks from ~1000 resident blocks
// and the gathers then miss L2 (C4: ~5x the compulsory DRAM bytes).
// Pass 1 counts rows per (bin, block) into counts[bin * nblk + block]; an
// exclusive scan of that bin-major array gives every block its start in
// every bin (bins are consecutive in `lists`); pass 2 scatters in row order
// (per-warp bin counts, prefixed across the block's warps in warp order).
constexpr int kOrdWarps = 8, kOrdRows = 256 * kBinRowsPerThread;
__global__ void __launch_bounds__(256) bin_block_counts(int64_t n, const int8_t* __restrict__ bin_of, int64_t nblk,
                                                        int32_t* __restrict__ counts) {
  __shared__ int32_t cnt[kNumBins];
  if (threadIdx.x < kNumBins) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kOrdRows;
#pragma unroll
  for (int q = 0; q < kBinRowsPerThread; ++q) {
    const int64_t j = j0 + q * 256 + threadIdx.x;
    const int b = j < n ? bin_of[j] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, b);
    if (b >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&cnt[b], __popc(grp));
  }
  __syncthreads();
  if (threadIdx.x < kNumBins) counts[static_cast<int64_t>(threadIdx.x) * nblk + blockIdx.x] = cnt[threadIdx.x];
}
__global__ void __launch_bounds__(256) scatter_bins_ordered(int64_t n, const int8_t* __restrict__ bin_of, int64_t nblk,
                                                            const int32_t* __restrict__ offs,
                                                            int32_t* __restrict__ lists) {
  __shared__ int32_t wcnt[kOrdWarps][kNumBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < kOrdWarps * kNumBins; t += 256) (&wcnt[0][0])[t] = 0;
  __syncthreads();
  // warp w owns rows j0 + w*128 .. +127 (4 groups of 32, in order)
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kOrdRows + static_cast<int64_t>(w) * 32 * kBinRowsPerThread;
  int b[kBinRowsPerThread];
#pragma unroll
  for (int q = 0; q < kBinRowsPerThread; ++q) {
    const int64_t j = j0 + q * 32 + lane;
    b[q] = j < n ? bin_of[j] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, b[q]);
    if (b[q] >= 0 && lane == __ffs(grp) - 1) wcnt[w][b[q]] += __popc(grp);  // one writer per (warp, bin) per q
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < kNumBins) {  // exclusive prefix over the warps, from the block's start in the bin
    int32_t run = offs[static_cast<int64_t>(threadIdx.x) * nblk + blockIdx.x];
    for (int ww = 0; ww < kOrdWarps; ++ww) {
      const int32_t c = wcnt[ww][threadIdx.x];
      wcnt[ww][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kBinRowsPerThread; ++q) {
    const unsigned grp = __match_any_sync(0xffffffffu, b[q]);
    const int leader = __ffs(grp) - 1;
    int32_t base = 0;
    if (b[q] >= 0) base = wcnt[w][b[q]];
    __syncwarp();
    if (b[q] >= 0) {
      lists[base + __popc(grp & ((1u << lane) - 1u))] = static_cast<int32_t>(j0 + q * 32 + lane);
      if (lane == leader) wcnt[w][b[q]] = base + __popc(grp);
    }
    __syncwarp();
  }
}

using SmemKernel = void (*)(Args, const int32_t*, int32_t, bool);

SmemKernel smem_kernel(int bin) {
  switch (bin - kFirstSmemBin) {
    case 0: return spgemm_smem<6>;
    case 1: return spgemm_smem<7>;
    case 2: return spgemm_smem<8>;
    case 3: return spgemm_smem<9>;
    case 4: return spgemm_smem<10>;
    case 5: return spgemm_smem<11>;
    default: return spgemm_smem<12>;
  }
}

int warps_for_bin(int bin) {
  int logs = bin - kFirstSmemBin + kMinLogSlots;
  int w = (200 * 1024) / smem_per_warp(logs);
  return std::max(1, std::min(8, w));
}

struct Plan {
  int32_t hist[kNumBins] = {};
  int32_t start[kNumBins + 1] = {};
  int32_t* lists = nullptr;   // device, rows grouped by bin
  int64_t products = 0;
  // global bin
  int64_t* goffs = nullptr;
  int8_t* glogs = nullptr;
  int32_t* gkey = nullptr;
  double* gval = nullptr;
  // tiny rows: G-entry staging slot per row, per tiny bin
  int32_t* tcol[kTinyBins] = {};
  double* tval[kTinyBins] = {};
  const int32_t* wbase = nullptr;  // window rows: first column of the window
  const int8_t* bin_of = nullptr;  // row -> bin
};

void launch_pass(const Args& g, const Plan& pl, bool numeric, cudaStream_t s, bool recompute = true,
                 bool short_rows = false) {
  for (int tb = 0; tb < kTinyBins; ++tb) {
    const int32_t tc = pl.hist[tb];
    if (!tc) continue;
    const int per_warp = 32 / kTinyG[tb];
    const int64_t warps = (tc + per_warp - 1) / per_warp;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((warps + 7) / 8, int64_t{num_sms()} * 8 * 16));
    const bool four = tb == 0 || short_rows;  // emit lanes per row: 4 or 8
    const int64_t rpb = four ? 64 : 32;       // rows per 256-thread block of the emit
    const unsigned egrid = static_cast<unsigned>(std::min<int64_t>((tc + rpb - 1) / rpb, int64_t{num_sms()} * 8 * 16));
    const int32_t* rows = pl.lists + pl.start[tb];
    switch (kTinyG[tb]) {
      case 8:
        if (numeric) spgemm_tiny_emit<8, 4><<<egrid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        else spgemm_tiny<8><<<grid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        break;
      case 16:
        if (numeric && four) spgemm_tiny_emit<16, 4><<<egrid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        else if (numeric) spgemm_tiny_emit<16, 8><<<egrid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        else spgemm_tiny<16><<<grid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        break;
      default:
        if (numeric && four) spgemm_tiny_emit<32, 4><<<egrid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        else if (numeric) spgemm_tiny_emit<32, 8><<<egrid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
        else spgemm_tiny<32><<<grid, 256, 0, s>>>(g, rows, tc, pl.tcol[tb], pl.tval[tb]);
    }
    SAIT_LAUNCHED();
  }
  if (numeric && g.stage_pos) {  // staged hash-table rows: one copy kernel over all of them
    const int32_t cnt = pl.start[kNumBins] - pl.start[kFirstSmemBin];
    if (cnt) {
      const unsigned grid = static_cast<unsigned>(std::min<int64_t>((g.n + 31) / 32, int64_t{num_sms()} * 8 * 16));
      spgemm_stage_emit<<<grid, 256, 0, s>>>(g, pl.bin_of);
      SAIT_LAUNCHED();
    }
    if (!recompute) return;
  }
  for (int b = kFirstSmemBin; b < kFirstSmemBin + kNumSmemBins; ++b) {
    int32_t cnt = pl.hist[b];
    if (!cnt) continue;
    int warps = warps_for_bin(b);
    int smem = warps * smem_per_warp(b - kFirstSmemBin + kMinLogSlots);
    SmemKernel k = smem_kernel(b);
    if (first_on_device(reinterpret_cast<const void*>(k)))
      SAIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    int blocks_per_sm = std::max(1, (228 * 1024) / (smem + 1024));
    int64_t want = (cnt + warps - 1) / warps;
    unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, int64_t{num_sms()} * blocks_per_sm * 4));
    k<<<grid, warps * 32, smem, s>>>(g, pl.lists + pl.start[b], cnt, numeric);
    SAIT_LAUNCHED();
  }
  for (int wb = 0; wb < kNumWinBins; ++wb) {
    const int b = kWinBin0 + wb;
    const int32_t cnt = pl.hist[b];
    if (!cnt) continue;
    const int Q = kWinQ[wb];
    static const bool zero_on = [] {  // SAIT_WIN_ZERO=0: the bitmap window for every epilogue
      const char* e = std::getenv("SAIT_WIN_ZERO");
      return !(e && std::atoi(e) == 0);
    }();
    // threshold builds with +I take the -0.0 window (ZeroWindow), sized to
    // the bin; other epilogues the bitmap window of 1024 R >= 128 Q slots
    const bool zero = zero_on && g.epi.add_identity && (g.epi.drop == 1 || g.epi.drop == 3) && g.epi.tau > 0.0;
    using WK = void (*)(Args, const int32_t*, int32_t, const int32_t*, bool);
    WK k;
    int per_warp, warps = 8;
    if (zero) {
      switch (Q) {
        case 4: k = spgemm_window_z<4>; break;
        case 5: k = spgemm_window_z<5>; break;
        case 6: k = spgemm_window_z<6>; break;
        case 7: k = spgemm_window_z<7>; break;
        default: k = spgemm_window_z<8>;
      }
      per_warp = zwindow_smem_per_warp(Q);
      // warps per CTA: the most resident warps per SM (228 KB of shared
      // memory, 1 KB reserved per CTA; 64 K registers, allocated per warp in
      // units of 256)
      cudaFuncAttributes fa{};
      SAIT_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(k)));
      const int reg_warps = 65536 / (((fa.numRegs * 32 + 255) / 256) * 256);
      int best = 0;
      for (int w = 8; w >= 1; --w) {
        const int res = std::min((228 * 1024) / (w * per_warp + 1024), reg_warps / w) * w;
        if (res > best) best = res, warps = w;
      }
    } else {  // (every window bin fits the 1024-slot bitmap window)
      k = spgemm_window<1>;
      per_warp = window_smem_per_warp(1);
      warps = window_warps(1);
    }
    const int smem = warps * per_warp;
    if (first_on_device(reinterpret_cast<const void*>(k)))
      SAIT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int blocks_per_sm = std::max(1, (228 * 1024) / (smem + 1024));
    const int64_t per_warp_rows = zero ? kRun : 1;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(
        (cnt + warps * per_warp_rows - 1) / (warps * per_warp_rows), int64_t{num_sms()} * blocks_per_sm * 4));
    k<<<grid, warps * 32, smem, s>>>(g, pl.lists + pl.start[b], cnt, pl.wbase, numeric);
    SAIT_LAUNCHED();
  }
  int32_t gc = pl.hist[kGlobalBin];
  if (gc) {
    unsigned grid = static_cast<unsigned>(std::min<int64_t>((gc + 7) / 8, num_sms() * 8));
    spgemm_global<<<grid, 256, 0, s>>>(g, pl.lists + pl.start[kGlobalBin], pl.goffs, pl.glogs, gc, pl.gkey,
                                        pl.gval, numeric);
    SAIT_LAUNCHED();
  }
}

}  // namespace

namespace {
// First step of a row-form recursion, C = drop(A I + I): every product is
// a_ik * 1.0 (= a_ik exactly) and A (= tT) holds no diagonal, so row i of C
// is A's row with 1.0 inserted at column i, filtered by the drop rule --
// the same entries and bits the generic pass produces, without planning,
// hashing or staging.  Thread per row.  Threshold / no-drop epilogues only
// (the caller keeps the generic pass for pattern drops).
__device__ __forceinline__ bool first_keep(const Epilogue& e, int32_t i, int32_t col, double v) {
  if (e.drop == 2) return in_pattern(e.pci, e.prp[i], e.prp[i + 1], col);
  if ((e.drop == 1 || e.drop == 3) && e.tau != 0.0) return col == i || fabs(v) >= e.tau;
  return true;
}
// G lanes per row (32/G rows per warp), the row's entries G at a time: the
// survivors' positions come from ballots of the keep flags; the diagonal
// goes right after the kept entries of columns < i (rows are sorted).
template <int G>
__device__ __forceinline__ unsigned group_ballot(bool p, int wl) {
  const unsigned b = __ballot_sync(0xffffffffu, p);
  return G == 32 ? b : (b >> (wl & ~(G - 1))) & ((1u << G) - 1u);
}
__global__ void first_step_count(int64_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                 const double* __restrict__ av, Epilogue e, int32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t r = static_cast<int32_t>(i);
  int32_t c = first_keep(e, r, r, 1.0) ? 1 : 0;
  for (int32_t q = arp[i]; q < arp[i + 1]; ++q) c += first_keep(e, r, aci[q], av[q]);
  cnt[i] = c;
}
template <int G>
__global__ void first_step_write(int64_t n, const int32_t* __restrict__ arp, const int32_t* __restrict__ aci,
                                 const double* __restrict__ av, Epilogue e, const int32_t* __restrict__ crp,
                                 int32_t* __restrict__ cci, double* __restrict__ cv) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const int wl = threadIdx.x & 31, lane = wl & (G - 1);
  const bool live = i < n;
  const int32_t r = static_cast<int32_t>(i);
  int32_t q0 = 0, q1 = 0, out = 0;
  if (live) {
    q0 = arp[i];
    q1 = arp[i + 1];
    out = crp[i];
  }
  const int32_t len = q1 - q0;
  const bool diag = live && first_keep(e, r, r, 1.0);
  bool placed = !diag;  // the diagonal written (or not kept)
  const unsigned below = (1u << lane) - 1u;
  auto put = [&](int32_t p, int32_t col, double v) {
    cci[p] = col;
    cv[p] = e.out_scale ? __dmul_rn(v, e.out_scale[col]) : v;
  };
  if constexpr (G == 1) {  // thread per row (short rows)
    if (!live) return;
    for (int32_t q = q0; q < q1; ++q) {
      const int32_t col = aci[q];
      if (!placed && col > r) {
        put(out++, r, 1.0);
        placed = true;
      }
      const double v = __dmul_rn(av[q], 1.0);
      if (first_keep(e, r, col, v)) put(out++, col, v);
    }
    if (!placed) put(out, r, 1.0);
  } else {
  for (int32_t o = 0; __any_sync(0xffffffffu, o < len); o += G) {
    const bool in = o + lane < len;
    const int32_t q = q0 + o + lane;
    const int32_t col = in ? aci[q] : INT32_MAX;
    const double v = in ? __dmul_rn(av[q], 1.0) : 0.0;
    const bool keep = in && first_keep(e, r, col, v);
    const unsigned km = group_ballot<G>(keep, wl);
    const unsigned after = group_ballot<G>(in && col > r, wl);  // a suffix of the chunk
    const bool here = !placed && after != 0u;  // the diagonal lands in this chunk, before `after`
    if (keep) put(out + __popc(km & below) + ((here && col > r) ? 1 : 0), col, v);
    if (here && lane == 0) put(out + __popc(km & ~after), r, 1.0);
    out += __popc(km) + (here ? 1 : 0);
    placed = placed || here;
  }
  if (live && !placed && lane == 0) put(out, r, 1.0);
  }
}
}  // namespace

SpgemmResult first_step_identity(const DevCsr& a, const Epilogue& epi, cudaStream_t s) {
  SpgemmResult res;
  const int64_t n = a.nrows;
  DevCsr& c = res.c;
  c.nrows = c.ncols = n;
  c.rp = dalloc<int32_t>(n + 1, s);
  int32_t* cnt = dalloc<int32_t>(n > 0 ? n : 1, s);
  const bool wide = a.nnz >= 12 * n;  // long rows: 4 lanes per row in the write pass (1.28 vs 3.6 ms at C4)
  if (n > 0) {
    first_step_count<<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, a.ci, a.v, epi, cnt);
    SAIT_LAUNCHED();
  }
  c.nnz = scan_counts(cnt, c.rp, n, s);
  dfree(cnt, s);
  if (c.nnz > INT32_MAX)
    throw Error(SAIT_ERR_NOMEM, "result has " + std::to_string(c.nnz) +
                                    " stored entries; the device CSR uses int32 indices (max 2^31-1)");
  c.ci = dalloc<int32_t>(c.nnz > 0 ? c.nnz : 1, s);
  c.v = dalloc<double>(c.nnz > 0 ? c.nnz : 1, s);
  if (n > 0) {
    if (wide)
      first_step_write<4><<<grid_for(n * 4, 256), 256, 0, s>>>(n, a.rp, a.ci, a.v, epi, c.rp, c.ci, c.v);
    else
      first_step_write<1><<<grid_for(n, 256), 256, 0, s>>>(n, a.rp, a.ci, a.v, epi, c.rp, c.ci, c.v);
    SAIT_LAUNCHED();
  }
  res.products = a.nnz;
  // vs M_0 = I (threshold or no drop): the diagonal always survives with
  // value 1.0, so M_1 == I exactly when nothing else survived
  res.changed = c.nnz != n;
  return res;
}

SpgemmResult spgemm_fused(const DevCsr& a, const DevCsr& b, const Epilogue& epi, cudaStream_t s) {
  if (a.ncols != b.nrows)
    throw_invalid("spgemm: inner dimensions " + std::to_string(a.ncols) + " and " + std::to_string(b.nrows) +
                  " do not match");
  SpgemmResult res;
  const int64_t n = a.nrows;
  DevCsr& c = res.c;
  c.nrows = n;
  c.ncols = b.ncols;
  c.rp = dalloc<int32_t>(n + 1, s);
  if (n == 0) {
    SAIT_CUDA(cudaMemsetAsync(c.rp, 0, sizeof(int32_t), s));
    c.ci = dalloc<int32_t>(1, s);
    c.v = dalloc<double>(1, s);
    res.changed = epi.qrp != nullptr ? false : true;
    return res;
  }
  Args g{};
  g.n = n;
  g.ncols = b.ncols;
  g.arp = a.rp;
  g.aci = a.ci;
  g.av = a.v;
  g.brp = b.rp;
  g.bci = b.ci;
  g.bv = b.v;
  g.epi = epi;

  // ---- plan: bin rows by product count
  Plan pl;
  int8_t* bin_of = dalloc<int8_t>(n, s);
  pl.bin_of = bin_of;
  int32_t* logs_of = dalloc<int32_t>(n, s);
  int32_t* hist = dalloc<int32_t>(2 * kNumBins, s);
  unsigned long long* total = dalloc<unsigned long long>(2, s);  // all products, hash-row products
  SAIT_CUDA(cudaMemsetAsync(hist, 0, 2 * kNumBins * sizeof(int32_t), s));
  SAIT_CUDA(cudaMemsetAsync(total, 0, 2 * sizeof(unsigned long long), s));
  static const int slack_pct = [] {
    const char* e = std::getenv("SAIT_HASH_SLACK");  // table slots per possible distinct column, in %
    return e ? std::max(101, std::atoi(e)) : 140;
  }();
  static const bool window_on = [] {  // SAIT_SPGEMM_WINDOW=0: hash tables only
    const char* e = std::getenv("SAIT_SPGEMM_WINDOW");
    return !(e && std::atoi(e) == 0);
  }();
  plan_rows<<<grid_for(n, 256), 256, 0, s>>>(g, bin_of, logs_of, hist, total, slack_pct, window_on);
  SAIT_LAUNCHED();
  unsigned long long htot[2] = {0, 0};
  read_back(s, {{pl.hist, hist, sizeof pl.hist}, {htot, total, sizeof htot}});
  const unsigned long long htotal = htot[0], hashed_products = htot[1];
  res.products = static_cast<int64_t>(htotal);
  for (int b2 = 0; b2 < kNumBins; ++b2) pl.start[b2 + 1] = pl.start[b2] + pl.hist[b2];
  pl.lists = dalloc<int32_t>(n, s);
  pl.wbase = logs_of;
  int32_t* cursor = hist + kNumBins;
  SAIT_CUDA(cudaMemcpyAsync(cursor, pl.start, kNumBins * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  for (int tb = 0; tb < kTinyBins; ++tb)
    if (pl.hist[tb]) {
      pl.tcol[tb] = dalloc<int32_t>(static_cast<int64_t>(pl.hist[tb]) * kTinyG[tb], s);
      pl.tval[tb] = dalloc<double>(static_cast<int64_t>(pl.hist[tb]) * kTinyG[tb], s);
    }
  static const int order_mode = [] {  // SAIT_BIN_ORDER: 0 atomic cursors, 1 always ordered, default: hash rows
    const char* e = std::getenv("SAIT_BIN_ORDER");
    return e ? std::atoi(e) : 2;
  }();
  const bool ordered =
      order_mode == 1 || (order_mode == 2 && pl.start[kNumBins] - pl.start[kFirstSmemBin] > 0);
  if (ordered) {
    const int64_t nblk = (n + kOrdRows - 1) / kOrdRows;
    int32_t* bc = dalloc<int32_t>(kNumBins * nblk, s);
    int32_t* bo = dalloc<int32_t>(kNumBins * nblk + 1, s);
    int64_t* btot = dalloc<int64_t>(1, s);
    bin_block_counts<<<static_cast<unsigned>(nblk), 256, 0, s>>>(n, bin_of, nblk, bc);
    SAIT_LAUNCHED();
    scan_counts_async(bc, bo, kNumBins * nblk, btot, s);
    dfree(btot, s);
    scatter_bins_ordered<<<static_cast<unsigned>(nblk), 256, 0, s>>>(n, bin_of, nblk, bo, pl.lists);
    SAIT_LAUNCHED();
    dfree(bc, s);
    dfree(bo, s);
  } else {
    scatter_bins<<<grid_for(n, 256 * kBinRowsPerThread), 256, 0, s>>>(n, bin_of, cursor, pl.lists);
    SAIT_LAUNCHED();
  }
  int32_t gc = pl.hist[kGlobalBin];
  if (gc) {
    // per-row global tables: gather the table sizes of the global-bin rows on
    // the device (only gc bytes cross PCIe), offsets on the host
    pl.glogs = dalloc<int8_t>(gc, s);
    gather_logs<<<grid_for(gc, 256), 256, 0, s>>>(pl.lists + pl.start[kGlobalBin], gc, logs_of, pl.glogs);
    SAIT_LAUNCHED();
    std::vector<int8_t> lg(gc);
    SAIT_CUDA(cudaMemcpyAsync(lg.data(), pl.glogs, gc * sizeof(int8_t), cudaMemcpyDeviceToHost, s));
    SAIT_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> offs(gc);
    int64_t tot = 0;
    for (int32_t q = 0; q < gc; ++q) {
      offs[q] = tot;
      tot += int64_t{1} << lg[q];
    }
    pl.goffs = dalloc<int64_t>(gc, s);
    pl.gkey = dalloc<int32_t>(tot, s);
    pl.gval = dalloc<double>(tot, s);
    SAIT_CUDA(cudaMemcpyAsync(pl.goffs, offs.data(), gc * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SAIT_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
  }

  // ---- count pass (hash-table rows staged), scan, numeric pass
  int32_t* counts = dalloc<int32_t>(n, s);
  g.ccount = counts;
  const int32_t hashed = pl.start[kNumBins] - pl.start[kFirstSmemBin];
  if (hashed && !std::getenv("SAIT_SPGEMM_NOSTAGE")) {
    // survivors of a row <= its products + 1; the staging area is sized from
    // the A operand (the previous iterate) and capped, rows beyond it fall
    // back to recomputation in the numeric pass
    int64_t cap = std::min<int64_t>({static_cast<int64_t>(hashed_products) + hashed,
                                     2 * a.nnz + n + (int64_t{1} << 20), int64_t{INT32_MAX}});
    if (const char* e = std::getenv("SAIT_SPGEMM_STAGE_CAP")) cap = std::min<int64_t>(cap, std::atoll(e));  // tests
    g.stage_cap = cap;
    g.stage_col = dalloc<int32_t>(cap, s);
    g.stage_val = dalloc<double>(cap, s);
    g.stage_pos = dalloc<int32_t>(n, s);
    g.stage_cursor = dalloc<unsigned long long>(1, s);
    SAIT_CUDA(cudaMemsetAsync(g.stage_cursor, 0, sizeof(unsigned long long), s));
  }
  launch_pass(g, pl, false, s);
  // one host round trip for the output size and the staging use
  int64_t* meta = reinterpret_cast<int64_t*>(total);  // {nnz, staged entries}; plan totals already read
  scan_counts_async(counts, c.rp, n, meta, s);
  if (g.stage_pos)
    SAIT_CUDA(cudaMemcpyAsync(meta + 1, g.stage_cursor, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
  int64_t hmeta[2] = {0, 0};
  read_back(s, {{hmeta, meta, sizeof hmeta}});
  if (hmeta[0] > INT32_MAX)
    throw Error(SAIT_ERR_NOMEM, "result has " + std::to_string(hmeta[0]) +
                                    " stored entries; the device CSR uses int32 indices (max 2^31-1)");
  c.nnz = hmeta[0];
  dfree(counts, s);
  c.ci = dalloc<int32_t>(c.nnz, s);
  c.v = dalloc<double>(c.nnz, s);
  int* changed = dalloc<int>(1, s);
  SAIT_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), s));
  g.ccount = nullptr;
  g.crp = c.rp;
  g.cci = c.ci;
  g.cv = c.v;
  g.changed = changed;
  // stabilized() compares the row pointers first (sait.cpp:19): a result of
  // another size has changed, and the numeric pass skips the value compare
  const bool compare = epi.qrp && !(epi.qnnz >= 0 && epi.qnnz != c.nnz);
  if (!compare) g.epi.qrp = g.epi.qci = nullptr, g.epi.qv = nullptr;
  const bool overflow = g.stage_pos && static_cast<unsigned long long>(hmeta[1]) >
                                           static_cast<unsigned long long>(g.stage_cap);
  launch_pass(g, pl, true, s, overflow, c.nnz <= 8 * n);
  if (compare) {
    int hc = 1;
    read_back(s, {{&hc, changed, sizeof hc}});
    res.changed = hc != 0;
  }
  dfree(changed, s);
  dfree(g.stage_col, s);
  dfree(g.stage_val, s);
  dfree(g.stage_pos, s);
  dfree(g.stage_cursor, s);
  dfree(bin_of, s);
  dfree(logs_of, s);
  dfree(hist, s);
  dfree(total, s);
  dfree(pl.lists, s);
  dfree(pl.goffs, s);
  dfree(pl.glogs, s);
  dfree(pl.gkey, s);
  dfree(pl.gval, s);
  for (int tb = 0; tb < kTinyBins; ++tb) {
    dfree(pl.tcol[tb], s);
    dfree(pl.tval[tb], s);
  }
  return res;
}

}  // namespace sait
