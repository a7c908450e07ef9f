// host_inputs.cpp — producers of the SAIT path's inputs (host C++):
//   * sait_ilu_k: level-of-fill ILU(k) by IKJ elimination (ilu.hpp:27,
//     ilu.cpp:98-173).  The path must see the SAME factors as the reference,
//     so the numeric phase performs the reference's operation sequence:
//     w[k] <- w[k] / u_kk, then w[j] <- w[j] - w[k] * u_kj for each j of
//     U(k,:) in the row's pattern, pivots k in increasing order, every product
//     rounded before the subtraction (compiled with -ffp-contract=off).
//   * seeded generators for BASELINE.json's synthetic problems.
// Compiled with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <queue>
#include <stdexcept>
#include <string>
#include <vector>

#include "sait_c.h"

namespace sait {
void set_last_error(const std::string& msg);  // capi.cu (sait_last_error)
}

namespace {


struct HostError : std::runtime_error {
  int code;
  HostError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <class F>
int host_guard(F&& f) {
  try {
    f();
    return SAIT_OK;
  } catch (const HostError& e) {
    sait::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    sait::set_last_error("out of host memory");
    return SAIT_ERR_NOMEM;
  }
}

struct Csr64 {
  int64_t nrows = 0, ncols = 0;
  std::vector<int64_t> rp{0}, ci;
  std::vector<double> v;
};

void emit(const Csr64& m, sait_host_csr* out) {
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  auto copy = [](const auto& vec) {
    using T = typename std::decay_t<decltype(vec)>::value_type;
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (vec.size() ? vec.size() : 1)));
    if (!p) throw std::bad_alloc();
    if (!vec.empty()) std::memcpy(p, vec.data(), sizeof(T) * vec.size());
    return p;
  };
  out->row_ptr = copy(m.rp);
  out->col_idx = copy(m.ci);
  out->values = copy(m.v);
}

// ----------------------------------------------------------------- ILU(k)

struct FillPattern {
  std::vector<int64_t> lp{0}, lc;           // strictly lower part per row
  std::vector<int64_t> up{0}, uc;           // upper part (diagonal first) per row
  std::vector<int> ul;                      // fill level of each U entry
};

// lev(i,j) = min over pivots k < min(i,j) of lev(i,k) + lev(k,j) + 1, entries
// of A at level 0, keep lev <= level.  Pivots are visited in increasing order
// through a min-heap; a pivot's level is final when it is popped because only
// smaller pivots can lower it.
FillPattern symbolic(const sait_host_csr* a, int level) {
  const int64_t n = a->nrows;
  FillPattern f;
  std::vector<int> lev(n, 0);
  std::vector<int64_t> mark(n, -1);
  std::vector<int64_t> cols;
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> pivots;
  for (int64_t i = 0; i < n; ++i) {
    cols.clear();
    bool diag = false;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) {
      const int64_t j = a->col_idx[e];
      diag = diag || j == i;
      mark[j] = i;
      lev[j] = 0;
      cols.push_back(j);
      if (j < i) pivots.push(j);
    }
    if (!diag)
      throw HostError(SAIT_ERR_INVALID_ARGUMENT, "ilu_k: structurally zero diagonal at row " + std::to_string(i));
    while (!pivots.empty()) {
      const int64_t k = pivots.top();
      pivots.pop();
      const int lk = lev[k];
      for (int64_t q = f.up[k]; q < f.up[k + 1]; ++q) {
        const int64_t j = f.uc[q];
        if (j == k) continue;
        const int cand = lk + f.ul[q] + 1;
        if (cand > level) continue;
        if (mark[j] == i) {
          lev[j] = std::min(lev[j], cand);
        } else {
          mark[j] = i;
          lev[j] = cand;
          cols.push_back(j);
          if (j < i) pivots.push(j);
        }
      }
    }
    std::sort(cols.begin(), cols.end());
    for (int64_t j : cols) {
      if (j < i) {
        f.lc.push_back(j);
      } else {
        f.uc.push_back(j);
        f.ul.push_back(lev[j]);
      }
    }
    f.lp.push_back(static_cast<int64_t>(f.lc.size()));
    f.up.push_back(static_cast<int64_t>(f.uc.size()));
  }
  return f;
}

void ilu(const sait_host_csr* a, int level, Csr64& L, Csr64& U) {
  if (a->nrows != a->ncols) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "ilu_k: matrix is not square");
  if (level < 0) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "ilu_k: negative fill level");
  const int64_t n = a->nrows;
  const int64_t nnz = a->row_ptr[n];
  double amax = 0.0;
  for (int64_t e = 0; e < nnz; ++e) amax = std::max(amax, std::fabs(a->values[e]));
  const double breakdown = 1e-14 * amax;
  FillPattern f = symbolic(a, level);
  L.nrows = L.ncols = U.nrows = U.ncols = n;
  L.ci.reserve(f.lc.size() + n);
  L.v.reserve(f.lc.size() + n);
  U.ci.reserve(f.uc.size());
  U.v.reserve(f.uc.size());
  std::vector<double> w(n, 0.0), pivot(n, 0.0);
  std::vector<int64_t> in_row(n, -1);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t p = f.lp[i]; p < f.lp[i + 1]; ++p) in_row[f.lc[p]] = i, w[f.lc[p]] = 0.0;
    for (int64_t p = f.up[i]; p < f.up[i + 1]; ++p) in_row[f.uc[p]] = i, w[f.uc[p]] = 0.0;
    for (int64_t e = a->row_ptr[i]; e < a->row_ptr[i + 1]; ++e) w[a->col_idx[e]] = a->values[e];
    for (int64_t p = f.lp[i]; p < f.lp[i + 1]; ++p) {
      const int64_t k = f.lc[p];
      const double mult = w[k] / pivot[k];
      w[k] = mult;
      for (int64_t q = U.rp[k]; q < U.rp[k + 1]; ++q) {
        const int64_t j = U.ci[q];
        if (j != k && in_row[j] == i) w[j] -= mult * U.v[q];
      }
    }
    for (int64_t p = f.lp[i]; p < f.lp[i + 1]; ++p) {
      L.ci.push_back(f.lc[p]);
      L.v.push_back(w[f.lc[p]]);
    }
    L.ci.push_back(i);  // explicit unit diagonal (ilu.cpp:156-157)
    L.v.push_back(1.0);
    L.rp.push_back(static_cast<int64_t>(L.ci.size()));
    const double piv = w[i];
    if (piv == 0.0 || std::fabs(piv) < breakdown) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%f", std::fabs(piv));
      throw HostError(SAIT_ERR_RUNTIME,
                      "ilu_k: pivot breakdown at row " + std::to_string(i) + " (|pivot| = " + buf + ")");
    }
    pivot[i] = piv;
    for (int64_t p = f.up[i]; p < f.up[i + 1]; ++p) {
      U.ci.push_back(f.uc[p]);
      U.v.push_back(w[f.uc[p]]);
    }
    U.rp.push_back(static_cast<int64_t>(U.ci.size()));
  }
}

// ------------------------------------------------------------- generators

uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t draw(uint64_t seed, uint64_t ctr) { return mix64(seed ^ mix64(ctr)); }
double unit53(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }        // [0,1)
double unit53_open0(uint64_t bits) { return static_cast<double>((bits >> 11) + 1) * 0x1.0p-53; }  // (0,1]

// Rows built in parallel chunks (OpenMP), concatenated in row order: each
// row's entries depend only on the row index, so the result is the same as a
// sequential build.
struct RowSink {
  std::vector<int64_t> ci;
  std::vector<double> v;
  std::vector<int64_t> cnt;
  void put(int64_t c, double x) {
    ci.push_back(c);
    v.push_back(x);
  }
};
template <class RowFn>
void build_rows_parallel(int64_t n, int64_t ncols, RowFn fn, sait_host_csr* out) {
  constexpr int64_t kChunk = 8192;
  const int64_t nch = (n + kChunk - 1) / kChunk;
  std::vector<RowSink> parts(static_cast<size_t>(nch));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nch; ++c) {
    RowSink& sk = parts[c];
    const int64_t r0 = c * kChunk, r1 = std::min(n, r0 + kChunk);
    sk.cnt.reserve(r1 - r0);
    for (int64_t i = r0; i < r1; ++i) {
      const size_t before = sk.ci.size();
      fn(i, sk);
      sk.cnt.push_back(static_cast<int64_t>(sk.ci.size() - before));
    }
  }
  std::vector<int64_t> base(static_cast<size_t>(nch) + 1, 0);
  for (int64_t c = 0; c < nch; ++c) base[c + 1] = base[c] + static_cast<int64_t>(parts[c].ci.size());
  const int64_t nnz = base[nch];
  out->nrows = n;
  out->ncols = ncols;
  out->row_ptr = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (n + 1)));
  out->col_idx = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (nnz ? nnz : 1)));
  out->values = static_cast<double*>(std::malloc(sizeof(double) * (nnz ? nnz : 1)));
  if (!out->row_ptr || !out->col_idx || !out->values) {
    std::free(out->row_ptr);
    std::free(out->col_idx);
    std::free(out->values);
    out->row_ptr = out->col_idx = nullptr;
    out->values = nullptr;
    throw std::bad_alloc();
  }
  out->row_ptr[0] = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nch; ++c) {
    const RowSink& sk = parts[c];
    int64_t at = base[c];
    const int64_t r0 = c * kChunk;
    for (size_t q = 0; q < sk.cnt.size(); ++q) {
      at += sk.cnt[q];
      out->row_ptr[r0 + static_cast<int64_t>(q) + 1] = at;
    }
    if (!sk.ci.empty()) {
      std::memcpy(out->col_idx + base[c], sk.ci.data(), sizeof(int64_t) * sk.ci.size());
      std::memcpy(out->values + base[c], sk.v.data(), sizeof(double) * sk.v.size());
    }
  }
}



}  // namespace

extern "C" {

int sait_ilu_k(const sait_host_csr* a, int level, sait_host_csr* lower, sait_host_csr* upper) {
  return host_guard([&] {
    if (!a || !lower || !upper) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "ilu_k: null argument");
    Csr64 L, U;
    ilu(a, level, L, U);
    emit(L, lower);
    emit(U, upper);
  });
}

int sait_problem_laplacian_2d(int64_t nx, sait_host_csr* out) {
  return host_guard([&] {
    if (nx < 1) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "laplacian_2d: nx must be >= 1");
    const int64_t n = nx * nx;
    build_rows_parallel(n, n, [nx](int64_t i, RowSink& b) {
      const int64_t y = i / nx, x = i % nx;
      if (y > 0) b.put(i - nx, -1.0);
      if (x > 0) b.put(i - 1, -1.0);
      b.put(i, 4.0);
      if (x + 1 < nx) b.put(i + 1, -1.0);
      if (y + 1 < nx) b.put(i + nx, -1.0);
    }, out);
  });
}

int sait_problem_laplacian_3d(int64_t m, sait_host_csr* out) {
  return host_guard([&] {
    if (m < 1) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "laplacian_3d: n must be >= 1");
    const int64_t plane = m * m, n = plane * m;
    build_rows_parallel(n, n, [m, plane](int64_t i, RowSink& b) {
      const int64_t z = i / plane, y = (i / m) % m, x = i % m;
      if (z > 0) b.put(i - plane, -1.0);
      if (y > 0) b.put(i - m, -1.0);
      if (x > 0) b.put(i - 1, -1.0);
      b.put(i, 6.0);
      if (x + 1 < m) b.put(i + 1, -1.0);
      if (y + 1 < m) b.put(i + m, -1.0);
      if (z + 1 < m) b.put(i + plane, -1.0);
    }, out);
  });
}

int sait_problem_convdiff_2d(int64_t nx, double bx, double by, sait_host_csr* out) {
  return host_guard([&] {
    if (nx < 1) throw HostError(SAIT_ERR_INVALID_ARGUMENT, "convdiff_2d: nx must be >= 1");
    const double h = 1.0 / static_cast<double>(nx + 1);
    // w[dy+1][dx+1]: 9-point isotropic diffusion / 6 + first-order upwind convection * h
    double w[3][3] = {{-1.0 / 6.0, -4.0 / 6.0, -1.0 / 6.0},
                      {-4.0 / 6.0, 20.0 / 6.0, -4.0 / 6.0},
                      {-1.0 / 6.0, -4.0 / 6.0, -1.0 / 6.0}};
    const double cx = h * bx, cy = h * by;
    if (cx >= 0) {
      w[1][1] += cx;
      w[1][0] -= cx;
    } else {
      w[1][1] -= cx;
      w[1][2] += cx;
    }
    if (cy >= 0) {
      w[1][1] += cy;
      w[0][1] -= cy;
    } else {
      w[1][1] -= cy;
      w[2][1] += cy;
    }
    const int64_t n = nx * nx;
    build_rows_parallel(n, n, [nx, &w](int64_t i, RowSink& b) {
      const int64_t y = i / nx, x = i % nx;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t xx = x + dx, yy = y + dy;
          if (xx < 0 || xx >= nx || yy < 0 || yy >= nx) continue;
          b.put(yy * nx + xx, w[dy + 1][dx + 1]);
        }
    }, out);
  });
}

int sait_problem_synthetic_lower(int64_t n, int64_t draws, double p, uint64_t seed, sait_host_csr* out) {
  return host_guard([&] {
    if (n < 1 || draws < 0 || !(p > 0.0 && p < 1.0))
      throw HostError(SAIT_ERR_INVALID_ARGUMENT, "synthetic_lower: bad parameters");
    const double lq = std::log1p(-p);
    const uint64_t s_off = seed * 2 + 1, s_val = seed * 2 + 2;
    build_rows_parallel(n, n, [&](int64_t i, RowSink& b) {
      thread_local std::vector<std::pair<int64_t, double>> row;
      row.clear();
      for (int64_t d = 0; i > 0 && d < draws; ++d) {
        const uint64_t ctr = static_cast<uint64_t>(i) * static_cast<uint64_t>(draws) + static_cast<uint64_t>(d);
        const double g = std::floor(std::log(unit53_open0(draw(s_off, ctr))) / lq);
        const int64_t off = g >= static_cast<double>(i) ? i : 1 + static_cast<int64_t>(g);
        const double u1 = unit53_open0(draw(s_val, 2 * ctr));
        const double u2 = unit53(draw(s_val, 2 * ctr + 1));
        const double val = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
        const int64_t c = i - std::min(off, i);
        auto it = std::lower_bound(row.begin(), row.end(), c,
                                   [](const std::pair<int64_t, double>& a, int64_t key) { return a.first < key; });
        if (it != row.end() && it->first == c) it->second += val;  // duplicates summed in draw order
        else row.insert(it, {c, val});
      }
      double sum_abs = 0.0;
      for (const auto& [c, v] : row) sum_abs += std::fabs(v);
      for (const auto& [c, v] : row) b.put(c, v);
      b.put(i, 1.5 * sum_abs + 1.0);
    }, out);
  });
}

void sait_fill_uniform_pm1(uint64_t seed, int64_t n, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * unit53(draw(seed, static_cast<uint64_t>(i))) - 1.0;
}

}  // extern "C"
