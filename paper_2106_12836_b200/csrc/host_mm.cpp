// host_mm.cpp — F4: Matrix Market ingestion (SPEC.md:373-381 mm_read, spec
// only in the reference) and the right-hand sides of the experiments
// (SPEC.md:382-389 make_rhs).  Host C++; the matrices then go to the device.
//
// mm_read: "%%MatrixMarket matrix coordinate real|integer general|symmetric";
// '%' lines skipped; 1-based indices; symmetric files expanded to full
// storage (each off-diagonal (i, j) followed by its mirror (j, i)); entries
// assembled with the reference's from_triplets rule (csr.cpp:10-58: stable
// order by (row, col), duplicates summed in input order).  Errors name the
// line: "mm_read: line N: ...".  mm_write emits the general form with
// %.17g values, so mm_read(mm_write(M)) == M bit for bit.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "sait_c.h"

namespace sait {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

struct MmError : std::runtime_error {
  int code;
  MmError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return SAIT_OK;
  } catch (const MmError& e) {
    sait::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    sait::set_last_error("out of host memory");
    return SAIT_ERR_NOMEM;
  }
}

[[noreturn]] void parse_error(int64_t line, const std::string& what) {
  throw MmError(SAIT_ERR_INVALID_ARGUMENT, "mm_read: line " + std::to_string(line) + ": " + what);
}

template <class T>
T* host_copy(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

std::string lower_word(const char*& p, const char* end) {
  while (p < end && (*p == ' ' || *p == '\t')) ++p;
  std::string w;
  while (p < end && *p != ' ' && *p != '\t' && *p != '\r' && *p != '\n') w += static_cast<char>(std::tolower(*p++));
  return w;
}

struct Reader {
  std::vector<char> buf;  // file bytes + a terminating NUL (strtoll stops there)
  size_t size = 0;        // file bytes
  size_t pos = 0;
  int64_t line = 0;
  // next line as [b, e) without the newline; false at end of file
  bool next(const char*& b, const char*& e) {
    if (pos >= size) return false;
    b = buf.data() + pos;
    const void* nl = std::memchr(b, '\n', size - pos);
    e = nl ? static_cast<const char*>(nl) : buf.data() + size;
    pos = static_cast<size_t>(e - buf.data()) + 1;
    if (e > b && e[-1] == '\r') --e;
    ++line;
    return true;
  }
};

bool blank(const char* b, const char* e) {
  for (; b < e; ++b)
    if (*b != ' ' && *b != '\t') return false;
  return true;
}

// integer field; advances p; false if none
bool read_i64(const char*& p, const char* e, int64_t& out) {
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  if (p >= e) return false;
  char* end = nullptr;
  errno = 0;
  const long long v = std::strtoll(p, &end, 10);
  if (end == p || errno == ERANGE || (end < e && *end != ' ' && *end != '\t')) return false;
  out = v;
  p = end;
  return true;
}

bool read_f64(const char*& p, const char* e, double& out) {
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  if (p >= e) return false;
  // strtod needs a terminated string: copy the token
  char tok[128];
  size_t k = 0;
  while (p < e && *p != ' ' && *p != '\t' && k + 1 < sizeof tok) tok[k++] = *p++;
  if (p < e && *p != ' ' && *p != '\t') return false;
  tok[k] = 0;
  char* end = nullptr;
  out = std::strtod(tok, &end);
  return end == tok + k && k > 0;
}

}  // namespace

extern "C" {

int sait_mm_read(const char* path, sait_host_csr* out) {
  return guard([&] {
    if (!path || !out) throw MmError(SAIT_ERR_INVALID_ARGUMENT, "mm_read: null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw MmError(SAIT_ERR_INVALID_ARGUMENT, std::string("mm_read: cannot open ") + path);
    Reader r;
    {
      std::fseek(f, 0, SEEK_END);
      const long size = std::ftell(f);
      std::fseek(f, 0, SEEK_SET);
      r.size = size > 0 ? static_cast<size_t>(size) : 0;
      r.buf.assign(r.size + 1, '\0');
      const size_t got = r.size ? std::fread(r.buf.data(), 1, r.size, f) : 0;
      std::fclose(f);
      if (got != r.size) throw MmError(SAIT_ERR_INVALID_ARGUMENT, std::string("mm_read: read error on ") + path);
    }
    const char *b = nullptr, *e = nullptr;
    if (!r.next(b, e)) parse_error(1, "empty file");
    // header
    {
      const char* p = b;
      const std::string banner = lower_word(p, e);
      const std::string object = lower_word(p, e), format = lower_word(p, e), field = lower_word(p, e),
                        symmetry = lower_word(p, e);
      if (banner != "%%matrixmarket") parse_error(r.line, "missing %%MatrixMarket banner");
      if (object != "matrix") parse_error(r.line, "object '" + object + "' is not 'matrix'");
      if (format != "coordinate") parse_error(r.line, "format '" + format + "' is not 'coordinate'");
      if (field == "complex" || field == "pattern")
        parse_error(r.line, "field '" + field + "' not supported (real or integer only)");
      if (field != "real" && field != "integer" && field != "double")
        parse_error(r.line, "unknown field '" + field + "'");
      if (symmetry != "general" && symmetry != "symmetric")
        parse_error(r.line, "symmetry '" + symmetry + "' not supported (general or symmetric only)");
      const bool sym = symmetry == "symmetric";
      // size line (after comments / blank lines)
      int64_t nrows = 0, ncols = 0, nnz = 0;
      while (true) {
        if (!r.next(b, e)) parse_error(r.line + 1, "missing size line");
        if (b < e && *b == '%') continue;
        if (blank(b, e)) continue;
        const char* q = b;
        if (!read_i64(q, e, nrows) || !read_i64(q, e, ncols) || !read_i64(q, e, nnz) || !blank(q, e))
          parse_error(r.line, "malformed size line (expected 'rows cols entries')");
        if (nrows < 0 || ncols < 0 || nnz < 0) parse_error(r.line, "negative size");
        if (sym && nrows != ncols) parse_error(r.line, "symmetric matrix must be square");
        break;
      }
      std::vector<int64_t> ri, cj;
      std::vector<double> vv;
      const size_t cap = static_cast<size_t>(sym ? 2 * nnz : nnz);
      ri.reserve(cap);
      cj.reserve(cap);
      vv.reserve(cap);
      int64_t seen = 0;
      while (r.next(b, e)) {
        if (b < e && *b == '%') continue;
        if (blank(b, e)) continue;
        if (seen == nnz) parse_error(r.line, "more entries than the size line states (" + std::to_string(nnz) + ")");
        const char* q = b;
        int64_t i = 0, j = 0;
        double v = 0.0;
        if (!read_i64(q, e, i) || !read_i64(q, e, j)) parse_error(r.line, "malformed entry indices");
        if (!read_f64(q, e, v) || !blank(q, e)) parse_error(r.line, "malformed entry value");
        if (i < 1 || i > nrows || j < 1 || j > ncols)
          parse_error(r.line, "index (" + std::to_string(i) + ", " + std::to_string(j) + ") out of bounds for " +
                                  std::to_string(nrows) + "x" + std::to_string(ncols));
        if (sym && j > i) parse_error(r.line, "symmetric file has an entry above the diagonal");
        ri.push_back(i - 1);
        cj.push_back(j - 1);
        vv.push_back(v);
        if (sym && i != j) {
          ri.push_back(j - 1);
          cj.push_back(i - 1);
          vv.push_back(v);
        }
        ++seen;
      }
      if (seen != nnz)
        parse_error(r.line, "file ends after " + std::to_string(seen) + " of " + std::to_string(nnz) + " entries");
      // from_triplets (csr.cpp:26-57): stable order by (row, col), duplicates summed in input order
      std::vector<int64_t> cnt(static_cast<size_t>(nrows) + 1, 0);
      for (int64_t x : ri) ++cnt[static_cast<size_t>(x) + 1];
      for (int64_t x = 0; x < nrows; ++x) cnt[x + 1] += cnt[x];
      std::vector<size_t> order(ri.size());
      {
        std::vector<int64_t> at(cnt.begin(), cnt.end() - 1);
        for (size_t k = 0; k < ri.size(); ++k) order[static_cast<size_t>(at[ri[k]]++)] = k;  // stable by row
      }
      std::vector<int64_t> rp(static_cast<size_t>(nrows) + 1, 0), ci;
      std::vector<double> val;
      ci.reserve(ri.size());
      val.reserve(ri.size());
      for (int64_t row = 0; row < nrows; ++row) {
        auto first = order.begin() + cnt[row], last = order.begin() + cnt[row + 1];
        std::stable_sort(first, last, [&](size_t a, size_t c) { return cj[a] < cj[c]; });
        int64_t cur = -1;
        for (auto it = first; it != last; ++it) {
          if (cj[*it] == cur) {
            val.back() += vv[*it];
          } else {
            cur = cj[*it];
            ci.push_back(cur);
            val.push_back(vv[*it]);
          }
        }
        rp[row + 1] = static_cast<int64_t>(ci.size());
      }
      out->nrows = nrows;
      out->ncols = ncols;
      out->row_ptr = host_copy(rp);
      out->col_idx = host_copy(ci);
      out->values = host_copy(val);
    }
  });
}

int sait_mm_write(const char* path, const sait_host_csr* m) {
  return guard([&] {
    if (!path || !m) throw MmError(SAIT_ERR_INVALID_ARGUMENT, "mm_write: null argument");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw MmError(SAIT_ERR_INVALID_ARGUMENT, std::string("mm_write: cannot open ") + path);
    const int64_t nnz = m->row_ptr[m->nrows];
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%lld %lld %lld\n", static_cast<long long>(m->nrows), static_cast<long long>(m->ncols),
                 static_cast<long long>(nnz));
    char line[96];
    for (int64_t i = 0; i < m->nrows; ++i)
      for (int64_t q = m->row_ptr[i]; q < m->row_ptr[i + 1]; ++q) {
        const double v = m->values ? m->values[q] : 1.0;
        const int len = std::snprintf(line, sizeof line, "%lld %lld %.17g\n", static_cast<long long>(i + 1),
                                      static_cast<long long>(m->col_idx[q] + 1), v);
        std::fwrite(line, 1, static_cast<size_t>(len), f);
      }
    if (std::fclose(f) != 0) throw MmError(SAIT_ERR_RUNTIME, std::string("mm_write: write error on ") + path);
  });
}

// mode 0 = ones-solution b = A * 1 (row sums in stored
// order); mode 1 = seeded random unit vector: x = uniform_pm1(seed), b = x /
// sqrt(sum x_i^2) (sum in index order).
int sait_make_rhs(const sait_host_csr* a, int mode, uint64_t seed, double* out) {
  return guard([&] {
    if (!a || !out) throw MmError(SAIT_ERR_INVALID_ARGUMENT, "make_rhs: null argument");
    if (a->nrows != a->ncols) throw MmError(SAIT_ERR_INVALID_ARGUMENT, "make_rhs: matrix is not square");
    const int64_t n = a->nrows;
    if (mode == 0) {
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t q = a->row_ptr[i]; q < a->row_ptr[i + 1]; ++q) s += a->values[q] * 1.0;
        out[i] = s;
      }
    } else if (mode == 1) {
      sait_fill_uniform_pm1(seed, n, out);
      double ss = 0.0;
      for (int64_t i = 0; i < n; ++i) ss += out[i] * out[i];
      const double nrm = std::sqrt(ss);
      if (nrm > 0.0)
        for (int64_t i = 0; i < n; ++i) out[i] /= nrm;
    } else {
      throw MmError(SAIT_ERR_INVALID_ARGUMENT, "make_rhs: mode must be 0 (ones-solution) or 1 (seeded-random)");
    }
  });
}

}  // extern "C"
