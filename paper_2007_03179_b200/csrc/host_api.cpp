// Host-side data-model entry points of the C ABI (gespmm.h): COO -> canonical
// CSR, the full canonical-CSR report, and the Matrix Market reader.  These sit
// on either side of the SpMM (ingestion), run once per matrix, and carry the
// reference's semantics and error texts so the C++ drop-in
// (include/gespmm/native_spmm.hpp) can offer the reference's functions:
//   from_coo / DedupPolicy    proj/include/spmm/csr.hpp:37-93
//   validate (all violations) proj/include/spmm/csr.hpp:107-153
//   parse_matrix_market       proj/include/spmm/matrix_market.hpp:60-160
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "gespmm/gespmm.h"
#include "launch.h"

using namespace gespmm;

namespace {

// ---- validate: every violation, in the reference's order and wording -------

struct Report {
  std::string text;  // violations separated by '\n'
  uint64_t count = 0;
  void add(const std::string& s) {
    if (count) text += '\n';
    text += s;
    ++count;
  }
};

void collect(const gespmm_csr_t& a, uint64_t rp_len, uint64_t ci_len, uint64_t v_len,
             Report& rep) {
  if (rp_len != uint64_t(a.n_rows) + 1) {
    rep.add("row_ptr length is " + std::to_string(rp_len) + ", expected n_rows+1 = " +
            std::to_string(uint64_t(a.n_rows) + 1));
    return;  // offsets unusable
  }
  if (ci_len != v_len)
    rep.add("col_ind length " + std::to_string(ci_len) + " != vals length " +
            std::to_string(v_len));
  const uint32_t* rp = a.row_ptr;
  if (rp[0] != 0) rep.add("row_ptr[0] = " + std::to_string(rp[0]) + ", expected 0");
  for (uint64_t i = 1; i < rp_len; ++i)
    if (rp[i] < rp[i - 1]) {
      rep.add("row_ptr non-decreasing violated at index " + std::to_string(i));
      return;
    }
  if (uint64_t(rp[a.n_rows]) != ci_len)
    rep.add("row_ptr[n_rows] = " + std::to_string(rp[a.n_rows]) + " != nnz = " +
            std::to_string(ci_len));
  // u32 positions, as the reference's CsrMatrix (nnz() is a u32)
  const uint32_t usable = uint32_t(std::min<uint64_t>(rp[a.n_rows], ci_len));
  for (uint32_t r = 0; r < a.n_rows; ++r) {
    const uint32_t lo = rp[r], hi = std::min(rp[r + 1], usable);
    for (uint32_t p = lo; p < hi; ++p) {
      const uint32_t c = a.col_ind[p];
      if (c >= a.n_cols)
        rep.add("col_ind[" + std::to_string(p) + "] = " + std::to_string(c) +
                " out of bounds (n_cols = " + std::to_string(a.n_cols) + ")");
      if (p > lo && c <= a.col_ind[p - 1])
        rep.add("columns not strictly increasing in row " + std::to_string(r) +
                " at position " + std::to_string(p));
    }
  }
}

// ---- Matrix Market ----------------------------------------------------------

struct MmError {
  uint64_t line;
  std::string what;
};

struct LineReader {
  const char* p;
  const char* end;
  uint64_t lineno = 0;
  bool next(std::string& out) {
    if (p >= end) return false;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
    const char* e = nl ? nl : end;
    out.assign(p, e);
    p = nl ? nl + 1 : end;
    ++lineno;
    if (!out.empty() && out.back() == '\r') out.pop_back();
    return true;
  }
};

std::vector<std::string> tokens(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string t;
  while (is >> t) out.push_back(t);
  return out;
}

bool to_u64(const std::string& s, uint64_t& v) {
  auto [q, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  return ec == std::errc() && q == s.data() + s.size();
}

bool to_f64(const std::string& s, double& v) {
  if (s.empty()) return false;
  char* e = nullptr;
  v = std::strtod(s.c_str(), &e);
  return e == s.c_str() + s.size();
}

struct MmHeader {
  uint64_t rows = 0, cols = 0, declared = 0;
  bool pattern = false, symmetric = false;
};

// Header and size line (matrix_market.hpp:67-110 semantics).
MmHeader read_header(LineReader& in) {
  std::string line;
  if (!in.next(line)) throw MmError{1, "empty input"};
  std::string low = line;
  for (auto& ch : low) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  const auto h = tokens(low);
  if (h.size() < 2 || h[0] != "%%matrixmarket" || h[1] != "matrix")
    throw MmError{in.lineno, "expected header '%%MatrixMarket matrix coordinate ...'"};
  if (h.size() < 3 || h[2] != "coordinate") {
    if (h.size() >= 3 && h[2] == "array")
      throw MmError{in.lineno, "'array' (dense) files are not supported, only 'coordinate'"};
    throw MmError{in.lineno, "expected 'coordinate' format in header"};
  }
  const std::string field = h.size() > 3 ? h[3] : "real";
  const std::string sym = h.size() > 4 ? h[4] : "general";
  if (field != "real" && field != "integer" && field != "pattern")
    throw MmError{in.lineno, "unsupported field '" + field + "' (want real, integer or pattern)"};
  if (sym != "general" && sym != "symmetric")
    throw MmError{in.lineno, "unsupported symmetry '" + sym + "' (want general or symmetric)"};
  MmHeader hd;
  hd.pattern = field == "pattern";
  hd.symmetric = sym == "symmetric";
  for (;;) {
    if (!in.next(line)) throw MmError{in.lineno + 1, "missing size line"};
    if (line.empty() || line[0] == '%') continue;
    const auto t = tokens(line);
    if (t.size() != 3 || !to_u64(t[0], hd.rows) || !to_u64(t[1], hd.cols) ||
        !to_u64(t[2], hd.declared))
      throw MmError{in.lineno, "size line must be '<rows> <cols> <nnz>'"};
    break;
  }
  if (hd.rows > 0xffffffffull || hd.cols > 0xffffffffull)
    throw MmError{in.lineno, "dimensions exceed 32-bit index range"};
  return hd;
}

// Entry lines; sink(r, c, v) per stored triple (mirrored for symmetric).
template <class Sink>
void read_entries(LineReader& in, const MmHeader& hd, Sink&& sink) {
  std::string line;
  uint64_t seen = 0;
  const size_t want = hd.pattern ? 2 : 3;
  while (seen < hd.declared) {
    if (!in.next(line))
      throw MmError{in.lineno + 1, "unexpected end of file: got " + std::to_string(seen) +
                                       " of " + std::to_string(hd.declared) + " entries"};
    if (line.empty() || line[0] == '%') continue;
    const auto t = tokens(line);
    if (t.size() != want)
      throw MmError{in.lineno, "expected " + std::to_string(want) + " fields, got " +
                                   std::to_string(t.size())};
    uint64_t r1 = 0, c1 = 0;
    if (!to_u64(t[0], r1) || !to_u64(t[1], c1)) throw MmError{in.lineno, "non-numeric index"};
    double v = 1.0;
    if (!hd.pattern && !to_f64(t[2], v)) throw MmError{in.lineno, "non-numeric value"};
    if (r1 < 1 || r1 > hd.rows || c1 < 1 || c1 > hd.cols)
      throw MmError{in.lineno, "index (" + t[0] + ", " + t[1] + ") outside declared " +
                                   std::to_string(hd.rows) + "x" + std::to_string(hd.cols)};
    const uint32_t r = uint32_t(r1 - 1), c = uint32_t(c1 - 1);
    sink(r, c, float(v));
    if (hd.symmetric && r != c) sink(c, r, float(v));
    ++seen;
  }
}

gespmm_status_t mm_fail(const MmError& e) {
  return set_error(GESPMM_EINVAL,
                   "matrix market: line " + std::to_string(e.line) + ": " + e.what);
}

}  // namespace

extern "C" {

uint64_t gespmm_validate_host(const gespmm_csr_t* a, uint64_t row_ptr_len, uint64_t col_ind_len,
                              uint64_t vals_len, char* msgs, uint64_t msgs_cap,
                              uint64_t* msgs_needed) {
  if (!a) return 0;
  Report rep;
  // a null row_ptr is a zero-length one (the length check reports it)
  collect(*a, a->row_ptr ? row_ptr_len : 0, col_ind_len, vals_len, rep);
  if (msgs_needed) *msgs_needed = rep.text.size() + 1;
  if (msgs && msgs_cap) {
    const size_t n = std::min<uint64_t>(rep.text.size(), msgs_cap - 1);
    std::memcpy(msgs, rep.text.data(), n);
    msgs[n] = '\0';
  }
  return rep.count;
}

gespmm_status_t gespmm_from_coo(uint32_t n_rows, uint32_t n_cols, uint64_t count,
                                const uint32_t* rows, const uint32_t* cols, const float* vals,
                                int32_t policy, uint32_t* row_ptr, uint32_t* col_ind,
                                float* out_vals, uint64_t* nnz) {
  if (policy != GESPMM_DEDUP_SUM && policy != GESPMM_DEDUP_LAST)
    return set_error(GESPMM_EINVAL, "from_coo: unknown dedup policy");
  if (count && (!rows || !cols || !vals)) return set_error(GESPMM_EINVAL, "from_coo: null input");
  for (uint64_t i = 0; i < count; ++i) {
    if (rows[i] >= n_rows || cols[i] >= n_cols) {
      std::ostringstream os;  // the reference formats the value with operator<<
      os << "coo entry (" << rows[i] << ", " << cols[i] << ", " << vals[i]
         << ") outside declared " << n_rows << "x" << n_cols << " bounds";
      return set_error(GESPMM_EINVAL, os.str());
    }
  }
  // counting sort by row (stable), then a stable sort by column inside each
  // row: input order survives within every duplicate run
  std::vector<uint64_t> start(size_t(n_rows) + 1, 0);
  for (uint64_t i = 0; i < count; ++i) ++start[rows[i] + 1];
  for (uint32_t r = 0; r < n_rows; ++r) start[r + 1] += start[r];
  std::vector<uint64_t> idx(count);
  {
    std::vector<uint64_t> fill(start.begin(), start.end() - 1);
    for (uint64_t i = 0; i < count; ++i) idx[fill[rows[i]]++] = i;
  }
  uint64_t out = 0;
  row_ptr[0] = 0;
  for (uint32_t r = 0; r < n_rows; ++r) {
    auto b = idx.begin() + int64_t(start[r]), e = idx.begin() + int64_t(start[r + 1]);
    std::stable_sort(b, e, [&](uint64_t x, uint64_t y) { return cols[x] < cols[y]; });
    for (auto it = b; it != e;) {
      const uint32_t c = cols[*it];
      float v = vals[*it];
      for (++it; it != e && cols[*it] == c; ++it)
        v = policy == GESPMM_DEDUP_SUM ? v + vals[*it] : vals[*it];
      col_ind[out] = c;
      out_vals[out] = v;
      ++out;
    }
    if (out > 0xffffffffull) return set_error(GESPMM_EINVAL, "from_coo: nnz exceeds 32-bit range");
    row_ptr[r + 1] = uint32_t(out);
  }
  if (nnz) *nnz = out;
  return GESPMM_OK;
}

gespmm_status_t gespmm_mtx_parse(const char* text, uint64_t len, uint32_t* n_rows,
                                 uint32_t* n_cols, uint64_t* n_entries, uint32_t* rows,
                                 uint32_t* cols, float* vals) {
  if (!text && len) return set_error(GESPMM_EINVAL, "matrix market: null input");
  LineReader in{text, text + len};
  try {
    const MmHeader hd = read_header(in);
    *n_rows = uint32_t(hd.rows);
    *n_cols = uint32_t(hd.cols);
    uint64_t k = 0;
    const uint64_t cap = rows ? *n_entries : 0;
    read_entries(in, hd, [&](uint32_t r, uint32_t c, float v) {
      if (rows && k < cap) {
        rows[k] = r;
        cols[k] = c;
        vals[k] = v;
      }
      ++k;
    });
    *n_entries = k;
  } catch (const MmError& e) {
    return mm_fail(e);
  }
  return GESPMM_OK;
}

}  // extern "C"
