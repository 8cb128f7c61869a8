// C++ drop-in for the reference's SpMM-like API (namespace spmm), running on the
// B200 through the C ABI in gespmm.h.  A reference user swaps
//     #include <spmm/spmm.hpp>            (reference proj/include/spmm/spmm.hpp)
// for
//     #include <gespmm/native_spmm.hpp>
// and links -lgespmm; the calls below keep the reference's names, argument
// meaning and spmm::Error texts.  Header-only; nothing here computes — every
// product goes through gespmm_spmm_host (the sm_100a kernels).
//
// Mirrored interfaces (under /root/reference/proj/include/spmm/):
//   Error                        common.hpp:17-21
//   CsrMatrix                    csr.hpp:22-35
//   DenseMatrix, make_random_dense, checksum   dense.hpp:14-72
//   ReduceOp, ops::sum/max, reduce_op_by_name   reduce_op.hpp:14-36 (+ mean, min)
//   KernelVariant, select_variant                kernel.hpp:44-98 (+ tuned)
//   FaultMode, ExecOptions                       kernel.hpp:167-186
//   native_spmm, ThroughputReport, bench         native.hpp:101-180
//   GraphGenSpec, gen_uniform_random, randomize_values  generate.hpp:14-80
//   CooEntry, CooEntries, DedupPolicy, from_coo, to_coo  csr.hpp:37-104
//   ValidationReport, validate, require_canonical        csr.hpp:107-158
//   KernelConfig, kMaxWarpSize, check_config             kernel.hpp:33, 77-92
//   MmParseError, parse_matrix_market, write_matrix_market  matrix_market.hpp:17-180
//   write_csr_cache, read_csr_cache, save_csr_cache, load_matrix  io.hpp:15-115
// Differences a reference user meets: ReduceOp::combine must be one of the
// built-in ops:: functions (the combine is fused into the device kernel, so
// a custom function pointer throws spmm::Error); mean and min are added;
// run_kernel (the SIMT simulator) and dense_reference (the brute-force
// oracle) are test instruments of the reference and are not offered here.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <istream>
#include <iterator>
#include <limits>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gespmm/gespmm.h"

namespace spmm {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what, gespmm_status_t st = GESPMM_EINVAL)
      : std::runtime_error(what), status(st) {}
  gespmm_status_t status;
};

namespace detail {
inline void check(gespmm_status_t st) {
  if (st != GESPMM_OK) throw Error(gespmm_last_error(), st);
}
}  // namespace detail

struct CsrMatrix {
  u32 n_rows = 0;
  u32 n_cols = 0;
  std::vector<u32> row_ptr;
  std::vector<u32> col_ind;
  std::vector<float> vals;

  CsrMatrix() : row_ptr(1, 0) {}
  CsrMatrix(u32 rows, u32 cols) : n_rows(rows), n_cols(cols), row_ptr(size_t(rows) + 1, 0) {}
  u32 nnz() const { return u32(col_ind.size()); }
  u32 row_len(u32 r) const { return row_ptr[r + 1] - row_ptr[r]; }
  double mean_degree() const { return n_rows ? double(nnz()) / n_rows : 0.0; }
};

struct DenseMatrix {
  u32 n_rows = 0;
  u32 n_cols = 0;
  std::vector<float> data;
  u32 base_alignment = 128;

  DenseMatrix() = default;
  DenseMatrix(u32 rows, u32 cols, float fill = 0.0f)
      : n_rows(rows), n_cols(cols), data(size_t(rows) * cols, fill) {}
  float& at(u32 r, u32 c) { return data[size_t(r) * n_cols + c]; }
  float at(u32 r, u32 c) const { return data[size_t(r) * n_cols + c]; }
  size_t size() const { return data.size(); }
  bool same_shape(const DenseMatrix& o) const { return n_rows == o.n_rows && n_cols == o.n_cols; }
  bool bitwise_equal(const DenseMatrix& o) const {
    return same_shape(o) &&
           (data.empty() || std::memcmp(data.data(), o.data.data(), data.size() * 4) == 0);
  }
};

inline void check_dense_valid(const DenseMatrix& m) {
  if (m.data.size() != size_t(m.n_rows) * m.n_cols)
    throw Error("dense matrix: data length does not match n_rows * n_cols");
  const u32 a = m.base_alignment;
  if (a == 0 || (a & (a - 1)) != 0 || a > 4096)
    throw Error("dense matrix: base_alignment must be a power of two <= 4096");
}

// reduce_op.hpp:14-36.  `combine` keeps the reference's function-pointer
// field; the device kernel fuses the combine, so only the built-in ops::
// functions are accepted (detail::reduce_code maps them to the ABI enum and
// throws for any other pointer).  `fold` is the host statement of the combine.
struct ReduceOp {
  std::string name;
  float init = 0.0f;
  float (*combine)(float, float) = nullptr;

  float fold(float acc, float x) const { return combine(acc, x); }
};

namespace ops {
inline float add_f32(float a, float b) { return a + b; }
inline float max_f32(float a, float b) { return a < b ? b : a; }
inline float min_f32(float a, float b) { return b < a ? b : a; }

inline ReduceOp sum() { return {"sum", 0.0f, &add_f32}; }
inline ReduceOp max() { return {"max", std::numeric_limits<float>::lowest(), &max_f32}; }
// mean folds like sum; the kernel divides by the row length at the end
inline ReduceOp mean() { return {"mean", 0.0f, &add_f32}; }
inline ReduceOp min() { return {"min", std::numeric_limits<float>::max(), &min_f32}; }
}  // namespace ops

namespace detail {
inline gespmm_reduce_t reduce_code(const ReduceOp& op) {
  if (op.combine == &ops::add_f32) return op.name == "mean" ? GESPMM_MEAN : GESPMM_SUM;
  if (op.combine == &ops::max_f32) return GESPMM_MAX;
  if (op.combine == &ops::min_f32) return GESPMM_MIN;
  throw Error("reduce op '" + op.name +
              "': the combine runs fused in the device kernel; only ops::add_f32 (sum, mean), "
              "ops::max_f32 and ops::min_f32 are supported");
}
}  // namespace detail

inline ReduceOp reduce_op_by_name(const std::string& name) {
  gespmm_reduce_t code;
  detail::check(gespmm_reduce_by_name(name.c_str(), &code));
  switch (code) {
    case GESPMM_SUM: return ops::sum();
    case GESPMM_MEAN: return ops::mean();
    case GESPMM_MAX: return ops::max();
    default: return ops::min();
  }
}

enum class KernelKind : u8 { Naive, Crc, CrcCwm, Tuned };

struct KernelVariant {
  KernelKind kind = KernelKind::Naive;
  u32 cf = 1;
  static KernelVariant naive() { return {KernelKind::Naive, 1}; }
  static KernelVariant crc() { return {KernelKind::Crc, 1}; }
  static KernelVariant crc_cwm(u32 cf) { return {KernelKind::CrcCwm, cf}; }
  static KernelVariant tuned() { return {KernelKind::Tuned, 1}; }
  u32 cf_effective() const { return kind == KernelKind::CrcCwm ? cf : 1; }
  std::string name() const {
    switch (kind) {
      case KernelKind::Naive: return "naive";
      case KernelKind::Crc: return "crc";
      case KernelKind::CrcCwm: return "crc-cwm";
      case KernelKind::Tuned: return "tuned";
    }
    return "?";
  }
  bool operator==(const KernelVariant&) const = default;
  gespmm_variant_t abi() const {
    switch (kind) {
      case KernelKind::Naive: return GESPMM_VARIANT_NAIVE;
      case KernelKind::Crc: return GESPMM_VARIANT_CRC;
      case KernelKind::CrcCwm: return GESPMM_VARIANT_CRC_CWM;
      default: return GESPMM_VARIANT_TUNED;
    }
  }
};

inline KernelVariant variant_by_name(const std::string& name, u32 cf = 2) {
  if (name == "naive") return KernelVariant::naive();
  if (name == "crc") return KernelVariant::crc();
  if (name == "crc-cwm") return KernelVariant::crc_cwm(cf);
  if (name == "tuned") return KernelVariant::tuned();
  throw Error("unknown kernel variant '" + name + "' (naive, crc, crc-cwm, tuned)");
}

// The reference's rule (N <= 32 -> crc, else crc-cwm(2)); tuned() is the B200 choice.
inline KernelVariant select_variant(u32 n) {
  int32_t v;
  u32 cf;
  gespmm_select_variant(n, &v, &cf);
  return v == GESPMM_VARIANT_CRC ? KernelVariant::crc() : KernelVariant::crc_cwm(cf);
}

// kernel.hpp:33, 77-92: the launch shape of the paper's kernels (warp size,
// warps per block, variant).  The device runs 32-lane warps; the config is
// checked with the reference's rules and messages.
inline constexpr u32 kMaxWarpSize = 64;

struct KernelConfig {
  u32 warp_size = 32;
  u32 warps_per_block = 8;
  KernelVariant variant = KernelVariant::naive();
};

inline void check_config(const KernelConfig& cfg) {
  const u32 ws = cfg.warp_size;
  if (ws < 4 || ws > kMaxWarpSize || (ws & (ws - 1)) != 0)
    throw Error("warp_size must be a power of two in [4, " + std::to_string(kMaxWarpSize) + "]");
  if (cfg.warps_per_block < 1) throw Error("warps_per_block must be >= 1");
  if (cfg.variant.kind == KernelKind::CrcCwm && cfg.variant.cf != 2 && cfg.variant.cf != 4 &&
      cfg.variant.cf != 8)
    throw Error("coarsening factor must be 2, 4 or 8");
}

enum class FaultMode : u8 { None, SkipTail };

struct ExecOptions {
  FaultMode fault = FaultMode::None;
  bool exact = true;
  gespmm_arg_kind_t arg_kind = GESPMM_ARG_EDGE;
  int32_t hub_threshold = 0;
};

namespace detail {
inline void precheck(const CsrMatrix& a, const DenseMatrix& b) {
  check_dense_valid(b);
  if (a.n_cols != b.n_rows)
    throw Error("spmm: dimension mismatch: A is " + std::to_string(a.n_rows) + "x" +
                    std::to_string(a.n_cols) + " but B has " + std::to_string(b.n_rows) + " rows",
                GESPMM_EDIM);
  const std::string pre = "spmm: matrix is not canonical CSR: ";
  if (a.row_ptr.size() != size_t(a.n_rows) + 1)
    throw Error(pre + "row_ptr length is " + std::to_string(a.row_ptr.size()) +
                    ", expected n_rows+1 = " + std::to_string(a.n_rows + 1),
                GESPMM_ENONCANON);
  if (a.col_ind.size() != a.vals.size())
    throw Error(pre + "col_ind length " + std::to_string(a.col_ind.size()) + " != vals length " +
                    std::to_string(a.vals.size()),
                GESPMM_ENONCANON);
}

inline DenseMatrix run(const CsrMatrix& a, const DenseMatrix& b, KernelVariant v,
                       const ReduceOp& op, const ExecOptions& ex, std::vector<int32_t>* arg) {
  precheck(a, b);
  gespmm_options_t o;
  gespmm_options_default(&o);
  o.variant = v.abi();
  o.cf = v.kind == KernelKind::CrcCwm ? v.cf : 2;
  o.exact = ex.exact ? 1 : 0;
  o.arg_kind = ex.arg_kind;
  o.fault_skip_tail = ex.fault == FaultMode::SkipTail;
  o.hub_threshold = ex.hub_threshold;
  o.validate = 1;
  const gespmm_csr_t csr{a.n_rows, a.n_cols, a.col_ind.size(), a.row_ptr.data(),
                         a.col_ind.data(), a.vals.data()};
  DenseMatrix c(a.n_rows, b.n_cols);
  if (arg) arg->assign(c.data.size(), -1);
  check(gespmm_spmm_host(&csr, b.data.data(), b.n_rows, b.n_cols, reduce_code(op), c.data.data(),
                         arg ? arg->data() : nullptr, &o));
  return c;
}
}  // namespace detail

// native.hpp:101-102.  `workers` is accepted for source compatibility.
inline DenseMatrix native_spmm(const CsrMatrix& a, const DenseMatrix& b, KernelVariant variant,
                               const ReduceOp& op, u32 workers = 0, ExecOptions exec = {}) {
  (void)workers;
  return detail::run(a, b, variant, op, exec, nullptr);
}

// SpMM-like max/min pooling with argmax/argmin (-1 where the seed survived).
inline std::pair<DenseMatrix, std::vector<int32_t>> native_spmm_arg(
    const CsrMatrix& a, const DenseMatrix& b, KernelVariant variant, const ReduceOp& op,
    ExecOptions exec = {}) {
  std::vector<int32_t> arg;
  DenseMatrix c = detail::run(a, b, variant, op, exec, &arg);
  return {std::move(c), std::move(arg)};
}

struct ThroughputReport {
  double elapsed_s = 0.0;
  double elapsed_mean_s = 0.0;
  u32 repeats = 0;
  u64 flops = 0;
  double gflops = 0.0;
  u64 output_checksum = 0;
};

inline u64 checksum(const DenseMatrix& m) {
  return gespmm_checksum(m.data.data(), m.n_rows, m.n_cols);
}

// native.hpp:156-180: median of `repeats` native_spmm wall times.
inline ThroughputReport bench(const CsrMatrix& a, const DenseMatrix& b, KernelVariant variant,
                              const ReduceOp& op, u32 workers = 0, u32 repeats = 9) {
  if (repeats < 1) throw Error("bench: repeats must be >= 1");
  ThroughputReport rep;
  rep.repeats = repeats;
  rep.flops = 2ull * a.nnz() * b.n_cols;
  std::vector<double> t;
  for (u32 r = 0; r < repeats; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    DenseMatrix c = native_spmm(a, b, variant, op, workers);
    t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    rep.output_checksum = checksum(c);
  }
  std::sort(t.begin(), t.end());
  rep.elapsed_s = t[(t.size() - 1) / 2];
  double s = 0;
  for (double x : t) s += x;
  rep.elapsed_mean_s = s / double(t.size());
  rep.gflops = rep.elapsed_s > 0 ? double(rep.flops) / rep.elapsed_s / 1e9 : 0.0;
  return rep;
}

inline DenseMatrix make_random_dense(u32 rows, u32 cols, u64 seed) {
  DenseMatrix m(rows, cols);
  if (!m.data.empty()) gespmm_make_random_dense(rows, cols, seed, m.data.data());
  return m;
}

inline void randomize_values(CsrMatrix& m, u64 seed) {
  if (!m.vals.empty()) gespmm_randomize_values(m.vals.data(), m.vals.size(), seed);
}

struct GraphGenSpec {
  u32 n_rows = 0;
  u64 nnz_target = 0;
  u64 seed = 0;
  bool self_loops = false;
};

inline CsrMatrix gen_uniform_random(const GraphGenSpec& spec) {
  CsrMatrix m(spec.n_rows, spec.n_rows);
  m.col_ind.resize(spec.nnz_target);
  m.vals.resize(spec.nnz_target);
  detail::check(gespmm_gen_uniform(spec.n_rows, spec.nnz_target, spec.seed, spec.self_loops,
                                   m.row_ptr.data(), m.col_ind.data(), m.vals.data()));
  return m;
}

// New: power-law (Chung-Lu style) generator for the Reddit/products shapes.
inline CsrMatrix gen_powerlaw(u32 rows, u64 nnz_target, u32 max_degree, double exponent,
                              u64 seed) {
  CsrMatrix m(rows, rows);
  detail::check(gespmm_gen_powerlaw(rows, nnz_target, max_degree, exponent, seed, 0,
                                    m.row_ptr.data(), nullptr, nullptr));
  m.col_ind.resize(m.row_ptr[rows]);
  m.vals.resize(m.row_ptr[rows]);
  detail::check(gespmm_gen_powerlaw(rows, nnz_target, max_degree, exponent, seed, 0,
                                    m.row_ptr.data(), m.col_ind.data(), m.vals.data()));
  return m;
}

// ---------------------------------------------------------------------------
// Data model: COO ingestion and the canonical-CSR report (csr.hpp:37-158),
// computed by the library (gespmm_from_coo / gespmm_validate_host).
// ---------------------------------------------------------------------------

struct CooEntry {
  u32 row = 0;
  u32 col = 0;
  float val = 0.0f;
  bool operator==(const CooEntry&) const = default;
};

struct CooEntries {
  u32 n_rows = 0;
  u32 n_cols = 0;
  std::vector<CooEntry> entries;
};

enum class DedupPolicy { Sum, Last };

inline CsrMatrix from_coo(const CooEntries& coo, DedupPolicy policy = DedupPolicy::Sum) {
  const size_t n = coo.entries.size();
  std::vector<u32> r(n), c(n);
  std::vector<float> v(n);
  for (size_t i = 0; i < n; ++i) {
    r[i] = coo.entries[i].row;
    c[i] = coo.entries[i].col;
    v[i] = coo.entries[i].val;
  }
  CsrMatrix m(coo.n_rows, coo.n_cols);
  m.col_ind.resize(n);
  m.vals.resize(n);
  u64 nnz = 0;
  detail::check(gespmm_from_coo(coo.n_rows, coo.n_cols, n, r.data(), c.data(), v.data(),
                                policy == DedupPolicy::Sum ? GESPMM_DEDUP_SUM : GESPMM_DEDUP_LAST,
                                m.row_ptr.data(), m.col_ind.data(), m.vals.data(), &nnz));
  m.col_ind.resize(nnz);
  m.vals.resize(nnz);
  return m;
}

inline CooEntries to_coo(const CsrMatrix& m) {
  CooEntries coo{m.n_rows, m.n_cols, {}};
  coo.entries.reserve(m.nnz());
  for (u32 r = 0; r < m.n_rows; ++r)
    for (u32 p = m.row_ptr[r]; p < m.row_ptr[r + 1]; ++p)
      coo.entries.push_back({r, m.col_ind[p], m.vals[p]});
  return coo;
}

struct ValidationReport {
  std::vector<std::string> violations;
  bool ok() const { return violations.empty(); }
};

inline ValidationReport validate(const CsrMatrix& m) {
  const gespmm_csr_t csr{m.n_rows, m.n_cols, m.col_ind.size(),
                         m.row_ptr.empty() ? nullptr : m.row_ptr.data(), m.col_ind.data(),
                         m.vals.data()};
  u64 need = 0;
  ValidationReport rep;
  if (gespmm_validate_host(&csr, m.row_ptr.size(), m.col_ind.size(), m.vals.size(), nullptr, 0,
                           &need) == 0)
    return rep;
  std::string text(need, '\0');
  gespmm_validate_host(&csr, m.row_ptr.size(), m.col_ind.size(), m.vals.size(), text.data(), need,
                       &need);
  text.resize(std::strlen(text.c_str()));
  std::istringstream is(text);
  for (std::string line; std::getline(is, line);) rep.violations.push_back(line);
  return rep;
}

inline void require_canonical(const CsrMatrix& m, const char* who) {
  const auto rep = validate(m);
  if (!rep.ok())
    throw Error(std::string(who) + ": matrix is not canonical CSR: " + rep.violations.front(),
                GESPMM_ENONCANON);
}

// ---------------------------------------------------------------------------
// File formats (matrix_market.hpp, io.hpp): parsing in the library
// (gespmm_mtx_parse, gespmm_csr1_*), streams and paths here.
// ---------------------------------------------------------------------------

class MmParseError : public Error {
 public:
  MmParseError(size_t line, const std::string& what)
      : Error("matrix market: line " + std::to_string(line) + ": " + what), line_(line) {}
  size_t line() const { return line_; }

 private:
  explicit MmParseError(const std::string& full, size_t line) : Error(full), line_(line) {}
  size_t line_;
  friend CooEntries parse_matrix_market(const std::string& text);
};

inline CooEntries parse_matrix_market(const std::string& text) {
  u32 rows = 0, cols = 0;
  u64 k = 0;
  auto fail = [] {
    const std::string msg = gespmm_last_error();
    const std::string pre = "matrix market: line ";
    size_t line = 0;
    if (msg.rfind(pre, 0) == 0) line = std::strtoull(msg.c_str() + pre.size(), nullptr, 10);
    throw MmParseError(msg, line);
  };
  if (gespmm_mtx_parse(text.data(), text.size(), &rows, &cols, &k, nullptr, nullptr, nullptr) !=
      GESPMM_OK)
    fail();
  std::vector<u32> r(k), c(k);
  std::vector<float> v(k);
  if (gespmm_mtx_parse(text.data(), text.size(), &rows, &cols, &k, r.data(), c.data(),
                       v.data()) != GESPMM_OK)
    fail();
  CooEntries coo{rows, cols, {}};
  coo.entries.reserve(k);
  for (u64 i = 0; i < k; ++i) coo.entries.push_back({r[i], c[i], v[i]});
  return coo;
}

inline CooEntries parse_matrix_market(std::istream& in) {
  return parse_matrix_market(
      std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()));
}

inline void write_matrix_market(std::ostream& out, const CooEntries& coo) {
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << coo.n_rows << " " << coo.n_cols << " " << coo.entries.size() << "\n";
  char buf[64];
  for (const auto& e : coo.entries) {
    std::snprintf(buf, sizeof(buf), "%u %u %.9g\n", e.row + 1, e.col + 1, double(e.val));
    out << buf;
  }
}

inline void write_matrix_market(std::ostream& out, const CsrMatrix& m) {
  write_matrix_market(out, to_coo(m));
}

// CSR1: "CSR1", u64 LE n_rows, n_cols, nnz, u32 row_ptr, u32 col_ind, f32 vals.
inline void write_csr_cache(std::ostream& out, const CsrMatrix& m) {
  auto put = [&](u64 v, int bytes) {
    char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = char((v >> (8 * i)) & 0xff);
    out.write(b, bytes);
  };
  out.write("CSR1", 4);
  put(m.n_rows, 8);
  put(m.n_cols, 8);
  put(m.nnz(), 8);
  for (u32 x : m.row_ptr) put(x, 4);
  for (u32 x : m.col_ind) put(x, 4);
  for (float f : m.vals) {
    u32 bits;
    std::memcpy(&bits, &f, 4);
    put(bits, 4);
  }
  if (!out) throw Error("csr cache: write failed");
}

inline void save_csr_cache(const std::filesystem::path& path, const CsrMatrix& m) {
  const gespmm_csr_t csr{m.n_rows, m.n_cols, m.col_ind.size(), m.row_ptr.data(),
                         m.col_ind.data(), m.vals.data()};
  detail::check(gespmm_csr1_write(path.c_str(), &csr));
}

namespace detail {
inline CsrMatrix read_csr1_file(const std::filesystem::path& path) {
  u32 rows = 0, cols = 0;
  u64 nnz = 0;
  check(gespmm_csr1_header(path.c_str(), &rows, &cols, &nnz));
  CsrMatrix m(rows, cols);
  m.col_ind.resize(nnz);
  m.vals.resize(nnz);
  check(gespmm_csr1_read_host(path.c_str(), m.row_ptr.data(), m.col_ind.data(), m.vals.data()));
  return m;
}
}  // namespace detail

// io.hpp:65-90 (no canonical check, as the reference); the same checks and
// messages as the library's file reader
inline CsrMatrix read_csr_cache(std::istream& in) {
  auto get = [&](u64& v, int bytes) {
    unsigned char b[8];
    if (!in.read(reinterpret_cast<char*>(b), bytes)) return false;
    v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
    return true;
  };
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, "CSR1", 4) != 0)
    throw Error("csr cache: bad magic (expected CSR1)");
  u64 rows, cols, nnz;
  if (!get(rows, 8) || !get(cols, 8) || !get(nnz, 8)) throw Error("csr cache: truncated header");
  if (rows > 0xffffffffull || cols > 0xffffffffull || nnz > 0xffffffffull)
    throw Error("csr cache: dimensions exceed 32-bit range");
  CsrMatrix m(static_cast<u32>(rows), static_cast<u32>(cols));
  m.col_ind.resize(nnz);
  m.vals.resize(nnz);
  u64 x;
  for (auto& v : m.row_ptr) {
    if (!get(x, 4)) throw Error("csr cache: truncated row_ptr");
    v = u32(x);
  }
  for (auto& v : m.col_ind) {
    if (!get(x, 4)) throw Error("csr cache: truncated col_ind");
    v = u32(x);
  }
  for (auto& f : m.vals) {
    if (!get(x, 4)) throw Error("csr cache: truncated vals");
    const u32 bits = u32(x);
    std::memcpy(&f, &bits, 4);
  }
  return m;
}

// io.hpp:100-115: .mtx (Matrix Market, duplicates summed) or .csr, then the
// canonical check with the reference's "load_matrix: ..." wording.
inline CsrMatrix load_matrix(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error("cannot open '" + path.string() + "'");
  const auto ext = path.extension().string();
  CsrMatrix m;
  if (ext == ".mtx") {
    m = from_coo(parse_matrix_market(in), DedupPolicy::Sum);
  } else if (ext == ".csr") {
    in.close();
    m = detail::read_csr1_file(path);
  } else {
    throw Error("unknown matrix extension '" + ext + "' (expected .mtx or .csr)");
  }
  require_canonical(m, "load_matrix");
  return m;
}

}  // namespace spmm
