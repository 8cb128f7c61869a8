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
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
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

// The combine is fused into the device kernel by name; `fold` is the host
// statement of it (used by the reduce-op law tests).
struct ReduceOp {
  std::string name;
  float init = 0.0f;
  gespmm_reduce_t code = GESPMM_SUM;
  float fold(float acc, float x) const {
    switch (code) {
      case GESPMM_MAX: return acc < x ? x : acc;
      case GESPMM_MIN: return x < acc ? x : acc;
      default: return acc + x;
    }
  }
};

namespace ops {
inline ReduceOp sum() { return {"sum", 0.0f, GESPMM_SUM}; }
inline ReduceOp max() { return {"max", std::numeric_limits<float>::lowest(), GESPMM_MAX}; }
inline ReduceOp mean() { return {"mean", 0.0f, GESPMM_MEAN}; }
inline ReduceOp min() { return {"min", std::numeric_limits<float>::max(), GESPMM_MIN}; }
}  // namespace ops

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
  check(gespmm_spmm_host(&csr, b.data.data(), b.n_rows, b.n_cols, op.code, c.data.data(),
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

}  // namespace spmm
