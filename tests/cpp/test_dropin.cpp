// C++ drop-in check: the reference's own test cases, written against
// <gespmm/native_spmm.hpp> exactly as a reference user would call them, run on
// the B200 through libgespmm.so.  Cases restate (under /root/reference/proj):
//   tests/test_kernels.cpp:26-166, tests/test_native.cpp:12-106,
//   tests/test_oracle.cpp:20-41, tests/test_reduce_op.cpp:24-46,
//   tests/test_simt.cpp:249-258 (error texts).
// The checker here is a plain ordered fold in this file (test code only).
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "gespmm/native_spmm.hpp"

using namespace spmm;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_fail;                                                          \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)

template <class F>
static std::string error_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.what();
  }
  return "";
}

static CsrMatrix coo(u32 rows, u32 cols, std::vector<std::tuple<u32, u32, float>> e) {
  std::sort(e.begin(), e.end(), [](auto& a, auto& b) {
    return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                            : std::get<1>(a) < std::get<1>(b);
  });
  CsrMatrix m(rows, cols);
  for (auto& [r, c, v] : e) {
    m.col_ind.push_back(c);
    m.vals.push_back(v);
    ++m.row_ptr[r + 1];
  }
  for (u32 r = 0; r < rows; ++r) m.row_ptr[r + 1] += m.row_ptr[r];
  return m;
}

// ordered fold, separate rounding (the contract every variant must meet)
static DenseMatrix fold_ref(const CsrMatrix& a, const DenseMatrix& b, const ReduceOp& op) {
  DenseMatrix c(a.n_rows, b.n_cols, op.init);
  for (u32 i = 0; i < a.n_rows; ++i)
    for (u32 p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p) {
      const float v = a.vals[p];
      for (u32 j = 0; j < b.n_cols; ++j) {
        volatile float x = v * b.at(a.col_ind[p], j);
        c.at(i, j) = op.fold(c.at(i, j), x);
      }
    }
  return c;
}

static const std::vector<KernelVariant> kAll = {
    KernelVariant::naive(),      KernelVariant::crc(),        KernelVariant::crc_cwm(2),
    KernelVariant::crc_cwm(4),   KernelVariant::crc_cwm(8),   KernelVariant::tuned()};

int main() {
  // identity reproduces B on every variant
  {
    const CsrMatrix a = coo(3, 3, {{0, 0, 1.f}, {1, 1, 1.f}, {2, 2, 1.f}});
    const DenseMatrix b = make_random_dense(3, 4, 11);
    for (auto& v : kAll) CHECK(native_spmm(a, b, v, ops::sum(), 3).bitwise_equal(b));
  }
  // single-row and hand cases
  {
    const CsrMatrix a = coo(1, 2, {{0, 0, 2.f}, {0, 1, 3.f}});
    DenseMatrix b(2, 2);
    b.at(0, 0) = b.at(1, 1) = 1.f;
    const DenseMatrix c = native_spmm(a, b, KernelVariant::naive(), ops::sum());
    CHECK(c.at(0, 0) == 2.f && c.at(0, 1) == 3.f);
    const CsrMatrix h = coo(2, 3, {{0, 0, 1.f}, {0, 2, 2.f}, {1, 1, 3.f}});
    const DenseMatrix ones(3, 2, 1.f);
    for (auto& v : kAll) {
      const DenseMatrix r = native_spmm(h, ones, v, ops::sum(), 1);
      CHECK(r.at(0, 0) == 3.f && r.at(0, 1) == 3.f && r.at(1, 0) == 3.f && r.at(1, 1) == 3.f);
    }
  }
  // empty rows produce the op seed
  {
    CsrMatrix a(3, 3);
    const DenseMatrix b = make_random_dense(3, 5, 3);
    for (auto& v : kAll) {
      for (float x : native_spmm(a, b, v, ops::sum()).data) CHECK(x == 0.0f);
      for (float x : native_spmm(a, b, v, ops::max()).data)
        CHECK(x == std::numeric_limits<float>::lowest());
      for (float x : native_spmm(a, b, v, ops::min()).data)
        CHECK(x == std::numeric_limits<float>::max());
    }
  }
  // max-pool hand case and its argmax
  {
    const CsrMatrix a = coo(3, 3, {{0, 1, 1.f}, {0, 2, 1.f}});
    DenseMatrix b(3, 1);
    b.at(1, 0) = 5.f;
    b.at(2, 0) = 3.f;
    for (auto& v : kAll) {
      auto [c, arg] = native_spmm_arg(a, b, v, ops::max());
      CHECK(c.at(0, 0) == 5.f && arg[0] == 0);
      CHECK(c.at(1, 0) == std::numeric_limits<float>::lowest() && arg[1] == -1);
      auto [cm, argm] = native_spmm_arg(a, b, v, ops::min(), {FaultMode::None, true,
                                                               GESPMM_ARG_COLUMN, 0});
      CHECK(cm.at(0, 0) == 3.f && argm[0] == 2);
    }
  }
  // cwm lane ownership, N = 64: C[0,0] = 2*1, C[0,32] = 2*33
  {
    const CsrMatrix a = coo(1, 1, {{0, 0, 2.f}});
    DenseMatrix b(1, 64);
    for (u32 j = 0; j < 64; ++j) b.at(0, j) = float(j + 1);
    for (auto& v : kAll) {
      const DenseMatrix c = native_spmm(a, b, v, ops::sum());
      CHECK(c.at(0, 0) == 2.f && c.at(0, 32) == 66.f);
    }
  }
  // randomized differential, seed 404 shape (test_kernels.cpp:118-137)
  {
    std::mt19937_64 rng(404);
    const u32 ns[] = {1, 5, 16, 33, 48, 64, 500};
    for (int it = 0; it < 25; ++it) {
      const u32 rows = 1 + u32(rng() % 200);
      const u64 nnz = rng() % (u64(rows) * (rows - 1) / 2 + 1);
      CsrMatrix a = gen_uniform_random({rows, nnz, rng(), (rng() & 1) != 0});
      randomize_values(a, rng());
      const u32 n = ns[rng() % 7];
      const DenseMatrix b = make_random_dense(rows, n, rng());
      const ReduceOp op = (it & 1) ? ops::max() : ops::sum();
      const DenseMatrix want = fold_ref(a, b, op);
      for (auto& v : kAll) CHECK(native_spmm(a, b, v, op, 1 + u32(rng() % 4)).bitwise_equal(want));
    }
  }
  // the reference's checksums on BASELINE configs 0-1 (tests/golden/golden.json)
  {
    struct Cfg { u32 rows; u64 nnz; u32 n; const char* op; u64 sum; };
    const Cfg cfgs[] = {{2708, 10556, 16, "sum", 0xfa17737d80a5e52eull},
                        {2708, 10556, 16, "max", 0x4e95c693783892a5ull},
                        {19717, 88648, 128, "sum", 0xabd0e8342dccbd56ull},
                        {19717, 88648, 128, "max", 0xd53351ef0a5d6b30ull}};
    for (const auto& c : cfgs) {
      CsrMatrix a = gen_uniform_random({c.rows, c.nnz, 1, false});
      randomize_values(a, 2);
      const DenseMatrix b = make_random_dense(c.rows, c.n, 42);
      const ReduceOp op = reduce_op_by_name(c.op);
      CHECK(checksum(native_spmm(a, b, select_variant(c.n), op)) == c.sum);
      CHECK(checksum(native_spmm(a, b, KernelVariant::tuned(), op)) == c.sum);
    }
  }
  // fault injection is detectable (test_kernels.cpp:153-166)
  {
    std::mt19937_64 rng(88);
    CsrMatrix a = gen_uniform_random({40, 300, rng(), false});
    randomize_values(a, rng());
    const DenseMatrix b = make_random_dense(40, 16, 2);
    const DenseMatrix want = fold_ref(a, b, ops::sum());
    for (auto& v : kAll)
      CHECK(!native_spmm(a, b, v, ops::sum(), 2, {FaultMode::SkipTail}).bitwise_equal(want));
  }
  // error texts (test_simt.cpp:249-258, native.hpp:110, reduce_op.hpp:35)
  {
    const CsrMatrix a = coo(2, 3, {{0, 0, 1.f}, {1, 1, 1.f}});
    CHECK(error_of([&] { native_spmm(a, DenseMatrix(4, 2), KernelVariant::crc(), ops::sum()); }) ==
          "spmm: dimension mismatch: A is 2x3 but B has 4 rows");
    CsrMatrix bad = a;
    bad.col_ind[1] = 0;
    bad.row_ptr = {0, 2, 2};
    CHECK(error_of([&] { native_spmm(bad, DenseMatrix(3, 2), KernelVariant::tuned(), ops::sum()); }) ==
          "spmm: matrix is not canonical CSR: columns not strictly increasing in row 0 at position 1");
    CHECK(error_of([&] { native_spmm(a, DenseMatrix(3, 0), KernelVariant::crc(), ops::sum()); }) ==
          "native_spmm: N must be >= 1");
    CHECK(error_of([&] { reduce_op_by_name("median"); }).find("unknown reduce op") == 0);
    CHECK(error_of([&] { native_spmm(a, DenseMatrix(3, 2), KernelVariant::crc_cwm(3), ops::sum()); }) ==
          "coarsening factor must be 2, 4 or 8");
  }
  // bench uses theoretical flops and a stable checksum (test_native.cpp:78-106)
  {
    CsrMatrix a = gen_uniform_random({128, 2000, 8, false});
    randomize_values(a, 9);
    const DenseMatrix b = make_random_dense(128, 48, 10);
    const ThroughputReport r1 = bench(a, b, KernelVariant::crc_cwm(2), ops::sum(), 4, 2);
    const ThroughputReport r2 = bench(a, b, KernelVariant::tuned(), ops::sum(), 1, 3);
    CHECK(r1.flops == 2ull * a.nnz() * 48 && r1.repeats == 2 && r1.gflops > 0);
    CHECK(r1.output_checksum == r2.output_checksum);
    CHECK(error_of([&] { bench(a, b, KernelVariant::naive(), ops::sum(), 1, 0); }) ==
          "bench: repeats must be >= 1");
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  if (g_fail == 0) std::printf("ALL PASS\n");
  return g_fail ? 1 : 0;
}
