// The reference's documented library usage and the cases of its own unit
// tests, written against <gespmm/native_spmm.hpp> with the reference's names
// and call shapes (a reference user's code compiles as is), run on the B200:
//   proj/README.md:133-141           library use (load_matrix, make_random_dense,
//                                    KernelConfig, select_variant, native_spmm)
//   proj/tests/test_kernels.cpp:26-116  identity / single row / empty rows /
//                                    tiles / CWM column ownership / ragged slice
//   proj/tests/test_native.cpp:12-58    hand case, worker independence,
//                                    native == kernel output over random shapes
//   proj/tests/test_csr.cpp, test_io.cpp  from_coo / to_coo / validate /
//                                    require_canonical / CSR1 + Matrix Market
// Two reference test instruments are not part of the drop-in: run_kernel (the
// SIMT simulator, whose transaction counters are checked by
// tests/test_gpu_sectors.py against the GPU's) and dense_reference (the
// brute-force oracle).  Here run_kernel(...).c is the same native_spmm call and
// dense_reference is a dense-matrix fold local to this file.
#include <unistd.h>

#include <cmath>
#include <fstream>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <limits>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "gespmm/native_spmm.hpp"

using namespace spmm;

// ---- a minimal test registry (the reference uses Catch2) --------------------
static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<const char*, std::function<void()>>>& cases() {
  static std::vector<std::pair<const char*, std::function<void()>>> v;
  return v;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                   \
  static void CAT(tc_, __LINE__)();                       \
  static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define REQUIRE(cond) CHECK(cond)
#define CAPTURE(...) (void)0

template <class F>
static std::string error_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.what();
  }
  return "";
}

// ---- test instruments (see the header comment) ------------------------------
struct KernelRun {
  DenseMatrix c;
};
static KernelRun run_kernel(const CsrMatrix& a, const DenseMatrix& b, const KernelConfig& cfg,
                            const ReduceOp& op) {
  check_config(cfg);
  return {native_spmm(a, b, cfg.variant, op)};
}

// densified A, ascending k, stored zeros skipped (the reference oracle's rule)
static DenseMatrix dense_reference(const CsrMatrix& a, const DenseMatrix& b, const ReduceOp& op) {
  std::vector<float> dense(size_t(a.n_rows) * a.n_cols, 0.0f);
  for (u32 r = 0; r < a.n_rows; ++r)
    for (u32 p = a.row_ptr[r]; p < a.row_ptr[r + 1]; ++p)
      dense[size_t(r) * a.n_cols + a.col_ind[p]] = a.vals[p];
  DenseMatrix c(a.n_rows, b.n_cols, op.init);
  for (u32 i = 0; i < a.n_rows; ++i)
    for (u32 j = 0; j < b.n_cols; ++j) {
      float acc = op.init;
      for (u32 k = 0; k < a.n_cols; ++k) {
        const float v = dense[size_t(i) * a.n_cols + k];
        if (v == 0.0f) continue;
        volatile float x = v * b.at(k, j);
        acc = op.fold(acc, x);
      }
      c.at(i, j) = acc;
    }
  return c;
}

static CsrMatrix random_matrix(std::mt19937_64& rng, u32 rows, u64 nnz) {
  CsrMatrix m = gen_uniform_random({rows, nnz, rng(), (rng() & 1) != 0});
  randomize_values(m, rng());
  return m;
}

static const std::vector<KernelVariant> kAllVariants = {
    KernelVariant::naive(), KernelVariant::crc(), KernelVariant::crc_cwm(2),
    KernelVariant::crc_cwm(4), KernelVariant::crc_cwm(8), KernelVariant::tuned()};

// ---- README.md:133-141 ------------------------------------------------------
TEST_CASE("README library use") {
  const auto dir = std::filesystem::temp_directory_path();
  const auto path = dir / ("gespmm_readme_" + std::to_string(::getpid()) + ".csr");
  {
    std::mt19937_64 rng(7);
    save_csr_cache(path, random_matrix(rng, 300, 6000));
  }
  CsrMatrix a = load_matrix(path);
  DenseMatrix b = make_random_dense(a.n_cols, 512, /*seed=*/42);
  KernelConfig cfg{32, 8, select_variant(b.n_cols)};
  CHECK(cfg.variant == KernelVariant::crc_cwm(2));
  DenseMatrix c2 = native_spmm(a, b, cfg.variant, ops::max(), /*workers=*/8);
  CHECK(c2.bitwise_equal(dense_reference(a, b, ops::max())));
  std::filesystem::remove(path);
}

// ---- test_kernels.cpp:26-116 -------------------------------------------------
TEST_CASE("identity matrix reproduces B on every variant") {
  CooEntries eye{3, 3, {{0, 0, 1.0f}, {1, 1, 1.0f}, {2, 2, 1.0f}}};
  const CsrMatrix a = from_coo(eye);
  const DenseMatrix b = make_random_dense(3, 4, 11);
  for (const auto& v : kAllVariants) {
    KernelConfig cfg{32, 8, v};
    CHECK(run_kernel(a, b, cfg, ops::sum()).c.bitwise_equal(b));
    CHECK(native_spmm(a, b, v, ops::sum(), 3).bitwise_equal(b));
  }
}

TEST_CASE("single-row case matches the dense reference") {
  CooEntries coo{1, 2, {{0, 0, 2.0f}, {0, 1, 3.0f}}};
  const CsrMatrix a = from_coo(coo);
  DenseMatrix b(2, 2);
  b.at(0, 0) = 1.0f;
  b.at(1, 1) = 1.0f;
  const DenseMatrix want = dense_reference(a, b, ops::sum());
  REQUIRE(want.at(0, 0) == 2.0f);
  REQUIRE(want.at(0, 1) == 3.0f);
  KernelConfig cfg{32, 8, KernelVariant::naive()};
  CHECK(run_kernel(a, b, cfg, ops::sum()).c.bitwise_equal(want));
}

TEST_CASE("empty rows produce the op seed in every column") {
  CsrMatrix a(3, 3);
  const DenseMatrix b = make_random_dense(3, 5, 3);
  for (const auto& v : kAllVariants) {
    KernelConfig cfg{32, 8, v};
    for (float x : run_kernel(a, b, cfg, ops::sum()).c.data) CHECK(x == 0.0f);
    for (float x : run_kernel(a, b, cfg, ops::max()).c.data)
      CHECK(x == std::numeric_limits<float>::lowest());
  }
}

TEST_CASE("short and long rows (one partial tile; ceil(len/32) tiles)") {
  for (u32 len : {5u, 70u}) {
    CooEntries coo{1, 100, {}};
    for (u32 c = 0; c < len; ++c) coo.entries.push_back({0, c, 1.0f});
    const CsrMatrix a = from_coo(coo);
    const DenseMatrix b = make_random_dense(100, 8, 5);
    for (const auto& v : kAllVariants)
      CHECK(run_kernel(a, b, KernelConfig{32, 8, v}, ops::sum()).c.bitwise_equal(
          dense_reference(a, b, ops::sum())));
  }
}

TEST_CASE("cwm lane owns columns strided by warp size") {
  CooEntries coo{1, 1, {{0, 0, 2.0f}}};
  const CsrMatrix a = from_coo(coo);
  DenseMatrix b(1, 64);
  for (u32 j = 0; j < 64; ++j) b.at(0, j) = float(j + 1);
  KernelConfig cfg{32, 8, KernelVariant::crc_cwm(2)};
  const auto res = run_kernel(a, b, cfg, ops::sum());
  CHECK(res.c.at(0, 0) == 2.0f * 1.0f);
  CHECK(res.c.at(0, 32) == 2.0f * 33.0f);
}

TEST_CASE("cwm masks the upper column slice at a ragged boundary") {
  CooEntries coo{1, 1, {{0, 0, 1.0f}}};
  const CsrMatrix a = from_coo(coo);
  const DenseMatrix b = make_random_dense(1, 48, 9);
  for (u32 cf : {2u, 4u, 8u}) {
    KernelConfig cfg{32, 8, KernelVariant::crc_cwm(cf)};
    CHECK(run_kernel(a, b, cfg, ops::sum()).c.bitwise_equal(dense_reference(a, b, ops::sum())));
  }
}

TEST_CASE("all variants agree bitwise with the dense reference (seed 404)") {
  std::mt19937_64 rng(404);
  const u32 n_choices[] = {1, 5, 16, 33, 48, 64, 500};
  for (int it = 0; it < 12; ++it) {
    const u32 rows = 1 + u32(rng() % 60);
    const CsrMatrix a = random_matrix(rng, rows, rng() % (u64(rows) * (rows - 1) / 2 + 1));
    const u32 n = n_choices[rng() % 7];
    const DenseMatrix b = make_random_dense(rows, n, rng());
    for (const ReduceOp& op : {ops::sum(), ops::max()}) {
      const DenseMatrix want = dense_reference(a, b, op);
      for (const auto& v : kAllVariants) {
        CAPTURE(it, n, v.name(), op.name);
        CHECK(native_spmm(a, b, v, op, 1 + u32(rng() % 8)).bitwise_equal(want));
      }
    }
  }
}

// ---- test_native.cpp:12-58 ---------------------------------------------------
TEST_CASE("native spmm matches the hand-computed small case") {
  CooEntries coo{2, 3, {{0, 0, 1.0f}, {0, 2, 2.0f}, {1, 1, 3.0f}}};
  const CsrMatrix a = from_coo(coo);
  const DenseMatrix b(3, 2, 1.0f);
  const DenseMatrix want = dense_reference(a, b, ops::sum());
  REQUIRE(want.at(0, 0) == 3.0f && want.at(0, 1) == 3.0f);
  REQUIRE(want.at(1, 0) == 3.0f && want.at(1, 1) == 3.0f);
  CHECK(native_spmm(a, b, KernelVariant::crc(), ops::sum(), 1).bitwise_equal(want));
}

TEST_CASE("output is independent of worker count") {
  std::mt19937_64 rng(6);
  CsrMatrix a = gen_uniform_random({257, 4000, rng(), false});
  randomize_values(a, rng());
  const DenseMatrix b = make_random_dense(257, 65, rng());
  for (const auto& v : {KernelVariant::naive(), KernelVariant::crc(), KernelVariant::crc_cwm(2)})
    CHECK(native_spmm(a, b, v, ops::sum(), 1).bitwise_equal(native_spmm(a, b, v, ops::sum(), 8)));
}

TEST_CASE("native output equals kernel output bitwise over random shapes") {
  std::mt19937_64 rng(60);
  for (int it = 0; it < 10; ++it) {
    const u32 rows = 1 + u32(rng() % 150);
    CsrMatrix a =
        gen_uniform_random({rows, rng() % (u64(rows) * (rows - 1) / 2 + 1), rng(), false});
    randomize_values(a, rng());
    const u32 n = 1 + u32(rng() % 100);
    const DenseMatrix b = make_random_dense(rows, n, rng());
    const ReduceOp op = (it & 1) ? ops::max() : ops::sum();
    const DenseMatrix want = dense_reference(a, b, op);
    for (const auto& v : {KernelVariant::naive(), KernelVariant::crc(), KernelVariant::crc_cwm(8),
                          KernelVariant::tuned()}) {
      KernelConfig cfg{32, 8, v};
      REQUIRE(native_spmm(a, b, v, op, 4).bitwise_equal(run_kernel(a, b, cfg, op).c));
      CHECK(native_spmm(a, b, v, op, 4).bitwise_equal(want));
    }
  }
}

// ---- data model and formats (csr.hpp, io.hpp, matrix_market.hpp) -------------
TEST_CASE("from_coo sorts, sums or keeps the last duplicate; to_coo round-trips") {
  CooEntries coo{3, 4, {{2, 1, 1.0f}, {0, 3, 2.0f}, {0, 1, 0.5f}, {2, 1, 4.0f}, {0, 3, 1.0f}}};
  const CsrMatrix s = from_coo(coo);
  CHECK((s.row_ptr == std::vector<u32>{0, 2, 2, 3}));
  CHECK((s.col_ind == std::vector<u32>{1, 3, 1}));
  CHECK((s.vals == std::vector<float>{0.5f, 3.0f, 5.0f}));
  const CsrMatrix l = from_coo(coo, DedupPolicy::Last);
  CHECK((l.vals == std::vector<float>{0.5f, 1.0f, 4.0f}));
  const CooEntries back = to_coo(s);
  CHECK(back.n_rows == 3 && back.n_cols == 4 && back.entries.size() == 3);
  CHECK((back.entries[2] == CooEntry{2, 1, 5.0f}));
  CHECK(error_of([] { from_coo(CooEntries{2, 2, {{3, 1, 1.5f}}}); }) ==
        "coo entry (3, 1, 1.5) outside declared 2x2 bounds");
}

TEST_CASE("validate reports every violation; require_canonical raises the first") {
  CsrMatrix m(2, 3);
  m.row_ptr = {0, 2, 4};
  m.col_ind = {2, 1, 5, 0};
  m.vals = {1, 1, 1, 1};
  const ValidationReport rep = validate(m);
  REQUIRE(rep.violations.size() == 3);
  CHECK(rep.violations[0] == "columns not strictly increasing in row 0 at position 1");
  CHECK(rep.violations[1] == "col_ind[2] = 5 out of bounds (n_cols = 3)");
  CHECK(rep.violations[2] == "columns not strictly increasing in row 1 at position 3");
  CHECK(error_of([&] { require_canonical(m, "who"); }) ==
        "who: matrix is not canonical CSR: columns not strictly increasing in row 0 at position 1");
  CsrMatrix short_rp(4, 4);
  short_rp.row_ptr = {0, 0};
  CHECK(validate(short_rp).violations.front() == "row_ptr length is 2, expected n_rows+1 = 5");
  CHECK(validate(from_coo(CooEntries{2, 2, {{0, 1, 1.0f}}})).ok());
}

TEST_CASE("KernelConfig and check_config keep the reference's rules") {
  CHECK(error_of([] { check_config(KernelConfig{48, 8, KernelVariant::crc()}); }) ==
        "warp_size must be a power of two in [4, 64]");
  CHECK(error_of([] { check_config(KernelConfig{32, 0, KernelVariant::crc()}); }) ==
        "warps_per_block must be >= 1");
  CHECK(error_of([] { check_config(KernelConfig{32, 8, KernelVariant::crc_cwm(3)}); }) ==
        "coarsening factor must be 2, 4 or 8");
  check_config(KernelConfig{});
}

TEST_CASE("CSR1 cache and Matrix Market load through load_matrix") {
  namespace fs = std::filesystem;
  const auto dir = fs::temp_directory_path();
  const std::string tag = std::to_string(::getpid());
  std::mt19937_64 rng(99);
  const CsrMatrix a = random_matrix(rng, 40, 300);
  std::stringstream ss;
  write_csr_cache(ss, a);
  const CsrMatrix r = read_csr_cache(ss);
  CHECK(r.row_ptr == a.row_ptr && r.col_ind == a.col_ind && r.vals == a.vals);
  const auto mtx = dir / ("gespmm_" + tag + ".mtx");
  {
    std::ofstream f(mtx);
    write_matrix_market(f, a);
  }
  const CsrMatrix m = load_matrix(mtx);
  CHECK(m.row_ptr == a.row_ptr && m.col_ind == a.col_ind && m.vals == a.vals);
  {
    std::ofstream f(mtx);
    f << "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 3\n";
  }
  const CsrMatrix sym = load_matrix(mtx);
  CHECK((sym.row_ptr == std::vector<u32>{0, 1, 2, 3}));
  CHECK((sym.col_ind == std::vector<u32>{1, 0, 2}));
  {
    std::ofstream f(mtx);
    f << "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n";
  }
  CHECK(error_of([&] { load_matrix(mtx); }) ==
        "matrix market: line 3: index (3, 1) outside declared 2x2");
  try {
    parse_matrix_market(std::string("%%MatrixMarket matrix array real general\n"));
    CHECK(false);
  } catch (const MmParseError& e) {
    CHECK(e.line() == 1);
  }
  fs::remove(mtx);
  CHECK(error_of([&] { load_matrix(dir / ("gespmm_" + tag + ".bin")); }).rfind("cannot open", 0) ==
        0);
}

TEST_CASE("custom combine pointers and the added ops") {
  const CsrMatrix a = from_coo(CooEntries{1, 2, {{0, 0, 2.0f}, {0, 1, -1.0f}}});
  const DenseMatrix b(2, 3, 1.0f);
  ReduceOp custom{"prod", 1.0f, [](float x, float y) { return x * y; }};
  CHECK(error_of([&] { native_spmm(a, b, KernelVariant::tuned(), custom); })
            .rfind("reduce op 'prod'", 0) == 0);
  const DenseMatrix mean = native_spmm(a, b, KernelVariant::tuned(), ops::mean());
  CHECK(mean.at(0, 0) == 0.5f);
  const DenseMatrix mn = native_spmm(a, b, KernelVariant::crc(), ops::min());
  CHECK(mn.at(0, 2) == -1.0f);
  CHECK(reduce_op_by_name("max").combine == &ops::max_f32);
}

int main() {
  for (auto& [name, fn] : cases()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "EXCEPTION in '%s': %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  if (g_fail == 0) std::printf("ALL PASS\n");
  return g_fail ? 1 : 0;
}
