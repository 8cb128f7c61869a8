// Host-side synthetic inputs and the output checksum (C ABI, see gespmm.h).
//
// Reference generators restated bit-exactly (under /root/reference/proj):
//   make_random_dense   include/spmm/dense.hpp:51-59
//   randomize_values    include/spmm/generate.hpp:73-80
//   gen_uniform_random  include/spmm/generate.hpp:39-69 (+ from_coo, csr.hpp:58-93)
//   checksum            include/spmm/dense.hpp:62-72
// New: gespmm_gen_powerlaw — a deterministic, multithreaded Chung-Lu-style
// power-law generator for the Reddit / ogbn-products shaped configs (the
// reference has no power-law generator).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "gespmm/gespmm.h"
#include "launch.h"

namespace {

// Fixed-point bounded draw (generate.hpp:30-32).
inline uint32_t bounded(std::mt19937_64& rng, uint32_t bound) {
  return static_cast<uint32_t>((static_cast<unsigned __int128>(rng()) * bound) >> 64);
}

inline uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Open-addressing set of u64 keys (the rejection set of gen_uniform; any set
// gives the same accepted sequence, this one is just faster than std's).
struct KeySet {
  std::vector<uint64_t> slots;
  uint64_t mask;
  explicit KeySet(uint64_t expected) {
    uint64_t cap = 16;
    while (cap < expected * 2 + 16) cap <<= 1;
    slots.assign(cap, ~0ull);
    mask = cap - 1;
  }
  bool insert(uint64_t key) {
    uint64_t h = key * 0x9E3779B97F4A7C15ull;
    for (uint64_t i = (h >> 17) & mask;; i = (i + 1) & mask) {
      if (slots[i] == key) return false;
      if (slots[i] == ~0ull) {
        slots[i] = key;
        return true;
      }
    }
  }
};

int clamp_threads(int t) {
  if (t <= 0) t = int(std::max(1u, std::thread::hardware_concurrency()));
  return std::min(t, 256);
}

}  // namespace

extern "C" {

void gespmm_make_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  std::mt19937_64 rng(seed);
  const uint64_t total = uint64_t(rows) * cols;
  for (uint64_t i = 0; i < total; ++i) {
    const uint32_t bits = static_cast<uint32_t>(rng() >> 40);  // 24 bits
    out[i] = static_cast<float>(bits) * 0x1p-23f - 1.0f;
  }
}

void gespmm_randomize_values(float* vals, uint64_t nnz, uint64_t seed) {
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < nnz; ++i) {
    const uint32_t bits = static_cast<uint32_t>(rng() >> 44) + 1;  // 1 .. 2^20
    float v = static_cast<float>(bits) * 0x1p-19f;                 // (0, 2]
    if (rng() & 1) v = -v;
    vals[i] = v;
  }
}

uint64_t gespmm_checksum(const float* data, uint32_t rows, uint32_t cols) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(data);
  const uint64_t n = uint64_t(rows) * cols * sizeof(float);
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h ^ ((uint64_t(rows) << 32) ^ cols);
}

gespmm_status_t gespmm_gen_uniform(uint32_t rows, uint64_t nnz, uint64_t seed, int32_t self_loops,
                                   uint32_t* row_ptr, uint32_t* col_ind, float* vals) {
  if (rows == 0) {
    if (nnz > 0) return gespmm::set_error(GESPMM_EINVAL, "graph gen: nnz_target > 0 with zero rows");
    row_ptr[0] = 0;
    return GESPMM_OK;
  }
  const uint64_t m = rows;
  const uint64_t feasible = self_loops ? m * m : m * (m - 1);
  if (nnz > feasible)
    return gespmm::set_error(
        GESPMM_EINVAL, "graph gen: nnz_target " + std::to_string(nnz) +
                           " exceeds feasible maximum " + std::to_string(feasible) +
                           (self_loops ? "" : " (self loops excluded)"));
  std::mt19937_64 rng(seed);
  KeySet taken(nnz);
  std::vector<uint64_t> keys;
  keys.reserve(nnz);
  while (keys.size() < nnz) {
    const uint32_t r = bounded(rng, rows);
    const uint32_t c = bounded(rng, rows);
    if (!self_loops && r == c) continue;
    const uint64_t key = uint64_t(r) * m + c;
    if (taken.insert(key)) keys.push_back(key);
  }
  // canonical order: (row, col) ascending; keys are distinct
  std::sort(keys.begin(), keys.end());
  std::memset(row_ptr, 0, sizeof(uint32_t) * (m + 1));
  for (uint64_t i = 0; i < nnz; ++i) {
    const uint32_t r = uint32_t(keys[i] / m);
    col_ind[i] = uint32_t(keys[i] % m);
    vals[i] = 1.0f;
    ++row_ptr[r + 1];
  }
  for (uint64_t r = 0; r < m; ++r) row_ptr[r + 1] += row_ptr[r];
  return GESPMM_OK;
}

gespmm_status_t gespmm_gen_powerlaw(uint32_t rows, uint64_t nnz_target, uint32_t max_degree,
                                    double exponent, uint64_t seed, int32_t threads,
                                    uint32_t* row_ptr, uint32_t* col_ind, float* vals) {
  if (rows < 2 || exponent <= 0.0)
    return gespmm::set_error(GESPMM_EINVAL, "powerlaw gen: need rows >= 2 and exponent > 0");
  const double mean = double(nnz_target) / rows;
  if (max_degree > rows - 1) max_degree = rows - 1;
  if (double(max_degree) < mean || mean > double(rows - 1))
    return gespmm::set_error(GESPMM_EINVAL,
                             "powerlaw gen: max_degree must be >= mean degree and <= rows-1");

  // rank weights w_r = (r + c)^-exponent, c chosen so the largest expected
  // degree is max_degree when the weights are scaled to nnz_target.
  auto max_for = [&](double c) {
    double sum = 0.0;
    for (uint32_t r = 0; r < rows; ++r) sum += std::pow(double(r) + c, -exponent);
    return double(nnz_target) * std::pow(c, -exponent) / sum;
  };
  double lo = 1e-6, hi = 1e12;
  for (int it = 0; it < 200 && hi / lo > 1.0 + 1e-9; ++it) {
    const double mid = std::sqrt(lo * hi);
    if (max_for(mid) > double(max_degree)) lo = mid; else hi = mid;
  }
  const double c = std::sqrt(lo * hi);
  std::vector<double> w(rows);
  double sum = 0.0;
  for (uint32_t r = 0; r < rows; ++r) sum += (w[r] = std::pow(double(r) + c, -exponent));
  const double scale = double(nnz_target) / sum;

  // integer degrees summing exactly to nnz_target: floors + largest remainders
  std::vector<uint32_t> deg_rank(rows);
  std::vector<std::pair<double, uint32_t>> frac(rows);
  uint64_t assigned = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    const double x = std::min(w[r] * scale, double(rows - 1));
    deg_rank[r] = uint32_t(std::floor(x));
    assigned += deg_rank[r];
    frac[r] = {x - std::floor(x), r};
  }
  std::stable_sort(frac.begin(), frac.end(),
                   [](const auto& a, const auto& b) { return a.first > b.first; });
  for (uint32_t i = 0; assigned < nnz_target && i < rows; ++i) {
    if (deg_rank[frac[i].second] < rows - 1) {
      ++deg_rank[frac[i].second];
      ++assigned;
    }
  }

  // random node ids for the ranks (hubs spread over the row space)
  std::vector<uint32_t> node_of_rank(rows), rank_of(rows);
  for (uint32_t r = 0; r < rows; ++r) node_of_rank[r] = r;
  uint64_t ps = seed ^ 0x5851F42D4C957F2Dull;
  for (uint32_t i = rows - 1; i > 0; --i) {
    const uint32_t j = uint32_t((static_cast<unsigned __int128>(splitmix(ps)) * (i + 1)) >> 64);
    std::swap(node_of_rank[i], node_of_rank[j]);
  }
  for (uint32_t r = 0; r < rows; ++r) rank_of[node_of_rank[r]] = r;

  row_ptr[0] = 0;
  for (uint32_t v = 0; v < rows; ++v) row_ptr[v + 1] = row_ptr[v] + deg_rank[rank_of[v]];
  if (!col_ind) return GESPMM_OK;  // sizing call

  // Vose alias table over node ids (weights w[rank_of[v]]), integer thresholds
  std::vector<uint32_t> alias(rows), thresh(rows);
  {
    std::vector<double> p(rows);
    for (uint32_t v = 0; v < rows; ++v) p[v] = w[rank_of[v]] / sum * rows;
    std::vector<uint32_t> small, large;
    small.reserve(rows);
    large.reserve(rows);
    for (uint32_t v = 0; v < rows; ++v) (p[v] < 1.0 ? small : large).push_back(v);
    while (!small.empty() && !large.empty()) {
      const uint32_t s = small.back(), l = large.back();
      small.pop_back();
      thresh[s] = uint32_t(std::min(4294967295.0, std::floor(p[s] * 4294967296.0)));
      alias[s] = l;
      p[l] = (p[l] + p[s]) - 1.0;
      if (p[l] < 1.0) {
        large.pop_back();
        small.push_back(l);
      }
    }
    for (uint32_t v : large) {
      thresh[v] = 0xffffffffu;
      alias[v] = v;
    }
    for (uint32_t v : small) {
      thresh[v] = 0xffffffffu;
      alias[v] = v;
    }
  }

  const int nt = clamp_threads(threads);
  auto work = [&](uint32_t r0, uint32_t r1) {
    std::vector<uint32_t> stamp(rows, 0xffffffffu);
    for (uint32_t row = r0; row < r1; ++row) {
      uint64_t s = seed * 0x9E3779B97F4A7C15ull ^ (uint64_t(row) + 1) * 0xD1B54A32D192ED03ull;
      const uint32_t d = row_ptr[row + 1] - row_ptr[row];
      uint32_t* out = col_ind + row_ptr[row];
      uint32_t got = 0;
      while (got < d) {
        const uint64_t u = splitmix(s);
        const uint32_t idx = uint32_t((static_cast<unsigned __int128>(u >> 32) * rows) >> 32);
        const uint32_t j = uint32_t(u) < thresh[idx] ? idx : alias[idx];
        if (j == row || stamp[j] == row) continue;
        stamp[j] = row;
        out[got++] = j;
      }
      std::sort(out, out + d);
      std::fill(vals + row_ptr[row], vals + row_ptr[row + 1], 1.0f);
    }
  };
  // split rows by nnz so hub rows do not serialise
  std::vector<std::thread> pool;
  const uint64_t total = row_ptr[rows];
  uint32_t begin = 0;
  for (int t = 0; t < nt; ++t) {
    const uint64_t target = total * uint64_t(t + 1) / uint64_t(nt);
    uint32_t end = begin;
    if (t == nt - 1) end = rows;
    else
      while (end < rows && row_ptr[end] < target) ++end;
    if (end > begin) pool.emplace_back(work, begin, end);
    begin = end;
  }
  for (auto& th : pool) th.join();
  return GESPMM_OK;
}

}  // extern "C"
