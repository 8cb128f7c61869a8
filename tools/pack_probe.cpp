// pack_probe: host cost and size of the col_ind upload codecs on the Reddit
// shape (run on the GPU box's host: it sets the e2e pipeline's packing budget).
//   u16  : the product's 16-bit gap codes (gespmm::pack_cols_block)
//   pfor : per-2048-position chunk bit width w (1..16) chosen for the fewest
//          bytes, gaps >= 2^w - 1 patched from a u16 side list
// Build: g++ -O3 -fopenmp -I include tools/pack_probe.cpp -L paper_2007_03179_b200 -lgespmm
#include <omp.h>
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "gespmm/gespmm.h"

namespace gespmm {
uint64_t pack_cols_block(const uint32_t*, const uint32_t*, uint32_t, uint32_t, uint16_t*, uint32_t*, uint64_t);
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <int W>
static inline void pack32(const uint32_t* g, uint32_t* out) {
  uint64_t acc = 0;
  int bits = 0, o = 0;
#pragma GCC unroll 32
  for (int i = 0; i < 32; ++i) {
    acc |= uint64_t(g[i]) << bits;
    bits += W;
    if (bits >= 32) { out[o++] = uint32_t(acc); acc >>= 32; bits -= 32; }
  }
}
typedef void (*Pack32)(const uint32_t*, uint32_t*);
static const Pack32 kPack[17] = {nullptr, pack32<1>, pack32<2>, pack32<3>, pack32<4>, pack32<5>, pack32<6>,
                                 pack32<7>, pack32<8>, pack32<9>, pack32<10>, pack32<11>, pack32<12>,
                                 pack32<13>, pack32<14>, pack32<15>, pack32<16>};

// one chunk: gaps -> width choice -> packed words; returns code bytes
static uint32_t pfor_chunk(const uint32_t* row_ptr, const uint32_t* col, uint64_t p0, uint32_t len, uint32_t& row,
                           uint32_t* words, uint16_t* side, uint32_t& n_side, uint8_t& w_out) {
  alignas(64) uint32_t g[2048 + 32];
  uint32_t i = 0;
  uint64_t p = p0;
  const uint64_t pend = p0 + len;
  while (p < pend) {
    while (row_ptr[row + 1] <= p) ++row;
    const uint64_t seg_end = std::min<uint64_t>(row_ptr[row + 1], pend);
    uint32_t prev;
    if (p == row_ptr[row]) { prev = col[p]; g[i++] = prev; ++p; }
    else prev = col[p - 1];
    for (; p < seg_end; ++p) { const uint32_t c = col[p]; g[i++] = c - prev - 1u; prev = c; }
  }
  uint32_t h[4][18] = {{0}};
  for (uint32_t k = 0; k < len; ++k) {
    const uint32_t x = std::min(g[k], 0xFFFEu) + 1u;
    ++h[k & 3][32 - __builtin_clz(x)];
  }
  uint32_t suffix[18] = {0};
  for (int bl = 16; bl >= 1; --bl) suffix[bl - 1] = suffix[bl] + h[0][bl] + h[1][bl] + h[2][bl] + h[3][bl];
  // suffix[w] = #(gap + 1 >= 2^w): the escapes at width w
  uint32_t best_w = 16, best = ~0u;
  for (uint32_t w = 1; w <= 16; ++w) {
    const uint32_t bytes = ((len * w + 31) / 32) * 4 + 2 * (w < 16 ? suffix[w] : 0);
    if (bytes < best) { best = bytes; best_w = w; }
  }
  const uint32_t w = best_w, lim = w < 16 ? (1u << w) - 1u : 0xFFFFu;
  uint32_t ns = 0;
  for (uint32_t k = 0; k < len; ++k) {
    const uint32_t x = g[k];
    side[ns] = uint16_t(std::min(x, 0xFFFFu));
    ns += x >= lim;
    g[k] = std::min(x, lim);
  }
  for (uint32_t k = len; k < ((len + 31) & ~31u); ++k) g[k] = 0;
  const Pack32 pk = kPack[w];
  for (uint32_t k = 0; k < len; k += 32) pk(g + k, words + (k / 32) * w);
  n_side = ns;
  w_out = uint8_t(w);
  return ((len * w + 31) / 32) * 4;
}

// u16 packer with a vectorisable inner loop: per row the first entry is its
// column, the rest (col[p] - col[p-1] - 1) computed without a carried
// dependency, clamped to 0xFFFF, with a running max; rows whose max reaches
// 0xFFFF get a scalar pass that records their escapes.
template <int DUMMY>
static inline uint64_t pack_rows_u16(const uint32_t* __restrict row_ptr, const uint32_t* __restrict col,
                                     uint32_t r0, uint32_t r1, uint64_t ps, uint16_t* __restrict enc,
                                     std::vector<uint32_t>& ex) {
  for (uint32_t r = r0; r < r1; ++r) {
    const uint64_t s = row_ptr[r], e = row_ptr[r + 1];
    if (s == e) continue;
    uint32_t mx = col[s] >= 0xFFFFu ? 0xFFFFu : 0u;
    enc[s - ps] = uint16_t(col[s] < 0xFFFFu ? col[s] : 0xFFFFu);
    const uint32_t* c = col + s;
    uint16_t* o = enc + (s - ps);
    const uint64_t n = e - s;
    for (uint64_t i = 1; i < n; ++i) {
      const uint32_t d = c[i] - c[i - 1] - 1u;
      mx = d > mx ? d : mx;
      o[i] = uint16_t(d < 0xFFFFu ? d : 0xFFFFu);
    }
    if (mx >= 0xFFFFu) {
      for (uint64_t i = 0; i < n; ++i)
        if (o[i] == 0xFFFFu) { ex.push_back(uint32_t(s + i - ps)); ex.push_back(c[i]); }
    }
  }
  return 0;
}
__attribute__((target("avx2"))) static uint64_t pack_rows_avx2(const uint32_t* rp, const uint32_t* col, uint32_t r0,
                                                               uint32_t r1, uint64_t ps, uint16_t* enc,
                                                               std::vector<uint32_t>& ex) {
  return pack_rows_u16<2>(rp, col, r0, r1, ps, enc, ex);
}
__attribute__((target("avx512f,avx512bw,avx512vl"))) static uint64_t pack_rows_avx512(
    const uint32_t* rp, const uint32_t* col, uint32_t r0, uint32_t r1, uint64_t ps, uint16_t* enc,
    std::vector<uint32_t>& ex) {
  return pack_rows_u16<3>(rp, col, r0, r1, ps, enc, ex);
}
static uint64_t pack_rows_base(const uint32_t* rp, const uint32_t* col, uint32_t r0, uint32_t r1, uint64_t ps,
                               uint16_t* enc, std::vector<uint32_t>& ex) {
  return pack_rows_u16<1>(rp, col, r0, r1, ps, enc, ex);
}

static double pack_fast_all(const std::vector<uint32_t>& rp, const std::vector<uint32_t>& ci,
                            const std::vector<uint32_t>& b, int blocks, int threads, std::vector<uint16_t>& enc,
                            int isa) {
  const double t0 = now_ms();
  for (int c = 0; c < blocks; ++c) {
    const uint32_t lo = b[c], hi = b[c + 1];
    const uint64_t ps = rp[lo], total = rp[hi] - ps;
    std::vector<uint32_t> cut(threads + 1, hi);
    cut[0] = lo;
    for (int t = 1; t < threads; ++t)
      cut[t] = std::max(cut[t - 1], uint32_t(std::lower_bound(rp.begin() + lo, rp.begin() + hi + 1,
                                                                uint32_t(ps + total * t / threads)) - rp.begin()));
    std::vector<std::vector<uint32_t>> ex(threads);
#pragma omp parallel num_threads(threads)
    {
      const int t = omp_get_thread_num();
      if (isa == 3) pack_rows_avx512(rp.data(), ci.data(), cut[t], cut[t + 1], ps, enc.data() + ps, ex[t]);
      else if (isa == 2) pack_rows_avx2(rp.data(), ci.data(), cut[t], cut[t + 1], ps, enc.data() + ps, ex[t]);
      else pack_rows_base(rp.data(), ci.data(), cut[t], cut[t + 1], ps, enc.data() + ps, ex[t]);
    }
  }
  return now_ms() - t0;
}

int main(int argc, char** argv) {
  const uint32_t m = 232965;
  const int blocks = argc > 1 ? atoi(argv[1]) : 12;
  const int threads = argc > 2 ? atoi(argv[2]) : std::max(1, int(std::thread::hardware_concurrency()) * 3 / 4);
  std::vector<uint32_t> rp(m + 1);
  if (gespmm_gen_powerlaw(m, 114800000ull, 21657, 1.0, 1, 0, rp.data(), nullptr, nullptr) != GESPMM_OK) return 1;
  const uint64_t nnz = rp[m];
  std::vector<uint32_t> ci(nnz);
  std::vector<float> v(nnz);
  if (gespmm_gen_powerlaw(m, 114800000ull, 21657, 1.0, 1, 0, rp.data(), ci.data(), v.data()) != GESPMM_OK) return 1;
  printf("nnz %lu, hw threads %u, packing threads %d\n", nnz, std::thread::hardware_concurrency(), threads);
  std::vector<uint32_t> b(blocks + 1);
  b[0] = 0; b[blocks] = m;
  for (int i = 1; i < blocks; ++i) b[i] = std::lower_bound(rp.begin(), rp.end(), uint32_t(nnz * i / blocks)) - rp.begin();
  std::vector<uint16_t> enc(nnz);
  std::vector<uint32_t> exc(nnz / 4 + 2);
  for (int rep = 0; rep < 3; ++rep) {
    const double t0 = now_ms();
    for (int c = 0; c < blocks; ++c)
      gespmm::pack_cols_block(rp.data(), ci.data(), b[c], b[c + 1], enc.data() + rp[b[c]], exc.data(), nnz / 8);
    const double t1 = now_ms();
    printf("u16 : %.2f ms total, %.3f ms per block, %.3f B/nnz\n", t1 - t0, (t1 - t0) / blocks, 2.0);
  }
  {
    std::vector<uint16_t> enc2(nnz);
    for (int isa = 1; isa <= 3; ++isa) {
      if (isa == 2 && !__builtin_cpu_supports("avx2")) continue;
      if (isa == 3 && !__builtin_cpu_supports("avx512bw")) continue;
      for (int rep = 0; rep < 3; ++rep) {
        const double ms = pack_fast_all(rp, ci, b, blocks, threads, enc2, isa);
        printf("u16 fast isa%d: %.2f ms total, %.3f ms per block%s\n", isa, ms, ms / blocks,
               rep == 2 ? (memcmp(enc2.data(), enc.data(), 2 * nnz) ? " MISMATCH" : " (== u16)") : "");
      }
    }
  }
  // pfor: chunk-aligned thread ranges within each block
  std::vector<uint32_t> words(nnz / 2 + 64 * 16);
  std::vector<uint16_t> side(nnz);
  std::vector<uint8_t> wv((nnz + 2047) / 2048 + blocks);
  for (int rep = 0; rep < 3; ++rep) {
    const double t0 = now_ms();
    uint64_t code_bytes = 0, side_n = 0, whist[17] = {0};
    for (int c = 0; c < blocks; ++c) {
      const uint64_t ps = rp[b[c]], pe = rp[b[c + 1]];
      const uint64_t nch = (pe - ps + 2047) / 2048;
      std::vector<uint64_t> tb(threads, 0), ts(threads, 0);
#pragma omp parallel num_threads(threads)
      {
        const int t = omp_get_thread_num();
        const uint64_t c0 = nch * t / threads, c1 = nch * (t + 1) / threads;
        uint32_t row = uint32_t(std::upper_bound(rp.begin() + b[c], rp.begin() + b[c + 1] + 1, uint32_t(ps + c0 * 2048)) - rp.begin()) - 1;
        uint32_t* wp = words.data() + (ps + c0 * 2048) / 2;   // worst case 16 bits per position
        uint16_t* sp = side.data() + ps + c0 * 2048;
        uint64_t bytes = 0, ns = 0;
        for (uint64_t ch = c0; ch < c1; ++ch) {
          const uint64_t p0 = ps + ch * 2048;
          const uint32_t len = uint32_t(std::min<uint64_t>(2048, pe - p0));
          uint32_t n_side = 0;
          uint8_t w = 0;
          const uint32_t by = pfor_chunk(rp.data(), ci.data(), p0, len, row, wp, sp, n_side, w);
          wp += by / 4; sp += n_side; bytes += by; ns += n_side;
          wv[ch] = w;
        }
        tb[t] = bytes; ts[t] = ns;
      }
      for (int t = 0; t < threads; ++t) { code_bytes += tb[t]; side_n += ts[t]; }
      for (uint64_t ch = 0; ch < nch; ++ch) whist[wv[ch]]++;
    }
    const double t1 = now_ms();
    printf("pfor: %.2f ms total, %.3f ms per block, %.3f B/nnz (codes %.3f + side %.3f)\n", t1 - t0, (t1 - t0) / blocks,
           (code_bytes + 2.0 * side_n) / nnz, double(code_bytes) / nnz, 2.0 * side_n / nnz);
    if (rep == 0) { printf("  width histogram (chunks):"); for (int w = 1; w <= 16; ++w) printf(" %d:%lu", w, whist[w]); printf("\n"); }
  }
  return 0;
}
