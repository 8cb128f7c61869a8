// Relocated hot rows: a frequency-chosen L2 working set for B (plan-time
// inspector + a per-execute row copy).
//
// When B is much larger than the 126 MB L2 (ogbn-products at N = 256: 2.5 GB),
// gathering every B row with evict_last makes L2 an LRU over B rows, and on a
// power-law column distribution LRU holds ~46% of the gathers in ~100 MB where
// the static top-by-frequency set of the same size holds ~60% (Che's
// approximation for the products generator; ncu: 45% measured).  The plan
// counts the gathers per column, picks the most-gathered columns whose rows fit
// a byte budget, and keeps
//   * a remapped copy of col_ind: a hot column becomes (1 << 31) | slot,
//     every other entry is unchanged (positions, and with them the fold order
//     and every result bit, are untouched);
//   * a contiguous buffer for those rows, refreshed from B at every execute
//     (one coalesced gather-copy: ~2 x budget bytes).
// The warp kernel then loads relocated rows from the buffer with evict_last
// and all others from B with evict_first: hot and cold are told apart by the
// staged column word itself, with no lookup (the experimental bitmap map,
// hotcols.cu, paid a dependent bitmap load per staged column and measured
// slower, profiles/r1_hot_map_v4.txt).
#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

constexpr uint32_t kHistBins = 1u << 16;  // column-count histogram, counts clipped
constexpr uint32_t kRelocBit = 0x80000000u;

__global__ void k_reloc_counts(const uint32_t* __restrict__ ci, uint64_t nnz,
                               uint32_t* __restrict__ counts) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(counts + __ldg(ci + i), 1u);
}

__global__ void k_reloc_hist(const uint32_t* __restrict__ counts, uint32_t k,
                             uint32_t* __restrict__ hist) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x)
    atomicAdd(hist + min(counts[c], kHistBins - 1), 1u);
}

// col'[i] = slot_of[col[i]] == ~0 ? col[i] : kRelocBit | slot
__global__ void k_reloc_remap(const uint32_t* __restrict__ ci, uint64_t nnz,
                              const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = __ldg(ci + i);
    const uint32_t s = __ldg(slot_of + c);
    out[i] = s == 0xffffffffu ? c : (kRelocBit | s);
  }
}

// b_hot[s][0:n] = b[list[s]][0:n]; one warp per row, VEC-wide lanes; the copy
// is written evict_last so the first gathers find it in L2.
template <int VEC>
__global__ void __launch_bounds__(256) k_reloc_refresh(const float* __restrict__ b, uint32_t ldb,
                                                       uint32_t n, const uint32_t* __restrict__ list,
                                                       uint32_t n_hot, float* __restrict__ out,
                                                       uint32_t ldh) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t keep;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  for (uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < n_hot;
       s += (gridDim.x * blockDim.x) >> 5) {
    const float* src = b + uint64_t(__ldg(list + s)) * ldb;
    float* dst = out + uint64_t(s) * ldh;
    for (uint32_t c = lane * VEC; c < n; c += 32 * VEC) {
      if constexpr (VEC == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src + c));
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst + c),
                     "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(keep)
                     : "memory");
      } else {
        const float v = __ldg(src + c);
        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(dst + c), "f"(v), "l"(keep)
                     : "memory");
      }
    }
  }
}

}  // namespace

cudaError_t build_hot_rows(const uint32_t* col_ind, uint64_t nnz, uint32_t k, uint32_t n,
                           uint64_t budget_rows, cudaStream_t st, HotRows* out) {
  *out = HotRows{};
  if (k == 0 || nnz == 0 || k >= kRelocBit || budget_rows == 0) return cudaSuccess;
  uint32_t *counts = nullptr, *hist = nullptr, *slot_of = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&counts), sizeof(uint32_t) * k);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&hist), sizeof(uint32_t) * kHistBins);
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * k, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kHistBins, st);
  std::vector<uint32_t> h(kHistBins), cnt(k);
  if (e == cudaSuccess) {
    k_reloc_counts<<<148 * 8, 256, 0, st>>>(col_ind, nnz, counts);
    k_reloc_hist<<<148 * 4, 256, 0, st>>>(counts, k, hist);
    note_launch();
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h.data(), hist, sizeof(uint32_t) * kHistBins, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(cnt.data(), counts, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  HotRows r;
  std::vector<uint32_t> slots, list;
  if (e == cudaSuccess) {
    // threshold t: the smallest count whose columns (count >= t) still fit the
    // budget; columns gathered at most once are never relocated
    uint64_t cols = 0;
    uint32_t t = kHistBins;
    for (uint32_t c = kHistBins - 1; c >= 2; --c) {
      if (cols + h[c] > budget_rows) break;
      cols += h[c];
      t = c;
    }
    slots.assign(k, 0xffffffffu);
    uint64_t gathered = 0;
    for (uint32_t c = 0; c < k; ++c)
      if (cnt[c] >= t) {
        slots[c] = uint32_t(list.size());
        list.push_back(c);
        gathered += cnt[c];
      }
    r.threshold = t;
    r.n_hot = uint32_t(list.size());
    r.hot_nnz_frac = double(gathered) / double(nnz);
  }
  if (e == cudaSuccess && r.n_hot) {
    r.ldh = n;
    e = cudaMalloc(reinterpret_cast<void**>(&slot_of), sizeof(uint32_t) * k);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&r.list), sizeof(uint32_t) * r.n_hot);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&r.col_ind), sizeof(uint32_t) * nnz);
    if (e == cudaSuccess)
      // one spare row: the copy starts at the offset congruent to B modulo the
      // row stride (place_hot_rows), so its rows are whole signed row offsets from B
      e = cudaMalloc(reinterpret_cast<void**>(&r.buf), sizeof(float) * uint64_t(r.n_hot + 1) * r.ldh);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(slot_of, slots.data(), sizeof(uint32_t) * k, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(r.list, list.data(), sizeof(uint32_t) * r.n_hot, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      k_reloc_remap<<<148 * 8, 256, 0, st>>>(col_ind, nnz, slot_of, r.col_ind);
      note_launch();
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (counts) cudaFree(counts);
  if (hist) cudaFree(hist);
  if (slot_of) cudaFree(slot_of);
  if (e != cudaSuccess) {
    free_hot_rows(&r);
    return e;
  }
  *out = r;
  return cudaSuccess;
}

bool place_hot_rows(const HotRows& h, const float* b, uint32_t ldb, const float** b_hot,
                    int32_t* hot_off) {
  if (!h.n_hot || ldb != h.ldh) return false;
  const uint64_t stride = uint64_t(ldb) * sizeof(float);
  const uint64_t bb = reinterpret_cast<uintptr_t>(b), base = reinterpret_cast<uintptr_t>(h.buf);
  const uint64_t shift = (bb % stride + stride - base % stride) % stride;  // base + shift = b (mod stride)
  const int64_t hot = int64_t(base + shift);
  const int64_t off = (hot - int64_t(bb)) / int64_t(stride);
  if (off < INT32_MIN || off + int64_t(h.n_hot) > INT32_MAX) return false;
  if (uint64_t(h.n_hot) * stride >= (1ull << 32)) return false;  // range policy sizes are 32-bit
  *b_hot = reinterpret_cast<const float*>(uintptr_t(hot));
  *hot_off = int32_t(off);
  return true;
}

cudaError_t refresh_hot_rows(const HotRows& h, const float* b, uint32_t ldb, uint32_t n,
                             const float* b_hot, cudaStream_t st) {
  if (!h.n_hot) return cudaSuccess;
  const bool v4 = n % 4 == 0 && ldb % 4 == 0 && (reinterpret_cast<uintptr_t>(b) & 15u) == 0 &&
                  (reinterpret_cast<uintptr_t>(b_hot) & 15u) == 0;
  const uint32_t blocks = std::min<uint32_t>((h.n_hot + 7) / 8, 148u * 8u);
  if (v4)
    k_reloc_refresh<4><<<blocks, 256, 0, st>>>(b, ldb, n, h.list, h.n_hot,
                                                const_cast<float*>(b_hot), ldb);
  else
    k_reloc_refresh<1><<<blocks, 256, 0, st>>>(b, ldb, n, h.list, h.n_hot,
                                                const_cast<float*>(b_hot), ldb);
  note_launch();
  return cudaGetLastError();
}

void free_hot_rows(HotRows* h) {
  if (h->col_ind) cudaFree(h->col_ind);
  if (h->list) cudaFree(h->list);
  if (h->buf) cudaFree(h->buf);
  *h = HotRows{};
}

}  // namespace gespmm
