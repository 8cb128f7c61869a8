// Frequency-aware L2 policy for the gathered B rows (plan-time inspector).
//
// When B is larger than what L2 can keep (ogbn-products at N=256: 2.5 GB of B
// against a 126 MB L2), marking every B load evict_last degenerates to LRU
// among B rows, and on a power-law column distribution LRU keeps many rows that
// are touched once.  The plan counts how often each column is gathered,
// picks the most-gathered columns whose rows fit a byte budget ("hot"), and
// emits a K-bit bitmap.  The warp kernel looks the bit up once per staged
// nonzero (phase 1 of the row cache) and gathers hot rows with evict_last and
// cold rows with evict_first, which approaches the static-optimal cache
// (top-C by frequency) instead of LRU.  Results are unaffected: this only
// changes cache-replacement hints.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

constexpr uint32_t kHistBins = 1u << 16;  // column-count histogram, counts clipped

__global__ void k_col_counts(const uint32_t* __restrict__ ci, uint64_t nnz,
                             uint32_t* __restrict__ counts) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(counts + __ldg(ci + i), 1u);
}

__global__ void k_count_hist(const uint32_t* __restrict__ counts, uint32_t k,
                             uint32_t* __restrict__ hist) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x)
    atomicAdd(hist + min(counts[c], kHistBins - 1), 1u);
}

// One thread per bitmap word: bit c set when column c is hot (count >= t).
__global__ void k_hot_bits(const uint32_t* __restrict__ counts, uint32_t k, uint32_t t,
                           uint32_t* __restrict__ bits) {
  const uint32_t words = (k + 31) / 32;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (uint32_t j = 0; j < 32; ++j) {
      const uint32_t c = w * 32 + j;
      if (c < k && counts[c] >= t) v |= 1u << j;
    }
    bits[w] = v;
  }
}

}  // namespace

cudaError_t build_hot_bitmap(const uint32_t* col_ind, uint64_t nnz, uint32_t k,
                             uint64_t budget_rows, cudaStream_t st, uint32_t** out_bits,
                             HotStats* stats) {
  *out_bits = nullptr;
  *stats = HotStats{};
  if (k == 0 || nnz == 0) return cudaSuccess;
  uint32_t *counts = nullptr, *hist = nullptr, *bits = nullptr;
  const uint32_t words = (k + 31) / 32;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(uint32_t) * k, st);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&hist), sizeof(uint32_t) * kHistBins, st);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&bits), sizeof(uint32_t) * words);
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * k, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kHistBins, st);
  std::vector<uint32_t> h(kHistBins);
  if (e == cudaSuccess) {
    k_col_counts<<<148 * 8, 256, 0, st>>>(col_ind, nnz, counts);
    k_count_hist<<<148 * 4, 256, 0, st>>>(counts, k, hist);
    note_launch();
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h.data(), hist, sizeof(uint32_t) * kHistBins, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    // threshold t: the smallest count whose columns (count >= t) still fit the
    // budget; columns of count 0 are never gathered and never hot.
    uint64_t cols = 0, gathered = 0;
    uint32_t t = kHistBins;
    for (uint32_t c = kHistBins - 1; c >= 1; --c) {
      if (cols + h[c] > budget_rows) break;
      cols += h[c];
      gathered += uint64_t(h[c]) * c;  // clipped bin undercounts: stats only
      t = c;
    }
    stats->threshold = t;
    stats->hot_cols = cols;
    stats->hot_nnz_frac = double(gathered) / double(nnz);
    k_hot_bits<<<(words + 255) / 256, 256, 0, st>>>(counts, k, t, bits);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (counts) cudaFreeAsync(counts, st);
  if (hist) cudaFreeAsync(hist, st);
  if (e != cudaSuccess) {
    if (bits) cudaFree(bits);
    return e;
  }
  *out_bits = bits;
  return cudaSuccess;
}

}  // namespace gespmm
