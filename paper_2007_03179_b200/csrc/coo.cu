// Device COO <-> CSR: the reference's ingestion step (from_coo / to_coo,
// /root/reference/proj/include/spmm/csr.hpp:37-104) on HBM-resident triples,
// so a graph that arrives as an edge list (a GNN dataloader's output, a
// Matrix Market file streamed to the device) becomes the kernels' canonical
// CSR without a host round trip.
//
// from_coo semantics, bit for bit (csr.hpp:54-93):
//   * the first triple outside the declared bounds, in input order, is the
//     error (with the reference's message, formatted on the host);
//   * entries are ordered by (row, col) with a STABLE sort, so each duplicate
//     run keeps input order: Sum folds it left to right in fp32
//     (v = v + next), Last keeps the final occurrence.
// Layout of the work: one 64-bit key row * n_cols + col per triple, a stable
// LSD radix sort of (key, value) pairs over only the key's significant bits,
// run heads flagged and scanned into output slots, one thread per run doing
// the ordered fold (runs are short; an adversarial run is still exact, just
// serial) and writing row_ptr where the row changes.  Temporaries (~28 bytes per
// triple + cub's) live in a grow-only per-device scratch.
#include <cub/cub.cuh>

#include <mutex>
#include <sstream>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

__global__ void k_coo_bounds(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                             uint64_t n, uint32_t n_rows, uint32_t n_cols,
                             unsigned long long* __restrict__ first_bad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (rows[i] >= n_rows || cols[i] >= n_cols) atomicMin(first_bad, (unsigned long long)i);
}

__global__ void k_coo_keys(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ cols,
                           uint64_t n, uint32_t n_cols, uint64_t* __restrict__ keys) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    keys[i] = uint64_t(rows[i]) * n_cols + cols[i];
}

__global__ void k_coo_heads(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* __restrict__ head) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// One thread per run head: the ordered fold of the run into its slot (the
// exclusive scan of heads).  row_ptr comes out of the same pass without
// atomics: the output is row-sorted, so a head that starts a new row writes
// row_ptr for every row since the previous run's row (empty rows included),
// and the last element writes the rows after the last non-empty one.
__global__ void k_coo_runs(const uint64_t* __restrict__ keys, const float* __restrict__ vals,
                           const uint32_t* __restrict__ head, const uint32_t* __restrict__ slot,
                           uint64_t n, uint32_t n_rows, uint32_t n_cols, int last,
                           uint32_t* __restrict__ col_ind, float* __restrict__ out_vals,
                           uint32_t* __restrict__ row_ptr) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const uint32_t row = uint32_t(k / n_cols);
    if (i == n - 1) {
      const uint32_t total = slot[i] + head[i];
      for (uint32_t r = row + 1; r <= n_rows; ++r) row_ptr[r] = total;
    }
    if (!head[i]) continue;
    float v = vals[i];
    for (uint64_t j = i + 1; j < n && keys[j] == k; ++j) v = last ? vals[j] : __fadd_rn(v, vals[j]);
    const uint32_t p = slot[i];
    col_ind[p] = uint32_t(k - uint64_t(row) * n_cols);
    out_vals[p] = v;
    const uint32_t first = i ? uint32_t(keys[i - 1] / n_cols) + 1 : 0u;
    for (uint32_t r = first; r <= row; ++r) row_ptr[r] = p;
  }
}

__global__ void k_coo_expand(const uint32_t* __restrict__ rp, uint32_t m, uint32_t* __restrict__ rows) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const uint32_t s = rp[r], e = rp[r + 1];
    for (uint32_t p = s + lane; p < e; p += 32) rows[p] = uint32_t(r);
  }
}

int bits_for(uint64_t max_value) {
  int b = 1;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

uint32_t grid_for(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return uint32_t(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

// Grow-only device scratch per device (the call holds its mutex until its
// work is complete): per-call stream-ordered allocations of ~2 GB at the
// Reddit scale were returned to the OS at each synchronisation and made every
// call pay the mapping again (58 ms per call, 7.7 ms of it kernels).
struct CooScratch {
  std::mutex mu;
  void* buf = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (buf) cudaFree(buf);
    buf = nullptr;
    cap = 0;
    const cudaError_t e = cudaMalloc(&buf, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
};
std::mutex g_coo_mu;
CooScratch* g_coo[64] = {};

CooScratch* coo_scratch() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_coo_mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!g_coo[dev]) g_coo[dev] = new CooScratch();
  return g_coo[dev];
}

}  // namespace

void release_coo_scratch() {
  int dev = 0;
  cudaGetDevice(&dev);
  CooScratch* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_coo_mu);
    if (dev >= 0 && dev < 64) s = g_coo[dev];
  }
  if (!s) return;
  std::lock_guard<std::mutex> lk(s->mu);
  if (s->buf) cudaFree(s->buf);
  s->buf = nullptr;
  s->cap = 0;
}

namespace {

// carves aligned pieces out of one buffer
struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t bytes) {
    T* p = reinterpret_cast<T*>(base + off);
    off += (bytes + 255) & ~size_t(255);
    return p;
  }
};

}  // namespace
}  // namespace gespmm

using namespace gespmm;

#define COO_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return set_error(e_ == cudaErrorMemoryAllocation ? GESPMM_ENOMEM : GESPMM_ECUDA, \
                       std::string(what) + ": CUDA error: " + cudaGetErrorString(e_)); \
  } while (0)

extern "C" gespmm_status_t gespmm_from_coo_device(uint32_t n_rows, uint32_t n_cols, uint64_t count,
                                                  const uint32_t* rows, const uint32_t* cols,
                                                  const float* vals, int32_t policy,
                                                  uint32_t* row_ptr, uint32_t* col_ind,
                                                  float* out_vals, uint64_t* nnz, void* stream) {
  const char* what = "from_coo";
  if (policy != GESPMM_DEDUP_SUM && policy != GESPMM_DEDUP_LAST)
    return set_error(GESPMM_EINVAL, "from_coo: unknown dedup policy");
  if (count && (!rows || !cols || !vals || !col_ind || !out_vals))
    return set_error(GESPMM_EINVAL, "from_coo: null input");
  if (!row_ptr) return set_error(GESPMM_EINVAL, "from_coo: null row_ptr");
  if (count > 0xffffffffull)  // the reference's nnz is a u32 (csr.hpp:32)
    return set_error(GESPMM_EINVAL, "from_coo: more than 2^32-1 triples");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint32_t g = grid_for(count);
  // temporaries: sizes first (cub's size queries run on the host)
  const int end_bit = count ? bits_for(uint64_t(n_rows) * n_cols - 1) : 1;
  size_t sort_bytes = 0, scan_bytes = 0;
  COO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint64_t*)nullptr,
                                           (uint64_t*)nullptr, (const float*)nullptr,
                                           (float*)nullptr, int64_t(count ? count : 1), 0,
                                           end_bit, st));
  COO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const uint32_t*)nullptr,
                                         (uint32_t*)nullptr, int64_t(count ? count : 1), st));
  const auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t need = al(8) + 2 * al(8 * count) + al(4 * count) + 2 * al(4 * count) +
                      al(sort_bytes) + al(scan_bytes);
  CooScratch* ws = coo_scratch();
  if (!ws) return set_error(GESPMM_EINVAL, "from_coo: device ordinal out of range");
  std::lock_guard<std::mutex> lk(ws->mu);
  COO_CUDA(ws->reserve(need));
  Carve cv{static_cast<char*>(ws->buf)};
  auto* d_bad = cv.take<unsigned long long>(8);
  auto* k_in = cv.take<uint64_t>(8 * count);
  auto* k_out = cv.take<uint64_t>(8 * count);
  auto* v_out = cv.take<float>(4 * count);
  auto* head = cv.take<uint32_t>(4 * count);
  auto* slot = cv.take<uint32_t>(4 * count);
  void* sort_tmp = cv.take<char>(sort_bytes);
  void* scan_tmp = cv.take<char>(scan_bytes);
  // 1. bounds, first offender in input order (the reference's loop order)
  if (count) {
    COO_CUDA(cudaMemsetAsync(d_bad, 0xff, sizeof(unsigned long long), st));
    k_coo_bounds<<<g, 256, 0, st>>>(rows, cols, count, n_rows, n_cols, d_bad);
    note_launch();
    COO_CUDA(cudaGetLastError());
    unsigned long long bad = 0;
    COO_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
    COO_CUDA(cudaStreamSynchronize(st));
    if (bad != ~0ull) {
      uint32_t r = 0, c = 0;
      float v = 0.0f;
      COO_CUDA(cudaMemcpy(&r, rows + bad, sizeof(r), cudaMemcpyDeviceToHost));
      COO_CUDA(cudaMemcpy(&c, cols + bad, sizeof(c), cudaMemcpyDeviceToHost));
      COO_CUDA(cudaMemcpy(&v, vals + bad, sizeof(v), cudaMemcpyDeviceToHost));
      std::ostringstream os;  // operator<< formatting of the reference (csr.hpp:64-66)
      os << "coo entry (" << r << ", " << c << ", " << v << ") outside declared " << n_rows << "x"
         << n_cols << " bounds";
      return set_error(GESPMM_EINVAL, os.str());
    }
  }
  uint64_t total = 0;
  if (count) {
    // 2. stable sort of (row * n_cols + col, value) over the key's significant bits
    k_coo_keys<<<g, 256, 0, st>>>(rows, cols, count, n_cols, k_in);
    note_launch();
    COO_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, k_in, k_out, vals, v_out,
                                             int64_t(count), 0, end_bit, st));
    note_launch();
    // 3. run heads -> output slots
    k_coo_heads<<<g, 256, 0, st>>>(k_out, count, head);
    note_launch();
    COO_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, head, slot, int64_t(count), st));
    note_launch();
    // 4. ordered fold per run; row_ptr from the row changes between runs
    k_coo_runs<<<g, 256, 0, st>>>(k_out, v_out, head, slot, count, n_rows, n_cols,
                                  policy == GESPMM_DEDUP_LAST, col_ind, out_vals, row_ptr);
    note_launch();
    COO_CUDA(cudaGetLastError());
    uint32_t last_slot = 0, last_head = 0;
    COO_CUDA(cudaMemcpyAsync(&last_slot, slot + count - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    COO_CUDA(cudaMemcpyAsync(&last_head, head + count - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    COO_CUDA(cudaStreamSynchronize(st));  // *nnz, and the scratch is free again
    total = uint64_t(last_slot) + last_head;
  } else {
    COO_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(uint32_t) * (size_t(n_rows) + 1), st));
    COO_CUDA(cudaStreamSynchronize(st));
  }
  if (nnz) *nnz = total;
  return GESPMM_OK;
}

extern "C" gespmm_status_t gespmm_to_coo_device(const gespmm_csr_t* a, uint32_t* rows, uint32_t* cols,
                                                float* vals, void* stream) {
  const char* what = "to_coo";
  if (!a) return set_error(GESPMM_EINVAL, "to_coo: null csr");
  if (a->nnz && (!rows || !cols || !vals)) return set_error(GESPMM_EINVAL, "to_coo: null output");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!a->nnz) return GESPMM_OK;
  k_coo_expand<<<grid_for(uint64_t(a->n_rows) * 32), 256, 0, st>>>(a->row_ptr, a->n_rows, rows);
  note_launch();
  COO_CUDA(cudaGetLastError());
  COO_CUDA(cudaMemcpyAsync(cols, a->col_ind, sizeof(uint32_t) * a->nnz, cudaMemcpyDeviceToDevice, st));
  COO_CUDA(cudaMemcpyAsync(vals, a->vals, sizeof(float) * a->nnz, cudaMemcpyDeviceToDevice, st));
  return GESPMM_OK;
}
