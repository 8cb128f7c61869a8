// GPU CSR transpose (A -> A^T as canonical CSR), for the GCN backward pass
// (grad_X = A^T · grad_Y).  The reference only has CPU COO round trips
// (/root/reference/proj/include/spmm/csr.hpp:58-104, from_coo/to_coo); this is
// the device equivalent of to_coo -> swap -> from_coo without duplicates.
//
// Deterministic: a *stable* LSD radix sort of (col, p) pairs keeps, inside each
// column, the nonzeros in ascending original position — i.e. ascending row —
// so A^T comes out canonical (strictly increasing columns per row) and
// identical run to run.
#include <cub/cub.cuh>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

// row index of every nonzero (warp per row)
__global__ void k_expand_rows(const uint32_t* __restrict__ rp, uint32_t m,
                              uint32_t* __restrict__ row_of) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const uint32_t s = rp[r], e = rp[r + 1];
    for (uint32_t p = s + lane; p < e; p += 32) row_of[p] = uint32_t(r);
  }
}

__global__ void k_iota(uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = uint32_t(i);
}

__global__ void k_count_cols(const uint32_t* __restrict__ ci, uint64_t nnz,
                             uint32_t* __restrict__ counts) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(counts + ci[i], 1u);
}

__global__ void k_gather_t(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ row_of,
                           const float* __restrict__ vals, uint64_t nnz,
                           uint32_t* __restrict__ t_col, float* __restrict__ t_val) {
  for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = perm[q];
    t_col[q] = row_of[p];
    t_val[q] = vals[p];
  }
}

int key_bits(uint32_t k) {
  int b = 1;
  while (b < 32 && (uint64_t(1) << b) < k) ++b;
  return b;
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

#define T_CUDA(call)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      for (void* p_ : bufs) if (p_) cudaFreeAsync(p_, st);                             \
      return set_error(e_ == cudaErrorMemoryAllocation ? GESPMM_ENOMEM : GESPMM_ECUDA, \
                       std::string("csr_transpose: CUDA error: ") + cudaGetErrorString(e_)); \
    }                                                                                  \
  } while (0)

extern "C" gespmm_status_t gespmm_csr_transpose_device(const gespmm_csr_t* a, uint32_t* t_row_ptr,
                                                       uint32_t* t_col_ind, float* t_vals,
                                                       void* stream) {
  if (!a) return set_error(GESPMM_EINVAL, "csr_transpose: null csr");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t nnz = a->nnz;
  const uint32_t m = a->n_rows, k = a->n_cols;
  if (nnz > 0xffffffffull) return set_error(GESPMM_EUNSUPPORTED, "csr_transpose: nnz >= 2^32");
  void* bufs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // counts -> exclusive scan -> t_row_ptr[0..k]
  uint32_t* counts = nullptr;
  T_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&counts), sizeof(uint32_t) * (size_t(k) + 1), st));
  bufs[0] = counts;
  T_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t(k) + 1), st));
  const int blocks = 148 * 8;
  if (nnz) {
    k_count_cols<<<blocks, 256, 0, st>>>(a->col_ind, nnz, counts);
    note_launch();
    T_CUDA(cudaGetLastError());
  }
  size_t scan_bytes = 0;
  T_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, t_row_ptr, int(k) + 1, st));
  void* scan_tmp = nullptr;
  T_CUDA(cudaMallocAsync(&scan_tmp, scan_bytes, st));
  bufs[1] = scan_tmp;
  T_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, t_row_ptr, int(k) + 1, st));
  note_launch();
  if (nnz) {
    uint32_t *row_of = nullptr, *idx_in = nullptr, *idx_out = nullptr, *keys_out = nullptr;
    T_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&row_of), sizeof(uint32_t) * nnz, st));
    bufs[2] = row_of;
    T_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&idx_in), sizeof(uint32_t) * nnz, st));
    bufs[3] = idx_in;
    T_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&idx_out), sizeof(uint32_t) * nnz, st));
    bufs[4] = idx_out;
    T_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&keys_out), sizeof(uint32_t) * nnz, st));
    bufs[5] = keys_out;
    k_expand_rows<<<blocks, 256, 0, st>>>(a->row_ptr, m, row_of);
    k_iota<<<blocks, 256, 0, st>>>(idx_in, nnz);
    note_launch();
    note_launch();
    T_CUDA(cudaGetLastError());
    size_t sort_bytes = 0;
    T_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, a->col_ind, keys_out, idx_in,
                                           idx_out, int64_t(nnz), 0, key_bits(k), st));
    void* sort_tmp = nullptr;
    T_CUDA(cudaMallocAsync(&sort_tmp, sort_bytes, st));
    T_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, a->col_ind, keys_out, idx_in,
                                           idx_out, int64_t(nnz), 0, key_bits(k), st));
    note_launch();
    cudaFreeAsync(sort_tmp, st);
    k_gather_t<<<blocks, 256, 0, st>>>(idx_out, row_of, a->vals, nnz, t_col_ind, t_vals);
    note_launch();
    T_CUDA(cudaGetLastError());
  }
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, st);
  return GESPMM_OK;
}
