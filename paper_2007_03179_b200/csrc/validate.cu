// Device-side canonical-CSR check.  Restates the invariants of the reference's
// validate() (/root/reference/proj/include/spmm/csr.hpp:112-153) as two
// data-parallel passes; the host (api.cu) turns the minima found here into the
// reference's first-violation message, in the reference's check order.
#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

struct Scratch {
  unsigned int first_decrease;
  unsigned int pad;
  unsigned long long first_bad_key;
  unsigned int bad_row;
  unsigned int bad_col;
};

// pass 1: row_ptr non-decreasing; first index i with row_ptr[i] < row_ptr[i-1]
__global__ void k_check_rowptr(const uint32_t* __restrict__ rp, uint32_t m, Scratch* s) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x + 1; i <= m;
       i += gridDim.x * blockDim.x) {
    if (rp[i] < rp[i - 1]) atomicMin(&s->first_decrease, i);
  }
}

// pass 2 (warp per row): every column in bounds and strictly increasing.
// Key 2p marks "out of bounds" at p, 2p+1 "not increasing" at p, so the
// minimum key is the reference's first violation (it checks bounds first).
__global__ void k_check_cols(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                             uint32_t m, uint32_t k, uint64_t usable, Scratch* s) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const uint64_t start = rp[r];
    uint64_t end = rp[r + 1];
    if (end > usable) end = usable;
    for (uint64_t p = start + lane; p < end; p += 32) {
      const uint32_t c = ci[p];
      unsigned long long key = ~0ull;
      if (c >= k) key = 2ull * p;
      else if (p > start && c <= ci[p - 1]) key = 2ull * p + 1;
      if (key != ~0ull) atomicMin(&s->first_bad_key, key);
    }
  }
}

// locate the row holding the first bad position (binary search over row_ptr)
__global__ void k_locate(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                         uint32_t m, Scratch* s) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (s->first_bad_key == ~0ull) return;
  const uint64_t p = s->first_bad_key >> 1;
  uint32_t lo = 0, hi = m;  // last r with rp[r] <= p and rp[r+1] > p
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (rp[mid] <= p) lo = mid; else hi = mid;
  }
  while (lo + 1 < m && rp[lo + 1] <= p) ++lo;  // skip empty rows sharing the offset
  s->bad_row = lo;
  s->bad_col = ci[p];
}

}  // namespace

cudaError_t validate_csr_device(uint32_t m, uint32_t k, uint64_t nnz, const uint32_t* row_ptr,
                                const uint32_t* col_ind, ValidateResult* out, cudaStream_t st) {
  Scratch* s = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&s), sizeof(Scratch), st);
  if (e != cudaSuccess) return e;
  Scratch init{0xffffffffu, 0u, ~0ull, 0u, 0u};
  e = cudaMemcpyAsync(s, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  uint32_t ends[2] = {0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ends[0], row_ptr, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ends[1], row_ptr + m, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && m > 0) {
    const uint32_t blocks = (m + 255) / 256 < 4096 ? (m + 255) / 256 : 4096;
    k_check_rowptr<<<blocks, 256, 0, st>>>(row_ptr, m, s);
    note_launch();
    e = cudaGetLastError();
  }
  Scratch host{};
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, s, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && host.first_decrease == 0xffffffffu && m > 0) {
    const uint64_t usable = ends[1] < nnz ? ends[1] : nnz;
    const uint64_t warps_needed = m;
    uint64_t blocks = (warps_needed + 7) / 8;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    k_check_cols<<<uint32_t(blocks), 256, 0, st>>>(row_ptr, col_ind, m, k, usable, s);
    k_locate<<<1, 32, 0, st>>>(row_ptr, col_ind, m, s);
    note_launch();
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(&host, s, sizeof(host), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFreeAsync(s, st);
  out->row_ptr0 = ends[0];
  out->row_ptr_last = ends[1];
  out->first_decrease = host.first_decrease;
  out->first_bad_key = host.first_bad_key;
  out->bad_row = host.bad_row;
  out->bad_col = host.bad_col;
  return e;
}

// ---- chunked column check (the host pipeline validates row blocks as their
// col_ind arrives; row_ptr itself is checked on the host) --------------------
struct ColCheck {
  Scratch* s = nullptr;
};

cudaError_t colcheck_begin(ColCheck** out, cudaStream_t st) {
  auto* c = new ColCheck();
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&c->s), sizeof(Scratch), st);
  if (e == cudaSuccess) {
    static const Scratch init{0xffffffffu, 0u, ~0ull, 0u, 0u};
    e = cudaMemcpyAsync(c->s, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  }
  if (e != cudaSuccess) {
    delete c;
    return e;
  }
  *out = c;
  return cudaSuccess;
}

cudaError_t colcheck_rows(ColCheck* c, const uint32_t* row_ptr_chunk, uint32_t m_chunk,
                          const uint32_t* col_ind, uint32_t k, uint64_t usable, cudaStream_t st) {
  if (m_chunk == 0) return cudaSuccess;
  uint64_t blocks = (uint64_t(m_chunk) + 7) / 8;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  k_check_cols<<<uint32_t(blocks), 256, 0, st>>>(row_ptr_chunk, col_ind, m_chunk, k, usable, c->s);
  note_launch();
  return cudaGetLastError();
}

cudaError_t colcheck_end(ColCheck* c, const uint32_t* row_ptr, const uint32_t* col_ind, uint32_t m,
                         uint64_t* first_bad_key, uint32_t* bad_row, uint32_t* bad_col,
                         cudaStream_t st) {
  Scratch host{};
  cudaError_t e = cudaSuccess;
  if (m > 0) {
    k_locate<<<1, 32, 0, st>>>(row_ptr, col_ind, m, c->s);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, c->s, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(c->s, st);
  delete c;
  *first_bad_key = e == cudaSuccess ? host.first_bad_key : ~0ull;
  *bad_row = host.bad_row;
  *bad_col = host.bad_col;
  return e;
}

}  // namespace gespmm
