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

// pass 2, position-parallel: every column in bounds and strictly increasing
// within its row.  Key 2p marks "out of bounds" at p, 2p+1 "not increasing"
// at p, so the minimum key is the reference's first violation (it checks
// bounds first).  Row starts come from a bitmap over positions (k_mark_starts),
// so a 20k-entry hub row costs the same as 600 short ones: one coalesced pass
// over col_ind, the predecessor from the neighbouring lane.
__global__ void k_mark_starts(const uint32_t* __restrict__ rp, uint32_t m, uint64_t usable,
                              uint32_t* __restrict__ bits) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = rp[r];
    if (p < usable) atomicOr(&bits[p >> 5], 1u << (p & 31));
  }
}

__global__ void k_check_positions(const uint32_t* __restrict__ ci, uint64_t ps, uint64_t pe,
                                  uint32_t k, const uint32_t* __restrict__ bits, Scratch* s) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  unsigned long long best = ~0ull;
  for (uint64_t base = (ps & ~31ull) + w0 * 32; base < pe; base += nwarps * 32) {
    const uint64_t p = base + lane;
    const bool in = p >= ps && p < pe;
    const uint32_t c = in ? ci[p] : 0u;
    uint32_t prev = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane == 0 && in && p > 0) prev = ci[p - 1];
    const bool start = (bits[base >> 5] >> lane) & 1u;
    if (in) {
      if (c >= k) best = min(best, 2ull * p);
      else if (!start && c <= prev) best = min(best, 2ull * p + 1);
    }
  }
  for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0 && best != ~0ull) atomicMin(&s->first_bad_key, best);
}

// bitmap of row starts + position check over [ps, pe) (positions global)
cudaError_t launch_colcheck(const uint32_t* rp, uint32_t m, const uint32_t* ci, uint32_t k,
                            uint64_t ps, uint64_t pe, uint64_t usable, uint32_t* bits, Scratch* s,
                            cudaStream_t st) {
  if (pe > usable) pe = usable;
  if (m == 0 || pe <= ps) return cudaSuccess;
  const uint64_t mb = (uint64_t(m) + 255) / 256;
  k_mark_starts<<<uint32_t(mb < 148 * 8 ? mb : 148 * 8), 256, 0, st>>>(rp, m, usable, bits);
  const uint64_t pb = (pe - ps + 255) / 256 + 1;
  k_check_positions<<<uint32_t(pb < 148 * 16 ? pb : 148 * 16), 256, 0, st>>>(ci, ps, pe, k, bits, s);
  note_launch();
  note_launch();
  return cudaGetLastError();
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
    uint32_t* bits = nullptr;
    const size_t bbytes = sizeof(uint32_t) * (usable / 32 + 1);
    e = cudaMallocAsync(reinterpret_cast<void**>(&bits), bbytes, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bits, 0, bbytes, st);
    if (e == cudaSuccess) e = launch_colcheck(row_ptr, m, col_ind, k, 0, usable, usable, bits, s, st);
    if (e == cudaSuccess) {
      k_locate<<<1, 32, 0, st>>>(row_ptr, col_ind, m, s);
      note_launch();
    }
    if (bits) cudaFreeAsync(bits, st);
    if (e == cudaSuccess) e = cudaGetLastError();
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
size_t colcheck_workspace_bytes(uint64_t nnz) {
  return 256 + sizeof(uint32_t) * (nnz / 32 + 1);
}

// `ws` (colcheck_workspace_bytes(nnz), caller-owned device memory, 256-byte
// aligned) holds the scratch minima and the bitmap: no allocation per call
// (stream-ordered allocations released at every sync made host calls stall).
cudaError_t colcheck_begin(ColCheck* c, uint64_t nnz, void* ws, cudaStream_t st) {
  c->scratch = ws;
  c->bits = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + 256);
  cudaError_t e = cudaMemsetAsync(c->bits, 0, sizeof(uint32_t) * (nnz / 32 + 1), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ws, 0xff, sizeof(Scratch), st);  // minima start at ~0
  return e;
}

unsigned long long* colcheck_key(ColCheck* c) {
  return &static_cast<Scratch*>(c->scratch)->first_bad_key;
}

cudaError_t colcheck_rows(ColCheck* c, const uint32_t* row_ptr_chunk, uint32_t m_chunk,
                          uint64_t ps, uint64_t pe, const uint32_t* col_ind, uint32_t k,
                          uint64_t usable, cudaStream_t st) {
  return launch_colcheck(row_ptr_chunk, m_chunk, col_ind, k, ps, pe, usable, c->bits,
                         static_cast<Scratch*>(c->scratch), st);
}

cudaError_t colcheck_end(ColCheck* c, const uint32_t* row_ptr, const uint32_t* col_ind, uint32_t m,
                         uint64_t* first_bad_key, uint32_t* bad_row, uint32_t* bad_col,
                         cudaStream_t st) {
  Scratch host{};
  cudaError_t e = cudaSuccess;
  if (m > 0) {
    k_locate<<<1, 32, 0, st>>>(row_ptr, col_ind, m, static_cast<Scratch*>(c->scratch));
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&host, c->scratch, sizeof(host), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  *first_bad_key = e == cudaSuccess ? host.first_bad_key : ~0ull;
  *bad_row = host.bad_row;
  *bad_col = host.bad_col;
  return e;
}

}  // namespace gespmm
