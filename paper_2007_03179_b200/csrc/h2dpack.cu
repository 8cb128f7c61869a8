// Packed column indices for the host entry's PCIe upload (device side).
//
// The host-buffer call is bound by the H2D copy (1.04 GB per Reddit step at
// ~55 GB/s).  Within a canonical CSR row the columns increase, so the host
// sends each col_ind block as 16-bit codes (h2dpack_host.cpp): the first
// entry of a row as its column, the others as (gap - 1), and 0xFFFF as an
// escape whose full 32-bit value travels in a small (position, value) list —
// lossless for ANY input, so non-canonical matrices still reach the device
// validation unchanged.  Here the block is rebuilt: exceptions are scattered
// into col_ind, then one segmented inclusive scan (segments restart at row
// starts — the validation's row-start bitmap — and at escapes) turns the codes
// back into columns.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/iterator/transform_output_iterator.h>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

struct SegVal {
  uint32_t v;
  uint32_t restart;
};

struct SegAdd {
  __host__ __device__ SegVal operator()(const SegVal& a, const SegVal& b) const {
    return b.restart ? b : SegVal{a.v + b.v, a.restart};
  }
};

struct Decode {
  const uint16_t* enc;
  const uint32_t* col;    // escaped values already scattered here
  const uint32_t* bits;   // row-start bitmap over global positions
  uint64_t ps;
  __host__ __device__ SegVal operator()(uint64_t i) const {
    const uint64_t p = ps + i;
    const uint32_t e = enc[i];
    const bool first = (bits[p >> 5] >> (p & 31u)) & 1u;
    if (e == 0xFFFFu) return SegVal{col[p], 1u};
    return first ? SegVal{e, 1u} : SegVal{e + 1u, 0u};
  }
};

struct TakeV {
  __host__ __device__ uint32_t operator()(const SegVal& s) const { return s.v; }
};

__global__ void k_scatter_exceptions(const uint2* __restrict__ exc, uint32_t n, uint64_t ps,
                                     uint32_t* __restrict__ col) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    col[ps + exc[i].x] = exc[i].y;
}

__global__ void k_mark_starts_p(const uint32_t* __restrict__ rp, uint32_t m, uint64_t usable,
                                uint32_t* __restrict__ bits) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < m;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = rp[r];
    if (p < usable) atomicOr(&bits[p >> 5], 1u << (p & 31));
  }
}

using DecodeIt = thrust::transform_iterator<Decode, thrust::counting_iterator<uint64_t>>;
using OutIt = thrust::transform_output_iterator<TakeV, uint32_t*>;

}  // namespace

size_t unpack_temp_bytes(uint64_t max_len) {
  size_t bytes = 0;
  DecodeIt in(thrust::counting_iterator<uint64_t>(0), Decode{nullptr, nullptr, nullptr, 0});
  OutIt out(static_cast<uint32_t*>(nullptr), TakeV{});
  cub::DeviceScan::InclusiveScan(nullptr, bytes, in, out, SegAdd{}, int(max_len));
  return bytes;
}

cudaError_t unpack_cols(const uint16_t* enc, const uint2* exc, uint32_t n_exc,
                        const uint32_t* row_ptr_block, uint32_t m_block, uint64_t ps, uint64_t pe,
                        uint64_t nnz, uint32_t* bits, uint32_t* col, void* temp, size_t temp_bytes,
                        cudaStream_t st) {
  if (pe <= ps) return cudaSuccess;
  if (pe - ps > 0x7fffffffull) return cudaErrorInvalidValue;
  const uint64_t mb = (uint64_t(m_block) + 255) / 256;
  if (m_block) {
    k_mark_starts_p<<<uint32_t(mb < 148 * 8 ? mb : 148 * 8), 256, 0, st>>>(row_ptr_block, m_block,
                                                                            nnz, bits);
    note_launch();
  }
  if (n_exc) {
    const uint32_t eb = (n_exc + 255) / 256;
    k_scatter_exceptions<<<eb < 148 * 8 ? eb : 148 * 8, 256, 0, st>>>(exc, n_exc, ps, col);
    note_launch();
  }
  DecodeIt in(thrust::counting_iterator<uint64_t>(0), Decode{enc, col, bits, ps});
  OutIt out(col + ps, TakeV{});
  size_t bytes = temp_bytes;
  cudaError_t e = cub::DeviceScan::InclusiveScan(temp, bytes, in, out, SegAdd{}, int(pe - ps), st);
  note_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace gespmm
