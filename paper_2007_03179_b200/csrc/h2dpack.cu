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

// Three passes over 2048-element chunks (one 256-thread CTA per chunk, 8
// consecutive elements per thread): per-chunk aggregates, one CTA scanning
// the aggregates into carries, then the chunk-local scan with its carry.  (A
// single cub::DeviceScan over a transform iterator of this 8-byte pair ran
// at ~80 G elements/s, 91 us per Reddit block; this reads the codes twice
// and writes the columns once.)
constexpr int kUnpackThreads = 256;
constexpr int kUnpackItems = 8;
constexpr uint32_t kUnpackChunk = kUnpackThreads * kUnpackItems;

using BlockScanT = cub::BlockScan<SegVal, kUnpackThreads>;
using BlockLoadT = cub::BlockLoad<uint16_t, kUnpackThreads, kUnpackItems, cub::BLOCK_LOAD_WARP_TRANSPOSE>;
using BlockStoreT = cub::BlockStore<uint32_t, kUnpackThreads, kUnpackItems, cub::BLOCK_STORE_WARP_TRANSPOSE>;
union UnpackSmem {
  typename BlockScanT::TempStorage scan;
  typename BlockLoadT::TempStorage load;
  typename BlockStoreT::TempStorage store;
};

// The chunk's codes, coalesced through shared memory into 8 consecutive
// elements per thread, decoded (row-start bit, escapes from col).
__device__ __forceinline__ void load_decode(const Decode& d, uint64_t len, UnpackSmem& sm,
                                            SegVal (&x)[kUnpackItems]) {
  const uint64_t c0 = uint64_t(blockIdx.x) * kUnpackChunk;
  const uint64_t rem = len - c0;
  const int valid = int(rem < kUnpackChunk ? rem : kUnpackChunk);
  uint16_t e[kUnpackItems];
  BlockLoadT(sm.load).Load(d.enc + c0, e, valid, uint16_t(0));
  __syncthreads();
  const uint64_t i0 = c0 + uint64_t(threadIdx.x) * kUnpackItems;
#pragma unroll
  for (int j = 0; j < kUnpackItems; ++j) {
    const uint64_t i = i0 + j;
    if (i >= len) {
      x[j] = SegVal{0u, 0u};
      continue;
    }
    const uint64_t p = d.ps + i;
    const bool first = (d.bits[p >> 5] >> (p & 31u)) & 1u;
    x[j] = e[j] == 0xFFFFu ? SegVal{d.col[p], 1u}
                           : (first ? SegVal{e[j], 1u} : SegVal{uint32_t(e[j]) + 1u, 0u});
  }
}

__global__ void __launch_bounds__(kUnpackThreads) k_unpack_agg(Decode d, uint64_t len,
                                                               SegVal* __restrict__ aggs) {
  __shared__ UnpackSmem sm;
  SegVal x[kUnpackItems];
  load_decode(d, len, sm, x);
  SegVal t{0u, 0u};
#pragma unroll
  for (int j = 0; j < kUnpackItems; ++j) t = SegAdd{}(t, x[j]);
  SegVal incl, total;
  BlockScanT(sm.scan).InclusiveScan(t, incl, SegAdd{}, total);
  if (threadIdx.x == 0) aggs[blockIdx.x] = total;
}

struct RunningPrefix {
  SegVal run;
  __device__ SegVal operator()(SegVal block_total) {
    const SegVal old = run;
    run = SegAdd{}(run, block_total);
    return old;
  }
};

// one CTA: exclusive segmented scan of the chunk aggregates (identity {0, 0}),
// 2048 aggregates per round (8 consecutive per thread)
__global__ void __launch_bounds__(kUnpackThreads) k_unpack_carry(const SegVal* __restrict__ aggs,
                                                                 uint32_t n, SegVal* __restrict__ carry) {
  __shared__ typename BlockScanT::TempStorage tmp;
  RunningPrefix pre{SegVal{0u, 0u}};
  for (uint32_t base = 0; base < n; base += kUnpackChunk) {
    const uint32_t c0 = base + threadIdx.x * kUnpackItems;
    SegVal x[kUnpackItems], ex[kUnpackItems];
#pragma unroll
    for (int j = 0; j < kUnpackItems; ++j)
      x[j] = c0 + j < n ? aggs[c0 + j] : SegVal{0u, 0u};
    BlockScanT(tmp).ExclusiveScan(x, ex, SegAdd{}, pre);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kUnpackItems; ++j)
      if (c0 + j < n) carry[c0 + j] = ex[j];
  }
}

// Writes the block's columns; with bad_key also runs the column part of the
// canonical check on them (k_check_positions' job, without re-reading col_ind):
// key 2p = column out of range at p, 2p + 1 = not increasing within its row.
__global__ void __launch_bounds__(kUnpackThreads) k_unpack_apply(Decode d, uint64_t len,
                                                                 const SegVal* __restrict__ carry,
                                                                 uint32_t* __restrict__ col,
                                                                 uint32_t k_cols,
                                                                 unsigned long long* bad_key) {
  __shared__ UnpackSmem sm;
  SegVal x[kUnpackItems];
  load_decode(d, len, sm, x);
  SegVal t{0u, 0u};
#pragma unroll
  for (int j = 0; j < kUnpackItems; ++j) t = SegAdd{}(t, x[j]);
  RunningPrefix pre{carry[blockIdx.x]};
  SegVal ex;
  BlockScanT(sm.scan).ExclusiveScan(t, ex, SegAdd{}, pre);
  uint32_t out[kUnpackItems];
  SegVal run = ex;
  unsigned long long worst = ~0ull;
  const uint64_t i0 = uint64_t(blockIdx.x) * kUnpackChunk + uint64_t(threadIdx.x) * kUnpackItems;
#pragma unroll
  for (int j = 0; j < kUnpackItems; ++j) {
    const uint32_t prev = run.v;  // the previous position's column
    run = SegAdd{}(run, x[j]);
    out[j] = run.v;
    if (bad_key && i0 + j < len) {
      const uint64_t p = d.ps + i0 + j;
      const bool first = (d.bits[p >> 5] >> (p & 31u)) & 1u;
      if (run.v >= k_cols) worst = min(worst, 2ull * p);
      else if (!first && run.v <= prev) worst = min(worst, 2ull * p + 1);
    }
  }
  if (bad_key) {
    for (int o = 16; o; o >>= 1) worst = min(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    if ((threadIdx.x & 31) == 0 && worst != ~0ull) atomicMin(bad_key, worst);
  }
  __syncthreads();  // scan storage is reused by the store
  const uint64_t c0 = uint64_t(blockIdx.x) * kUnpackChunk;
  const uint64_t rem = len - c0;
  BlockStoreT(sm.store).Store(col + d.ps + c0, out, int(rem < kUnpackChunk ? rem : kUnpackChunk));
}

}  // namespace

size_t unpack_temp_bytes(uint64_t max_len) {
  const uint64_t chunks = (max_len + kUnpackChunk - 1) / kUnpackChunk;
  return size_t(2 * chunks + 2) * sizeof(SegVal);
}

cudaError_t unpack_cols(const uint16_t* enc, const uint2* exc, uint32_t n_exc,
                        const uint32_t* row_ptr_block, uint32_t m_block, uint64_t ps, uint64_t pe,
                        uint64_t nnz, uint32_t* bits, uint32_t* col, void* temp, size_t temp_bytes,
                        cudaStream_t st, uint32_t k_cols, unsigned long long* bad_key) {
  if (pe <= ps) return cudaSuccess;
  const uint64_t len = pe - ps;
  const uint64_t chunks = (len + kUnpackChunk - 1) / kUnpackChunk;
  if (chunks > 0x7fffffffull || temp_bytes < size_t(2 * chunks) * sizeof(SegVal))
    return cudaErrorInvalidValue;
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
  SegVal* aggs = static_cast<SegVal*>(temp);
  SegVal* carry = aggs + chunks;
  const Decode d{enc, col, bits, ps};
  k_unpack_agg<<<uint32_t(chunks), kUnpackThreads, 0, st>>>(d, len, aggs);
  k_unpack_carry<<<1, kUnpackThreads, 0, st>>>(aggs, uint32_t(chunks), carry);
  k_unpack_apply<<<uint32_t(chunks), kUnpackThreads, 0, st>>>(d, len, carry, col, k_cols, bad_key);
  note_launch();
  note_launch();
  note_launch();
  return cudaGetLastError();
}

}  // namespace gespmm
