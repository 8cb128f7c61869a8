// The paper's Algorithms 1-3 on sm_100a with the reference's launch geometry
// (/root/reference/proj/include/spmm/kernel.hpp:100-136): one warp per
// (row, column tile), warps numbered row-major, tile width 32*cf, lane l owns
// columns col_base + l + c*32 for c < cf, 8 warps per block.  These are the
// ablation baselines (naive -> CRC -> CRC+CWM) measured on B200; the product
// path is the tuned kernel in kernels_tuned.cu.  All three produce results
// bit-identical to the reference's ordered fold.
#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

constexpr int kWarpsPerBlock = 8;  // KernelConfig::warps_per_block (kernel.hpp:79)
constexpr int kBatch = 4;          // nonzeros gathered per batch in every variant

// Algorithm 1 (kernel.hpp:197-224): per nonzero, warp-uniform loads of the
// column index and value, then one unit-stride B load per lane.
template <int OP, bool FAST>
__global__ void __launch_bounds__(256) k_naive(SpmmArgs a) {
  if (aborted(a)) return;
  using R = Reduce<OP>;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t total = uint64_t(a.n_sched) * a.n_tiles;
  if (warp >= total) return;
  const Policies pol = make_policies(a.hints);
  const uint32_t row = uint32_t(warp / a.n_tiles);
  const uint32_t col = uint32_t(warp % a.n_tiles) * 32u + lane;
  const bool active = col < a.n;
  const uint32_t start = a.row_ptr[row];
  const uint32_t full_end = a.row_ptr[row + 1];
  const uint32_t end = faulted_end(start, full_end, a.skip_tail);
  float acc = R::init();
  int32_t who = -1;
  // Batches of kBatch nonzeros: the B loads of a batch are issued before any
  // fold (the same memory-level parallelism every variant gets, so the
  // ablation compares the algorithms, not the compiler's scheduling).  Every
  // load is predicated exactly like the reference's masks (past-the-end slots
  // and columns >= N issue nothing), so the kernel's L1 sector counts equal
  // the reference simulator's transaction counts (tools/sector_parity.py).
  const float* bcol = a.b + col;
  for (uint32_t p = start; p < end; p += kBatch) {
    uint32_t k[kBatch];
    float v[kBatch], bv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      k[u] = 0u;
      v[u] = 0.0f;
      if (p + u < end) {
        k[u] = __ldg(a.col_ind + p + u);  // warp-uniform (broadcast) loads
        v[u] = __ldg(a.vals + p + u);
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      bv[u] = 0.0f;
      if (active && p + u < end) bv[u] = ld_keep<1>(bcol + uint64_t(k[u]) * a.n, pol.keep).x[0];
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (active && p + u < end)
        R::template fold<FAST>(acc, who, v[u], bv[u], a.arg_col ? int32_t(k[u]) : int32_t(p + u));
  }
  if (active) {
    const uint64_t o = uint64_t(row) * a.n + col;
    acc = finish<OP>(acc, full_end - start);
    st_stream<1>(a.c + o, &acc, pol.stream);
    if (R::kHasArg && a.arg) st_stream_i32<1>(a.arg + o, &who, pol.stream);
  }
}

// Algorithms 2 and 3 (kernel.hpp:234-278, 287-343): phase 1 stages a 32-wide
// tile of (col, val) into the warp's shared tile with one coalesced load per
// array; phase 2 consumes it sequentially, each staged nonzero feeding CF
// column slices of 32 lanes.  CF = 1 is plain CRC.
template <int OP, bool FAST, int CF>
__global__ void __launch_bounds__(256) k_crc(SpmmArgs a) {
  if (aborted(a)) return;
  using R = Reduce<OP>;
  __shared__ uint32_t s_col[kWarpsPerBlock][32];
  __shared__ float s_val[kWarpsPerBlock][32];
  const uint32_t wib = threadIdx.x >> 5;
  const uint64_t warp = uint64_t(blockIdx.x) * kWarpsPerBlock + wib;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t total = uint64_t(a.n_sched) * a.n_tiles;
  if (warp >= total) return;  // warp-uniform
  const Policies pol = make_policies(a.hints);
  const uint32_t row = uint32_t(warp / a.n_tiles);
  const uint32_t col_base = uint32_t(warp % a.n_tiles) * (32u * CF);
  const uint32_t start = a.row_ptr[row];
  const uint32_t full_end = a.row_ptr[row + 1];
  const uint32_t end = faulted_end(start, full_end, a.skip_tail);

  float acc[CF];
  int32_t who[CF];
#pragma unroll
  for (int c = 0; c < CF; ++c) {
    acc[c] = R::init();
    who[c] = -1;
  }
  for (uint32_t ptr = start; ptr < end; ptr += 32) {
    const uint32_t tile_n = min(32u, end - ptr);
    if (lane < tile_n) {  // phase 1
      s_col[wib][lane] = ld_stream_u32(a.col_ind + ptr + lane, pol.stream);
      s_val[wib][lane] = ld_stream_f32(a.vals + ptr + lane, pol.stream);
    }
    __syncwarp();
    for (uint32_t kk = 0; kk < tile_n; kk += kBatch) {  // phase 2, kBatch at a time
      float bv[kBatch][CF];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const uint32_t k = s_col[wib][min(kk + u, tile_n - 1)];
        const float* brow = a.b + uint64_t(k) * a.n;
#pragma unroll
        for (int c = 0; c < CF; ++c) {
          const uint32_t col = col_base + c * 32u + lane;
          bv[u][c] = 0.0f;
          if (kk + u < tile_n && col < a.n) bv[u][c] = ld_keep<1>(brow + col, pol.keep).x[0];
        }
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (kk + u < tile_n) {
          const uint32_t k = s_col[wib][kk + u];
          const float v = s_val[wib][kk + u];
          const int32_t pos = a.arg_col ? int32_t(k) : int32_t(ptr + kk + u);
#pragma unroll
          for (int c = 0; c < CF; ++c)
            if (col_base + c * 32u + lane < a.n) R::template fold<FAST>(acc[c], who[c], v, bv[u][c], pos);
        }
      }
    }
    __syncwarp();
  }
  const uint32_t row_len = full_end - start;
#pragma unroll
  for (int c = 0; c < CF; ++c) {
    const uint32_t col = col_base + c * 32u + lane;
    if (col < a.n) {
      const uint64_t o = uint64_t(row) * a.n + col;
      float out = finish<OP>(acc[c], row_len);
      st_stream<1>(a.c + o, &out, pol.stream);
      if (R::kHasArg && a.arg) st_stream_i32<1>(a.arg + o, &who[c], pol.stream);
    }
  }
}

template <int OP, bool FAST>
cudaError_t launch_op(int variant, uint32_t cf, const SpmmArgs& a, cudaStream_t s) {
  const uint64_t warps = uint64_t(a.n_sched) * a.n_tiles;
  const uint64_t blocks64 = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks64 == 0) return cudaSuccess;
  if (blocks64 > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const dim3 grid{uint32_t(blocks64)}, block{32 * kWarpsPerBlock};
  if (variant == GESPMM_VARIANT_NAIVE) {
    k_naive<OP, FAST><<<grid, block, 0, s>>>(a);
  } else if (variant == GESPMM_VARIANT_CRC) {
    k_crc<OP, FAST, 1><<<grid, block, 0, s>>>(a);
  } else {
    switch (cf) {
      case 2: k_crc<OP, FAST, 2><<<grid, block, 0, s>>>(a); break;
      case 4: k_crc<OP, FAST, 4><<<grid, block, 0, s>>>(a); break;
      default: k_crc<OP, FAST, 8><<<grid, block, 0, s>>>(a); break;
    }
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace

uint32_t faithful_tiles(int variant, uint32_t cf, uint32_t n) {
  const uint32_t width = 32u * (variant == GESPMM_VARIANT_CRC_CWM ? cf : 1u);
  return (n + width - 1) / width;
}

cudaError_t launch_faithful(int variant, uint32_t cf, int op, bool fast, const SpmmArgs& a,
                            cudaStream_t s) {
  switch (op) {
    case kSum: return fast ? launch_op<kSum, true>(variant, cf, a, s)
                           : launch_op<kSum, false>(variant, cf, a, s);
    case kMean: return fast ? launch_op<kMean, true>(variant, cf, a, s)
                            : launch_op<kMean, false>(variant, cf, a, s);
    case kMax: return launch_op<kMax, false>(variant, cf, a, s);
    default: return launch_op<kMin, false>(variant, cf, a, s);
  }
}

}  // namespace gespmm
