// Diagnostic kernels for the roofline report (not on the SpMM path).
//
// k_gather: the pure gather ceiling of an index stream — for each idx[i] the
// warp reads row idx[i] of B (N = 128 floats, one float4 per lane) and adds it
// into a register accumulator: the L2->SM traffic of the SpMM with no multiply,
// no per-row output and no row structure.  Run on the SpMM's own col_ind it
// bounds what any kernel with one B-row gather per nonzero can reach.
#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

template <int U>
__global__ void __launch_bounds__(256, 3) k_gather(const uint32_t* __restrict__ idx,
                                                   uint64_t count, const float* __restrict__ b,
                                                   uint32_t n, float* __restrict__ sink,
                                                   int hints) {
  const Policies pol = make_policies(hints);
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t chunks = (count + 31) / 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (uint64_t ch = warp; ch < chunks; ch += warps) {
    const uint64_t base = ch * 32;
    const uint32_t mine = base + lane < count ? ld_stream_u32(idx + base + lane, pol.stream) : 0u;
    const uint64_t left = count - base;
    const uint32_t valid = left < 32 ? uint32_t(left) : 32u;
#pragma unroll 1
    for (uint32_t kk = 0; kk < 32; kk += U) {
      Vec<4> v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = __shfl_sync(0xffffffffu, mine, int(kk + u));
        v[u] = ld_keep<4>(b + uint64_t(k) * n + lane * 4, pol.keep);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (kk + u < valid)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] += v[u].x[e];
    }
  }
  sink[warp * 32 + lane] = acc[0] + acc[1] + acc[2] + acc[3];
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

extern "C" gespmm_status_t gespmm_diag_gather(const uint32_t* idx, uint64_t count,
                                              const float* b, uint32_t n, float* sink,
                                              int32_t blocks, int32_t hints, void* stream) {
  if (n != 128) return set_error(GESPMM_EUNSUPPORTED, "diag_gather: n must be 128");
  if (blocks <= 0) blocks = 148 * 3;
  k_gather<8><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(idx, count, b, n, sink,
                                                                     hints);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(GESPMM_ECUDA, std::string("diag_gather: CUDA error: ") + cudaGetErrorString(e));
  return GESPMM_OK;
}

// k_gather_hub: the same gather, but rows idx < hub_rows are served from a
// shared-memory copy of B's first hub_rows rows (loaded once per persistent
// CTA) — measures what a static smem hub cache buys over L1/L2 gathers.
namespace gespmm {
namespace {
template <int U>
__global__ void __launch_bounds__(1024, 1) k_gather_hub(const uint32_t* __restrict__ idx,
                                                        uint64_t count, const float* __restrict__ b,
                                                        uint32_t hub_rows, float* __restrict__ sink) {
  extern __shared__ __align__(16) float s_hub[];
  const Policies pol = make_policies(1);
  for (uint32_t i = threadIdx.x; i < hub_rows * 32u; i += blockDim.x)
    reinterpret_cast<float4*>(s_hub)[i] = reinterpret_cast<const float4*>(b)[i];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t chunks = (count + 31) / 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (uint64_t ch = warp; ch < chunks; ch += warps) {
    const uint64_t base = ch * 32;
    const uint32_t mine = base + lane < count ? ld_stream_u32(idx + base + lane, pol.stream) : 0u;
#pragma unroll 1
    for (uint32_t kk = 0; kk < 32; kk += U) {
      Vec<4> v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = __shfl_sync(0xffffffffu, mine, int(kk + u));
        if (k < hub_rows) {
          const float4 t = reinterpret_cast<const float4*>(s_hub)[k * 32u + lane];
          v[u].x[0] = t.x; v[u].x[1] = t.y; v[u].x[2] = t.z; v[u].x[3] = t.w;
        } else {
          v[u] = ld_keep<4>(b + uint64_t(k) * 128u + lane * 4, pol.keep);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] += v[u].x[e];
    }
  }
  sink[warp * 32 + lane] = acc[0] + acc[1] + acc[2] + acc[3];
}
}  // namespace
}  // namespace gespmm

extern "C" gespmm_status_t gespmm_diag_gather_hub(const uint32_t* idx, uint64_t count,
                                                  const float* b, uint32_t hub_rows, float* sink,
                                                  int32_t blocks, void* stream) {
  if (hub_rows > 400) return set_error(GESPMM_EUNSUPPORTED, "diag_gather_hub: hub_rows <= 400");
  if (blocks <= 0) blocks = 148;
  const size_t smem = size_t(hub_rows) * 512;
  cudaFuncSetAttribute(k_gather_hub<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  k_gather_hub<8><<<blocks, 1024, smem, static_cast<cudaStream_t>(stream)>>>(idx, count, b,
                                                                            hub_rows, sink);
  note_launch();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_error(GESPMM_ECUDA, std::string("diag_gather_hub: CUDA error: ") + cudaGetErrorString(e));
  return GESPMM_OK;
}

// k_gather_mode: the gather ceiling under different load paths, to choose how
// the SpMM moves B rows (N = 128, 512 B per row).  Each warp takes a
// contiguous range of the index stream, in batches of 8 rows:
//   mode 0  LDG.128 per lane, L1-allocating (what k_warp does)
//   mode 1  LDG.128 per lane, L1::no_allocate
//   mode 2  cp.async.cg 16 B per lane (LDGSTS, L1 bypass) into a per-warp
//           double-buffered smem ring, then LDS.128
//   mode 3  cp.async.bulk (TMA bulk copy, one 512-B row per issuing lane,
//           mbarrier complete_tx) into the ring, then LDS.128
namespace gespmm {
namespace {

constexpr int kModeWarps = 8;
constexpr int kModeBatch = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void __launch_bounds__(32 * kModeWarps) k_gather_mode(const uint32_t* __restrict__ idx,
                                                                 uint64_t count,
                                                                 const float* __restrict__ b,
                                                                 float* __restrict__ sink) {
  extern __shared__ __align__(128) float s_ring[];  // [warps][2][8][128]
  __shared__ __align__(8) uint64_t s_bar[kModeWarps][2];
  const Policies pol = make_policies(1);
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t per = (count + warps - 1) / warps;
  const uint64_t beg = min(count, warp * per), end = min(count, beg + per);
  const uint64_t batches = (end - beg + kModeBatch - 1) / kModeBatch;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float* ring = s_ring + size_t(wib) * 2 * kModeBatch * 128;
  if (MODE == 0 || MODE == 1) {
    for (uint64_t bt = 0; bt < batches; ++bt) {
      const uint64_t i0 = beg + bt * kModeBatch;
      const uint32_t mine = (lane < kModeBatch && i0 + lane < end) ? ld_stream_u32(idx + i0 + lane, pol.stream) : 0u;
      float4 v[kModeBatch];
#pragma unroll
      for (int u = 0; u < kModeBatch; ++u) {
        const uint32_t k = __shfl_sync(0xffffffffu, mine, u);
        const float* p = b + uint64_t(k) * 128u + lane * 4;
        if (MODE == 0)
          asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
              : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p), "l"(pol.keep));
        else
          asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
              : "=f"(v[u].x), "=f"(v[u].y), "=f"(v[u].z), "=f"(v[u].w) : "l"(p), "l"(pol.keep));
      }
#pragma unroll
      for (int u = 0; u < kModeBatch; ++u) {
        acc[0] += v[u].x; acc[1] += v[u].y; acc[2] += v[u].z; acc[3] += v[u].w;
      }
    }
  } else {
    const uint32_t bar0 = smem_u32(&s_bar[wib][0]);
    if (MODE == 3 && lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    auto issue = [&](uint64_t bt) {
      const uint64_t i0 = beg + bt * kModeBatch;
      const uint32_t buf = uint32_t(bt & 1);
      float* dst = ring + buf * kModeBatch * 128;
      if (MODE == 2) {
        const uint32_t mine = (lane < kModeBatch && i0 + lane < end) ? ld_stream_u32(idx + i0 + lane, pol.stream) : 0u;
#pragma unroll
        for (int u = 0; u < kModeBatch; ++u) {
          const uint32_t k = __shfl_sync(0xffffffffu, mine, u);
          const float* src = b + uint64_t(k) * 128u + lane * 4;
          asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
                       ::"r"(smem_u32(dst + u * 128 + lane * 4)), "l"(src), "l"(pol.keep) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      } else {
        const uint32_t bar = bar0 + buf * 8;
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                       ::"r"(bar), "r"(uint32_t(kModeBatch * 512)) : "memory");
        __syncwarp();
        if (lane < kModeBatch) {
          const uint32_t k = i0 + lane < end ? ld_stream_u32(idx + i0 + lane, pol.stream) : 0u;
          const float* src = b + uint64_t(k) * 128u;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                       " [%0], [%1], 512, [%2], %3;"
                       ::"r"(smem_u32(dst + lane * 128)), "l"(src), "r"(bar), "l"(pol.keep) : "memory");
        }
      }
    };
    uint32_t phase[2] = {0u, 0u};
    if (batches) issue(0);
    for (uint64_t bt = 0; bt < batches; ++bt) {
      if (bt + 1 < batches) issue(bt + 1);
      const uint32_t buf = uint32_t(bt & 1);
      if (MODE == 2) {
        if (bt + 1 < batches) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
      } else {
        const uint32_t bar = bar0 + buf * 8;
        uint32_t done = 0;
        while (!done)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar), "r"(phase[buf]) : "memory");
        phase[buf] ^= 1u;
      }
      const uint64_t left = end - (beg + bt * kModeBatch);
      const float* src = ring + buf * kModeBatch * 128;
#pragma unroll
      for (int u = 0; u < kModeBatch; ++u) {
        if (uint64_t(u) < left) {
          const float4 t = *reinterpret_cast<const float4*>(src + u * 128 + lane * 4);
          acc[0] += t.x; acc[1] += t.y; acc[2] += t.z; acc[3] += t.w;
        }
      }
      __syncwarp();  // ring slot reads done before it is refilled
    }
  }
  sink[warp * 32 + lane] = acc[0] + acc[1] + acc[2] + acc[3];
}

}  // namespace
}  // namespace gespmm

extern "C" gespmm_status_t gespmm_diag_gather_mode(const uint32_t* idx, uint64_t count,
                                                   const float* b, float* sink, int32_t blocks,
                                                   int32_t mode, void* stream) {
  if (blocks <= 0) blocks = 148 * 3;
  const size_t smem = size_t(kModeWarps) * 2 * kModeBatch * 512;
  auto st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
#define GESPMM_M(M)                                                                          \
  case M:                                                                                    \
    e = cudaFuncSetAttribute(k_gather_mode<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             int(smem));                                                     \
    if (e == cudaSuccess) {                                                                  \
      k_gather_mode<M><<<blocks, 32 * kModeWarps, smem, st>>>(idx, count, b, sink);          \
      e = cudaGetLastError();                                                                \
    }                                                                                        \
    break;
  switch (mode) {
    GESPMM_M(0) GESPMM_M(1) GESPMM_M(2) GESPMM_M(3)
    default: return set_error(GESPMM_EINVAL, "diag_gather_mode: mode 0..3");
  }
#undef GESPMM_M
  note_launch();
  if (e != cudaSuccess)
    return set_error(GESPMM_ECUDA, std::string("diag_gather_mode: CUDA error: ") + cudaGetErrorString(e));
  return GESPMM_OK;
}
