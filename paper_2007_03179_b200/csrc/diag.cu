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
