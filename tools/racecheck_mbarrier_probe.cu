// racecheck_mbarrier_probe: is compute-sanitizer racecheck able to follow an
// mbarrier handoff between warps?  Warp 1 writes a shared buffer (plain st or
// cp.async + wait_all), arrives on an mbarrier with release semantics; warp 0
// waits on the phase (acquire) and reads.  Correct by the PTX memory model;
// mode 2 uses __syncthreads instead (racecheck's native barrier) as control.
// nvcc -gencode arch=compute_100a,code=sm_100a -o racecheck_mbarrier_probe racecheck_mbarrier_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(const float* g, float* out, int mode) {
  __shared__ float buf[32 * 16];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    for (int i = 0; i < 16; ++i) {
      if (mode == 1) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(&buf[i * 32 + lane]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(g + i * 32 + lane) : "memory");
      } else {
        buf[i * 32 + lane] = g[i * 32 + lane];
      }
    }
    if (mode == 1) asm volatile("cp.async.wait_all;" ::: "memory");
    if (mode != 2) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
  }
  if (mode == 2) __syncthreads();
  if (warp == 0) {
    if (mode != 2) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(b) : "memory");
    }
    float s = 0.f;
    for (int i = 0; i < 16; ++i) s += buf[i * 32 + lane];
    out[lane] = s;
  }
}

int main() {
  float *g, *o;
  cudaMalloc(&g, 4 * 512);
  cudaMalloc(&o, 4 * 32);
  cudaMemset(g, 0, 4 * 512);
  const char* names[3] = {"st.shared + mbarrier", "cp.async + wait_all + mbarrier", "__syncthreads"};
  for (int mode = 0; mode < 3; ++mode) {
    k<<<1, 64>>>(g, o, mode);
    cudaDeviceSynchronize();
    printf("mode %d (%s): %s\n", mode, names[mode], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
