// Multi-GPU plumbing of the fused all-gather epilogue: the cross-rank barrier
// over peer-mapped signal words, and peer-shareable buffers with their CUDA IPC
// handles.  The data path itself is the SpMM epilogue (store_replicas,
// common.cuh); this file only orders it across ranks.
#include <cstring>
#include <string>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Signals {
  uint32_t* p[GESPMM_MAX_GATHER_DSTS];
};

// One warp; lane p < world talks to rank p.  The system-scope fence makes
// every store this rank issued before the barrier (the previous kernel's
// peer stores are ordered before this kernel by the stream) visible before
// the signal; acquire loads order the caller's later reads after the peers'.
__global__ void k_peer_barrier(Signals s, int rank, int world, uint32_t epoch,
                               uint64_t timeout_ns, int32_t* error) {
  const int p = int(threadIdx.x);
  if (p >= world) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(s.p[p] + rank), "r"(epoch)
               : "memory");
  const uint32_t* mine = s.p[rank] + p;
  const uint64_t t0 = globaltimer_ns();
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if (v == epoch) break;
    if (globaltimer_ns() - t0 > timeout_ns) {
      if (error) atomicExch(error, 1);
      break;
    }
    __nanosleep(200);
  }
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

namespace {

gespmm_status_t cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return GESPMM_OK;
  return set_error(e == cudaErrorMemoryAllocation ? GESPMM_ENOMEM : GESPMM_ECUDA,
                   std::string(where) + ": CUDA error: " + cudaGetErrorString(e));
}
}  // namespace

extern "C" {

gespmm_status_t gespmm_peer_barrier(uint32_t* const* signals, int32_t rank, int32_t world,
                                    uint32_t epoch, uint32_t timeout_ms, int32_t* error,
                                    void* stream) {
  if (!signals) return set_error(GESPMM_EINVAL, "peer_barrier: null signals");
  if (world < 1 || world > GESPMM_MAX_GATHER_DSTS || rank < 0 || rank >= world)
    return set_error(GESPMM_EINVAL, "peer_barrier: bad rank/world");
  Signals s{};
  for (int p = 0; p < world; ++p) {
    if (!signals[p]) return set_error(GESPMM_EINVAL, "peer_barrier: null signal word");
    s.p[p] = signals[p];
  }
  const uint64_t ns = uint64_t(timeout_ms ? timeout_ms : 60000u) * 1000000ull;
  k_peer_barrier<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(s, rank, world, epoch, ns, error);
  note_launch();
  return cuda_status(cudaGetLastError(), "peer_barrier");
}

gespmm_status_t gespmm_peer_alloc(uint64_t bytes, void** out) {
  if (!out) return set_error(GESPMM_EINVAL, "peer_alloc: null out");
  *out = nullptr;
  return cuda_status(cudaMalloc(out, bytes ? bytes : 1), "peer_alloc");
}

gespmm_status_t gespmm_peer_free(void* ptr) { return cuda_status(cudaFree(ptr), "peer_free"); }

gespmm_status_t gespmm_ipc_get_handle(void* ptr, unsigned char out[64]) {
  if (!ptr || !out) return set_error(GESPMM_EINVAL, "ipc_get_handle: null argument");
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  const gespmm_status_t st = cuda_status(cudaIpcGetMemHandle(&h, ptr), "ipc_get_handle");
  if (st == GESPMM_OK) std::memcpy(out, &h, sizeof(h));
  return st;
}

gespmm_status_t gespmm_ipc_open_handle(const unsigned char handle[64], void** out) {
  if (!handle || !out) return set_error(GESPMM_EINVAL, "ipc_open_handle: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  *out = nullptr;
  return cuda_status(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess),
                     "ipc_open_handle");
}

gespmm_status_t gespmm_ipc_close(void* ptr) {
  return cuda_status(cudaIpcCloseMemHandle(ptr), "ipc_close");
}

}  // extern "C"
