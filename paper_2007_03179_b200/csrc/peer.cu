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

// ---------------------------------------------------------------------------
// Single-process NVLS multicast buffers (driver API through
// cudaGetDriverEntryPoint: no libcuda link dependency).  A multicast object
// with this process's device(s) bound to one physical allocation: stores to
// the multicast VA (multimem.st) land in every bound device's memory.  On an
// NVSwitch node the cross-process version of the same object comes from
// symmetric memory (exported handles); this one validates the epilogue's
// multicast store path on whatever the process can see.
// ---------------------------------------------------------------------------
#include <cuda.h>

#include <map>
#include <mutex>

namespace {

struct McFns {
  bool ok = false;
  decltype(&cuMulticastCreate) create = nullptr;
  decltype(&cuMulticastAddDevice) add_device = nullptr;
  decltype(&cuMulticastBindMem) bind_mem = nullptr;
  decltype(&cuMulticastUnbind) unbind = nullptr;
  decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
  decltype(&cuMemCreate) mem_create = nullptr;
  decltype(&cuMemRelease) mem_release = nullptr;
  decltype(&cuMemGetAllocationGranularity) mem_gran = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuDeviceGetAttribute) dev_attr = nullptr;
};

const McFns& mc_fns() {
  static McFns f;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** p) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, p, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *p;
    };
    f.ok = get("cuMulticastCreate", reinterpret_cast<void**>(&f.create)) &&
           get("cuMulticastAddDevice", reinterpret_cast<void**>(&f.add_device)) &&
           get("cuMulticastBindMem", reinterpret_cast<void**>(&f.bind_mem)) &&
           get("cuMulticastUnbind", reinterpret_cast<void**>(&f.unbind)) &&
           get("cuMulticastGetGranularity", reinterpret_cast<void**>(&f.mc_gran)) &&
           get("cuMemCreate", reinterpret_cast<void**>(&f.mem_create)) &&
           get("cuMemRelease", reinterpret_cast<void**>(&f.mem_release)) &&
           get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&f.mem_gran)) &&
           get("cuMemAddressReserve", reinterpret_cast<void**>(&f.reserve)) &&
           get("cuMemAddressFree", reinterpret_cast<void**>(&f.addr_free)) &&
           get("cuMemMap", reinterpret_cast<void**>(&f.map)) &&
           get("cuMemUnmap", reinterpret_cast<void**>(&f.unmap)) &&
           get("cuMemSetAccess", reinterpret_cast<void**>(&f.set_access)) &&
           get("cuDeviceGetAttribute", reinterpret_cast<void**>(&f.dev_attr));
  });
  return f;
}

struct McBuffer {
  CUmemGenericAllocationHandle mem = 0, mc = 0;
  CUdeviceptr uc = 0, mcva = 0;
  size_t size = 0;
  int dev = 0;
};
std::mutex g_mc_mu;
std::map<void*, McBuffer> g_mc;

gespmm_status_t drv_status(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return GESPMM_OK;
  return set_error(r == CUDA_ERROR_NOT_SUPPORTED ? GESPMM_EUNSUPPORTED : GESPMM_ECUDA,
                   std::string("multicast: ") + what + " failed (CUresult " + std::to_string(int(r)) + ")");
}

}  // namespace

extern "C" {

gespmm_status_t gespmm_multicast_alloc(uint64_t bytes, void** uc_ptr, void** mc_ptr) {
  if (!uc_ptr || !mc_ptr) return set_error(GESPMM_EINVAL, "multicast_alloc: null out");
  *uc_ptr = *mc_ptr = nullptr;
  const McFns& f = mc_fns();
  if (!f.ok) return set_error(GESPMM_EUNSUPPORTED, "multicast: driver entry points unavailable");
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_status(ce, "multicast_alloc");
  int supported = 0;
  f.dev_attr(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, CUdevice(dev));
  if (!supported) return set_error(GESPMM_EUNSUPPORTED, "multicast: device does not support multicast");
  McBuffer b;
  b.dev = dev;
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  mp.size = bytes ? bytes : 1;
  size_t mg = 0;
  gespmm_status_t s = drv_status(f.mc_gran(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "granularity");
  if (s != GESPMM_OK) return s;
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  size_t ag = 0;
  if ((s = drv_status(f.mem_gran(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity")) != GESPMM_OK)
    return s;
  const size_t g = mg > ag ? mg : ag;
  b.size = (mp.size + g - 1) / g * g;
  mp.size = b.size;
  auto fail_cleanup = [&](gespmm_status_t st) {
    if (b.mcva) { f.unmap(b.mcva, b.size); f.addr_free(b.mcva, b.size); }
    if (b.uc) { f.unmap(b.uc, b.size); f.addr_free(b.uc, b.size); }
    if (b.mc && b.mem) f.unbind(b.mc, CUdevice(dev), 0, b.size);
    if (b.mc) f.mem_release(b.mc);
    if (b.mem) f.mem_release(b.mem);
    return st;
  };
  {
    // the driver may insist on an exportable handle type even for a one-process team
    CUresult r = CUDA_ERROR_INVALID_VALUE;
    for (CUmemAllocationHandleType ht :
         {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC}) {
      mp.handleTypes = ht;
      r = f.create(&b.mc, &mp);
      if (r == CUDA_SUCCESS) break;
    }
    if (r != CUDA_SUCCESS) {
      // measured on the gpurun boxes: the device reports multicast support but
      // the container has no NVSwitch/IMEX device nodes, and every create is
      // refused with CUDA_ERROR_INVALID_VALUE (tools/multicast_probe.py)
      return fail_cleanup(set_error(GESPMM_EUNSUPPORTED,
                                    "multicast: the driver refused the multicast object (CUresult " +
                                        std::to_string(int(r)) +
                                        "; no NVSwitch fabric access in this process?)"));
    }
  }
  if ((s = drv_status(f.add_device(b.mc, CUdevice(dev)), "add device")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.mem_create(&b.mem, b.size, &ap, 0), "physical allocation")) != GESPMM_OK)
    return fail_cleanup(s);
  if ((s = drv_status(f.bind_mem(b.mc, 0, b.mem, 0, b.size, 0), "bind")) != GESPMM_OK) return fail_cleanup(s);
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((s = drv_status(f.reserve(&b.uc, b.size, g, 0, 0), "reserve")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.map(b.uc, b.size, 0, b.mem, 0), "map")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.set_access(b.uc, b.size, &acc, 1), "access")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.reserve(&b.mcva, b.size, g, 0, 0), "reserve mc")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.map(b.mcva, b.size, 0, b.mc, 0), "map mc")) != GESPMM_OK) return fail_cleanup(s);
  if ((s = drv_status(f.set_access(b.mcva, b.size, &acc, 1), "access mc")) != GESPMM_OK) return fail_cleanup(s);
  *uc_ptr = reinterpret_cast<void*>(b.uc);
  *mc_ptr = reinterpret_cast<void*>(b.mcva);
  std::lock_guard<std::mutex> lk(g_mc_mu);
  g_mc[*uc_ptr] = b;
  return GESPMM_OK;
}

gespmm_status_t gespmm_multicast_free(void* uc_ptr) {
  McBuffer b;
  {
    std::lock_guard<std::mutex> lk(g_mc_mu);
    auto it = g_mc.find(uc_ptr);
    if (it == g_mc.end()) return set_error(GESPMM_EINVAL, "multicast_free: unknown buffer");
    b = it->second;
    g_mc.erase(it);
  }
  const McFns& f = mc_fns();
  cudaDeviceSynchronize();
  f.unmap(b.mcva, b.size);
  f.addr_free(b.mcva, b.size);
  f.unmap(b.uc, b.size);
  f.addr_free(b.uc, b.size);
  f.unbind(b.mc, CUdevice(b.dev), 0, b.size);
  f.mem_release(b.mc);
  f.mem_release(b.mem);
  return GESPMM_OK;
}

}  // extern "C"
