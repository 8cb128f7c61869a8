// Packed column indices for the host entry's PCIe upload (host side; the
// device side and the format are described in h2dpack.cu).  Encoding runs on
// most host threads (OpenMP) while the copy engine moves the previous block.
#include <cuda_runtime_api.h>
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>

#include <atomic>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace gespmm {
namespace {

// One thread's rows: a row's first entry is its column, every other entry
// (col[p] - col[p-1] - 1) clamped to 0xFFFF.  The inner loop has no carried
// dependency (it re-reads the previous column instead of keeping it), so it
// vectorises; a running max flags the rows that need escapes (a gap >= 0xFFFF,
// or a decrease, which wraps to a huge value — non-canonical input keeps its
// exact columns), and only those rows get the scalar pass that records them.
// Measured on the box's host (tools/pack_probe.cpp, 12 threads, Reddit
// blocks): 1.04 ms per block for the scalar loop with the carried previous
// column, 0.75 ms for this one at SSE2, 0.69 ms at AVX2.
template <int ISA>
inline void pack_rows_impl(const uint32_t* __restrict row_ptr, const uint32_t* __restrict col, uint32_t r0,
                           uint32_t r1, uint64_t ps, uint16_t* __restrict enc, std::vector<uint32_t>& ex) {
  for (uint32_t r = r0; r < r1; ++r) {
    const uint64_t s = row_ptr[r], e = row_ptr[r + 1];
    if (s == e) continue;
    const uint32_t* c = col + s;
    uint16_t* o = enc + (s - ps);
    const uint64_t n = e - s;
    uint32_t mx = c[0];
    o[0] = uint16_t(c[0] < 0xFFFFu ? c[0] : 0xFFFFu);
    for (uint64_t i = 1; i < n; ++i) {
      const uint32_t d = c[i] - c[i - 1] - 1u;
      mx = d > mx ? d : mx;
      o[i] = uint16_t(d < 0xFFFFu ? d : 0xFFFFu);
    }
    if (mx >= 0xFFFFu) {
      for (uint64_t i = 0; i < n; ++i)
        if (o[i] == 0xFFFFu) {
          ex.push_back(uint32_t(s + i - ps));
          ex.push_back(c[i]);
        }
    }
  }
}

using PackRows = void (*)(const uint32_t*, const uint32_t*, uint32_t, uint32_t, uint64_t, uint16_t*,
                          std::vector<uint32_t>&);

__attribute__((target("avx2"))) void pack_rows_avx2(const uint32_t* rp, const uint32_t* col, uint32_t r0,
                                                    uint32_t r1, uint64_t ps, uint16_t* enc,
                                                    std::vector<uint32_t>& ex) {
  pack_rows_impl<2>(rp, col, r0, r1, ps, enc, ex);
}
void pack_rows_base(const uint32_t* rp, const uint32_t* col, uint32_t r0, uint32_t r1, uint64_t ps,
                    uint16_t* enc, std::vector<uint32_t>& ex) {
  pack_rows_impl<1>(rp, col, r0, r1, ps, enc, ex);
}

PackRows pick_pack_rows() {
  __builtin_cpu_init();
  return __builtin_cpu_supports("avx2") ? pack_rows_avx2 : pack_rows_base;
}

}  // namespace

// three quarters of the host threads unless OMP_NUM_THREADS says otherwise:
// with every core packing, the packing contends with the copy engine's reads
// of host memory and with the CUDA driver threads (Reddit, 16 cores: 17.9 ms
// at 16 threads, 16.3 ms at 12, 16.7-19.3 ms at 8; tools/e2e_threads.py)
// GESPMM_PACK_THREADS overrides; under torchrun (LOCAL_WORLD_SIZE set, which
// also forces OMP_NUM_THREADS=1) the host's threads are split between ranks
int pack_threads() {
  static const int nt = [] {
    if (const char* e = std::getenv("GESPMM_PACK_THREADS")) return std::max(1, std::atoi(e));
    const char* lws = std::getenv("LOCAL_WORLD_SIZE");
    if (std::getenv("OMP_NUM_THREADS") && !lws) return std::max(1, omp_get_max_threads());
    const int hw = int(std::thread::hardware_concurrency());
    const int mine = std::max(1, hw > 4 ? hw * 3 / 4 : hw);
    return lws ? std::max(1, mine / std::max(1, std::atoi(lws))) : mine;
  }();
  return nt;
}

// Keeps the packing threads busy until every stream in `streams` has drained.
// Measured on the box (tools/e2e_env.py, Reddit host call, 3 processes each):
// when the packer finishes (~10 ms into a ~17 ms call) and the host goes idle,
// the remaining H2D/D2H copies and kernels slow down (the last block lands
// ~2.3 ms after the previous one instead of ~1.1 ms), 17.3-17.8 ms per call;
// with the OpenMP threads spinning (OMP_WAIT_POLICY=active) 16.2-16.5 ms.  So
// after the last block is enqueued the pool polls the streams instead of
// sleeping.  GESPMM_HOST_POLL=0 turns it off, =N polls with N threads.
void host_poll(void* const* streams, int n) {
  static const int np = [] {
    const char* e = std::getenv("GESPMM_HOST_POLL");
    return e ? std::max(0, std::atoi(e)) : -1;
  }();
  const int threads = np < 0 ? pack_threads() : np;
  if (threads == 0 || n == 0) return;
  std::atomic<bool> done{false};
#pragma omp parallel num_threads(threads)
  {
    if (omp_get_thread_num() == 0) {
      for (int i = 0; i < n; ++i)
        while (cudaStreamQuery(static_cast<cudaStream_t>(streams[i])) == cudaErrorNotReady) _mm_pause();
      done.store(true, std::memory_order_release);
    } else {
      while (!done.load(std::memory_order_acquire)) _mm_pause();
    }
  }
}

// Encodes positions [row_ptr[lo], row_ptr[hi]) of rows [lo, hi) into enc
// (relative positions) and appends escaped (relative position, value) pairs to
// exc in position order.  Returns the number of exceptions, or UINT64_MAX when
// they exceed max_exc (the caller then sends the block raw).
uint64_t pack_cols_block(const uint32_t* row_ptr, const uint32_t* col_ind, uint32_t lo,
                         uint32_t hi, uint16_t* enc, uint32_t* exc /* pairs */, uint64_t max_exc) {
  const uint64_t ps = row_ptr[lo];
  const int nt = pack_threads();
  // rows split by nnz across threads
  std::vector<uint32_t> cut(size_t(nt) + 1, hi);
  cut[0] = lo;
  const uint64_t total = uint64_t(row_ptr[hi]) - ps;
  for (int t = 1; t < nt; ++t) {
    const uint64_t target = ps + total * uint64_t(t) / uint64_t(nt);
    const uint32_t* it = std::lower_bound(row_ptr + lo, row_ptr + hi + 1, uint32_t(target));
    cut[size_t(t)] = std::max(cut[size_t(t) - 1], uint32_t(std::min<ptrdiff_t>(it - row_ptr, hi)));
  }
  std::vector<std::vector<uint32_t>> local(static_cast<size_t>(nt));
  static const PackRows pack_rows = pick_pack_rows();
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num();
    pack_rows(row_ptr, col_ind, cut[size_t(t)], cut[size_t(t) + 1], ps, enc, local[size_t(t)]);
  }
  uint64_t n = 0;
  for (const auto& v : local) n += v.size() / 2;
  if (n > max_exc) return UINT64_MAX;
  uint64_t off = 0;
  for (const auto& v : local) {
    if (!v.empty()) std::memcpy(exc + off, v.data(), v.size() * sizeof(uint32_t));
    off += v.size();
  }
  return n;
}

}  // namespace gespmm
