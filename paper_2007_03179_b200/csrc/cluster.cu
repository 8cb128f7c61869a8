// k_warp_cluster — the row-per-warp SpMM with the hottest B rows held in the
// distributed shared memory of a thread-block cluster (opt-in plan option
// cluster_hot; N = 128, float4 lanes, one row per warp).
//
// On a power-law graph a few thousand columns carry a large share of the
// gathers (Reddit shape: the top 3.4k columns 24%, the top 6.8k 35%), but
// L1 holds only ~400 B rows per SM.  Here every CTA of a cluster of CS CTAs
// (one CTA per SM, 28 warps, ~213 KB of shared memory each) keeps 426 distinct
// hot B rows, so a cluster caches CS x 426 rows; a gather of a hot column reads
// the owning CTA's shared memory through DSMEM (`mapa` + `ld.shared::cluster`),
// a path whose bandwidth adds to the L2 -> SM crossbar's (the kernel's bound).
// The plan remaps col_ind once: hot columns become (1 << 31) | slot, slot s
// living in CTA s % CS at row s / CS.  Rows are walked in the plan's LPT order
// by persistent warps pulling from a counter.  Fold order per output element
// is the CSR order, so results stay bit-identical.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

constexpr int kClWarps = 28;                 // 28 x 32 threads x 72 registers fill one SM
#ifndef GESPMM_CL_HOT_ROWS
#define GESPMM_CL_HOT_ROWS 416
#endif
constexpr int kClHotRows = GESPMM_CL_HOT_ROWS;  // hot B rows (512 B) per CTA
constexpr size_t kClHotBytes = size_t(kClHotRows) * 512;
constexpr size_t kClStageBytes = size_t(kClWarps) * 2 * 32 * 8;   // per-warp (col, val) tiles
constexpr uint32_t kHot = 0x80000000u;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ Vec<4> ld_dsmem4(uint32_t local_addr, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  Vec<4> v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x[0]), "=f"(v.x[1]), "=f"(v.x[2]), "=f"(v.x[3])
               : "r"(remote)
               : "memory");
  return v;
}

struct ClusterArgs {
  const uint32_t* hot_list;   // slot -> column (n_hot entries)
  uint32_t n_hot;
  uint32_t* counter;          // row-unit counter (zeroed before the launch)
};

template <int OP, bool FAST, int CS>
__global__ void __launch_bounds__(kClWarps * 32, 1) k_warp_cluster(SpmmArgs a, ClusterArgs c) {
  using R = Reduce<OP>;
  constexpr int U = 8;
  extern __shared__ __align__(128) unsigned char cl_smem[];
  float4* hot = reinterpret_cast<float4*>(cl_smem);                          // [kClHotRows][32]
  uint32_t* s_col = reinterpret_cast<uint32_t*>(cl_smem + kClHotBytes);      // [warps][2][32]
  float* s_val = reinterpret_cast<float*>(cl_smem + kClHotBytes + kClStageBytes / 2);
  const uint32_t rank = cluster_rank();
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const Policies pol = args_policies(a);

  // this CTA's hot rows: slots rank, rank + CS, ...
  for (uint32_t i = threadIdx.x; i < uint32_t(kClHotRows) * 32u; i += blockDim.x) {
    const uint32_t j = i >> 5, s = j * CS + rank;
    if (s < c.n_hot) {
      const uint32_t col = c.hot_list[s];
      hot[i] = *reinterpret_cast<const float4*>(a.b + uint64_t(col) * a.ldb + (i & 31u) * 4u);
    }
  }
  cluster_sync_all();  // every CTA's slice is in place before any DSMEM read

  const uint32_t hot_base = static_cast<uint32_t>(__cvta_generic_to_shared(hot)) + lane * 16u;
  uint32_t* my_col = s_col + wib * 64;
  float* my_val = s_val + wib * 64;
  const char* bl = reinterpret_cast<const char*>(a.b + lane * 4u);
  const uint32_t stride = a.ldb * 4u;
  for (;;) {
    uint32_t unit = 0;
    if (lane == 0) unit = atomicAdd(c.counter, 1u);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= a.n_sched) break;
    const uint32_t row = a.order ? a.order[unit] : unit;
    const uint32_t start = a.row_ptr[row], full_end = a.row_ptr[row + 1];
    const uint32_t len = faulted_end(start, full_end, a.skip_tail) - start;
    const uint32_t* ci = a.col_ind + start;
    const float* vs = a.vals + start;
    float acc[4];
    int32_t who[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[e] = R::init();
      who[e] = -1;
    }
    uint32_t kn = 0;
    float vn = 0.0f;
    if (lane < len) {
      kn = ld_stream_u32(ci + lane, pol.stream);
      vn = ld_stream_f32(vs + lane, pol.stream);
    }
    __syncwarp();
    my_col[lane] = kn;
    my_val[lane] = vn;
    uint32_t buf = 0;
    for (uint32_t off = 0; off < len; off += 32) {
      uint32_t k2 = 0;
      float v2 = 0.0f;
      if (off + 32 + lane < len) {
        k2 = ld_stream_u32(ci + off + 32 + lane, pol.stream);
        v2 = ld_stream_f32(vs + off + 32 + lane, pol.stream);
      }
      __syncwarp();
      const uint32_t* cs = my_col + buf * 32;
      const float* vsm = my_val + buf * 32;
      const uint32_t chunk = min(32u, len - off);
      for (uint32_t kk = 0; kk < chunk; kk += U) {
        uint32_t k[U];
        float v[U];
#pragma unroll
        for (int q = 0; q < U; q += 4) {
          const uint4 c4 = *reinterpret_cast<const uint4*>(cs + kk + q);
          const float4 v4 = *reinterpret_cast<const float4*>(vsm + kk + q);
          k[q] = c4.x; k[q + 1] = c4.y; k[q + 2] = c4.z; k[q + 3] = c4.w;
          v[q] = v4.x; v[q + 1] = v4.y; v[q + 2] = v4.z; v[q + 3] = v4.w;
        }
        Vec<4> bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (k[u] & kHot) {  // warp-uniform: every lane holds the same staged entry
            const uint32_t s = k[u] & ~kHot;
            bv[u] = ld_dsmem4(hot_base + (s / CS) * 512u, s % CS);
          } else {
            bv[u] = ld_keep<4>(reinterpret_cast<const float*>(bl + uint64_t(k[u]) * stride), pol.keep);
          }
        }
        const int32_t rem = int32_t(chunk - kk);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u < rem) {
            // column args name the original column, not the remapped slot
            const int32_t pos =
                a.arg_col ? int32_t((k[u] & kHot) ? c.hot_list[k[u] & ~kHot] : k[u])
                          : int32_t(start + off + kk + u);
            fold_vec<OP, FAST, 4>(acc, who, v[u], bv[u].x, pos);
          }
        }
      }
      buf ^= 1u;
      my_col[buf * 32 + lane] = k2;
      my_val[buf * 32 + lane] = v2;
    }
    float out[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) out[e] = finish<OP>(acc[e], full_end - start);
    const uint64_t o = uint64_t(row) * a.ld + lane * 4u;
    st_stream<4>(a.c + o, out, pol.stream);
    if (R::kHasArg && a.arg) st_stream_i32<4>(a.arg + o, who, pol.stream);
    if (a.n_peer || a.c_mc) store_replicas<4, R::kHasArg>(a, o, out, who);
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its slice
}

__global__ void k_remap_cols(const uint32_t* __restrict__ ci, uint64_t nnz,
                             const uint32_t* __restrict__ map, uint32_t* __restrict__ out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = map[__ldg(ci + i)];
}

__global__ void k_count_cols_cl(const uint32_t* __restrict__ ci, uint64_t nnz,
                                uint32_t* __restrict__ counts) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(counts + __ldg(ci + i), 1u);
}

template <int CS>
cudaError_t launch_cs(int op, bool fast, const SpmmArgs& a, const ClusterArgs& c, cudaStream_t st,
                      int* clusters_out) {
  const size_t smem = kClHotBytes + kClStageBytes;
  auto pick = [&](auto kernel) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
    if (CS > 8) {
      e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kClWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    cfg.gridDim = dim3(CS * 148);
    e = cudaOccupancyMaxActiveClusters(&clusters, kernel, &cfg);
    if (e != cudaSuccess) return e;
    if (clusters <= 0) return cudaErrorInvalidConfiguration;
    *clusters_out = clusters;
    cfg.gridDim = dim3(uint32_t(CS * clusters));
    e = cudaLaunchKernelEx(&cfg, kernel, a, c);
    note_launch();
    return e;
  };
  switch (op) {
    case kSum: return fast ? pick(k_warp_cluster<kSum, true, CS>) : pick(k_warp_cluster<kSum, false, CS>);
    case kMean: return fast ? pick(k_warp_cluster<kMean, true, CS>) : pick(k_warp_cluster<kMean, false, CS>);
    case kMax: return pick(k_warp_cluster<kMax, false, CS>);
    default: return pick(k_warp_cluster<kMin, false, CS>);
  }
}

}  // namespace

uint32_t cluster_hot_rows(int cs) { return uint32_t(cs) * uint32_t(kClHotRows); }

// Plan-time: the top-(CS x kClHotRows) columns by gather count become hot; slot
// order by descending count so the heaviest rows spread round-robin over the
// cluster's CTAs.  Produces the remapped col_ind and the slot -> column list.
cudaError_t build_cluster_hot(const uint32_t* col_ind, uint64_t nnz, uint32_t k, int cs,
                              cudaStream_t st, ClusterHot* out) {
  *out = ClusterHot{};
  if (nnz == 0 || k == 0) return cudaSuccess;
  uint32_t* counts = nullptr;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&counts), sizeof(uint32_t) * k);
  if (e != cudaSuccess) return e;
  std::vector<uint32_t> h(k);
  e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * k, st);
  if (e == cudaSuccess) {
    k_count_cols_cl<<<148 * 8, 256, 0, st>>>(col_ind, nnz, counts);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), counts, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(counts);
  if (e != cudaSuccess) return e;
  const uint32_t cap = std::min<uint32_t>(cluster_hot_rows(cs), k);
  std::vector<uint32_t> idx(k);
  std::iota(idx.begin(), idx.end(), 0u);
  std::partial_sort(idx.begin(), idx.begin() + cap, idx.end(),
                    [&](uint32_t x, uint32_t y) { return h[x] != h[y] ? h[x] > h[y] : x < y; });
  uint32_t n_hot = 0;
  uint64_t hot_nnz = 0;
  std::vector<uint32_t> map(k), list;
  for (uint32_t c = 0; c < k; ++c) map[c] = c;
  for (uint32_t s = 0; s < cap && h[idx[s]] > 1; ++s) {  // a once-gathered row gains nothing
    map[idx[s]] = kHot | s;
    list.push_back(idx[s]);
    hot_nnz += h[idx[s]];
    ++n_hot;
  }
  uint32_t* d_map = nullptr;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&d_map), sizeof(uint32_t) * k)) != cudaSuccess) return e;
  e = cudaMalloc(reinterpret_cast<void**>(&out->col_ind), sizeof(uint32_t) * nnz);
  if (e == cudaSuccess && n_hot)
    e = cudaMalloc(reinterpret_cast<void**>(&out->hot_list), sizeof(uint32_t) * n_hot);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_map, map.data(), sizeof(uint32_t) * k, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && n_hot)
    e = cudaMemcpyAsync(out->hot_list, list.data(), sizeof(uint32_t) * n_hot,
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    k_remap_cols<<<148 * 8, 256, 0, st>>>(col_ind, nnz, d_map, out->col_ind);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&out->counter), sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_map);
  out->n_hot = n_hot;
  out->cs = cs;
  out->hot_nnz_frac = double(hot_nnz) / double(nnz);
  return e;
}

void free_cluster_hot(ClusterHot* h) {
  if (h->col_ind) cudaFree(h->col_ind);
  if (h->hot_list) cudaFree(h->hot_list);
  if (h->counter) cudaFree(h->counter);
  *h = ClusterHot{};
}

cudaError_t launch_cluster_warp(const ClusterHot& h, int op, bool fast, const SpmmArgs& a0,
                                cudaStream_t st, int* clusters) {
  SpmmArgs a = a0;
  a.col_ind = h.col_ind;
  ClusterArgs c{h.hot_list, h.n_hot, h.counter};
  cudaError_t e = cudaMemsetAsync(h.counter, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  switch (h.cs) {
    case 16: return launch_cs<16>(op, fast, a, c, st, clusters);
    case 4: return launch_cs<4>(op, fast, a, c, st, clusters);
    case 2: return launch_cs<2>(op, fast, a, c, st, clusters);
    default: return launch_cs<8>(op, fast, a, c, st, clusters);
  }
}

}  // namespace gespmm
