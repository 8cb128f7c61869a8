// Tuned B200 SpMM-like kernels (the product path).
//
// k_warp — row per (sub)warp.  Coalesced Row Caching: the LPR lanes that own a
//   row load the next LPR*E (col, val) pairs of the row with E coalesced loads
//   each (E = 2 for 4-lane rows, else 1; prefetched one chunk ahead) into a
//   per-warp shared tile and read them back with broadcast LDS.128, so
//   col_ind/vals are read once per row tile.  Lanes own VEC contiguous columns
//   and gather B rows with 16-byte (float4) loads.  Coarse-grained Warp
//   Merging: each lane owns CF column sub-tiles, so one staged nonzero feeds
//   CF vector gathers.  U nonzeros are gathered before any is folded (memory-
//   level parallelism), then folded in ascending position: every output
//   element is still reduced by one thread in CSR order, so results are
//   bit-identical to the reference fold (kernel.hpp:287-343) in exact mode.
//
// k_hub — row per CTA for hub rows (the rows whose single-warp time would
//   bound a launch): producer warps stream the row's B slices into a
//   shared-memory ring with LDGSTS + mbarriers, consumer warps fold them in
//   order (see the comment at the kernel).
//
// k_cta — row per CTA for hub rows the ring cannot address (N % 4 != 0,
//   misaligned B/C).  The CTA stages the row's sparse segment into shared
//   memory (double-buffered), and its warps split the COLUMNS of the row (never
//   the nonzeros), keeping the per-element ascending fold and with it
//   bit-exactness; a deeper gather batch (32 scalar or 8 vector loads per lane)
//   gives the hub the latency hiding a single warp cannot.
//
// k_split_combine / k_split_refresh — split hub rows (max/min, fast-mode
//   sum/mean): k_warp folds each hub row's segments into partial rows, the
//   combine folds the partials in segment order; the refresh rebuilds the
//   segments' virtual row_ptr from the live row_ptr for a cached plan.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include <cuda.h>  // CUtensorMap (the type only; encoded through the runtime's driver entry point)

#include "common.cuh"
#include "launch.h"

namespace gespmm {
namespace {

constexpr unsigned kFull = 0xffffffffu;
enum : int { kHotOff = 0, kHotMap = 1, kHotReloc = 2 };  // k_warp's B-row placement modes
// the hot-row modes were measured slower: compiled only into the
// experimental library
#ifdef GESPMM_EXPERIMENTAL
constexpr bool kExpBuild = true;
#else
constexpr bool kExpBuild = false;
#endif

template <int N>
struct Pack;  // staged-entry read width: N consecutive (col) or (val) words
template <>
struct Pack<1> {
  using U = uint32_t;
  using F = float;
};
template <>
struct Pack<2> {
  using U = uint2;
  using F = float2;
};
template <>
struct Pack<4> {
  using U = uint4;
  using F = float4;
};

constexpr int kWarpBlock = 4;  // warps per CTA (CF=1 sum: 64 registers, 8 CTAs = 32 warps/SM)

// max/min carry 2*CF*VEC accumulator registers (value + arg): 6 CTAs per SM
// (85 registers; 4 at CF=4) instead of spilling under the 7-CTA cap.
template <int OP, int CF, int LPR = 32>
// CF=4 sum/mean shapes (low-degree rows, e.g. Pubmed): 6 CTAs per SM; 7 or 8
// (<= 64 registers, spills) measured no faster on Pubmed N=128 (14.4 vs
// 14.4/15.2/16.4 us median)
#ifndef GESPMM_CF4_BLOCKS
#define GESPMM_CF4_BLOCKS 6
#endif
// CF=1 sum/mean (the Reddit N=128 shape): 8 CTAs per SM fit 64 registers
// without spills: 32 warps/SM, best step 2.80 vs 2.84 ms at 7 CTAs
#ifndef GESPMM_CF1_BLOCKS
#define GESPMM_CF1_BLOCKS 8
#endif
#ifndef GESPMM_CF2_BLOCKS
#define GESPMM_CF2_BLOCKS 7
#endif
#ifndef GESPMM_ARG_BLOCKS
#define GESPMM_ARG_BLOCKS 6
#endif
constexpr int warp_min_blocks() {
#ifdef GESPMM_NARROW_BLOCKS
  if (LPR <= 16 && CF == 1 && !Reduce<OP>::kHasArg) return GESPMM_NARROW_BLOCKS;
#endif
  return Reduce<OP>::kHasArg ? (CF >= 4 ? 4 : GESPMM_ARG_BLOCKS)
                             : (CF >= 4 ? GESPMM_CF4_BLOCKS
                                        : (CF == 1 ? GESPMM_CF1_BLOCKS : GESPMM_CF2_BLOCKS));
}

template <int LPR, int CF>
#ifndef GESPMM_U_NARROW
#define GESPMM_U_NARROW 8
#endif
#ifndef GESPMM_U_WIDE
#define GESPMM_U_WIDE 8  // gather batch of full-warp CF=1 rows (A/B builds: 16 with fewer CTAs/SM)
#endif
#ifndef GESPMM_STAGE_MIN
#define GESPMM_STAGE_MIN 8  // staged entries per row per chunk, at least
#endif
struct WarpGeom {
  static constexpr int RPW = 32 / LPR;                     // rows per warp
  // staged entries per lane per chunk: 4-lane rows (N = 16) stage 8 entries
  // per row per chunk, not 4, so a chunk's col/val round trip is hidden behind
  // 8 gathers in flight (Reddit shape N=16: 2.65 ms at 4 per chunk)
  // (scalar 1- and 2-lane rows, N < 4, keep one entry per lane)
  static constexpr int E = (LPR >= GESPMM_STAGE_MIN || LPR < 4) ? 1 : GESPMM_STAGE_MIN / LPR;
  static constexpr int CH = LPR * E;                       // entries per row per chunk
  static constexpr int U0 = (LPR == 16 ? GESPMM_U_NARROW : (LPR == 32 && CF == 1 ? GESPMM_U_WIDE : 8)) / CF;
  static constexpr int U = U0 < CH ? U0 : CH;              // gather batch; CH % U == 0
  static constexpr int W = U < 4 ? U : 4;                  // LDS width (entries per read)
  static_assert(CH % U == 0 && U % W == 0 && E <= (GESPMM_STAGE_MIN / 4 > 1 ? GESPMM_STAGE_MIN / 4 : 1),
                "batch geometry");
};

// Relocated hot rows: a remapped column with bit 31 set is slot s of the plan's
// copy, which starts hot_off rows (of B's stride) from B; the staged index
// becomes that signed row offset, so the gather needs no select.
__device__ __forceinline__ uint32_t reloc_index(const SpmmArgs& a, uint32_t k) {
  return (k & 0x80000000u) ? uint32_t(int32_t(k & 0x7fffffffu) + a.hot_off) : k;
}
// One L2 policy for every gather, from the launch parameters (a uniform
// register, no per-load move): the address-range policy resolved on the host
// side (resolve_range_policy), or the fractional keep (reloc_mode 0, A/B).
__device__ __forceinline__ uint64_t reloc_policy(const SpmmArgs& a, const Policies& pol) {
  return a.reloc_mode == 0 ? pol.keep : a.pol_hot;
}

// Row metadata of one (sub)warp unit for this lane: the row, its CSR range,
// and this lane's entry of the row's first staged chunk.
struct UnitMeta {
  uint32_t row, start, full_end;
  uint32_t k0[GESPMM_STAGE_MIN / 4 > 1 ? GESPMM_STAGE_MIN / 4 : 1];  // this lane's chunk-0
  float v0[GESPMM_STAGE_MIN / 4 > 1 ? GESPMM_STAGE_MIN / 4 : 1];     // entries (WarpGeom::E)
  bool row_ok;
};

template <int LPR>
__device__ __forceinline__ void unit_rows(const SpmmArgs& a, uint32_t group, UnitMeta& m) {
  const uint32_t sidx = group * (32 / LPR) + (threadIdx.x & 31) / LPR;
  m.row_ok = sidx < a.n_sched;
  m.row = m.row_ok ? (a.order ? a.order[sidx] : sidx) : 0u;
  m.start = m.full_end = 0;
  if (m.row_ok) {
    m.start = a.row_ptr[m.row];
    m.full_end = a.row_ptr[m.row + 1];
  }
}

// Issues this lane's chunk-0 (col, val) loads; slots past the row end hold
// column 0 (a valid row).
template <int LPR, int E, int HOT>
__device__ __forceinline__ void unit_chunk0(const SpmmArgs& a, const Policies& pol, UnitMeta& m) {
  const uint32_t sl = (threadIdx.x & 31) % LPR;
  const uint32_t len = faulted_end(m.start, m.full_end, a.skip_tail) - m.start;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const uint32_t i = uint32_t(j * LPR) + sl;
    m.k0[j] = 0;
    m.v0[j] = 0.0f;
    if (i < len) {
      m.k0[j] = ld_stream_u32(a.col_ind + m.start + i, pol.stream);
      m.v0[j] = ld_stream_f32(a.vals + m.start + i, pol.stream);
      if (HOT == kHotMap) m.k0[j] |= cold_mark(a.hot, m.k0[j]);
      if (HOT == kHotReloc) m.k0[j] = reloc_index(a, m.k0[j]);
    }
  }
}

// One (row group, column tile) unit: Coalesced Row Caching of the row's
// sparse segment through the per-warp double-buffered shared tile, CF column
// sub-tiles per lane (warp merging), U gathers in flight, ordered fold.
// HOT = kHotMap: the plan carries a hot-column map (bit 31 of a staged column
// marks a cold B row, loaded with the cold policy).  HOT = kHotReloc: the
// plan relocated the most-gathered B rows into its own contiguous copy
// (a.b_hot, refreshed every execute) and a.col_ind is its remapped copy, where
// bit 31 marks a relocated row and the low bits are its slot; those rows are
// gathered from the copy with evict_last, every other row from B with the cold
// policy, so L2 keeps the static top-by-frequency set instead of LRU's.
// HOT = kHotOff: every gather uses one policy register, so no per-load
// descriptor selection is emitted.
template <int OP, bool FAST, int VEC, int LPR, int CF, int HOT>
__device__ __forceinline__ void warp_unit(const SpmmArgs& a, const Policies& pol, uint32_t tile,
                                          const UnitMeta& m, uint32_t* my_col, float* my_val) {
  using R = Reduce<OP>;
  using G = WarpGeom<LPR, CF>;
  constexpr int RPW = G::RPW, U = G::U, W = G::W, E = G::E, CH = G::CH;
  constexpr uint32_t TILE = 32u * E;                // staged entries per buffer
  constexpr uint32_t SUB = uint32_t(VEC * LPR);     // columns per sub-tile
  constexpr uint32_t TW = SUB * CF;                 // columns per tile
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t sub = lane / LPR;
  const uint32_t sl = lane % LPR;
  const bool row_ok = m.row_ok;
  const uint32_t row = m.row, start = m.start, full_end = m.full_end;
  const uint32_t len = faulted_end(start, full_end, a.skip_tail) - start;
  const uint32_t maxlen = RPW == 1 ? len : __reduce_max_sync(kFull, len);

  const uint32_t col0 = tile * TW + sl * uint32_t(VEC);
  bool colok[CF];
  const char* bbase[CF];  // byte base of the lane's sub-tile (masked lanes: see below)
  float acc[CF][VEC];
  int32_t who[CF][VEC];
#pragma unroll
  for (int c = 0; c < CF; ++c) {
    colok[c] = row_ok && (col0 + c * SUB) < a.n;
#ifdef GESPMM_AB_MASK0
    bbase[c] = reinterpret_cast<const char*>(a.b + (colok[c] ? col0 + c * SUB : 0u));
#else
    // lanes past N re-read the row's last vector: it lies in a line the
    // quarter-warp's active lanes touch anyway, where column 0 added a line
    // (one more L1 wavefront per gathered row at N = 44)
    bbase[c] = reinterpret_cast<const char*>(a.b + (colok[c] ? col0 + c * SUB : a.n - uint32_t(VEC)));
#endif
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      acc[c][e] = R::init();
      who[c][e] = -1;
    }
  }
  bool all_cols = true;  // every sub-tile of every row of the warp in range (warp-uniform)
#pragma unroll
  for (int c = 0; c < CF; ++c) all_cols = all_cols && colok[c];
  all_cols = __all_sync(kFull, all_cols);
  const uint32_t stride = a.ldb * 4u;  // bytes per B row (B < 4 GiB per row index * stride)
  uint64_t pol_hot = pol.keep;
  if constexpr (HOT == kHotReloc) pol_hot = reloc_policy(a, pol);
  const uint32_t* ci = a.col_ind + start;
  const float* vs = a.vals + start;

  __syncwarp();  // the previous unit's reads of the tile are done
  const uint32_t slot = sub * uint32_t(CH) + sl;  // this lane's first entry in a buffer
#pragma unroll
  for (int j = 0; j < E; ++j) {  // phase 1 of chunk 0
    my_col[slot + j * LPR] = m.k0[j];
    my_val[slot + j * LPR] = m.v0[j];
  }
  uint32_t buf = 0;
  for (uint32_t off = 0; off < maxlen; off += CH) {
    // issue the next chunk's sparse loads before consuming this one
    uint32_t kn[E];
    float vn[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      kn[j] = 0;
      vn[j] = 0.0f;
      const uint32_t nxt = off + CH + uint32_t(j * LPR) + sl;
      if (nxt < len) {
        kn[j] = ld_stream_u32(ci + nxt, pol.stream);
        vn[j] = ld_stream_f32(vs + nxt, pol.stream);
        if (HOT == kHotMap) kn[j] |= cold_mark(a.hot, kn[j]);
        if (HOT == kHotReloc) kn[j] = reloc_index(a, kn[j]);
      }
    }
    __syncwarp();
    const uint32_t* cs = my_col + buf * TILE + sub * CH;
    const float* vsm = my_val + buf * TILE + sub * CH;
    const uint32_t chunk = min(uint32_t(CH), maxlen - off);
    for (uint32_t kk = 0; kk < chunk; kk += U) {
      uint32_t k[U];
      float v[U];
#pragma unroll
      for (int q = 0; q < U; q += W) {
        const typename Pack<W>::U c4 = *reinterpret_cast<const typename Pack<W>::U*>(cs + kk + q);
        const typename Pack<W>::F v4 = *reinterpret_cast<const typename Pack<W>::F*>(vsm + kk + q);
        const uint32_t* cp = reinterpret_cast<const uint32_t*>(&c4);
        const float* vp = reinterpret_cast<const float*>(&v4);
#pragma unroll
        for (int t = 0; t < W; ++t) {
          k[q + t] = cp[t];
          v[q + t] = vp[t];
        }
      }
      // all U*CF gathers issued before any fold (memory-level parallelism);
      // unpredicated: past-the-end slots re-read a valid row.
      Vec<VEC> bv[U][CF];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t pu = pol.keep;
        if constexpr (HOT == kHotReloc) {
          // staged index already relative to B (relocated rows: negative or
          // past K, inside the plan's copy): signed row offset, one policy
          // register (address-range policy: the copy evict_last)
#pragma unroll
          for (int c = 0; c < CF; ++c)
            bv[u][c] = ld_keep<VEC>(reinterpret_cast<const float*>(
                                        bbase[c] + int64_t(int32_t(k[u])) * int32_t(stride)),
                                    pol_hot);
          continue;
        }
        if (HOT == kHotMap) {
          // bit 31 of a staged column marks a cold B row (hot-column map).  With
          // one row per warp the mark is warp-uniform (vote), and with the
          // policies in launch parameters the choice is a uniform select.
          const bool cold = RPW == 1 ? __any_sync(kFull, k[u] & kColdBit) : (k[u] & kColdBit);
          k[u] &= ~kColdBit;
          pu = cold ? pol.cold : pol.keep;
        }
#pragma unroll
        for (int c = 0; c < CF; ++c)
          bv[u][c] = ld_keep<VEC>(
              reinterpret_cast<const float*>(bbase[c] + uint64_t(k[u]) * stride), pu);
      }
      const int32_t rem = int32_t(len - off - kk);  // entries left in this row (may be <= 0)
      const int32_t pos0 = int32_t(start + off + kk);
      if (rem >= U && all_cols) {
        // full batch, every sub-tile in range: no per-element predicates
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t pos = a.arg_col ? int32_t(k[u]) : pos0 + u;
#pragma unroll
          for (int c = 0; c < CF; ++c) fold_vec<OP, FAST, VEC>(acc[c], who[c], v[u], bv[u][c].x, pos);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u < rem) {
            const int32_t pos = a.arg_col ? int32_t(k[u]) : pos0 + u;
#pragma unroll
            for (int c = 0; c < CF; ++c)
              if (colok[c]) fold_vec<OP, FAST, VEC>(acc[c], who[c], v[u], bv[u][c].x, pos);
          }
        }
      }
    }
    buf ^= 1u;
#pragma unroll
    for (int j = 0; j < E; ++j) {  // phase 1 of the next chunk (buffer last read
      my_col[buf * TILE + slot + j * LPR] = kn[j];  // before this iteration's __syncwarp)
      my_val[buf * TILE + slot + j * LPR] = vn[j];
    }
  }

  const uint32_t row_len = full_end - start;
#pragma unroll
  for (int c = 0; c < CF; ++c) {
    if (!colok[c]) continue;
    float out[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) out[e] = finish<OP>(acc[c][e], row_len);
    const uint64_t o = uint64_t(row) * a.ld + col0 + c * SUB;
    st_stream<VEC>(a.c + o, out, pol.stream);
    if (R::kHasArg && a.arg) st_stream_i32<VEC>(a.arg + o, who[c], pol.stream);
    if (a.n_peer || a.c_mc) store_replicas<VEC, R::kHasArg>(a, o, out, who[c]);
  }
}

template <int OP, bool FAST, int VEC, int LPR, int CF, int HOT>
__global__ void __launch_bounds__(32 * kWarpBlock, warp_min_blocks<OP, CF, LPR>()) k_warp(SpmmArgs a) {
  // Staged sparse tile, double-buffered per warp: phase 1 writes E (col, val)
  // per lane, phase 2 reads them back with broadcast LDS of W entries — 2/W
  // shared-pipe wavefronts per nonzero instead of two shuffles.
  __shared__ __align__(16) uint32_t s_col[kWarpBlock][2][32 * WarpGeom<LPR, CF>::E];
  __shared__ __align__(16) float s_val[kWarpBlock][2][32 * WarpGeom<LPR, CF>::E];
  const uint32_t wib = threadIdx.x >> 5;
  const uint64_t unit = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t groups = (uint64_t(a.n_sched) + WarpGeom<LPR, CF>::RPW - 1) / WarpGeom<LPR, CF>::RPW;
  // dependents (an overlap_prev plan next on the stream) may launch once every
  // CTA of this grid has started; they wait for its completion before their
  // first B read (griddepcontrol.wait below), so this only overlaps launches
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (unit >= groups * a.n_tiles) return;  // warp-uniform exit
  if (aborted(a)) return;
  const Policies pol = args_policies(a);
  // (group, tile) without a 64-bit division in the common cases
  uint32_t group, tile;
  if (a.n_tiles == 1) {
    group = uint32_t(unit);
    tile = 0;
  } else if (unit <= 0xffffffffull) {
    group = uint32_t(unit) / a.n_tiles;
    tile = uint32_t(unit) - group * a.n_tiles;
  } else {
    group = uint32_t(unit / a.n_tiles);
    tile = uint32_t(unit % a.n_tiles);
  }
  UnitMeta m;
  unit_rows<LPR>(a, group, m);
  unit_chunk0<LPR, WarpGeom<LPR, CF>::E, HOT>(a, pol, m);
  // overlap_prev: row schedule, row_ptr and the first (col, val) chunk are in
  // flight; B and C belong to the previous kernel until it has completed
  if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  warp_unit<OP, FAST, VEC, LPR, CF, HOT>(a, pol, tile, m, &s_col[wib][0][0], &s_val[wib][0][0]);
}

template <int OP, bool FAST, int VEC, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_cta(SpmmArgs a) {
  using R = Reduce<OP>;
  constexpr int THREADS = WARPS * 32;
  constexpr int CHUNK = 256;                 // staged nonzeros per phase
  constexpr int PER_T = CHUNK / THREADS;     // staged entries per thread
  constexpr int U = 32 / VEC;                // gather batch per lane
  constexpr uint32_t TW = uint32_t(WARPS * 32 * VEC);
  static_assert(CHUNK % THREADS == 0 && CHUNK % U == 0, "chunk geometry");
  __shared__ uint2 s_kv[2][CHUNK];

  const uint32_t unit = blockIdx.x;
  const uint32_t sidx = unit / a.n_tiles;
  const uint32_t tile = unit % a.n_tiles;
  if (sidx >= a.n_sched || aborted(a)) return;
  const Policies pol = make_policies(a.hints);
  const uint32_t row = a.order ? a.order[sidx] : sidx;
  const uint32_t start = a.row_ptr[row];
  const uint32_t full_end = a.row_ptr[row + 1];
  const uint32_t len = faulted_end(start, full_end, a.skip_tail) - start;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t col0 = tile * TW + warp * (32u * VEC) + lane * uint32_t(VEC);
  const bool colok = col0 < a.n;
  const uint32_t* ci = a.col_ind + start;
  const float* vs = a.vals + start;

  float acc[VEC];
  int32_t who[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) {
    acc[e] = R::init();
    who[e] = -1;
  }

  // stage chunk 0
#pragma unroll
  for (int t = 0; t < PER_T; ++t) {
    const uint32_t i = threadIdx.x + t * THREADS;
    if (i < len)
      s_kv[0][i] = make_uint2(ld_stream_u32(ci + i, pol.stream),
                              __float_as_uint(ld_stream_f32(vs + i, pol.stream)));
  }
  __syncthreads();

  const float* bcol = a.b + col0;
  // lanes past N re-read the row's last vector (a line the active lanes touch)
  const float* bsafe = colok ? bcol : a.b + (a.n - uint32_t(VEC));
  for (uint32_t off = 0, buf = 0; off < len; off += CHUNK, buf ^= 1u) {
    // issue the next chunk's sparse loads before consuming this one
    uint2 nxt[PER_T];
#pragma unroll
    for (int t = 0; t < PER_T; ++t) {
      const uint32_t i = off + CHUNK + threadIdx.x + t * THREADS;
      nxt[t] = make_uint2(0u, 0u);
      if (i < len)
        nxt[t] = make_uint2(ld_stream_u32(ci + i, pol.stream),
                            __float_as_uint(ld_stream_f32(vs + i, pol.stream)));
    }
    const uint32_t n_cur = min(uint32_t(CHUNK), len - off);
    for (uint32_t kk = 0; kk < n_cur; kk += U) {
      uint2 kv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) kv[u] = s_kv[buf][kk + u];
      // unpredicated gathers (slots past the chunk re-read the batch's first
      // row, lanes past N re-read the row's last vector, bsafe): predicated loads let ptxas interleave
      // them with the folds, and the U loads in flight collapse to ~1
      Vec<VEC> bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = (kk + u < n_cur) ? kv[u].x : kv[0].x;
        bv[u] = ld_keep<VEC>(bsafe + uint64_t(k) * a.ldb, pol.keep);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kk + u < n_cur) {
          const int32_t pos = a.arg_col ? int32_t(kv[u].x) : int32_t(start + off + kk + u);
          const float v = __uint_as_float(kv[u].y);
#pragma unroll
          for (int e = 0; e < VEC; ++e) R::template fold<FAST>(acc[e], who[e], v, bv[u].x[e], pos);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < PER_T; ++t) s_kv[buf ^ 1u][threadIdx.x + t * THREADS] = nxt[t];
    __syncthreads();
  }

  if (colok) {
    float out[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) out[e] = finish<OP>(acc[e], full_end - start);
    const uint64_t o = uint64_t(row) * a.ld + col0;
    st_stream<VEC>(a.c + o, out, pol.stream);
    if (R::kHasArg && a.arg) st_stream_i32<VEC>(a.arg + o, who, pol.stream);
    if (a.n_peer || a.c_mc) store_replicas<VEC, R::kHasArg>(a, o, out, who);
  }
}

// k_hub — row per CTA for hub rows, fed by a shared-memory ring.  The ring
//   holds S stages of G nonzeros: for each nonzero the B-row slice of this
//   column tile (512*VEC bytes) plus its (col, val).  kHubProducers producer
//   warps fill stages round-robin with cp.async (LDGSTS, 16 B per lane, L1
//   bypassed), each stage's completion tracked by an mbarrier through
//   cp.async.mbarrier.arrive; one consumer warp owns the tile's 32*VEC columns
//   (VEC per lane) and folds the stages in ascending position — the
//   per-element ordered fold, bit-exact like every other kernel.  Narrow tiles
//   (VEC = 1: 32 columns) spread one hub row over N/32 SMs.  With ~64 KB of
//   gathers in flight per CTA a 21k-nonzero row is no longer bound by one
//   warp's 8-deep load batch (~1.6 ms), which otherwise caps a row shard's
//   step time from below (row-sharded multi-GPU, the pipelined host entry).
//   (A first version issued one TMA bulk copy per nonzero from a single
//   producer warp: 0.87 ms for a 21,657-nonzero row — the per-SM bulk-copy
//   engine keeps too few 512-B copies in flight; tools/longrow_probe.py.)
//   Needs N % 4 == 0 and 16-byte aligned B/C (16-byte copy units).
#ifndef GESPMM_HUB_PRODUCERS
#define GESPMM_HUB_PRODUCERS 4
#endif
constexpr int kHubProducers = GESPMM_HUB_PRODUCERS;  // producer (LDGSTS) warps
// Two ring geometries (BIG = the hub kernel carries the step, launched ahead of
// the warp kernel; small = a side job next to it): 16 nonzeros per stage in a
// 32 KB ring, or 32 per stage in 64 KB.  Fewer, larger stages halve the barrier
// round trips per nonzero (8-way Reddit shard 0.69 -> 0.58 ms) but the larger
// ring takes L1 capacity from a warp kernel running alongside (2-way shard 1.63
// -> 1.82 ms, products 4-way 3.69 -> 4.01 ms; profiles/r1_shard_emulation.md).
#ifndef GESPMM_HUB_BIG_GROUP
#define GESPMM_HUB_BIG_GROUP 32  // A/B builds: nonzeros per stage of the big ring
#endif
#ifndef GESPMM_HUB_BIG_KB
#define GESPMM_HUB_BIG_KB 64
#endif
template <bool BIG>
struct HubRing {
  static constexpr int GROUP = BIG ? GESPMM_HUB_BIG_GROUP : 16;  // nonzeros per stage (one full/empty pair)
  static constexpr int BYTES = (BIG ? GESPMM_HUB_BIG_KB : 32) * 1024;
};

template <int VEC, bool BIG, int C>
struct HubGeom {
  static constexpr int G = HubRing<BIG>::GROUP;
  static constexpr int RING = HubRing<BIG>::BYTES;
  static constexpr int TW = 32 * C * VEC;                      // columns per tile
  static constexpr int ROW_BYTES = TW * 4;                     // bytes per staged B slice
  static constexpr int CHUNKS = ROW_BYTES / 16;                // 16-byte copies per slice
  static constexpr int STAGES = RING / (ROW_BYTES * G);
  static_assert(STAGES >= kHubProducers, "every producer warp needs a stage of its own");
  static_assert((G * CHUNKS) % 32 == 0, "a stage is whole warp-wide copy rounds");
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
  // .cg (L2 only): staging through L1 (.ca) measured much slower
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

template <int VEC>
__device__ __forceinline__ Vec<VEC> lds_vec(const float* p) {
  Vec<VEC> r;
  if constexpr (VEC == 4) {
    const float4 f = *reinterpret_cast<const float4*>(p);
    r.x[0] = f.x;
    r.x[1] = f.y;
    r.x[2] = f.z;
    r.x[3] = f.w;
  } else if constexpr (VEC == 2) {
    const float2 f = *reinterpret_cast<const float2*>(p);
    r.x[0] = f.x;
    r.x[1] = f.y;
  } else {
    r.x[0] = p[0];
  }
  return r;
}

template <int OP, bool FAST, int VEC, bool BIG, int C>
__global__ void __launch_bounds__(32 * (C + kHubProducers))
k_hub(SpmmArgs a) {
  using R = Reduce<OP>;
  using H = HubGeom<VEC, BIG, C>;
  constexpr int S = H::STAGES, G = H::G;
  extern __shared__ __align__(128) unsigned char hub_smem[];
  float* ring = reinterpret_cast<float*>(hub_smem);                       // [S][G][TW]
  float* s_val = reinterpret_cast<float*>(hub_smem + H::RING);            // [S*G]
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_val + S * G);           // [S*G]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_col + S * G);            // full[S], empty[S]

  __shared__ uint32_t s_unit;
  if (aborted(a)) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }
  const Policies pol = args_policies(a);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + S);
  const uint32_t n_units = a.n_sched * a.n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      // full: one arrival per producer lane; empty: one arrival per consumer lane
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(full0 + 8 * i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * i),
                   "r"(32 * C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }

  // The warp kernel queued behind this one (programmatic dependent launch,
  // disjoint rows, no data dependence) may start now: these CTAs hold their
  // SM slots first, the warp kernel fills what is left.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // Units (hub row, column tile) in schedule (LPT) order.  Persistent launch
  // (a.work != null): CTAs pull units from a counter, so a few CTAs per SM
  // leave room for the warp kernel running alongside; otherwise one unit per
  // CTA.  Ring stages and barrier phases run on across units (gbase).
  uint32_t gbase = 0;
  for (uint32_t iter = 0;; ++iter) {
    if (threadIdx.x == 0)
      s_unit = a.work ? atomicAdd(a.work, 1u) : (iter == 0 ? blockIdx.x : 0xffffffffu);
    __syncthreads();
    const uint32_t unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t sidx = unit / a.n_tiles;
    const uint32_t tile = unit - sidx * a.n_tiles;
    const uint32_t row = a.order ? a.order[sidx] : sidx;
    const uint32_t start = a.row_ptr[row];
    const uint32_t full_end = a.row_ptr[row + 1];
    const uint32_t len = faulted_end(start, full_end, a.skip_tail) - start;
    const uint32_t col0 = tile * uint32_t(H::TW);
    const uint32_t tw = min(uint32_t(H::TW), a.n - col0);      // valid columns of this tile
    const uint32_t chunks = tw / 4u;                            // 16-byte copies per slice
    const uint32_t groups = (len + G - 1) / G;

    if (warp >= uint32_t(C)) {
      // ---- producer warp pw fills groups q = pw, pw + P, ...; the group's
      // (col, val) are loaded one group ahead of the copies they address.
      const uint32_t pw = warp - uint32_t(C);
      const uint32_t* ci = a.col_ind + start;
      const float* vs = a.vals + start;
      const char* bsrc = reinterpret_cast<const char*>(a.b + col0);
      const uint64_t stride = uint64_t(a.ldb) * 4u;
      uint32_t q = pw;
      uint32_t kn = 0;
      if (q < groups && q * G + lane < len && lane < uint32_t(G))
        kn = ld_stream_u32(ci + q * G + lane, pol.stream);
      for (; q < groups; q += kHubProducers) {
        const uint32_t kcur = kn;
        const uint32_t qn = q + kHubProducers;
        kn = 0;
        if (qn < groups && lane < uint32_t(G) && qn * G + lane < len)
          kn = ld_stream_u32(ci + qn * G + lane, pol.stream);
        const uint32_t ga = gbase + q;
        const uint32_t st = ga % S, round = ga / S;
        if (round > 0) mbar_wait(empty0 + 8 * st, (round - 1) & 1u);
        const uint32_t cnt = min(uint32_t(G), len - q * G);
        const uint32_t e0 = st * G;
        if (lane < cnt) {
          cp_async4(smem_addr(s_val + e0 + lane), vs + q * G + lane);
          cp_async4(smem_addr(s_col + e0 + lane), ci + q * G + lane);
        }
        // the group's G x CHUNKS 16-byte pieces, spread over the lanes: piece c
        // is entry c / CHUNKS, bytes 16 * (c % CHUNKS) of its B slice
        const uint32_t slot = smem_addr(ring + size_t(e0) * H::TW);
#pragma unroll
        for (int j = 0; j < (G * H::CHUNKS) / 32; ++j) {
          const uint32_t c = lane + 32u * uint32_t(j);
          const uint32_t e = c / uint32_t(H::CHUNKS), piece = c % uint32_t(H::CHUNKS);
          const uint32_t k = __shfl_sync(0xffffffffu, kcur, int(e));
          if (e < cnt && piece < chunks)
            cp_async16(slot + c * 16u, bsrc + uint64_t(k) * stride + piece * 16u, pol.keep);
        }
#ifdef GESPMM_HUB_ASYNC_ARRIVE
        // the stage completes when every lane's copies land (no producer stall)
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full0 + 8 * st)
                     : "memory");
#else
        // each lane waits for its own copies, then arrives with release
        // semantics: the same completion point (a producer warp has nothing
        // else to issue until the ring frees its next stage), expressed as an
        // ordinary barrier handoff that compute-sanitizer's racecheck can follow
        asm volatile("cp.async.wait_all;" ::: "memory");
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(full0 + 8 * st)
                     : "memory");
#endif
      }
    } else {
      // ---- consumer warps: thread t owns columns col0 + t*VEC .. +VEC
      const uint32_t t = threadIdx.x;                    // 0 .. 32*C-1
      const bool colok = t * uint32_t(VEC) < tw;
      float acc[VEC];
      int32_t who[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc[e] = R::init();
        who[e] = -1;
      }
      for (uint32_t q = 0; q < groups; ++q) {
        const uint32_t ga = gbase + q;
        const uint32_t st = ga % S;
        mbar_wait(full0 + 8 * st, (ga / S) & 1u);
        const uint32_t cnt = min(uint32_t(G), len - q * G);
        const float* slot = ring + size_t(st) * G * H::TW + t * VEC;
        if (colok) {
          if (cnt == uint32_t(G)) {
            // every shared-memory read of the stage first (G loads in flight),
            // then the ordered fold
            Vec<VEC> bv[G];
            float vv[G];
#pragma unroll
            for (int e = 0; e < G; ++e) {
              bv[e] = lds_vec<VEC>(slot + e * H::TW);
              vv[e] = s_val[st * G + e];
            }
#pragma unroll
            for (int e = 0; e < G; ++e) {
              const int32_t pos =
                  a.arg_col ? int32_t(s_col[st * G + e]) : int32_t(start + q * G + e);
              fold_vec<OP, FAST, VEC>(acc, who, vv[e], bv[e].x, pos);
            }
          } else {
            for (uint32_t e = 0; e < cnt; ++e) {
              const Vec<VEC> bv = lds_vec<VEC>(slot + e * H::TW);
              const float v = s_val[st * G + e];
              const int32_t pos =
                  a.arg_col ? int32_t(s_col[st * G + e]) : int32_t(start + q * G + e);
              fold_vec<OP, FAST, VEC>(acc, who, v, bv.x, pos);
            }
          }
        }
        // every consumer lane releases its own reads of the stage (32 * C
        // arrivals): the producer's acquire then orders each lane's reads
        // before the next round's copies directly, which compute-sanitizer's
        // racecheck verifies (with one arrival per warp after __syncwarp it
        // could not follow lanes 1..31 and reported every stage)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * st)
                     : "memory");
      }
      if (colok) {
        float out[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) out[e] = finish<OP>(acc[e], full_end - start);
        const uint64_t o = uint64_t(row) * a.ld + col0 + t * VEC;
        st_stream<VEC>(a.c + o, out, pol.stream);
        if (R::kHasArg && a.arg) st_stream_i32<VEC>(a.arg + o, who, pol.stream);
        if (a.n_peer || a.c_mc) store_replicas<VEC, R::kHasArg>(a, o, out, who);
      }
    }
    gbase += groups;
    __syncthreads();  // the unit is done (and s_unit read) before the next fetch
  }
}

// k_hub_g4 — the same ring fed by the tensor-memory accelerator instead of
//   LDGSTS: one producer warp, and per stage G/4 lanes each issue one
//   cp.async.bulk.tensor.2d ... tile::gather4 (four B rows, the tile's TW
//   columns each, straight into the stage; a tensor map over B, box {TW, 1})
//   with mbarrier complete_tx accounting.  The staged bytes enter shared memory
//   through the TMA unit, not the LSU pipe, and the four LDGSTS producer warps
//   (and their per-lane address math) go away.  Columns past the slice width
//   and rows past K are zero-filled by the unit (never folded: colok / cnt).
//   The consumer side and with it the per-element ascending fold are k_hub's.
template <int OP, bool FAST, int VEC, bool BIG, int C>
__global__ void __launch_bounds__(32 * (C + 1))
k_hub_g4(SpmmArgs a, const __grid_constant__ CUtensorMap tmap) {
  using R = Reduce<OP>;
  using H = HubGeom<VEC, BIG, C>;
  constexpr int S = H::STAGES, G = H::G;
  constexpr uint32_t OP_BYTES = 4u * uint32_t(H::ROW_BYTES);  // one gather4: 4 B slices
  static_assert(G % 4 == 0 && G / 4 <= 32, "a stage is whole gather4 ops, one per lane");
  extern __shared__ __align__(128) unsigned char hub_smem[];
  float* ring = reinterpret_cast<float*>(hub_smem);                       // [S][G][TW]
  float* s_val = reinterpret_cast<float*>(hub_smem + H::RING);            // [S*G]
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_val + S * G);           // [S*G]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_col + S * G);            // full[S], empty[S]

  __shared__ uint32_t s_unit;
  if (aborted(a)) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    return;
  }
  const Policies pol = args_policies(a);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = smem_addr(bars), empty0 = smem_addr(bars + S);
  const uint32_t n_units = a.n_sched * a.n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      // full: the producer's arrive.expect_tx (+ the stage's bytes); empty:
      // one arrival per consumer lane
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8 * i), "r"(32 * C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == uint32_t(C) && lane == 0)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  uint32_t gbase = 0;
  for (uint32_t iter = 0;; ++iter) {
    if (threadIdx.x == 0)
      s_unit = a.work ? atomicAdd(a.work, 1u) : (iter == 0 ? blockIdx.x : 0xffffffffu);
    __syncthreads();
    const uint32_t unit = s_unit;
    if (unit >= n_units) break;
    const uint32_t sidx = unit / a.n_tiles;
    const uint32_t tile = unit - sidx * a.n_tiles;
    const uint32_t row = a.order ? a.order[sidx] : sidx;
    const uint32_t start = a.row_ptr[row];
    const uint32_t full_end = a.row_ptr[row + 1];
    const uint32_t len = faulted_end(start, full_end, a.skip_tail) - start;
    const uint32_t col0 = tile * uint32_t(H::TW);
    const uint32_t tw = min(uint32_t(H::TW), a.n - col0);
    const uint32_t groups = (len + G - 1) / G;

    if (warp == uint32_t(C)) {
      // ---- producer warp: group q's (col, val) are loaded one group ahead
      const uint32_t* ci = a.col_ind + start;
      const float* vs = a.vals + start;
      uint32_t kn = 0;
      float vn = 0.0f;
      if (groups && lane < uint32_t(G) && lane < len) {
        kn = ld_stream_u32(ci + lane, pol.stream);
        vn = ld_stream_f32(vs + lane, pol.stream);
      }
      for (uint32_t q = 0; q < groups; ++q) {
        const uint32_t kcur = kn;
        const float vcur = vn;
        const uint32_t nx = (q + 1) * uint32_t(G) + lane;
        kn = 0;
        vn = 0.0f;
        if (lane < uint32_t(G) && nx < len) {
          kn = ld_stream_u32(ci + nx, pol.stream);
          vn = ld_stream_f32(vs + nx, pol.stream);
        }
        const uint32_t ga = gbase + q;
        const uint32_t st = ga % S, round = ga / S;
        if (round > 0) mbar_wait(empty0 + 8 * st, (round - 1) & 1u);
        const uint32_t cnt = min(uint32_t(G), len - q * G);
        const uint32_t e0 = st * G;
        if (lane < cnt) {
          s_val[e0 + lane] = vcur;
          s_col[e0 + lane] = kcur;
        }
        __syncwarp();
        // slots past the row end gather the group's first row again (never folded)
        const uint32_t k_first = __shfl_sync(kFull, kcur, 0);
        const uint32_t kk = lane < cnt ? kcur : k_first;
        const uint32_t r0 = __shfl_sync(kFull, kk, int(4 * (lane & 7u) + 0));
        const uint32_t r1 = __shfl_sync(kFull, kk, int(4 * (lane & 7u) + 1));
        const uint32_t r2 = __shfl_sync(kFull, kk, int(4 * (lane & 7u) + 2));
        const uint32_t r3 = __shfl_sync(kFull, kk, int(4 * (lane & 7u) + 3));
        const uint32_t n_ops = (cnt + 3u) / 4u;
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * st),
                       "r"(n_ops * OP_BYTES)
                       : "memory");
        __syncwarp();
        if (lane < n_ops) {
          const uint32_t dst = smem_addr(ring + size_t(e0 + 4 * lane) * H::TW);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(col0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
              "r"(full0 + 8 * st), "l"(pol.keep)
              : "memory");
        }
      }
    } else {
      // ---- consumer warps (k_hub's): thread t owns columns col0 + t*VEC .. +VEC
      const uint32_t t = threadIdx.x;
      const bool colok = t * uint32_t(VEC) < tw;
      float acc[VEC];
      int32_t who[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        acc[e] = R::init();
        who[e] = -1;
      }
      for (uint32_t q = 0; q < groups; ++q) {
        const uint32_t ga = gbase + q;
        const uint32_t st = ga % S;
        mbar_wait(full0 + 8 * st, (ga / S) & 1u);
        const uint32_t cnt = min(uint32_t(G), len - q * G);
        const float* slot = ring + size_t(st) * G * H::TW + t * VEC;
        if (colok) {
          if (cnt == uint32_t(G)) {
            Vec<VEC> bv[G];
            float vv[G];
#pragma unroll
            for (int e = 0; e < G; ++e) {
              bv[e] = lds_vec<VEC>(slot + e * H::TW);
              vv[e] = s_val[st * G + e];
            }
#pragma unroll
            for (int e = 0; e < G; ++e) {
              const int32_t pos =
                  a.arg_col ? int32_t(s_col[st * G + e]) : int32_t(start + q * G + e);
              fold_vec<OP, FAST, VEC>(acc, who, vv[e], bv[e].x, pos);
            }
          } else {
            for (uint32_t e = 0; e < cnt; ++e) {
              const Vec<VEC> bv = lds_vec<VEC>(slot + e * H::TW);
              const float v = s_val[st * G + e];
              const int32_t pos =
                  a.arg_col ? int32_t(s_col[st * G + e]) : int32_t(start + q * G + e);
              fold_vec<OP, FAST, VEC>(acc, who, v, bv.x, pos);
            }
          }
        }
        // every consumer lane releases its own reads of the stage (32 * C
        // arrivals): the producer's acquire then orders each lane's reads
        // before the next round's copies directly, which compute-sanitizer's
        // racecheck verifies (with one arrival per warp after __syncwarp it
        // could not follow lanes 1..31 and reported every stage)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * st)
                     : "memory");
      }
      if (colok) {
        float out[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) out[e] = finish<OP>(acc[e], full_end - start);
        const uint64_t o = uint64_t(row) * a.ld + col0 + t * VEC;
        st_stream<VEC>(a.c + o, out, pol.stream);
        if (R::kHasArg && a.arg) st_stream_i32<VEC>(a.arg + o, who, pol.stream);
        if (a.n_peer || a.c_mc) store_replicas<VEC, R::kHasArg>(a, o, out, who);
      }
    }
    gbase += groups;
    __syncthreads();
  }
}

template <int VEC, bool BIG, int C>
constexpr size_t hub_smem_bytes() {
  using H = HubGeom<VEC, BIG, C>;
  return size_t(H::RING) + size_t(H::STAGES) * H::G * 8 + size_t(H::STAGES) * 16;
}

// ---- dispatch tables ------------------------------------------------------

template <class K>
cudaError_t launch_ex(K kernel, dim3 g, dim3 b, cudaStream_t st, const SpmmArgs& a,
                      const cudaAccessPolicyWindow* window, bool pdl = false) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  cfg.numAttrs = 0;
  if (window) {
    attr[cfg.numAttrs].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[cfg.numAttrs].val.accessPolicyWindow = *window;
    ++cfg.numAttrs;
  }
  if (pdl) {  // programmatic dependent launch: may start once the previous kernel triggers
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

// Shared-memory carve-out preference for the warp kernel (percent of the
// unified L1/shared array; GESPMM_WARP_CARVEOUT, <0 = driver default).
int warp_carveout() {
  static const int v = [] {
    const char* e = std::getenv("GESPMM_WARP_CARVEOUT");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

template <class K>
void apply_carveout(K kernel) {
  const int c = warp_carveout();
  if (c >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
}

template <int OP, bool FAST>
cudaError_t warp_dispatch(const WarpShape& s, const SpmmArgs& a, cudaStream_t st,
                          const cudaAccessPolicyWindow* window, bool pdl) {
  const uint32_t rpw = 32u / uint32_t(s.lpr);
  const uint64_t groups = (uint64_t(a.n_sched) + rpw - 1) / rpw;
  const uint64_t warps = groups * a.n_tiles;
  const uint64_t blocks = (warps + kWarpBlock - 1) / kWarpBlock;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const dim3 b{32 * kWarpBlock};
  // shapes without a hot-row mode gather B directly through the caller's col_ind
  SpmmArgs plain = a;
  if (plain.col_ind_orig) plain.col_ind = plain.col_ind_orig;
  plain.b_hot = nullptr;
#define GESPMM_W(V, L, F)                                                                    \
  if (s.vec == V && s.lpr == L && s.cf == F) {                                               \
    constexpr int kMap = (kExpBuild && L == 32) ? kHotMap : kHotOff;   /* full-warp rows only */ \
    constexpr int kReloc = (kExpBuild && L == 32) ? kHotReloc : kHotOff;                     \
    const dim3 g{uint32_t(blocks)};                                                          \
    apply_carveout(k_warp<OP, FAST, V, L, F, kHotOff>);                                      \
    const cudaError_t e =                                                                    \
        (kReloc == kHotReloc && a.b_hot) ? launch_ex(k_warp<OP, FAST, V, L, F, kReloc>, g, b, st, a, window, pdl) \
        : (kMap == kHotMap && a.hot) ? launch_ex(k_warp<OP, FAST, V, L, F, kMap>, g, b, st, a, window, pdl) \
                             : launch_ex(k_warp<OP, FAST, V, L, F, kHotOff>, g, b, st, plain, window, pdl); \
    note_launch();                                                                           \
    return e;                                                                                \
  }
  GESPMM_W(4, 4, 1) GESPMM_W(4, 8, 1) GESPMM_W(4, 16, 1) GESPMM_W(4, 32, 1)
  GESPMM_W(4, 32, 2) GESPMM_W(4, 32, 4)
  GESPMM_W(4, 4, 2) GESPMM_W(4, 8, 2) GESPMM_W(4, 8, 4) GESPMM_W(4, 16, 2) GESPMM_W(4, 16, 4)
  GESPMM_W(2, 32, 1) GESPMM_W(2, 32, 2) GESPMM_W(2, 32, 4)
  GESPMM_W(1, 1, 1) GESPMM_W(1, 2, 1) GESPMM_W(1, 4, 1) GESPMM_W(1, 8, 1)
  GESPMM_W(1, 16, 1) GESPMM_W(1, 32, 1) GESPMM_W(1, 32, 2) GESPMM_W(1, 32, 4)
#undef GESPMM_W
  return cudaErrorInvalidValue;
}

template <int OP, bool FAST>
cudaError_t cta_dispatch(const CtaShape& s, const SpmmArgs& a, cudaStream_t st) {
  const uint64_t blocks = uint64_t(a.n_sched) * a.n_tiles;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  const dim3 g{uint32_t(blocks)};
#define GESPMM_C(V, W)                                          \
  if (s.vec == V && s.warps == W) {                             \
    k_cta<OP, FAST, V, W><<<g, dim3(W * 32), 0, st>>>(a);       \
    note_launch();                                              \
    return cudaGetLastError();                                  \
  }
  GESPMM_C(1, 1) GESPMM_C(1, 2) GESPMM_C(1, 4) GESPMM_C(1, 8)
  GESPMM_C(4, 2) GESPMM_C(4, 4) GESPMM_C(4, 8)
#undef GESPMM_C
  return cudaErrorInvalidValue;
}

// Persistent hub launches pull units from a counter zeroed on the launch's
// stream right before it.  Plans and the host entry's workspace own their
// counters (SpmmArgs::work, one per launch site), so a captured graph or a
// second stream never shares one; only a caller without one (none in the
// library today) falls back to this per-device ring.
struct HubCounters {
  uint32_t* d = nullptr;
  std::atomic<uint32_t> next{0};
};
constexpr uint32_t kHubCounterRing = 256;

cudaError_t hub_counter(uint32_t** out, cudaStream_t st) {
  static std::mutex mu;
  static HubCounters per_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  HubCounters& h = per_dev[dev];
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!h.d &&
        (e = cudaMalloc(reinterpret_cast<void**>(&h.d), sizeof(uint32_t) * kHubCounterRing)) !=
            cudaSuccess)
      return e;
  }
  uint32_t* c = h.d + (h.next.fetch_add(1) % kHubCounterRing);
  *out = c;
  return cudaMemsetAsync(c, 0, sizeof(uint32_t), st);
}

int sm_count_of_current_device() {
  static std::mutex mu;
  static int sms[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lk(mu);
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] > 0 ? sms[dev] : 148;
}

// cudaFuncSetAttribute once per (kernel instance, device); not stream-ordered,
// so concurrent first calls from two host threads are serialised.
template <typename K>
cudaError_t set_smem_once(K kernel, size_t bytes, bool* done) {
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

// Hub ring feed: the LDGSTS producer warps (default) or TMA gather4
// (GESPMM_HUB_FEED=g4).  gather4 measured at about half the LDGSTS feed's
// rate: ~135 clk per 4-row op per SM whatever the row width, i.e. ~15 B/clk
// per SM at 512-B slices (LDGSTS ~27); 8-way Reddit shard 0.594 vs 0.528 ms,
// one 21,657-nonzero row 0.367 vs 0.213 ms (profiles/r2/hub_g4_ab.md).
bool hub_feed_g4() {
  static const bool v = [] {
    const char* e = std::getenv("GESPMM_HUB_FEED");
    return e && std::string(e) == "g4";
  }();
  return v;
}

// 2-D tensor map over B (rows of `n` floats at pitch `ldb`, kb rows) with a
// {tw, 1} box: the gather4 source.  cuTensorMapEncodeTiled through the
// runtime's driver entry point (no libcuda link dependency).
bool encode_b_map(const float* b, uint32_t n, uint32_t ldb, uint32_t kb, uint32_t tw,
                  CUtensorMap* out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<Encode>(p);
  }();
  if (!enc || tw == 0 || tw > 256 || (reinterpret_cast<uintptr_t>(b) & 15u) || (ldb % 4u) ||
      n == 0 || kb == 0)
    return false;
  const cuuint64_t dims[2] = {n, kb};
  const cuuint64_t strides[1] = {cuuint64_t(ldb) * 4u};
  const cuuint32_t box[2] = {tw, 1};
  const cuuint32_t estr[2] = {1, 1};
  return enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(b), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int OP, bool FAST>
cudaError_t hub_dispatch(int vec, int cons, bool big, const SpmmArgs& a0, cudaStream_t st) {
  const uint64_t units = uint64_t(a0.n_sched) * a0.n_tiles;
  if (units == 0) return cudaSuccess;
  if (units > 0x7fffffffull) return cudaErrorInvalidConfiguration;
  SpmmArgs a = a0;
  // persistent: at most 2 CTAs per SM when the hub kernel runs next to the
  // warp kernel (side job), so the warp kernel keeps most of each SM; one CTA
  // per unit (as many as fit) when it runs alone ahead of it (big: the hub
  // rows carry the launch).  GESPMM_HUB_PERSIST=n forces n per SM (0 = one
  // CTA per unit) in both modes.
  static const int per_sm_env = [] {
    const char* e = std::getenv("GESPMM_HUB_PERSIST");
    return e ? std::atoi(e) : -1;
  }();
  const int per_sm = per_sm_env >= 0 ? per_sm_env : (big ? 0 : 2);
  uint64_t blocks = units;
  if (per_sm > 0) {
    const cudaError_t ec = a0.work ? cudaMemsetAsync(a.work, 0, sizeof(uint32_t), st)
                                   : hub_counter(&a.work, st);
    if (ec != cudaSuccess) return ec;
    blocks = std::min<uint64_t>(units, uint64_t(per_sm) * uint64_t(sm_count_of_current_device()));
  } else {
    a.work = nullptr;
  }
  // TMA gather4 feed when a tensor map over B can be encoded (B rows known,
  // 16-byte row pitch and base: the caller's tma test)
  CUtensorMap tmap;
  const bool g4 = hub_feed_g4() && a.kb > 0 &&
                  encode_b_map(a.b, a.n, a.ldb, a.kb, uint32_t(32 * cons * vec), &tmap);
#define GESPMM_H(V, BIG, C)                                                                \
  if (vec == V && big == BIG && cons == C) {                                               \
    const size_t sm = hub_smem_bytes<V, BIG, C>();                                         \
    if (g4) {                                                                              \
      static bool attr_g4[64] = {};                                                        \
      const cudaError_t e0 = set_smem_once(k_hub_g4<OP, FAST, V, BIG, C>, sm, attr_g4);    \
      if (e0 != cudaSuccess) return e0;                                                    \
      k_hub_g4<OP, FAST, V, BIG, C><<<dim3(uint32_t(blocks)), dim3(32 * (C + 1)), sm, st>>>(a, tmap); \
    } else {                                                                               \
      static bool attr_done[64] = {};                                                      \
      const cudaError_t e0 = set_smem_once(k_hub<OP, FAST, V, BIG, C>, sm, attr_done);     \
      if (e0 != cudaSuccess) return e0;                                                    \
      k_hub<OP, FAST, V, BIG, C><<<dim3(uint32_t(blocks)), dim3(32 * (C + kHubProducers)), sm, st>>>(a); \
    }                                                                                      \
    note_launch();                                                                         \
    return cudaGetLastError();                                                             \
  }
  // tile of 32 * C * V columns: one consumer warp with V-wide lanes, or C
  // consumer warps sharing the tile's columns (fewer instructions per warp
  // per nonzero, folds on C schedulers at once)
  GESPMM_H(1, false, 1) GESPMM_H(2, false, 1) GESPMM_H(4, false, 1)
  GESPMM_H(1, true, 1) GESPMM_H(2, true, 1) GESPMM_H(4, true, 1)
  GESPMM_H(1, false, 2) GESPMM_H(2, false, 2) GESPMM_H(1, false, 4)
  GESPMM_H(1, true, 2) GESPMM_H(2, true, 2) GESPMM_H(1, true, 4)
#undef GESPMM_H
  return cudaErrorInvalidValue;
}

__global__ void k_range_policy(const void* base, uint32_t bytes, int mode, uint64_t* out) {
  uint64_t p;
  if (mode == 1)
    asm("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
        : "=l"(p)
        : "l"(base), "r"(bytes), "r"(bytes));
  else
    asm("createpolicy.range.global.L2::evict_last.b64 %0, [%1], %2, %3;"
        : "=l"(p)
        : "l"(base), "r"(bytes), "r"(bytes));
  out[0] = p;
}

__global__ void k_policies(int hints, uint64_t* out) {
  const Policies p = make_policies(hints);
  out[0] = p.keep;
  out[1] = p.cold;
  out[2] = p.stream;
}

// Split hub rows (order-insensitive folds): a hub row's nonzeros were cut into
// segments, each folded by k_warp into its own partial row (value, and the
// position of the element that last replaced it for max/min).  One thread per
// (hub row, column) folds the partials in segment order — for max/min with
// the fold's own strict compare, so the earliest position among equal maxima
// survives and the result is bit-identical to the sequential fold; for sum /
// mean (fast mode only) in segment order (a different, tolerance-level
// rounding).  Then the row's epilogue: mean's division, C, arg, replicas.
// hubs[3h..3h+2] = (row, first partial row, partial rows).
template <int OP>
__global__ void __launch_bounds__(256) k_split_combine(SpmmArgs a, const uint32_t* __restrict__ hubs,
                                                       uint32_t n_hub, const float* __restrict__ part,
                                                       const int32_t* __restrict__ part_arg) {
  using R = Reduce<OP>;
  const uint64_t total = uint64_t(n_hub) * a.n;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t h = uint32_t(i / a.n), col = uint32_t(i - uint64_t(h) * a.n);
    const uint32_t row = hubs[3 * h], v0 = hubs[3 * h + 1], k = hubs[3 * h + 2];
    float acc = R::init();
    int32_t who = -1;
    for (uint32_t j = 0; j < k; ++j) {
      const uint64_t q = uint64_t(v0 + j) * a.n + col;
      const float x = part[q];
      if constexpr (OP == kSum || OP == kMean) {
        acc = __fadd_rn(acc, x);
      } else if constexpr (OP == kMax) {
        if (acc < x) {
          acc = x;
          who = part_arg[q];
        }
      } else {
        if (x < acc) {
          acc = x;
          who = part_arg[q];
        }
      }
    }
    const float out = finish<OP>(acc, a.row_ptr[row + 1] - a.row_ptr[row]);
    const uint64_t o = uint64_t(row) * a.ld + col;
    a.c[o] = out;
    if (R::kHasArg && a.arg) a.arg[o] = who;
    if (a.n_peer || a.c_mc) store_replicas<1, R::kHasArg>(a, o, &out, &who);
  }
}

__global__ void __launch_bounds__(256) k_split_refresh(const uint32_t* __restrict__ row_ptr,
                                                       const uint32_t* __restrict__ hubs,
                                                       uint32_t n_hub, uint32_t seg_len,
                                                       uint32_t* __restrict__ vptr) {
  for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < n_hub; h += gridDim.x * blockDim.x) {
    const uint32_t row = hubs[3 * h], v0 = hubs[3 * h + 1], k = hubs[3 * h + 2];
    const uint32_t lo = row_ptr[row], hi = row_ptr[row + 1];
    const uint32_t d = hi - lo;
    for (uint32_t j = 0; j < k; ++j) {
      const uint64_t off = uint64_t(j) * seg_len;
      vptr[v0 + j] = lo + uint32_t(off < d ? off : d);
    }
    vptr[v0 + k] = hi;
  }
}

}  // namespace

cudaError_t resolve_range_policy(const void* base, uint32_t bytes, int mode, uint64_t* out,
                                 cudaStream_t st) {
  struct Key {
    int dev;
    const void* base;
    uint32_t bytes;
    int mode;
    bool operator<(const Key& o) const {
      return std::tie(dev, base, bytes, mode) < std::tie(o.dev, o.base, o.bytes, o.mode);
    }
  };
  static std::mutex mu;
  static std::map<Key, uint64_t> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const Key key{dev, base, bytes, mode};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  uint64_t* d = nullptr;
  uint64_t v = 0;
  if ((e = cudaMalloc(reinterpret_cast<void**>(&d), sizeof(v))) != cudaSuccess) return e;
  k_range_policy<<<1, 1, 0, st>>>(base, bytes, mode, d);
  note_launch();
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 64) cache.clear();
  cache[key] = v;
  *out = v;
  return cudaSuccess;
}

cudaError_t resolve_policies(SpmmArgs* a, cudaStream_t st) {
  struct Entry {
    bool ok = false;
    uint64_t v[3] = {0, 0, 0};
  };
  static std::mutex mu;
  static Entry cache[64][3];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const int h = a->hints < 0 ? 0 : (a->hints > 2 ? 2 : a->hints);
  if (dev < 0 || dev >= 64) {
    a->pol_valid = 0;
    return cudaSuccess;
  }
  std::lock_guard<std::mutex> lk(mu);
  Entry& en = cache[dev][h];
  if (!en.ok) {
    uint64_t* d = nullptr;
    if ((e = cudaMalloc(reinterpret_cast<void**>(&d), sizeof(en.v))) != cudaSuccess) return e;
    k_policies<<<1, 1, 0, st>>>(h, d);
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(en.v, d, sizeof(en.v), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return e;
    en.ok = true;
  }
  a->pol_keep = en.v[0];
  a->pol_cold = en.v[1];
  a->pol_stream = en.v[2];
  a->pol_valid = 1;
  return cudaSuccess;
}

bool tuned_shape_supported(const WarpShape& s) {
  static const int table[][3] = {{4, 4, 1},  {4, 8, 1},  {4, 16, 1}, {4, 32, 1}, {4, 32, 2},
                                 {4, 32, 4}, {4, 4, 2},  {4, 8, 2},  {4, 8, 4},  {4, 16, 2},
                                 {4, 16, 4}, {2, 32, 1}, {2, 32, 2}, {2, 32, 4}, {1, 1, 1},
                                 {1, 2, 1},  {1, 4, 1},  {1, 8, 1},  {1, 16, 1}, {1, 32, 1},
                                 {1, 32, 2}, {1, 32, 4}};
  for (const auto& t : table)
    if (t[0] == s.vec && t[1] == s.lpr && t[2] == s.cf) return true;
  return false;
}

// N -> (VEC, LPR, CF): the smallest sub-warp whose VEC-wide lanes cover N
// (several short rows per warp when N < 128), then the CWM merge factor so a
// warp covers up to 4 sub-tiles of one row before the row is re-staged.
// rows_per_warp > 1 (low-degree matrices, where the per-row prologue and
// epilogue outweigh the few gathers of a row): float4 lanes only, LPR shrunk
// so that several rows share a warp, each lane covering up to 4 sub-tiles.
WarpShape pick_warp_shape(uint32_t n, bool vec4_ok, bool vec2_ok, int rows_per_warp) {
  WarpShape s;
  s.vec = vec4_ok ? 4 : (vec2_ok ? 2 : 1);
  if (n < 16 || (s.vec == 2 && n < 64)) s.vec = 1;  // narrow rows: scalar lanes waste less
  const uint32_t lanes = (n + uint32_t(s.vec) - 1) / uint32_t(s.vec);
  if (rows_per_warp > 1 && s.vec == 4 && lanes >= 8 && lanes <= 64) {
    uint32_t lpr = 32u / uint32_t(rows_per_warp);
    lpr = std::max<uint32_t>(4, std::min<uint32_t>(16, lpr));
    while (lanes > lpr * 4u) lpr *= 2;  // CF <= 4
    uint32_t cf = (lanes + lpr - 1) / lpr;
    cf = cf >= 4 ? 4 : (cf >= 2 ? 2 : 1);
    WarpShape t;
    t.vec = 4;
    t.lpr = int(lpr);
    t.cf = int(cf);
    if (lpr < 32 && tuned_shape_supported(t)) return t;
  }
  if (lanes >= 32) {
    s.lpr = 32;
    const uint32_t sub = 32u * uint32_t(s.vec);
    const uint32_t tiles = (n + sub - 1) / sub;
    s.cf = tiles >= 4 ? 4 : (tiles >= 2 ? 2 : 1);
  } else {
    int l = 1;
    while (uint32_t(l) < lanes) l <<= 1;
    if (s.vec == 4 && l < 4) l = 4;
    s.lpr = l;
    s.cf = 1;
  }
  return s;
}

bool cta_shape_supported(const CtaShape& s) {
  return (s.vec == 1 && (s.warps == 1 || s.warps == 2 || s.warps == 4 || s.warps == 8)) ||
         (s.vec == 4 && (s.warps == 2 || s.warps == 4 || s.warps == 8));
}

// Hub rows: split the columns over as many warps as give every lane a column
// (scalar lanes up to 256 columns), wider lanes beyond that.
CtaShape pick_cta_shape(uint32_t n, bool vec4_ok, bool /*vec2_ok*/) {
  CtaShape s;
  if (n <= 256 || !vec4_ok) {
    s.vec = 1;
    const uint32_t w = (n + 31) / 32;
    s.warps = w >= 8 ? 8 : (w >= 4 ? 4 : (w >= 2 ? 2 : 1));
  } else {
    s.vec = 4;
    const uint32_t w = (n + 127) / 128;
    s.warps = w >= 8 ? 8 : (w >= 4 ? 4 : 2);
  }
  return s;
}

cudaError_t launch_tuned_warp(const WarpShape& s, int op, bool fast, const SpmmArgs& a,
                              cudaStream_t st, const cudaAccessPolicyWindow* w, bool pdl) {
  switch (op) {
    case kSum: return fast ? warp_dispatch<kSum, true>(s, a, st, w, pdl) : warp_dispatch<kSum, false>(s, a, st, w, pdl);
    case kMean: return fast ? warp_dispatch<kMean, true>(s, a, st, w, pdl) : warp_dispatch<kMean, false>(s, a, st, w, pdl);
    case kMax: return warp_dispatch<kMax, false>(s, a, st, w, pdl);
    default: return warp_dispatch<kMin, false>(s, a, st, w, pdl);
  }
}

// Widest lanes (fewest sparse-row re-reads) whose column tiles still put >= 2
// CTAs on every SM across the hub rows; a handful of hub rows get 32-column
// tiles, spreading each over N/32 SMs.
int hub_vec(uint32_t n, uint32_t n_hub) {
  if (const char* e = std::getenv("GESPMM_HUB_VEC")) {  // tuning experiments
    const int v = std::atoi(e);
    if (v == 1 || v == 2 || v == 4) return v;
  }
  for (int v : {4, 2}) {
    const uint64_t tw = 32u * uint64_t(v);
    const uint64_t tiles = (uint64_t(n) + tw - 1) / tw;
    if (uint64_t(n_hub) * tiles >= 2ull * 148ull) return v;
  }
  return 1;
}
// Consumer warps sharing a tile of 32 * width columns (the lane width shrinks
// accordingly): 2 when the hub kernel leads the step (the consumer's fold rate
// bounds it: 8-way Reddit shard 0.578 -> 0.541 ms, 4000 rows x 2000 nonzeros
// 9.1 -> 10.8 TB/s), 1 as a side job (4-way shard 1.006 vs 1.088 ms with 2).
// GESPMM_HUB_SPLIT = 1, 2 or 4 forces it (tuning experiments).
int hub_split(int width, bool big) {
  static const int forced = [] {
    const char* e = std::getenv("GESPMM_HUB_SPLIT");
    return e ? std::atoi(e) : 0;
  }();
  int c = (forced == 1 || forced == 2 || forced == 4) ? forced : (big ? 2 : 1);
  while (c > width) c >>= 1;
  return c;
}
uint32_t hub_tile_width(uint32_t n, uint32_t n_hub) {
  return uint32_t(32 * hub_vec(n, n_hub));
}

cudaError_t launch_tuned_hub(int op, bool fast, const SpmmArgs& a, cudaStream_t st, bool big) {
  const int w = hub_vec(a.n, a.n_sched);  // tile = 32 * w columns
  const int c = hub_split(w, big);
  const int v = w / c;
  switch (op) {
    case kSum: return fast ? hub_dispatch<kSum, true>(v, c, big, a, st) : hub_dispatch<kSum, false>(v, c, big, a, st);
    case kMean: return fast ? hub_dispatch<kMean, true>(v, c, big, a, st) : hub_dispatch<kMean, false>(v, c, big, a, st);
    case kMax: return hub_dispatch<kMax, false>(v, c, big, a, st);
    default: return hub_dispatch<kMin, false>(v, c, big, a, st);
  }
}

cudaError_t launch_split_combine(int op, const SpmmArgs& a, const uint32_t* hubs, uint32_t n_hub,
                                 const float* part, const int32_t* part_arg, cudaStream_t st) {
  if (!n_hub || !a.n) return cudaSuccess;
  const uint64_t total = uint64_t(n_hub) * a.n;
  const uint64_t want = (total + 255) / 256;
  const uint32_t g = uint32_t(want < 148 * 8 ? want : 148 * 8);
  switch (op) {
    case kSum: k_split_combine<kSum><<<g, 256, 0, st>>>(a, hubs, n_hub, part, part_arg); break;
    case kMean: k_split_combine<kMean><<<g, 256, 0, st>>>(a, hubs, n_hub, part, part_arg); break;
    case kMax: k_split_combine<kMax><<<g, 256, 0, st>>>(a, hubs, n_hub, part, part_arg); break;
    default: k_split_combine<kMin><<<g, 256, 0, st>>>(a, hubs, n_hub, part, part_arg); break;
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_split_refresh(const uint32_t* row_ptr, const uint32_t* hubs, uint32_t n_hub,
                                 uint32_t seg_len, uint32_t* vptr, cudaStream_t st) {
  if (!n_hub) return cudaSuccess;
  const uint32_t g = (n_hub + 255) / 256;
  k_split_refresh<<<g < 148 ? g : 148, 256, 0, st>>>(row_ptr, hubs, n_hub, seg_len, vptr);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_tuned_cta(const CtaShape& s, int op, bool fast, const SpmmArgs& a,
                             cudaStream_t st) {
  switch (op) {
    case kSum: return fast ? cta_dispatch<kSum, true>(s, a, st) : cta_dispatch<kSum, false>(s, a, st);
    case kMean: return fast ? cta_dispatch<kMean, true>(s, a, st) : cta_dispatch<kMean, false>(s, a, st);
    case kMax: return cta_dispatch<kMax, false>(s, a, st);
    default: return cta_dispatch<kMin, false>(s, a, st);
  }
}

}  // namespace gespmm
