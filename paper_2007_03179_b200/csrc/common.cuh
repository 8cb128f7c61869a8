// Shared device-side pieces of the B200 GE-SpMM kernels: the fused reduce
// functors (replacing the reference's function-pointer ReduceOp,
// /root/reference/proj/include/spmm/reduce_op.hpp:14-28) and cache-hinted
// loads/stores (sm_100a PTX).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gespmm/gespmm.h"

namespace gespmm {

// ---------------------------------------------------------------------------
// Reduce ops, fused in-register.  Each output element is folded by exactly one
// thread in ascending CSR position, so with separate round-to-nearest multiply
// and combine (exact mode) every variant is bit-identical to the reference's
// ordered fold (kernel.hpp:218/271/331: acc = op.fold(acc, v * b)).
// ---------------------------------------------------------------------------
enum : int { kSum = GESPMM_SUM, kMean = GESPMM_MEAN, kMax = GESPMM_MAX, kMin = GESPMM_MIN };

template <int OP>
struct Reduce;

template <>
struct Reduce<kSum> {
  static constexpr bool kHasArg = false;
  __device__ __forceinline__ static float init() { return 0.0f; }
  template <bool FAST>
  __device__ __forceinline__ static void fold(float& acc, int32_t&, float v, float b, int32_t) {
    if (FAST)
      acc = __fmaf_rn(v, b, acc);
    else
      acc = __fadd_rn(acc, __fmul_rn(v, b));  // FMUL + FADD, never contracted
  }
};

template <>
struct Reduce<kMean> : Reduce<kSum> {};

template <>
struct Reduce<kMax> {
  static constexpr bool kHasArg = true;
  __device__ __forceinline__ static float init() { return -3.402823466e+38f; }  // lowest()
  template <bool FAST>
  __device__ __forceinline__ static void fold(float& acc, int32_t& who, float v, float b,
                                              int32_t pos) {
    const float x = __fmul_rn(v, b);
    // reference max_f32(a, b) = a < b ? b : a  (reduce_op.hpp:25): strict, so
    // ties keep the earlier element and NaN products never enter.
    if (acc < x) {
      acc = x;
      who = pos;
    }
  }
};

template <>
struct Reduce<kMin> {
  static constexpr bool kHasArg = true;
  __device__ __forceinline__ static float init() { return 3.402823466e+38f; }  // max()
  template <bool FAST>
  __device__ __forceinline__ static void fold(float& acc, int32_t& who, float v, float b,
                                              int32_t pos) {
    const float x = __fmul_rn(v, b);
    if (x < acc) {
      acc = x;
      who = pos;
    }
  }
};

// Packed pair update for sum/mean (sm_100a FADD2 / FFMA2).  Exact mode keeps
// the two products as scalar FMULs and only packs the adds: FMUL+FMUL+FADD2
// is never contracted by ptxas (a packed mul followed by a packed add is).
__device__ __forceinline__ void add2_rn(float& a0, float& a1, float p0, float p1) {
  asm("{\n\t.reg .b64 ra, rp;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rp, {%2, %3};\n\t"
      "add.rn.f32x2 ra, ra, rp;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(p0), "f"(p1));
}
__device__ __forceinline__ void fma2_rn(float& a0, float& a1, float v, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rv;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
      "mov.b64 rv, {%4, %4};\n\tfma.rn.f32x2 ra, rv, rb, ra;\n\tmov.b64 {%0, %1}, ra;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(b0), "f"(b1), "f"(v));
}

// Fold one staged nonzero (value v, position pos) into VEC accumulators.
template <int OP, bool FAST, int VEC>
__device__ __forceinline__ void fold_vec(float* acc, int32_t* who, float v, const float* b,
                                         int32_t pos) {
  if constexpr ((OP == kSum || OP == kMean) && VEC % 2 == 0) {
#pragma unroll
    for (int e = 0; e < VEC; e += 2) {
      if (FAST)
        fma2_rn(acc[e], acc[e + 1], v, b[e], b[e + 1]);
      else
        add2_rn(acc[e], acc[e + 1], __fmul_rn(v, b[e]), __fmul_rn(v, b[e + 1]));
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) Reduce<OP>::template fold<FAST>(acc[e], who[e], v, b[e], pos);
  }
}

// mean = sum / float(row length); an empty row keeps the sum seed.
template <int OP>
__device__ __forceinline__ float finish(float acc, uint32_t row_len) {
  if (OP == kMean && row_len > 0) return __fdiv_rn(acc, static_cast<float>(row_len));
  return acc;
}

// ---------------------------------------------------------------------------
// L2 cache policies.  B (the gathered dense rows, re-read ~nnz/K times) is
// kept with evict_last; the streamed CSR arrays and the written C use
// evict_first so they do not push B out of the 126 MB L2.  With hints off both
// policies are evict_normal (same code path).
// ---------------------------------------------------------------------------
struct Policies {
  uint64_t keep;    // for B (hot rows when the plan has a hot-column map)
  uint64_t cold;    // for B rows outside the hot-column map
  uint64_t stream;  // for CSR and C
};

__device__ __forceinline__ Policies make_policies(int hints) {
  Policies p;
  if (hints) {
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p.keep));
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p.stream));
    if (hints == 2)
      asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p.cold));
    else
      p.cold = p.stream;
  } else {
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p.keep));
    p.stream = p.keep;
    p.cold = p.keep;
  }
  return p;
}

// Hot-column map lookup (plan-time bitmap, hotcols.cu): bit 31 of the staged
// column marks a COLD column, so an absent map leaves every column "hot".
constexpr uint32_t kColdBit = 0x80000000u;
__device__ __forceinline__ uint32_t cold_mark(const uint32_t* __restrict__ hot, uint32_t k) {
  return ((__ldg(hot + (k >> 5)) >> (k & 31u)) & 1u) ? 0u : kColdBit;
}

// Streamed sparse arrays: read once, do not allocate in L1.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* ptr, uint64_t pol) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
      : "=r"(r)
      : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_stream_f32(const float* ptr, uint64_t pol) {
  float r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
      : "=f"(r)
      : "l"(ptr), "l"(pol));
  return r;
}

// Gathered dense rows of B: L1-allocating (hub rows hit), L2 evict_last.
template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  float x[1];
};
template <>
struct Vec<2> {
  float x[2];
};
template <>
struct Vec<4> {
  float x[4];
};

template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_keep(const float* ptr, uint64_t pol);

template <>
__device__ __forceinline__ Vec<1> ld_keep<1>(const float* ptr, uint64_t pol) {
  Vec<1> r;
  asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r.x[0]) : "l"(ptr), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ Vec<2> ld_keep<2>(const float* ptr, uint64_t pol) {
  Vec<2> r;
  asm("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
      : "=f"(r.x[0]), "=f"(r.x[1])
      : "l"(ptr), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ Vec<4> ld_keep<4>(const float* ptr, uint64_t pol) {
  Vec<4> r;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
      : "l"(ptr), "l"(pol));
  return r;
}

// Output stores: written once, streamed past L1, evict_first in L2.
template <int VEC>
__device__ __forceinline__ void st_stream(float* ptr, const float* v, uint64_t pol);
template <>
__device__ __forceinline__ void st_stream<1>(float* ptr, const float* v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(ptr),
               "f"(v[0]), "l"(pol)
               : "memory");
}
template <>
__device__ __forceinline__ void st_stream<2>(float* ptr, const float* v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(ptr),
               "f"(v[0]), "f"(v[1]), "l"(pol)
               : "memory");
}
template <>
__device__ __forceinline__ void st_stream<4>(float* ptr, const float* v, uint64_t pol) {
  asm volatile(
      "st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "l"(pol)
      : "memory");
}

template <int VEC>
__device__ __forceinline__ void st_stream_i32(int32_t* ptr, const int32_t* v, uint64_t pol);
template <>
__device__ __forceinline__ void st_stream_i32<1>(int32_t* ptr, const int32_t* v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(ptr),
               "r"(v[0]), "l"(pol)
               : "memory");
}
template <>
__device__ __forceinline__ void st_stream_i32<2>(int32_t* ptr, const int32_t* v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(ptr),
               "r"(v[0]), "r"(v[1]), "l"(pol)
               : "memory");
}
template <>
__device__ __forceinline__ void st_stream_i32<4>(int32_t* ptr, const int32_t* v, uint64_t pol) {
  asm volatile(
      "st.global.L1::no_allocate.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "l"(pol)
      : "memory");
}

// SkipTail fault hook (reference kernel.hpp:174-180 faulted_row_end, ws = 32).
__device__ __forceinline__ uint32_t faulted_end(uint32_t start, uint32_t end, int skip_tail) {
  if (!skip_tail || end <= start) return end;
  const uint32_t tiles = (end - start + 31u) >> 5;
  return start + (tiles - 1u) * 32u;
}

// Launch parameters shared by every SpMM kernel.
// ---------------------------------------------------------------------------
// Fused all-gather epilogue (multi-GPU stacked layers): the
// output row is also stored to peer-mapped replicas of C on the other ranks
// (NVLink P2P stores through UVA), or once through an NVLS multicast address
// (multimem.st: the NVSwitch fans the store out to every member GPU).  Plain
// stores, no L2 policy: the lines live in the peer's L2, not ours.
// ---------------------------------------------------------------------------
constexpr int kMaxPeers = GESPMM_MAX_GATHER_DSTS - 1;

template <int VEC>
__device__ __forceinline__ void st_peer(float* ptr, const float* v) {
  if constexpr (VEC == 4) {
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3])
                 : "memory");
  } else if constexpr (VEC == 2) {
    asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(ptr), "f"(v[0]), "f"(v[1]) : "memory");
  } else {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(ptr), "f"(v[0]) : "memory");
  }
}
template <int VEC>
__device__ __forceinline__ void st_peer_i32(int32_t* ptr, const int32_t* v) {
  st_peer<VEC>(reinterpret_cast<float*>(ptr), reinterpret_cast<const float*>(v));
}
template <int VEC>
__device__ __forceinline__ void st_multicast(float* ptr, const float* v) {
  if constexpr (VEC == 4) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ptr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
                 : "memory");
  } else if constexpr (VEC == 2) {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(ptr), "f"(v[0]),
                 "f"(v[1])
                 : "memory");
  } else {
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(ptr), "f"(v[0]) : "memory");
  }
}
// ptxas takes vector multimem.st only for float types: the int32 arg lanes go
// as their bit patterns (a store never alters them).
template <int VEC>
__device__ __forceinline__ void st_multicast_i32(int32_t* ptr, const int32_t* v) {
  st_multicast<VEC>(reinterpret_cast<float*>(ptr), reinterpret_cast<const float*>(v));
}

struct SpmmArgs {
  const uint32_t* row_ptr;
  const uint32_t* col_ind;
  const float* vals;
  const float* b;
  float* c;
  int32_t* arg;
  const uint32_t* order;  // row schedule (nullable -> identity)
  uint32_t n_sched;       // rows in the schedule
  uint32_t n;             // dense width N (of this launch's column slice)
  uint32_t ld;            // row stride of C and arg in elements (>= n)
  uint32_t ldb;           // row stride of B in elements (>= n): ld, or the plan's re-pitched copy
  uint32_t n_tiles;       // column tiles per row
  uint32_t kb;            // rows of B (the gathered operand; A's n_cols), 0 = not given
  int arg_col;            // arg = col_ind[p] instead of p
  int skip_tail;
  int hints;              // 0 off, 1 B evict_last / CSR,C evict_first, 2 = 1 with cold B evict_normal
  const uint32_t* hot;    // hot-column bitmap (nullable): cold B rows use the cold policy
  // Relocated hot rows (nullable): the plan's contiguous copy of the most-gathered
  // B rows (row stride ldh), addressed by col_ind entries with bit 31 set.
  const float* b_hot;   // start of the copy (row stride ldb, congruent to b modulo the stride)
  int32_t hot_off;      // (b_hot - b) / row stride
  uint32_t hot_bytes;   // bytes of the copy (< 4 GiB)
  int reloc_mode;       // L2 policy of the gathers: 1 range (copy evict_last), 0 keep for all
  uint64_t pol_hot;     // the range policy word (resolve_range_policy)
  const uint32_t* col_ind_orig;  // host-side: the caller's col_ind when col_ind is the remap
  // L2 policies resolved once on the device (resolve_policies) and passed as
  // launch parameters: they then live in uniform registers, so a per-gather
  // choice between two of them is a uniform select, not a per-load descriptor
  // move.  pol_valid = 0 -> the kernel creates them itself (make_policies).
  uint64_t pol_keep, pol_cold, pol_stream;
  int pol_valid;
  // Fused all-gather epilogue: n_peer replicas of C (and arg) on other ranks,
  // each addressed like c (same row offsets and ld); c_mc/arg_mc: multicast
  // addresses of C/arg (nullable).  n_peer = 0 and c_mc = null: local only.
  int n_peer;
  float* c_peer[kMaxPeers];
  int32_t* arg_peer[kMaxPeers];
  float* c_mc;
  int32_t* arg_mc;
  uint32_t* work;  // hub kernel: unit counter of a persistent launch (zeroed before it), or null
  // Host entry's pipelined validation: the column check of a row block runs
  // just before its kernels on the same stream; a kernel returns at once when
  // this key (the first violation found so far, ~0 = none) is set, so
  // non-canonical columns are never dereferenced.  Null: no check.
  const unsigned long long* abort_if;
  // overlap_prev plans: launched as a programmatic dependent of the previous
  // kernel; every warp executes griddepcontrol.wait after its A-side prologue
  // and before its first B gather (1), or never waits (0: the hub-then-warp
  // pair, whose rows are disjoint and whose B was complete before either ran).
  int pdl_wait;
};

__device__ __forceinline__ bool aborted(const SpmmArgs& a) {
  return a.abort_if && *reinterpret_cast<const volatile unsigned long long*>(a.abort_if) != ~0ull;
}

// Epilogue replicas of one output vector (element offset o from c / arg).
template <int VEC, bool ARG>
__device__ __forceinline__ void store_replicas(const SpmmArgs& a, uint64_t o, const float* out,
                                               const int32_t* who) {
  for (int p = 0; p < a.n_peer; ++p) {
    st_peer<VEC>(a.c_peer[p] + o, out);
    if (ARG && a.arg_peer[p]) st_peer_i32<VEC>(a.arg_peer[p] + o, who);
  }
  if (a.c_mc) {
    st_multicast<VEC>(a.c_mc + o, out);
    if (ARG && a.arg_mc) st_multicast_i32<VEC>(a.arg_mc + o, who);
  }
}

__device__ __forceinline__ Policies args_policies(const SpmmArgs& a) {
  if (a.pol_valid) {
    Policies p;
    p.keep = a.pol_keep;
    p.cold = a.pol_cold;
    p.stream = a.pol_stream;
    return p;
  }
  return make_policies(a.hints);
}

}  // namespace gespmm
