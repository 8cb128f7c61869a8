// C-ABI implementation: argument checks with the reference's error texts,
// plans (inspector: degree distribution -> kernel shape + row schedule),
// the device and host-buffer entry points.
//
// Reference behaviour mirrored (file:line under /root/reference/proj):
//   check_spmm_inputs   include/spmm/simt.hpp:373-380 (dims, then canonical)
//   require_canonical   include/spmm/csr.hpp:155-158  ("<who>: matrix is not canonical CSR: ...")
//   native_spmm         include/spmm/native.hpp:101-143 (M==0 -> empty, N==0 -> error)
//   check_config        include/spmm/kernel.hpp:83-92  (cf in {2,4,8})
//   select_variant      include/spmm/kernel.hpp:96-98
//   reduce_op_by_name   include/spmm/reduce_op.hpp:32-36
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys/ncu timelines
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace gespmm {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {

thread_local std::string t_err;

gespmm_status_t fail(gespmm_status_t st, const std::string& msg) {
  t_err = msg;
  return st;
}

gespmm_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? GESPMM_ENOMEM : GESPMM_ECUDA,
              std::string(where) + ": CUDA error: " + cudaGetErrorString(e));
}

#define GESPMM_CUDA(call, where)                     \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Formats the first violation in the order the reference checks
// (csr.hpp:112-153); returns GESPMM_OK when canonical.
gespmm_status_t validation_status(const ValidateResult& r, uint32_t m, uint32_t k, uint64_t nnz,
                                  const char* who) {
  char buf[256];
  const std::string pre = std::string(who) + ": matrix is not canonical CSR: ";
  if (r.row_ptr0 != 0) {
    std::snprintf(buf, sizeof buf, "row_ptr[0] = %u, expected 0", r.row_ptr0);
    return fail(GESPMM_ENONCANON, pre + buf);
  }
  if (r.first_decrease != 0xffffffffu) {
    std::snprintf(buf, sizeof buf, "row_ptr non-decreasing violated at index %u", r.first_decrease);
    return fail(GESPMM_ENONCANON, pre + buf);
  }
  if (uint64_t(r.row_ptr_last) != nnz) {
    std::snprintf(buf, sizeof buf, "row_ptr[n_rows] = %u != nnz = %llu", r.row_ptr_last,
                  (unsigned long long)nnz);
    return fail(GESPMM_ENONCANON, pre + buf);
  }
  if (r.first_bad_key != ~0ull) {
    const unsigned long long p = r.first_bad_key >> 1;
    if ((r.first_bad_key & 1ull) == 0)
      std::snprintf(buf, sizeof buf, "col_ind[%llu] = %u out of bounds (n_cols = %u)", p,
                    r.bad_col, k);
    else
      std::snprintf(buf, sizeof buf, "columns not strictly increasing in row %u at position %llu",
                    r.bad_row, p);
    return fail(GESPMM_ENONCANON, pre + buf);
  }
  (void)m;
  return GESPMM_OK;
}

gespmm_status_t check_opts(const gespmm_options_t& o) {
#ifndef GESPMM_EXPERIMENTAL
  // options that were measured slower on B200 ship only in the
  // experimental build (GESPMM_EXPERIMENTAL=1 python -m paper_2007_03179_b200._build)
  const char* exp_opt = o.cluster_hot ? "cluster_hot"
                        : o.l2_hot_mb > 0 ? "l2_hot_mb"
                        : o.col_slices > 1 ? "col_slices"
                        : o.l2_persist ? "l2_persist"
                        : o.hot_rows_mb > 0 ? "hot_rows_mb" : nullptr;
  if (exp_opt)
    return fail(GESPMM_EUNSUPPORTED, std::string(exp_opt) +
                                         " is an experimental option (measured slower, DESIGN.md "
                                         "§2); this library was built without GESPMM_EXPERIMENTAL");
#endif
  if (o.cluster_hot != 0 && o.cluster_hot != 2 && o.cluster_hot != 4 && o.cluster_hot != 8 &&
      o.cluster_hot != 16)
    return fail(GESPMM_EINVAL, "cluster_hot must be 0, 2, 4, 8 or 16");
  if (o.variant < GESPMM_VARIANT_TUNED || o.variant > GESPMM_VARIANT_CRC_CWM)
    return fail(GESPMM_EINVAL, "unknown kernel variant " + std::to_string(o.variant) +
                                   " (naive, crc, crc-cwm, tuned)");
  if (o.variant == GESPMM_VARIANT_CRC_CWM && o.cf != 2 && o.cf != 4 && o.cf != 8)
    return fail(GESPMM_EINVAL, "coarsening factor must be 2, 4 or 8");
  if (o.tuned_cf != 0 && o.tuned_cf != 1 && o.tuned_cf != 2 && o.tuned_cf != 4)
    return fail(GESPMM_EINVAL, "tuned_cf must be 0 (auto), 1, 2 or 4");
  if (o.arg_kind != GESPMM_ARG_EDGE && o.arg_kind != GESPMM_ARG_COLUMN)
    return fail(GESPMM_EINVAL, "arg_kind must be edge (0) or column (1)");
  if (o.rows_per_warp != 0 && o.rows_per_warp != 1 && o.rows_per_warp != 2 &&
      o.rows_per_warp != 4 && o.rows_per_warp != 8)
    return fail(GESPMM_EINVAL, "rows_per_warp must be 0 (auto), 1, 2, 4 or 8");
  return GESPMM_OK;
}

gespmm_status_t check_op(gespmm_reduce_t op, const int32_t* arg) {
  if (op < GESPMM_SUM || op > GESPMM_MIN)
    return fail(GESPMM_EINVAL, "unknown reduce op " + std::to_string(int(op)) +
                                   " (built-ins: sum, mean, max, min)");
  if (arg && op != GESPMM_MAX && op != GESPMM_MIN)
    return fail(GESPMM_EINVAL, "arg indices are defined for max and min only");
  return GESPMM_OK;
}

// arg is int32 (C ABI): an edge arg is a CSR position < nnz, a column arg a
// column < n_cols; either must fit, or the call is refused rather than
// writing wrapped indices.
gespmm_status_t check_arg_range(const int32_t* arg, uint64_t nnz, uint32_t n_cols,
                                int32_t arg_kind) {
  if (!arg) return GESPMM_OK;
  const bool column = arg_kind == GESPMM_ARG_COLUMN;
  const uint64_t bound = column ? uint64_t(n_cols) : nnz;
  if (bound > uint64_t(INT32_MAX) + 1)
    return fail(GESPMM_EINVAL, std::string("arg: ") + (column ? "column" : "CSR position") +
                                   " indices up to " + std::to_string(bound - 1) +
                                   " do not fit the int32 arg" +
                                   (column ? "" : " (use arg_kind = column)"));
  return GESPMM_OK;
}

}  // namespace

gespmm_status_t set_error(gespmm_status_t st, const std::string& msg) { return fail(st, msg); }

gespmm_status_t validate_device_as(const gespmm_csr_t* a, cudaStream_t st, const char* who) {
  ValidateResult r{};
  GESPMM_CUDA(validate_csr_device(a->n_rows, a->n_cols, a->nnz, a->row_ptr, a->col_ind, &r, st),
              "validate");
  return validation_status(r, a->n_rows, a->n_cols, a->nnz, who);
}

// ---------------------------------------------------------------------------
// Plans
// ---------------------------------------------------------------------------

// Tuned-kernel shapes for one (n, options): the column slicing and, per slice
// width, the vectorised shapes with their scalar-lane fallbacks.
struct TunedShapes {
  uint32_t n = 0;
  uint32_t slices = 1;   // column slices, traversed slice-major
  uint32_t slice_w = 0;  // columns per slice (the last one may be narrower)
  int rpw = 1;           // rows per warp requested for float4 lanes
  WarpShape warp_v, warp_s;
  CtaShape cta_v, cta_s;
};

struct Plan {
  gespmm_csr_t a{};
  uint32_t n = 0;
  gespmm_reduce_t op = GESPMM_SUM;
  gespmm_options_t o{};
  int device = 0;
  // tuned
  TunedShapes sh;            // kernel shapes + column slicing
  uint32_t n_hub = 0;        // order[0, n_hub) -> row-per-CTA
  uint32_t hub_threshold = 0;
  bool hub_pdl = false;      // hub rows carry >= kHubPdlShare of the nonzeros
  uint32_t* d_order = nullptr;
  uint32_t* d_work = nullptr;  // hub kernel unit counters, one per column slice (plan-owned)
  uint32_t* d_hot = nullptr;  // hot-column bitmap (frequency-aware L2 policy), nullable
  HotStats hot{};
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::string desc;
  uint32_t max_degree = 0;
  double mean_degree = 0.0;
  ClusterHot ch;             // cluster-DSMEM hot-row cache (o.cluster_hot), col_ind copy
  HotRows hr;                // relocated hot rows (o.hot_rows_mb), col_ind copy
  // Split hub rows (max/min, or fast-mode sum/mean): each hub row's nonzeros
  // cut into segments of seg_len, folded by k_warp into partial rows, then
  // combined in segment order (k_split_combine) instead of the k_hub ring.
  bool split = false;
  uint32_t seg_len = 0, n_seg = 0, n_vrows = 0;
  uint32_t* d_vptr = nullptr;       // virtual row_ptr over segments
  uint32_t* d_seg_order = nullptr;  // the segments' virtual rows
  uint32_t* d_hubs = nullptr;       // per hub row: (row, first virtual row, segments)
  float* d_part = nullptr;          // partial rows [n_vrows][n]
  int32_t* d_part_arg = nullptr;    // their arg (max/min)

  ~Plan() {
#ifdef GESPMM_EXPERIMENTAL
    free_cluster_hot(&ch);
#endif
#ifdef GESPMM_EXPERIMENTAL
    free_hot_rows(&hr);
#endif
    if (d_order) cudaFree(d_order);
    if (d_work) cudaFree(d_work);
    for (void* q : {static_cast<void*>(d_vptr), static_cast<void*>(d_seg_order),
                    static_cast<void*>(d_hubs), static_cast<void*>(d_part),
                    static_cast<void*>(d_part_arg)})
      if (q) cudaFree(q);
    if (d_hot) cudaFree(d_hot);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
  }
};

namespace {

// Row-per-CTA only for rows so long that one warp walking them would outlast
// the rest of the launch.  Measured on B200 (Reddit shape, N=128): with the LPT
// row schedule the warp kernel alone runs 3.05 ms, while peeling the 1687 rows
// of degree >= 7884 onto the CTA kernel made the step 6.04 ms (the CTA kernel
// moves 4x more load instructions per byte and competes for the same SMs).
// A warp sustains ~1/3500 of the chip's gather rate, so a row is a tail risk
// only beyond ~nnz/1024 nonzeros.
// Hub rows: a row of degree d on one warp costs ~d * L * CF / 8 (one L2 round
// trip L ~ 0.7 us per batch of 8/CF gathers), while a launch over `nnz`
// nonzeros is gather-bound at ~nnz * 4N / 19 TB/s.  Rows whose single-warp
// time would exceed 1/2.5 of the launch go to the ring-fed row-per-CTA kernel
// (k_hub: a 21,657-nonzero row in ~0.2 ms instead of ~1.7 ms) — unless even
// the longest row fits comfortably in the launch.  So the threshold scales
// with the work per launch: no hub rows on the whole Reddit shape, ~7k on a
// 1/2 row shard, 2048 (the floor) on a 1/8 shard or one block of the
// pipelined host entry.  Measured with tools/shard_emulation.py
// (profiles/r1_shard_emulation.md): the 1-GPU step unchanged, the 8-shard step
// 1.51 -> 0.52 ms.
uint32_t auto_hub_threshold(uint32_t n, uint64_t nnz, int cf, uint32_t k, int dev,
                            uint32_t tile_cols, uint32_t max_degree) {
  if (n < 8) return 0xffffffffu;  // too narrow for a CTA per row
  // the warp kernel moves whole lane tiles (N = 44 -> 64 columns of float4 lanes)
  const uint32_t moved = std::max(n, tile_cols);
  // gather rate: ~19 TB/s while B (mostly) fits the L2, ~9.5 TB/s once the
  // gathers miss to HBM (ogbn-products N=256: B = 2.5 GB)
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  const double b_bytes = double(k) * double(n) * 4.0;
  const double rate = (l2 > 0 && b_bytes > 1.5 * double(l2)) ? 9.5e12 : 19e12;
  // narrow tiles are not byte-bound: below ~90 columns the warp kernel runs at
  // ~18 ps per nonzero whatever the width (Reddit shape, 115M nonzeros: N=24/32
  // 1.8 ms, N=44/48/64 2.1-2.3 ms; tools/gcn_width_probe.py).  Without this
  // floor N=32 got ~2600 hub rows and took 3.1 ms instead of 1.7 ms.
  const double t_launch = std::max(double(nnz) * 4.0 * double(moved) / rate, double(nnz) * 18e-12);
  const double t_nnz = 0.7e-6 * double(cf < 1 ? 1 : cf) / 8.0;
  // no hub rows while the longest row's warp time stays well inside the launch
  // (whole Reddit: 0.61 of it; products half-shard: 0.47): a side-stream hub
  // kernel there only disturbs the warp kernel
  if (double(max_degree) * t_nnz <= 0.75 * t_launch) return 0xffffffffu;
  // narrow lane tiles (N < 128) fold fewer columns per staged nonzero in k_hub:
  // fewer, longer hub rows there (GCN N=44: 2.07 ms at threshold 12k, 2.93 ms at 7k)
  double f = moved >= 128 ? 2.5 : 1.5;  // GESPMM_HUB_FACTOR overrides (shard_emulation.py)
  if (const char* e = std::getenv("GESPMM_HUB_FACTOR")) f = std::max(0.05, std::atof(e));
  const double t = std::max(2048.0, t_launch / (f * t_nnz));
  return t >= 4294967295.0 ? 0xffffffffu : uint32_t(t);
}

// Hub threshold when the ring runs alone ahead of the warp kernel (exact
// sum/mean plans whose hub rows carry >= kHubPdlShare of the nonzeros): the
// step is then the ring phase plus the warp phase, and the warp phase ends
// with its longest row (LPT), so rows stay on warps only while one of them
// takes at most alpha (0.5) of the warp phase.  Scans the degree-descending
// order for the first row that satisfies it.  Measured on Reddit shards
// (tools/r2_floor.sh, tools/r2_alpha.sh, profiles/r2/hubseq/): 8 shards best
// at ~1024 (0.466 ms; the launch-wide rule gave 2048: 0.503 ms), 4 shards flat
// between 2800 and 4096 (0.843-0.831 ms); alpha 0.35/0.5/0.6/0.7 -> 2/4/8
// shards 1.60/0.87/0.49, 1.57/0.84/0.46, 1.52/0.83/0.48, 1.55/0.83/0.49 ms.
constexpr double kSeqAlpha = 0.5;
uint32_t seq_hub_threshold(const std::vector<uint32_t>& deg, const std::vector<uint32_t>& order,
                           uint64_t total, uint32_t n, uint32_t tile_cols, int cf, uint32_t k,
                           int dev) {
  const uint32_t moved = std::max(n, tile_cols);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  const double b_bytes = double(k) * double(n) * 4.0;
  const double rate = (l2 > 0 && b_bytes > 1.5 * double(l2)) ? 9.5e12 : 19e12;
  const double t_nnz = 0.7e-6 * double(cf < 1 ? 1 : cf) / 8.0;
  uint64_t cum = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    const double rest = double(total - cum);
    const double warp_phase = std::max(rest * 4.0 * double(moved) / rate, rest * 18e-12);
    const uint32_t d = deg[order[i]];
    if (double(d) * t_nnz <= kSeqAlpha * warp_phase) return std::max<uint32_t>(256u, d + 1u);
    cum += d;
  }
  return 256u;
}

// Round-2 hub schedule for exact plans (ring first and alone, warp kernel
// after it, seq_hub_threshold); GESPMM_HUB_SEQ=0 restores round 1's.
bool hub_ring_first() {
  static const bool on = [] {
    const char* e = std::getenv("GESPMM_HUB_SEQ");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Frequency-aware L2 policy budget (bytes of B rows kept evict_last), 0 = off.
// Opt-in (l2_hot_mb > 0).  History on B200 (profiles/r1_hot_sweep.txt,
// profiles/r1_kernel_v4.txt): with the per-load policy select of the first
// kernel it helped products N=256 max+arg (14.49 -> 13.70 ms); once the
// un-mapped kernel dropped that select (one loop-invariant policy register,
// check-free full batches) the map-less kernel is faster (13.14 ms) than the
// mapped one (17.2 ms: the cold/hot branch costs registers and spills at 6
// CTAs/SM), so auto = off.
uint64_t hot_budget_bytes(const gespmm_options_t& o, uint32_t k, uint32_t n, int dev) {
  (void)n;
  (void)dev;
  if (o.l2_hot_mb <= 0 || k >= 0x80000000u) return 0;  // bit 31 of a staged column is the mark
  return uint64_t(o.l2_hot_mb) << 20;
}

// Relocated hot rows (hotrows.cu): budget in bytes of B rows, 0 = off.
// Opt-in (hot_rows_mb > 0, experimental build).  Measured on B200 (products
// N=256 max+arg, profiles/r2/reloc_products.md): DRAM reads 71.4 -> 61.6 GB
// per step, yet 12.3 -> 12.8-13.0 ms for every budget and L2 policy tried
// (address-range evict_last, + evict_first outside, or one keep policy).
// Column args would report the remapped ids, so edge args only.
uint64_t hot_rows_budget(const gespmm_options_t& o, uint32_t k, uint32_t n, int dev) {
  (void)n;
  (void)dev;
#ifndef GESPMM_EXPERIMENTAL
  (void)o;
  (void)k;
  return 0;
#else
  if (o.hot_rows_mb <= 0 || k >= 0x80000000u || o.arg_kind == GESPMM_ARG_COLUMN) return 0;
  return uint64_t(o.hot_rows_mb) << 20;
#endif
}

// Column slices (slice-major traversal).  The kernels fold each output
// element in one thread in CSR order whatever the slice, so slicing only
// changes which columns of B are live at a time: B/S instead of B.  Measured
// on B200 (profiles/r1_col_slices.txt) it never pays: products N=256 max+arg
// 13.5 ms at S=1 -> 15.9 / 18.2 / 30.0 ms at S=2/4/8 (the CSR stream and the
// per-row work repeat per slice and narrower gathers cost more per byte than
// the extra L2 hits save); Reddit N=128 3.0 -> 4.1 ms at S=2.  Auto = off;
// explicit S stays available.
uint32_t pick_slices(const gespmm_options_t& o, uint32_t /*k*/, uint32_t n, int /*dev*/) {
  if (o.col_slices >= 1) return std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(o.col_slices), n));
  return 1;
}

TunedShapes make_shapes(const gespmm_options_t& o, uint32_t k, uint32_t n, int dev,
                        double mean_degree) {
  TunedShapes t;
  t.n = n;
  t.slices = pick_slices(o, k, n, dev);
  uint32_t w = (n + t.slices - 1) / t.slices;
  // slice offsets keep the lanes' vector alignment (float4 at N % 4 == 0,
  // float2 at even N; an odd offset made float2 loads fault — fuzz test)
  if (n % 4 == 0) w = (w + 3) & ~3u;
  else if (n % 2 == 0) w = (w + 1) & ~1u;
  t.slice_w = std::max<uint32_t>(1, std::min(w, n));
  t.slices = (n + t.slice_w - 1) / t.slice_w;
  const uint32_t sw = t.slice_w;
  const bool n4 = n % 4 == 0, n2 = n % 2 == 0;
  // low-degree matrices share a warp between rows: 2 rows at N >= 64, 4 below
  // (Pubmed, warm graph replay per SpMM, tools/r2_rpw.sh: N=128 8.62 -> 8.13 us
  // at 2 rows (lpr 16, cf 2) vs 4 (lpr 8, cf 4); N=64 6.27 -> 6.08; N=256 equal;
  // N=32 best at 4 rows, lpr 8: 4.47 vs 6.01 us at 2)
  t.rpw = o.rows_per_warp > 0 ? o.rows_per_warp : (mean_degree <= 16.0 ? (sw >= 64 ? 2 : 4) : 1);
  t.warp_v = pick_warp_shape(sw, n4, !n4 && n2, t.rpw);
  t.warp_s = pick_warp_shape(sw, false, false);
  if (o.tuned_cf > 0) {  // explicit CWM merge factor for the warp kernel (tuning)
    for (WarpShape* ws : {&t.warp_v, &t.warp_s}) {
      WarpShape u = *ws;
      u.cf = o.tuned_cf;
      if (u.lpr == 32 && tuned_shape_supported(u)) *ws = u;
    }
  }
  t.cta_v = pick_cta_shape(sw, n4, n2);
  t.cta_s = pick_cta_shape(sw, false, false);
  return t;
}

// Launches the tuned kernels over the rows `order[0, n_hub + n_rest)` (hub
// rows first, row-per-CTA) for every column slice, slice-major.  `a` carries
// the full-width B/C/arg pointers with ld = row stride.  With `side` the hub
// kernel overlaps the warp kernel of the same slice on that stream.
// How the hub kernel shares the GPU with the warp kernel: when the hub rows
// carry a large share of the nonzeros (a 1/8 row shard of a power-law graph:
// ~35%), the hub kernel goes first on the same stream and the warp kernel
// follows as a programmatic dependent launch, so the hub CTAs (the critical
// path) are resident from the start; with a small share, the hub kernel runs
// on a high-priority side stream and its CTAs take SM slots as warp CTAs
// retire, which disturbs the warp kernel less (profiles/r1_shard_emulation.md).
constexpr double kHubPdlShare = 0.25;

gespmm_status_t launch_tuned_rows(const TunedShapes& t, int op, bool fast, const SpmmArgs& a0,
                                  const uint32_t* order, uint32_t n_hub, uint32_t n_rest,
                                  cudaStream_t st, cudaStream_t side, cudaEvent_t fork,
                                  cudaEvent_t join, const cudaAccessPolicyWindow* winp,
                                  bool hub_pdl, uint32_t* work, bool chain = false,
                                  bool pdl_overlap = false) {
  SpmmArgs a = a0;
  // overlap_prev: only a single-kernel execute chains onto the previous kernel
  chain = chain && n_hub == 0 && t.slices == 1;
  GESPMM_CUDA(resolve_policies(&a, st), "spmm");
  const bool v_ok = aligned(a.b, 16) && aligned(a.c, 16) && (!a.arg || aligned(a.arg, 16));
  const bool v2_ok = aligned(a.b, 8) && aligned(a.c, 8) && (!a.arg || aligned(a.arg, 8));
  const bool n4 = t.n % 4 == 0, n2 = t.n % 2 == 0;
  for (uint32_t j = 0; j < t.slices; ++j) {
    const uint32_t off = j * t.slice_w;
    const uint32_t w = std::min(t.slice_w, t.n - off);
    const bool narrow = w != t.slice_w;  // ragged last slice
    WarpShape wv = narrow ? pick_warp_shape(w, n4, !n4 && n2, t.rpw) : t.warp_v;
    WarpShape wsc = narrow ? pick_warp_shape(w, false, false) : t.warp_s;
    const CtaShape cv = narrow ? pick_cta_shape(w, n4, n2) : t.cta_v;
    const CtaShape csc = narrow ? pick_cta_shape(w, false, false) : t.cta_s;
    // the slice's own offset must keep the vector alignment too
    const bool sv_ok = v_ok && off % 4 == 0, sv2_ok = v2_ok && off % 2 == 0;
    const WarpShape& ws = sv_ok ? wv : wsc;
    const CtaShape& cs = sv_ok ? cv : csc;
    const WarpShape& wsel = (ws.vec == 2 && !sv2_ok) ? wsc : ws;
    SpmmArgs sa = a;
    sa.b = a.b + off;
    sa.c = a.c + off;
    sa.arg = a.arg ? a.arg + off : nullptr;
    for (int q = 0; q < a.n_peer; ++q) {
      sa.c_peer[q] = a.c_peer[q] + off;
      sa.arg_peer[q] = a.arg_peer[q] ? a.arg_peer[q] + off : nullptr;
    }
    sa.c_mc = a.c_mc ? a.c_mc + off : nullptr;
    sa.b_hot = a.b_hot ? a.b_hot + off : nullptr;
    sa.arg_mc = a.arg_mc ? a.arg_mc + off : nullptr;
    sa.n = w;
    bool hub_then_pdl = false, side_used = false;
    if (n_hub) {
      SpmmArgs h = sa;
      if (h.col_ind_orig) {  // hub kernels gather B directly through the caller's col_ind
        h.col_ind = h.col_ind_orig;
        h.b_hot = nullptr;
      }
      h.order = order;
      h.n_sched = n_hub;
      h.work = work ? work + j : nullptr;  // caller-owned counter of this launch site
      // TMA-ring hub kernel when bulk copies can address the B slices (16-byte
      // units: N % 4 == 0, ld % 4 == 0, 16-byte aligned B/C/arg at this offset)
      static const bool force_cta = [] {  // GESPMM_HUB_KCTA=1: A/B against the LDG CTA kernel
        const char* e = std::getenv("GESPMM_HUB_KCTA");
        return e && e[0] == '1';
      }();
      const bool tma = !force_cta && w % 4 == 0 && a.ld % 4 == 0 && a.ldb % 4 == 0 &&
                       aligned(sa.b, 16) &&
                       aligned(sa.c, 16) && (!sa.arg || aligned(sa.arg, 16));
      const uint32_t tw = tma ? hub_tile_width(w, n_hub) : uint32_t(cs.vec * cs.warps * 32);
      h.n_tiles = (w + tw - 1) / tw;
      // When the hub rows carry the launch (>= kHubPdlShare of its nonzeros:
      // a 1/4 or 1/8 row shard of a power-law graph), the hub kernel runs
      // first and alone, one CTA per unit, and the warp kernel follows in
      // stream order.  Round 1 ran them together (the warp kernel as a
      // programmatic dependent launch, the hub kernel capped at 2 persistent
      // CTAs per SM); measured in round 2 (tools/r2_hubseq.sh, Reddit N=128,
      // emulated shards): 4 shards 0.973 -> 0.833 ms, 8 shards 0.526 ->
      // 0.499 ms — the ring's 128 KB of shared memory per SM took L1 and
      // occupancy from the warp kernel next to it.  GESPMM_HUB_SEQ=0 restores
      // the round-1 scheme (overlapped launch, side stream, launch-wide
      // threshold).
      if (tma && (hub_pdl || !side)) {
        GESPMM_CUDA(launch_tuned_hub(op, fast, h, st, true), "spmm");
        hub_then_pdl = !hub_ring_first();
      } else {
        cudaStream_t hs = side ? side : st;
        if (side) {
          GESPMM_CUDA(cudaEventRecord(fork, st), "spmm");
          GESPMM_CUDA(cudaStreamWaitEvent(side, fork, 0), "spmm");
        }
        if (tma)
          GESPMM_CUDA(launch_tuned_hub(op, fast, h, hs, false), "spmm");
        else
          GESPMM_CUDA(launch_tuned_cta(cs, op, fast, h, hs), "spmm");
        if (side) {
          GESPMM_CUDA(cudaEventRecord(join, side), "spmm");
          side_used = true;
        }
      }
    }
    sa.order = order + n_hub;
    sa.n_sched = n_rest;
    sa.n_tiles = (w + wsel.tile_width() - 1) / wsel.tile_width();
    sa.pdl_wait = chain ? 1 : 0;
    if (n_rest)
      GESPMM_CUDA(launch_tuned_warp(wsel, op, fast, sa, st, winp,
                                    hub_then_pdl || chain || pdl_overlap), "spmm");
    if (side_used) GESPMM_CUDA(cudaStreamWaitEvent(st, join, 0), "spmm");
  }
  return GESPMM_OK;
}

// Split hub rows instead of the k_hub ring when the fold does not depend on
// the order of its partial results: max/min (strict compare + earliest
// position among ties = the sequential fold's result) always; sum/mean only
// in fast mode (the partial sums reassociate the fold within the tolerance).
// Not with the SkipTail fault hook (per-row tail) or column slices.
// GESPMM_HUB_SEGMENTS=0 keeps the ring (A/B).
bool split_eligible(const Plan& p) {
  static const bool off = [] {
    const char* e = std::getenv("GESPMM_HUB_SEGMENTS");
    return e && e[0] == '0';
  }();
  if (off || p.o.fault_skip_tail || p.sh.slices != 1 || p.o.variant != GESPMM_VARIANT_TUNED)
    return false;
  if (p.op == GESPMM_MAX || p.op == GESPMM_MIN) return true;
  return p.o.exact == 0;
}

// Inspector: degree-descending row schedule (stable counting sort) so heavy
// rows start first (LPT) and sub-warps pair rows of similar length; rows with
// degree >= threshold are peeled off for the row-per-CTA kernel.
gespmm_status_t build_tuned(Plan& p, const uint32_t* host_rp, cudaStream_t st) {
  const uint32_t m = p.a.n_rows;
  std::vector<uint32_t> deg(m);
  uint32_t maxd = 0;
  for (uint32_t r = 0; r < m; ++r) {
    deg[r] = host_rp[r + 1] - host_rp[r];
    maxd = std::max(maxd, deg[r]);
  }
  p.max_degree = maxd;
  p.mean_degree = m ? double(host_rp[m]) / m : 0.0;
  p.sh = make_shapes(p.o, p.a.n_cols, p.n, p.device, p.mean_degree);
  const uint32_t sw = p.sh.slice_w;
  std::vector<uint32_t> count(size_t(maxd) + 2, 0);
  for (uint32_t r = 0; r < m; ++r) ++count[maxd - deg[r]];
  uint64_t acc = 0;
  for (auto& c : count) {
    const uint64_t t = c;
    c = uint32_t(acc);
    acc += t;
  }
  std::vector<uint32_t> order(m);
  for (uint32_t r = 0; r < m; ++r) order[count[maxd - deg[r]]++] = r;

  const int32_t ht = p.o.hub_threshold;
  p.hub_threshold = ht > 0 ? uint32_t(ht)
                           : (ht < 0 ? 0xffffffffu
                                     : auto_hub_threshold(sw, host_rp[m], p.sh.warp_v.cf,
                                                          p.a.n_cols, p.device,
                                                          p.sh.warp_v.tile_width(), maxd));
  uint32_t n_hub = 0;
  uint64_t hub_nnz = 0;
  while (n_hub < m && deg[order[n_hub]] >= p.hub_threshold) hub_nnz += deg[order[n_hub++]];
  p.n_hub = n_hub;
  p.hub_pdl = host_rp[m] && double(hub_nnz) >= kHubPdlShare * double(host_rp[m]);
  // exact plans with hub rows always run the ring first and alone (even when
  // the hub rows carry < kHubPdlShare: 2 Reddit shards 1.714 ms with the ring
  // as a side job, 1.566 ms ring-first; tools/r2_alpha.sh)
  const bool seq_always = hub_ring_first();
  if (ht == 0 && n_hub && seq_always && !split_eligible(p) && sw >= 8) {
    // the ring will run alone first (launch_tuned_rows): re-pick the threshold
    p.hub_threshold = seq_hub_threshold(deg, order, host_rp[m], sw, p.sh.warp_v.tile_width(),
                                        p.sh.warp_v.cf, p.a.n_cols, p.device);
    n_hub = 0;
    hub_nnz = 0;
    while (n_hub < m && deg[order[n_hub]] >= p.hub_threshold) hub_nnz += deg[order[n_hub++]];
    p.n_hub = n_hub;
    p.hub_pdl = seq_always || double(hub_nnz) >= kHubPdlShare * double(host_rp[m]);
  }
  if (n_hub && split_eligible(p)) {
    // segments of at most half the hub threshold: each one's single-warp time
    // is then at most half of what made a row a hub row
    const uint32_t t = p.hub_threshold == 0xffffffffu ? 4096u : p.hub_threshold;
    p.seg_len = std::max<uint32_t>(256, (t / 2 + 63) & ~63u);
    // (segment-length sweep, profiles/r2/split/seglen_*: 512 / half the
    // threshold / 2048 within 2%, 4096 slower)
    std::vector<uint32_t> vptr, seg, hubs;
    for (uint32_t i = 0; i < n_hub; ++i) {
      const uint32_t r = order[i], d = deg[r];
      const uint32_t k = (d + p.seg_len - 1) / p.seg_len;
      const uint32_t base = uint32_t(vptr.size());
      for (uint32_t j = 0; j <= k; ++j) vptr.push_back(host_rp[r] + std::min(j * p.seg_len, d));
      for (uint32_t j = 0; j < k; ++j) seg.push_back(base + j);
      hubs.insert(hubs.end(), {r, base, k});
    }
    p.split = true;
    p.n_seg = uint32_t(seg.size());
    p.n_vrows = uint32_t(vptr.size());
    const bool arg_op = p.op == GESPMM_MAX || p.op == GESPMM_MIN;
    const auto up = [&](uint32_t** dst, const std::vector<uint32_t>& v) {
      cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), sizeof(uint32_t) * v.size());
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(*dst, v.data(), sizeof(uint32_t) * v.size(), cudaMemcpyHostToDevice, st);
      return e;
    };
    GESPMM_CUDA(up(&p.d_vptr, vptr), "plan_create");
    GESPMM_CUDA(up(&p.d_seg_order, seg), "plan_create");
    GESPMM_CUDA(up(&p.d_hubs, hubs), "plan_create");
    GESPMM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.d_part),
                           sizeof(float) * size_t(p.n_vrows) * p.n), "plan_create");
    if (arg_op)
      GESPMM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.d_part_arg),
                             sizeof(int32_t) * size_t(p.n_vrows) * p.n), "plan_create");
    GESPMM_CUDA(cudaStreamSynchronize(st), "plan_create");
  }

  // Rows of at most two staged chunks gain nothing from the LPT schedule:
  // the identity order saves the schedule load in front of every row.
  const bool identity = n_hub == 0 && maxd <= 64;
  if (m && !identity) {
    GESPMM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.d_order), sizeof(uint32_t) * m),
                "plan_create");
    GESPMM_CUDA(cudaMemcpyAsync(p.d_order, order.data(), sizeof(uint32_t) * m,
                                cudaMemcpyHostToDevice, st),
                "plan_create");
    GESPMM_CUDA(cudaStreamSynchronize(st), "plan_create");
  }
  if (n_hub) {
    // hub rows are the critical path: their CTAs dispatch ahead of the warp
    // kernel's whenever an SM frees up
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    GESPMM_CUDA(cudaStreamCreateWithPriority(&p.side, cudaStreamNonBlocking, hi_prio), "plan_create");
    GESPMM_CUDA(cudaEventCreateWithFlags(&p.ev_fork, cudaEventDisableTiming), "plan_create");
    GESPMM_CUDA(cudaEventCreateWithFlags(&p.ev_join, cudaEventDisableTiming), "plan_create");
    GESPMM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.d_work), sizeof(uint32_t) * p.sh.slices),
                "plan_create");
  }
#ifdef GESPMM_EXPERIMENTAL
  if (p.o.cluster_hot > 0 && p.n == 128 && p.a.nnz) {
    // every row goes through the cluster kernel (LPT order, persistent warps)
    if (!p.d_order && m) {
      GESPMM_CUDA(cudaMalloc(reinterpret_cast<void**>(&p.d_order), sizeof(uint32_t) * m),
                  "plan_create");
      GESPMM_CUDA(cudaMemcpyAsync(p.d_order, order.data(), sizeof(uint32_t) * m,
                                  cudaMemcpyHostToDevice, st), "plan_create");
    }
    GESPMM_CUDA(build_cluster_hot(p.a.col_ind, p.a.nnz, p.a.n_cols, p.o.cluster_hot, st, &p.ch),
                "plan_create");
  }
  const uint64_t hot_budget = hot_budget_bytes(p.o, p.a.n_cols, p.n, p.device);
  if (hot_budget && p.o.l2_hints && p.a.nnz) {
    GESPMM_CUDA(build_hot_bitmap(p.a.col_ind, p.a.nnz, p.a.n_cols,
                                 hot_budget / (uint64_t(sw) * sizeof(float)), st, &p.d_hot,
                                 &p.hot),
                "plan_create");
  }
#endif
#ifdef GESPMM_EXPERIMENTAL
  const uint64_t reloc = hot_rows_budget(p.o, p.a.n_cols, p.n, p.device);
  if (reloc && p.a.nnz && p.n)
    GESPMM_CUDA(build_hot_rows(p.a.col_ind, p.a.nnz, p.a.n_cols, p.n,
                               reloc / (uint64_t(p.n) * sizeof(float)), st, &p.hr),
                "plan_create");
#endif
  char buf[512];
  int len = std::snprintf(buf, sizeof buf,
                "tuned: warp(vec=%d,lpr=%d,cf=%d) rows=%u; cta(vec=%d,warps=%d) hub_rows=%u "
                "(deg>=%u); mean_deg=%.1f max_deg=%u",
                p.sh.warp_v.vec, p.sh.warp_v.lpr, p.sh.warp_v.cf, m - n_hub, p.sh.cta_v.vec,
                p.sh.cta_v.warps,
                n_hub, p.hub_threshold, p.mean_degree, maxd);
  if (p.d_hot && len > 0 && size_t(len) < sizeof buf)
    std::snprintf(buf + len, sizeof buf - size_t(len),
                  "; l2 hot map %.0f MB: %llu cols (gathered>=%u) = %.1f%% of gathers",
                  double(p.o.l2_hot_mb) * 1.048576, (unsigned long long)p.hot.hot_cols, p.hot.threshold,
                  100.0 * p.hot.hot_nnz_frac);
  len = int(std::strlen(buf));
  if (size_t(len) < sizeof buf)
    std::snprintf(buf + len, sizeof buf - size_t(len), "; %s",
                  identity ? "identity order" : "degree-sorted (LPT) order");
  len = int(std::strlen(buf));
  if (p.ch.col_ind && size_t(len) < sizeof buf) {
    std::snprintf(buf + len, sizeof buf - size_t(len),
                  "; cluster DSMEM cache: %u hot rows in clusters of %d = %.1f%% of gathers",
                  p.ch.n_hot, p.ch.cs, 100.0 * p.ch.hot_nnz_frac);
    len = int(std::strlen(buf));
  }
  if (p.hr.n_hot && size_t(len) < sizeof buf) {
    std::snprintf(buf + len, sizeof buf - size_t(len),
                  "; relocated hot rows %.1f MB: %u cols (gathered>=%u) = %.1f%% of gathers",
                  double(p.hr.n_hot) * p.hr.ldh * 4.0 / 1048576.0, p.hr.n_hot, p.hr.threshold,
                  100.0 * p.hr.hot_nnz_frac);
    len = int(std::strlen(buf));
  }
  if (p.sh.slices > 1 && size_t(len) < sizeof buf)
    std::snprintf(buf + len, sizeof buf - size_t(len), "; %u column slices of %u", p.sh.slices, sw);
  len = int(std::strlen(buf));
  if (p.split && size_t(len) < sizeof buf)
    std::snprintf(buf + len, sizeof buf - size_t(len),
                  "; hub rows split: %u segments of <= %u nonzeros, ordered combine", p.n_seg,
                  p.seg_len);
  p.desc = buf;
  return GESPMM_OK;
}

gespmm_status_t plan_create_impl(const gespmm_csr_t* a, uint32_t n, gespmm_reduce_t op,
                                 const gespmm_options_t* opts, cudaStream_t st,
                                 const uint32_t* host_rp, Plan** out) {
  gespmm_options_t o;
  if (opts) o = *opts; else gespmm_options_default(&o);
  gespmm_status_t s = check_opts(o);
  if (s != GESPMM_OK) return s;
  s = check_op(op, nullptr);
  if (s != GESPMM_OK) return s;
  if (n == 0 && a->n_rows != 0) return fail(GESPMM_EINVAL, "native_spmm: N must be >= 1");
  auto p = std::make_unique<Plan>();
  p->a = *a;
  p->n = n;
  p->op = op;
  p->o = o;
  cudaGetDevice(&p->device);
  if (o.variant == GESPMM_VARIANT_TUNED && a->n_rows > 0) {
    std::vector<uint32_t> tmp;
    if (!host_rp) {
      tmp.resize(size_t(a->n_rows) + 1);
      GESPMM_CUDA(cudaMemcpyAsync(tmp.data(), a->row_ptr, sizeof(uint32_t) * tmp.size(),
                                  cudaMemcpyDeviceToHost, st),
                  "plan_create");
      GESPMM_CUDA(cudaStreamSynchronize(st), "plan_create");
      host_rp = tmp.data();
    }
    s = build_tuned(*p, host_rp, st);
    if (s != GESPMM_OK) return s;
  } else {
    char buf[128];
    const char* names[] = {"tuned", "naive", "crc", "crc-cwm"};
    std::snprintf(buf, sizeof buf, "%s(cf=%u)", names[o.variant],
                  o.variant == GESPMM_VARIANT_CRC_CWM ? o.cf : 1u);
    p->desc = buf;
  }
  *out = p.release();
  return GESPMM_OK;
}

// Persisting-L2 set-aside, raised once per device to the hardware maximum
// when a plan asks for it (opt-in: this is device-wide state).
struct PersistLimits {
  size_t max_window = 0;
  size_t set_aside = 0;
};
std::mutex g_persist_mu;
PersistLimits g_persist[64];
bool g_persist_init[64] = {};

PersistLimits persist_limits(int dev) {
  std::lock_guard<std::mutex> lk(g_persist_mu);
  if (dev < 0 || dev >= 64) return {};
  if (!g_persist_init[dev]) {
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(max_persist)) == cudaSuccess) {
      size_t got = 0;
      cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
      g_persist[dev].set_aside = got;
    }
    g_persist[dev].max_window = size_t(max_window);
    g_persist_init[dev] = true;
  }
  return g_persist[dev];
}

gespmm_status_t plan_execute_impl(Plan& p, const float* b, float* c, int32_t* arg,
                                  cudaStream_t st, const SpmmArgs* rep = nullptr) {
  gespmm_status_t s = check_op(p.op, arg);
  if (s == GESPMM_OK) s = check_arg_range(arg, p.a.nnz, p.a.n_cols, p.o.arg_kind);
  if (s != GESPMM_OK) return s;
  if (p.a.n_rows == 0) return GESPMM_OK;
  SpmmArgs args{};
  args.row_ptr = p.a.row_ptr;
  args.col_ind = p.a.col_ind;
  args.vals = p.a.vals;
  args.b = b;
  args.c = c;
  args.arg = arg;
  args.n = p.n;
  args.kb = p.a.n_cols;
  args.arg_col = p.o.arg_kind == GESPMM_ARG_COLUMN;
  args.skip_tail = p.o.fault_skip_tail;
  args.hints = p.o.l2_hints;
  args.hot = p.d_hot;
  if (rep) {  // fused all-gather epilogue (tuned plans only, checked by the caller)
    args.n_peer = rep->n_peer;
    for (int q = 0; q < rep->n_peer; ++q) {
      args.c_peer[q] = rep->c_peer[q];
      args.arg_peer[q] = rep->arg_peer[q];
    }
    args.c_mc = rep->c_mc;
    args.arg_mc = rep->arg_mc;
  }
  const bool fast = p.o.exact == 0;
  if (p.o.variant != GESPMM_VARIANT_TUNED) {
    args.order = nullptr;
    args.n_sched = p.a.n_rows;
    args.ld = args.ldb = p.n;
    args.n_tiles = faithful_tiles(p.o.variant, p.o.cf, p.n);
    GESPMM_CUDA(launch_faithful(p.o.variant, p.o.cf, p.op, fast, args, st), "spmm");
    return GESPMM_OK;
  }
  args.ld = args.ldb = p.n;
#ifdef GESPMM_EXPERIMENTAL
  if (p.ch.col_ind && aligned(b, 16) && aligned(c, 16) && (!arg || aligned(arg, 16))) {
    args.order = p.d_order;
    args.n_sched = p.a.n_rows;
    args.n_tiles = 1;
    GESPMM_CUDA(resolve_policies(&args, st), "spmm");
    int clusters = 0;
    GESPMM_CUDA(launch_cluster_warp(p.ch, p.op, fast, args, st, &clusters), "spmm");
    return GESPMM_OK;
  }
#endif
  cudaAccessPolicyWindow win{};
  const cudaAccessPolicyWindow* winp = nullptr;
  if (p.o.l2_persist == 2) persist_limits(p.device);  // set-aside only, no window
  if (p.o.l2_persist == 1) {
    const size_t b_bytes = size_t(p.a.n_cols) * args.ldb * sizeof(float);
    const PersistLimits lim = persist_limits(p.device);
    if (lim.max_window > 0 && lim.set_aside > 0 && b_bytes > 0) {
      win.base_ptr = const_cast<float*>(b);
      win.num_bytes = std::min(b_bytes, lim.max_window);
      win.hitRatio = float(std::min(1.0, double(lim.set_aside) / double(win.num_bytes)));
      win.hitProp = cudaAccessPropertyPersisting;
      win.missProp = cudaAccessPropertyStreaming;
      winp = &win;
    }
  }
#ifdef GESPMM_EXPERIMENTAL
  const float* b_hot = nullptr;
  int32_t hot_off = 0;
  if (p.hr.n_hot && place_hot_rows(p.hr, b, args.ldb, &b_hot, &hot_off)) {
    // relocated hot rows: refresh the copy from this B, gather through the remap
    GESPMM_CUDA(refresh_hot_rows(p.hr, b, args.ldb, p.n, b_hot, st), "spmm");
    args.col_ind_orig = args.col_ind;
    args.col_ind = p.hr.col_ind;
    args.b_hot = b_hot;
    args.hot_off = hot_off;
    args.hot_bytes = uint32_t(uint64_t(p.hr.n_hot) * args.ldb * sizeof(float));
    static const int mode = [] {
      const char* e = std::getenv("GESPMM_RELOC_POLICY");  // A/B: 0 keep, 1 range+evict_first, 2 range
      return e ? std::atoi(e) : 1;
    }();
    args.reloc_mode = mode;
    if (mode != 0)
      GESPMM_CUDA(resolve_range_policy(b_hot, args.hot_bytes, mode, &args.pol_hot, st), "spmm");
  }
#endif
  if (p.split) {
    // the hub rows' segments first (equal-length work units, the long pole of
    // the row schedule) into partial rows; the rows below the threshold (LPT
    // order) follow as a programmatic dependent launch (disjoint outputs,
    // both run together); then the ordered combine (a normal launch: after
    // both).  Rest-first put the segments behind the whole rest grid (its
    // last CTA triggers the dependent launch): products 8 shards 1.81 ms.
    SpmmArgs sg = args;
    sg.row_ptr = p.d_vptr;
    sg.c = p.d_part;
    sg.arg = args.arg ? p.d_part_arg : nullptr;
    sg.ld = p.n;
    sg.n_peer = 0;
    sg.c_mc = nullptr;
    sg.arg_mc = nullptr;
    const int seg_op = p.op == GESPMM_MEAN ? GESPMM_SUM : p.op;  // mean divides in the combine
    gespmm_status_t s2 = launch_tuned_rows(p.sh, seg_op, fast, sg, p.d_seg_order, 0, p.n_seg, st,
                                           nullptr, nullptr, nullptr, winp, false, nullptr);
    if (s2 != GESPMM_OK) return s2;
    s2 = launch_tuned_rows(p.sh, p.op, fast, args, p.d_order + p.n_hub, 0, p.a.n_rows - p.n_hub,
                           st, nullptr, nullptr, nullptr, winp, false, nullptr, false, true);
    if (s2 != GESPMM_OK) return s2;
    GESPMM_CUDA(launch_split_combine(p.op, args, p.d_hubs, p.n_hub, p.d_part,
                                     args.arg ? p.d_part_arg : nullptr, st), "spmm");
    return GESPMM_OK;
  }
  return launch_tuned_rows(p.sh, p.op, fast, args, p.d_order, p.n_hub, p.a.n_rows - p.n_hub, st,
                           p.side, p.ev_fork, p.ev_join, winp, p.hub_pdl, p.d_work,
                           p.o.overlap_prev != 0 && !winp);
}

// Small LRU of plans for the plan-less device entry point: keyed by the CSR
// arrays, shape, op, options, device and stream (a plan's hub counters and
// split partials are per-execute scratch, so two streams never share one).
// A cached plan keeps a row schedule derived from row_ptr, and every schedule
// covers every row exactly once, so a stale entry (row_ptr mutated in place,
// or a new CSR at a recycled address) can only cost speed; the one piece of
// plan state that holds row_ptr values, a split plan's virtual row_ptr over
// hub-row segments, is rebuilt from the live row_ptr on every cache hit
// (launch_split_refresh).  Plans that snapshot col_ind (cluster_hot's
// remapped copy, relocated hot rows) are never cached: the call builds and
// drops one each time.
struct CacheEntry {
  gespmm_csr_t a;
  uint32_t n;
  gespmm_reduce_t op;
  gespmm_options_t o;
  int device;
  cudaStream_t stream;
  std::shared_ptr<Plan> plan;  // shared: a caller keeps its plan alive past an eviction
};
std::mutex g_cache_mu;
std::list<CacheEntry> g_cache;
constexpr size_t kCacheCap = 16;

std::shared_ptr<Plan> cached_plan(const gespmm_csr_t* a, uint32_t n, gespmm_reduce_t op,
                  const gespmm_options_t& o, cudaStream_t st, const uint32_t* host_rp,
                  gespmm_status_t* status) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
    if (it->device == dev && it->stream == st && it->n == n && it->op == op &&
        std::memcmp(&it->a, a, sizeof(*a)) == 0 && std::memcmp(&it->o, &o, sizeof(o)) == 0) {
      g_cache.splice(g_cache.begin(), g_cache, it);
      std::shared_ptr<Plan> hit = g_cache.front().plan;
      *status = GESPMM_OK;
      if (hit->split) {
        const cudaError_t e = launch_split_refresh(a->row_ptr, hit->d_hubs, hit->n_hub,
                                                   hit->seg_len, hit->d_vptr, st);
        if (e != cudaSuccess) {
          *status = cuda_fail(e, "spmm");
          return nullptr;
        }
      }
      return hit;
    }
  }
  Plan* p = nullptr;
  *status = plan_create_impl(a, n, op, &o, st, host_rp, &p);
  if (*status != GESPMM_OK) return nullptr;
  std::shared_ptr<Plan> sp(p);
  g_cache.push_front(CacheEntry{*a, n, op, o, dev, st, sp});
  if (g_cache.size() > kCacheCap) g_cache.pop_back();
  return sp;
}

// Grow-only device staging for the host-buffer entry point: buffers, a
// compute stream and copy-in / copy-out streams with per-chunk events.
constexpr int kMaxChunks = 16;
struct Workspace {
  std::mutex mu;
  cudaStream_t stream = nullptr, in = nullptr, out = nullptr;
  cudaStream_t side = nullptr;  // hub-row kernels next to the warp kernel of a block
  cudaEvent_t ev_b = nullptr, ev_in[kMaxChunks] = {}, ev_done[kMaxChunks] = {};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // device: row_ptr, col_ind, vals, B, C, arg, order, validation scratch +
  // row-start bitmap, packed codes, packed exceptions, scan temp, hub counters
  void* buf[12] = {};
  size_t cap[12] = {};
  // pinned host staging: packed codes, packed exceptions, row schedule
  void* hbuf[3] = {};
  size_t hcap[3] = {};
  cudaError_t reserve(int i, size_t bytes) {
    if (bytes <= cap[i]) return cudaSuccess;
    if (buf[i]) cudaFree(buf[i]);
    buf[i] = nullptr;
    cap[i] = 0;
    cudaError_t e = cudaMalloc(&buf[i], bytes);
    if (e == cudaSuccess) cap[i] = bytes;
    return e;
  }
  cudaError_t reserve_host(int i, size_t bytes) {
    if (bytes <= hcap[i]) return cudaSuccess;
    if (hbuf[i]) cudaFreeHost(hbuf[i]);
    hbuf[i] = nullptr;
    hcap[i] = 0;
    cudaError_t e = cudaHostAlloc(&hbuf[i], bytes, cudaHostAllocDefault);
    if (e == cudaSuccess) hcap[i] = bytes;
    return e;
  }
};
std::mutex g_ws_mu;
Workspace* g_ws[64] = {};

Workspace* workspace() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if (!g_ws[dev]) {
    auto* w = new Workspace();
    cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&w->in, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&w->out, cudaStreamNonBlocking);
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    cudaStreamCreateWithPriority(&w->side, cudaStreamNonBlocking, hi_prio);
    cudaEventCreateWithFlags(&w->ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->ev_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&w->ev_b, cudaEventDisableTiming);
    for (int i = 0; i < kMaxChunks; ++i) {
      cudaEventCreateWithFlags(&w->ev_in[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&w->ev_done[i], cudaEventDisableTiming);
    }
    g_ws[dev] = w;
  }
  return g_ws[dev];
}

// Frees the host entry's grow-only buffers of the current device (the next
// call reallocates them).
void release_host_workspace() {
  int dev = 0;
  cudaGetDevice(&dev);
  Workspace* w = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (dev >= 0 && dev < 64) w = g_ws[dev];
  }
  if (!w) return;
  std::lock_guard<std::mutex> lk(w->mu);  // no host-entry call in flight on this device
  for (size_t i = 0; i < sizeof(w->buf) / sizeof(w->buf[0]); ++i)
    if (w->buf[i]) {
      cudaFree(w->buf[i]);
      w->buf[i] = nullptr;
      w->cap[i] = 0;
    }
  for (size_t i = 0; i < sizeof(w->hbuf) / sizeof(w->hbuf[0]); ++i)
    if (w->hbuf[i]) {
      cudaFreeHost(w->hbuf[i]);
      w->hbuf[i] = nullptr;
      w->hcap[i] = 0;
    }
}

// GESPMM_TRACE=1: host-side phase timestamps of the host entry point (stderr).
// NVTX range for the lifetime of a scope (nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Trace {
  bool on = false;
  std::chrono::steady_clock::time_point t0;
  Trace() {
    const char* e = std::getenv("GESPMM_TRACE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) const {
    nvtxMarkA(what);  // a no-op unless a profiler is attached
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[gespmm] %8.3f ms  %s\n", ms, what);
  }
  // device timeline: timing events recorded on the streams, printed by dump()
  // relative to the first one (after the streams are synchronised)
  mutable std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void dev(const std::string& what, cudaStream_t s) const {
    if (!on) return;
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    ev.emplace_back(what, e);
  }
  void dump() const {
    if (!on) return;
    for (auto& [what, e] : ev) {
      float ms = 0.0f;
      cudaEventSynchronize(e);
      cudaEventElapsedTime(&ms, ev.front().second, e);
      std::fprintf(stderr, "[gespmm] device %8.3f ms  %s\n", ms, what.c_str());
    }
    for (auto& pr : ev) cudaEventDestroy(pr.second);
    ev.clear();
  }
};

// Host-side row_ptr checks (csr.hpp:118-131 order): row_ptr[0], monotonicity,
// row_ptr[M] == nnz.  Column checks run on the device per row block.
gespmm_status_t host_rowptr_status(const gespmm_csr_t* a, const char* who) {
  ValidateResult r{};
  r.row_ptr0 = a->row_ptr[0];
  r.row_ptr_last = a->row_ptr[a->n_rows];
  r.first_decrease = 0xffffffffu;
  for (uint32_t i = 1; i <= a->n_rows; ++i)
    if (a->row_ptr[i] < a->row_ptr[i - 1]) {
      r.first_decrease = i;
      break;
    }
  r.first_bad_key = ~0ull;
  return validation_status(r, a->n_rows, a->n_cols, a->nnz, who);
}

gespmm_status_t device_validate(const gespmm_csr_t* a, cudaStream_t st, const char* who) {
  ValidateResult r{};
  GESPMM_CUDA(validate_csr_device(a->n_rows, a->n_cols, a->nnz, a->row_ptr, a->col_ind, &r, st),
              "validate");
  return validation_status(r, a->n_rows, a->n_cols, a->nnz, who);
}

}  // namespace
}  // namespace gespmm

using namespace gespmm;

extern "C" {

void gespmm_options_default(gespmm_options_t* o) {
  std::memset(o, 0, sizeof(*o));
  o->variant = GESPMM_VARIANT_TUNED;
  o->cf = 2;
  o->exact = 1;
  o->arg_kind = GESPMM_ARG_EDGE;
  o->validate = 1;
  o->fault_skip_tail = 0;
  o->l2_hints = 1;
  o->hub_threshold = 0;
  o->l2_persist = 0;
}

const char* gespmm_last_error(void) { return t_err.c_str(); }

int32_t gespmm_abi_version(void) { return GESPMM_ABI_VERSION; }

void gespmm_release_workspace(void) {
  release_host_workspace();
  release_coo_scratch();
}

int32_t gespmm_build_flags(void) {
#ifdef GESPMM_EXPERIMENTAL
  return GESPMM_BUILD_EXPERIMENTAL;
#else
  return 0;
#endif
}

uint64_t gespmm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

gespmm_status_t gespmm_validate_device(const gespmm_csr_t* a, void* stream) {
  if (!a) return fail(GESPMM_EINVAL, "null csr");
  return device_validate(a, static_cast<cudaStream_t>(stream), "spmm");
}

gespmm_status_t gespmm_validate_device_as(const gespmm_csr_t* a, void* stream, const char* who) {
  if (!a) return fail(GESPMM_EINVAL, "null csr");
  return validate_device_as(a, static_cast<cudaStream_t>(stream), who ? who : "spmm");
}

gespmm_status_t gespmm_plan_create(const gespmm_csr_t* a, uint32_t n, gespmm_reduce_t op,
                                   const gespmm_options_t* opts, void* stream,
                                   gespmm_plan_t* out) {
  if (!a || !out) return fail(GESPMM_EINVAL, "null argument");
  Plan* p = nullptr;
  gespmm_status_t s = plan_create_impl(a, n, op, opts, static_cast<cudaStream_t>(stream),
                                       nullptr, &p);
  if (s != GESPMM_OK) return s;
  *out = reinterpret_cast<gespmm_plan_t>(p);
  return GESPMM_OK;
}

gespmm_status_t gespmm_plan_execute(gespmm_plan_t plan, const float* b, float* c, int32_t* arg,
                                    void* stream) {
  if (!plan) return fail(GESPMM_EINVAL, "null plan");
  const NvtxRange nvtx("gespmm_plan_execute");
  return plan_execute_impl(*reinterpret_cast<Plan*>(plan), b, c, arg,
                           static_cast<cudaStream_t>(stream));
}

gespmm_status_t gespmm_plan_execute_gather(gespmm_plan_t plan, const float* b,
                                           float* const* c_dsts, int32_t* const* arg_dsts,
                                           int32_t n_dsts, float* c_multicast,
                                           int32_t* arg_multicast, void* stream) {
  if (!plan || !c_dsts) return fail(GESPMM_EINVAL, "null argument");
  Plan& p = *reinterpret_cast<Plan*>(plan);
  if (n_dsts < 1 || n_dsts > GESPMM_MAX_GATHER_DSTS)
    return fail(GESPMM_EINVAL, "gather: n_dsts must be in [1, " +
                                   std::to_string(GESPMM_MAX_GATHER_DSTS) + "]");
  if (p.o.variant != GESPMM_VARIANT_TUNED)
    return fail(GESPMM_EUNSUPPORTED, "gather: the fused all-gather epilogue needs a tuned plan");
  const bool has_arg = p.op == GESPMM_MAX || p.op == GESPMM_MIN;
  int32_t* arg0 = (arg_dsts && has_arg) ? arg_dsts[0] : nullptr;
  SpmmArgs rep{};
  rep.n_peer = n_dsts - 1;
  for (int q = 1; q < n_dsts; ++q) {
    if (!c_dsts[q]) return fail(GESPMM_EINVAL, "gather: null destination");
    // replicas share the local C's alignment class, so the chosen vector
    // width is valid for every destination
    if ((reinterpret_cast<uintptr_t>(c_dsts[q]) ^ reinterpret_cast<uintptr_t>(c_dsts[0])) % 16)
      return fail(GESPMM_EINVAL, "gather: destinations must share the local C's 16-byte alignment");
    rep.c_peer[q - 1] = c_dsts[q];
    rep.arg_peer[q - 1] = (arg_dsts && has_arg) ? arg_dsts[q] : nullptr;
    if (rep.arg_peer[q - 1] && (!arg0 || (reinterpret_cast<uintptr_t>(rep.arg_peer[q - 1]) ^
                                          reinterpret_cast<uintptr_t>(arg0)) % 16))
      return fail(GESPMM_EINVAL, "gather: arg replicas need a local arg with the same 16-byte alignment");
  }
  rep.c_mc = c_multicast;
  rep.arg_mc = has_arg ? arg_multicast : nullptr;
  if (c_multicast &&
      (reinterpret_cast<uintptr_t>(c_multicast) ^ reinterpret_cast<uintptr_t>(c_dsts[0])) % 16)
    return fail(GESPMM_EINVAL, "gather: multicast address must share the local C's 16-byte alignment");
  return plan_execute_impl(p, b, c_dsts[0], arg0, static_cast<cudaStream_t>(stream), &rep);
}

const char* gespmm_plan_describe(gespmm_plan_t plan) {
  return plan ? reinterpret_cast<Plan*>(plan)->desc.c_str() : "";
}

int32_t gespmm_plan_launches(gespmm_plan_t plan) {
  if (!plan) return 0;
  const Plan* p = reinterpret_cast<Plan*>(plan);
  if (p->a.n_rows == 0) return 0;
  if (p->o.variant != GESPMM_VARIANT_TUNED) return 1;
  // the same branches as plan_execute_impl / launch_tuned_rows: one cluster
  // launch, or per column slice a hub launch and a warp launch
  if (p->ch.col_ind) return 1;
  if (p->split) return (p->a.n_rows > p->n_hub ? 1 : 0) + 2;  // rows, segments, combine
  const int32_t per_slice = (p->n_hub ? 1 : 0) + (p->a.n_rows > p->n_hub ? 1 : 0);
  return per_slice * int32_t(p->sh.slices) + (p->hr.n_hot ? 1 : 0);  // + the hot-row refresh
}

void gespmm_plan_destroy(gespmm_plan_t plan) { delete reinterpret_cast<Plan*>(plan); }

gespmm_status_t gespmm_spmm_device(const gespmm_csr_t* a, const float* b, uint32_t n,
                                   gespmm_reduce_t op, float* c, int32_t* arg,
                                   const gespmm_options_t* opts, void* stream) {
  if (!a) return fail(GESPMM_EINVAL, "null csr");
  gespmm_options_t o;
  if (opts) o = *opts; else gespmm_options_default(&o);
  gespmm_status_t s = check_opts(o);
  if (s != GESPMM_OK) return s;
  s = check_op(op, arg);
  if (s == GESPMM_OK) s = check_arg_range(arg, a->nnz, a->n_cols, o.arg_kind);
  if (s != GESPMM_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (o.validate) {
    s = device_validate(a, st, "spmm");
    if (s != GESPMM_OK) return s;
  }
  if (a->n_rows == 0) return GESPMM_OK;
  if (n == 0) return fail(GESPMM_EINVAL, "native_spmm: N must be >= 1");
  o.validate = 0;  // not part of the plan identity
  if (o.cluster_hot > 0 || o.hot_rows_mb > 0) {  // snapshots col_ind: a fresh plan per call, never cached
    Plan* fresh = nullptr;
    s = plan_create_impl(a, n, op, &o, st, nullptr, &fresh);
    if (s != GESPMM_OK) return s;
    std::unique_ptr<Plan> own(fresh);
    s = plan_execute_impl(*own, b, c, arg, st);
    if (s == GESPMM_OK) GESPMM_CUDA(cudaStreamSynchronize(st), "spmm");  // before the free
    return s;
  }
  const std::shared_ptr<Plan> p = cached_plan(a, n, op, o, st, nullptr, &s);
  if (!p) return s;
  return plan_execute_impl(*p, b, c, arg, st);
}

gespmm_status_t gespmm_spmm_host(const gespmm_csr_t* a, const float* b, uint32_t b_rows,
                                 uint32_t n, gespmm_reduce_t op, float* c, int32_t* arg,
                                 const gespmm_options_t* opts) {
  // Row-block pipeline: B and row_ptr go first; then for each nnz-balanced
  // row block its col_ind/vals H2D (copy-in stream) -> column validation +
  // kernel (compute stream) -> C rows D2H (copy-out stream), so the kernels and
  // the D2H hide under the CSR upload.  On an error status the contents of c
  // (and arg) are unspecified.
  if (!a) return fail(GESPMM_EINVAL, "null csr");
  const NvtxRange nvtx("gespmm_spmm_host");
  const Trace tr;
  gespmm_options_t o;
  if (opts) o = *opts; else gespmm_options_default(&o);
  gespmm_status_t s = check_op(op, arg);
  if (s == GESPMM_OK) s = check_arg_range(arg, a->nnz, a->n_cols, o.arg_kind);
  if (s != GESPMM_OK) return s;
  if (a->n_cols != b_rows) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "spmm: dimension mismatch: A is %ux%u but B has %u rows",
                  a->n_rows, a->n_cols, b_rows);
    return fail(GESPMM_EDIM, buf);
  }
  if (o.validate) {
    tr.mark("enter");
    s = host_rowptr_status(a, "spmm");
    if (s != GESPMM_OK) return s;
  }
  s = check_opts(o);
  if (s != GESPMM_OK) return s;
  const uint64_t m = a->n_rows, nnz = a->nnz;
  if (m == 0) return GESPMM_OK;
  if (n == 0) {
    // the reference validates columns before reporting N (native.hpp:103-110)
    if (o.validate && nnz) {
      Workspace* ws0 = workspace();
      std::lock_guard<std::mutex> lk0(ws0->mu);
      GESPMM_CUDA(ws0->reserve(0, sizeof(uint32_t) * (m + 1)), "spmm");
      GESPMM_CUDA(ws0->reserve(1, sizeof(uint32_t) * nnz), "spmm");
      GESPMM_CUDA(cudaMemcpyAsync(ws0->buf[0], a->row_ptr, sizeof(uint32_t) * (m + 1),
                                  cudaMemcpyHostToDevice, ws0->stream), "spmm");
      GESPMM_CUDA(cudaMemcpyAsync(ws0->buf[1], a->col_ind, sizeof(uint32_t) * nnz,
                                  cudaMemcpyHostToDevice, ws0->stream), "spmm");
      gespmm_csr_t d0 = *a;
      d0.row_ptr = static_cast<const uint32_t*>(ws0->buf[0]);
      d0.col_ind = static_cast<const uint32_t*>(ws0->buf[1]);
      s = device_validate(&d0, ws0->stream, "spmm");
      if (s != GESPMM_OK) return s;
    }
    return fail(GESPMM_EINVAL, "native_spmm: N must be >= 1");
  }
  Workspace* ws = workspace();
  std::lock_guard<std::mutex> lk(ws->mu);
  const uint64_t bsz = uint64_t(b_rows) * n, csz = m * n;
  GESPMM_CUDA(ws->reserve(0, sizeof(uint32_t) * (m + 1)), "spmm");
  GESPMM_CUDA(ws->reserve(1, sizeof(uint32_t) * std::max<uint64_t>(nnz, 1)), "spmm");
  GESPMM_CUDA(ws->reserve(2, sizeof(float) * std::max<uint64_t>(nnz, 1)), "spmm");
  GESPMM_CUDA(ws->reserve(3, sizeof(float) * std::max<uint64_t>(bsz, 1)), "spmm");
  GESPMM_CUDA(ws->reserve(4, sizeof(float) * csz), "spmm");
  if (arg) GESPMM_CUDA(ws->reserve(5, sizeof(int32_t) * csz), "spmm");
  GESPMM_CUDA(ws->reserve(6, sizeof(uint32_t) * m), "spmm");
  auto* d_rp = static_cast<uint32_t*>(ws->buf[0]);
  auto* d_ci = static_cast<uint32_t*>(ws->buf[1]);
  auto* d_v = static_cast<float*>(ws->buf[2]);
  auto* d_b = static_cast<float*>(ws->buf[3]);
  auto* d_c = static_cast<float*>(ws->buf[4]);
  auto* d_arg = arg ? static_cast<int32_t*>(ws->buf[5]) : nullptr;
  auto* d_order = static_cast<uint32_t*>(ws->buf[6]);
  tr.mark("workspace ready");

  // ---- copy-in stream: row_ptr, B first (every block needs them)
  tr.dev("start (copy-in stream)", ws->in);
  GESPMM_CUDA(cudaMemcpyAsync(d_rp, a->row_ptr, sizeof(uint32_t) * (m + 1),
                              cudaMemcpyHostToDevice, ws->in), "spmm");
  if (bsz)
    GESPMM_CUDA(cudaMemcpyAsync(d_b, b, sizeof(float) * bsz, cudaMemcpyHostToDevice, ws->in),
                "spmm");

  // ---- row blocks balanced by nnz (binary search on the host row_ptr)
  // pipeline depth: more blocks shrink the un-overlapped tail (last block's
  // kernel + C copy-out) but each block's compute carries its hub rows' critical
  // path; with the packed upload (~0.9 ms of copy per block at 16 blocks) the
  // per-block compute (~0.8 ms) nears the copy once clocks drop under the power
  // cap, so 12 blocks keep a margin (Reddit: 16.2-16.5 ms vs 16.4-17.1 at 16).
  // (the paper's Alg. 1-3 kernels keep 8: their hub rows bound every block)
  const bool tuned_v = o.variant == GESPMM_VARIANT_TUNED;
  int chunks = (tuned_v && nnz >= (uint64_t(32) << 20)) ? 12 : (nnz >= (uint64_t(8) << 20) ? 8 : 1);
  if (const char* e = std::getenv("GESPMM_CHUNKS")) {  // pipeline depth experiments
    const int v = std::atoi(e);
    if (v >= 1 && v <= kMaxChunks && nnz >= uint64_t(v)) chunks = v;
  }
  // taper: the last two blocks carry half a block's nonzeros each, so less is
  // left after the final copy.  Round 1 measured it within the noise; with the
  // host polling through the tail (host_poll) the noise is gone and it is
  // 0.1-0.2 ms faster (Reddit: 16.16/16.28 vs 16.40/16.46 ms median,
  // profiles/r2/e2e_taper.txt).  GESPMM_TAPER=0 turns it off.
  static const bool taper = [] {
    const char* e = std::getenv("GESPMM_TAPER");
    return !(e && e[0] == '0');
  }();
  double wsum = 0.0, wcum[kMaxChunks + 1] = {0.0};
  for (int i = 0; i < chunks; ++i) {
    wsum += (taper && chunks >= 4 && i >= chunks - 2) ? 0.5 : 1.0;
    wcum[i + 1] = wsum;
  }
  uint32_t bound[kMaxChunks + 1];
  bound[0] = 0;
  for (int i = 1; i < chunks; ++i) {
    const uint64_t target = uint64_t(double(nnz) * (wcum[i] / wsum));
    const uint32_t* it = std::lower_bound(a->row_ptr, a->row_ptr + m + 1, uint32_t(target));
    bound[i] = std::max<uint32_t>(bound[i - 1], uint32_t(std::min<uint64_t>(it - a->row_ptr, m)));
  }
  bound[chunks] = uint32_t(m);

  // ---- schedule (tuned): per block, local rows in descending degree (LPT);
  //      rows at or above the hub threshold first, for the row-per-CTA kernel
  const bool tuned = o.variant == GESPMM_VARIANT_TUNED;
  uint32_t hub_count[kMaxChunks] = {};
  uint64_t hub_nnz[kMaxChunks] = {};
  TunedShapes shapes;
  uint32_t* d_work = nullptr;  // hub kernel counters: one per (block, column slice)
  if (tuned) {
    int dev = 0;
    GESPMM_CUDA(cudaGetDevice(&dev), "spmm");
    shapes = make_shapes(o, a->n_cols, n, dev, m ? double(nnz) / double(m) : 0.0);
    GESPMM_CUDA(ws->reserve(11, sizeof(uint32_t) * size_t(kMaxChunks) * shapes.slices), "spmm");
    d_work = static_cast<uint32_t*>(ws->buf[11]);
    const int32_t ht = o.hub_threshold;
    uint32_t maxd = 0;
    for (uint64_t r = 0; r < m; ++r) maxd = std::max(maxd, a->row_ptr[r + 1] - a->row_ptr[r]);
    // every row block is its own launch: the threshold follows the block's work
    const uint32_t hub_t =
        ht > 0 ? uint32_t(ht)
               : (ht < 0 ? 0xffffffffu
                         : auto_hub_threshold(shapes.slice_w, nnz / uint64_t(chunks),
                                              shapes.warp_v.cf, a->n_cols, dev,
                                              shapes.warp_v.tile_width(), maxd));
    GESPMM_CUDA(ws->reserve_host(2, sizeof(uint32_t) * m), "spmm");
    uint32_t* order = static_cast<uint32_t*>(ws->hbuf[2]);  // pinned: no sync after its copy
    std::vector<uint32_t> count(size_t(maxd) + 2);
    for (int ch = 0; ch < chunks; ++ch) {
      std::fill(count.begin(), count.end(), 0u);
      const uint32_t lo = bound[ch], hi = bound[ch + 1];
      for (uint32_t r = lo; r < hi; ++r) ++count[maxd - (a->row_ptr[r + 1] - a->row_ptr[r])];
      uint32_t acc = lo;
      for (auto& cnt : count) {
        const uint32_t t = cnt;
        cnt = acc;
        acc += t;
      }
      for (uint32_t r = lo; r < hi; ++r) {
        const uint32_t d = a->row_ptr[r + 1] - a->row_ptr[r];
        order[count[maxd - d]++] = r - lo;  // local id within the block
        if (d >= hub_t) {
          ++hub_count[ch];
          hub_nnz[ch] += d;
        }
      }
    }
    GESPMM_CUDA(cudaMemcpyAsync(d_order, order, sizeof(uint32_t) * m, cudaMemcpyHostToDevice,
                                ws->in), "spmm");
  }
  tr.mark("row_ptr+B enqueued, schedule built");
  tr.dev("row_ptr + B (+ order) landed", ws->in);
  GESPMM_CUDA(cudaEventRecord(ws->ev_b, ws->in), "spmm");
  GESPMM_CUDA(cudaStreamWaitEvent(ws->stream, ws->ev_b, 0), "spmm");
  // packed column indices on the upload (h2dpack.cu): auto for large inputs
  bool pack = o.h2d_pack > 0 || (o.h2d_pack == 0 && nnz >= (uint64_t(8) << 20));
  if (const char* e = std::getenv("GESPMM_H2D_PACK")) pack = std::atoi(e) != 0;
  // the encoder walks the host row_ptr: only once it is known to be sound
  // (validate=1 checked it above; otherwise a silent pass decides)
  const bool rp_sound = o.validate || host_rowptr_status(a, "spmm") == GESPMM_OK;
  pack = pack && rp_sound && nnz > 0 && nnz < 0x7fffffffull;
  uint16_t *h_enc = nullptr, *d_enc = nullptr;
  uint32_t *h_exc = nullptr, *d_exc = nullptr, *bits = nullptr;
  void* scan_tmp = nullptr;
  size_t scan_bytes = 0;
  if (pack) {
    uint64_t max_blk = 0;
    for (int ch = 0; ch < chunks; ++ch)
      max_blk = std::max<uint64_t>(max_blk, a->row_ptr[bound[ch + 1]] - a->row_ptr[bound[ch]]);
    scan_bytes = unpack_temp_bytes(max_blk);
    GESPMM_CUDA(ws->reserve_host(0, sizeof(uint16_t) * nnz), "spmm");
    GESPMM_CUDA(ws->reserve_host(1, sizeof(uint32_t) * (nnz / 4 + 2)), "spmm");
    GESPMM_CUDA(ws->reserve(8, sizeof(uint16_t) * nnz), "spmm");
    GESPMM_CUDA(ws->reserve(9, sizeof(uint32_t) * (nnz / 4 + 2)), "spmm");
    GESPMM_CUDA(ws->reserve(10, std::max<size_t>(scan_bytes, 1)), "spmm");
    h_enc = static_cast<uint16_t*>(ws->hbuf[0]);
    h_exc = static_cast<uint32_t*>(ws->hbuf[1]);
    d_enc = static_cast<uint16_t*>(ws->buf[8]);
    d_exc = static_cast<uint32_t*>(ws->buf[9]);
    scan_tmp = ws->buf[10];
  }
  ColCheck cc_view;
  ColCheck* cc = nullptr;
  if ((o.validate || pack) && nnz) {
    GESPMM_CUDA(ws->reserve(7, colcheck_workspace_bytes(nnz)), "spmm");
    bits = reinterpret_cast<uint32_t*>(static_cast<char*>(ws->buf[7]) + 256);
    if (o.validate) {
      cc = &cc_view;
      GESPMM_CUDA(colcheck_begin(cc, nnz, ws->buf[7], ws->stream), "spmm");
    } else {
      GESPMM_CUDA(cudaMemsetAsync(bits, 0, sizeof(uint32_t) * (nnz / 32 + 1), ws->stream), "spmm");
    }
  }
  uint64_t exc_off = 0;  // exception pairs used so far

  const bool fast = o.exact == 0;
  for (int ch = 0; ch < chunks; ++ch) {
    const uint32_t lo = bound[ch], hi = bound[ch + 1];
    const uint64_t ps = a->row_ptr[lo], pe = a->row_ptr[hi];
    uint64_t nexc = UINT64_MAX;  // exceptions of this block when it travels packed
    if (pe > ps && pack) {
      tr.mark("pack block");
      nexc = pack_cols_block(a->row_ptr, a->col_ind, lo, hi, h_enc + ps, h_exc + 2 * exc_off,
                             (pe - ps) / 8);
    }
    if (pe > ps && nexc != UINT64_MAX) {
      GESPMM_CUDA(cudaMemcpyAsync(d_enc + ps, h_enc + ps, sizeof(uint16_t) * (pe - ps),
                                  cudaMemcpyHostToDevice, ws->in), "spmm");
      if (nexc)
        GESPMM_CUDA(cudaMemcpyAsync(d_exc + 2 * exc_off, h_exc + 2 * exc_off,
                                    sizeof(uint32_t) * 2 * nexc, cudaMemcpyHostToDevice, ws->in),
                    "spmm");
    } else if (pe > ps) {
      GESPMM_CUDA(cudaMemcpyAsync(d_ci + ps, a->col_ind + ps, sizeof(uint32_t) * (pe - ps),
                                  cudaMemcpyHostToDevice, ws->in), "spmm");
    }
    if (pe > ps) {
      GESPMM_CUDA(cudaMemcpyAsync(d_v + ps, a->vals + ps, sizeof(float) * (pe - ps),
                                  cudaMemcpyHostToDevice, ws->in), "spmm");
    }
    tr.dev("block " + std::to_string(ch) + " CSR landed", ws->in);
    GESPMM_CUDA(cudaEventRecord(ws->ev_in[ch], ws->in), "spmm");
    GESPMM_CUDA(cudaStreamWaitEvent(ws->stream, ws->ev_in[ch], 0), "spmm");
    const bool packed_blk = pe > ps && nexc != UINT64_MAX;
    if (packed_blk) {
      // the unpack also runs the column check on the rebuilt columns
      GESPMM_CUDA(unpack_cols(d_enc + ps, reinterpret_cast<const uint2*>(d_exc + 2 * exc_off),
                              uint32_t(nexc), d_rp + lo, hi - lo, ps, pe, nnz, bits, d_ci,
                              scan_tmp, scan_bytes, ws->stream, a->n_cols,
                              cc ? colcheck_key(cc) : nullptr),
                  "spmm");
      exc_off += nexc;
    }
    if (cc && !packed_blk)
      GESPMM_CUDA(colcheck_rows(cc, d_rp + lo, hi - lo, ps, pe, d_ci, a->n_cols, nnz, ws->stream),
                  "spmm");
    SpmmArgs args{};
    args.abort_if = cc ? colcheck_key(cc) : nullptr;  // skip the block's kernels on a violation
    args.row_ptr = d_rp + lo;  // positions stay global; rows and outputs are block-local
    args.col_ind = d_ci;
    args.vals = d_v;
    args.b = d_b;
    args.c = d_c + uint64_t(lo) * n;
    args.arg = d_arg ? d_arg + uint64_t(lo) * n : nullptr;
    args.n = n;
    args.kb = a->n_cols;
    args.ld = args.ldb = n;
    args.arg_col = o.arg_kind == GESPMM_ARG_COLUMN;
    args.skip_tail = o.fault_skip_tail;
    args.hints = o.l2_hints;
    if (hi > lo) {
      if (!tuned) {
        args.order = nullptr;
        args.n_sched = hi - lo;
        args.n_tiles = faithful_tiles(o.variant, o.cf, n);
        GESPMM_CUDA(launch_faithful(o.variant, o.cf, op, fast, args, ws->stream), "spmm");
      } else {
        const uint32_t nh = hub_count[ch];
        const bool pdl = double(hub_nnz[ch]) >= kHubPdlShare * double(pe - ps);
        s = launch_tuned_rows(shapes, op, fast, args, d_order + lo, nh, hi - lo - nh, ws->stream,
                              ws->side, ws->ev_fork, ws->ev_join, nullptr, pdl,
                              d_work + size_t(ch) * shapes.slices);
        if (s != GESPMM_OK) return s;
      }
    }
    tr.dev("block " + std::to_string(ch) + " computed", ws->stream);
    GESPMM_CUDA(cudaEventRecord(ws->ev_done[ch], ws->stream), "spmm");
    GESPMM_CUDA(cudaStreamWaitEvent(ws->out, ws->ev_done[ch], 0), "spmm");
    const uint64_t rows = hi - lo;
    if (rows) {
      GESPMM_CUDA(cudaMemcpyAsync(c + uint64_t(lo) * n, d_c + uint64_t(lo) * n,
                                  sizeof(float) * rows * n, cudaMemcpyDeviceToHost, ws->out),
                  "spmm");
      if (arg)
        GESPMM_CUDA(cudaMemcpyAsync(arg + uint64_t(lo) * n, d_arg + uint64_t(lo) * n,
                                    sizeof(int32_t) * rows * n, cudaMemcpyDeviceToHost, ws->out),
                    "spmm");
      tr.dev("block " + std::to_string(ch) + " C copied out", ws->out);
    }
  }
  tr.dev("all C rows copied out", ws->out);
  tr.mark("all blocks enqueued");
  {
    void* drain[2] = {ws->stream, ws->out};
    host_poll(drain, 2);
  }
  tr.mark("streams drained");
  if (cc) {
    uint64_t key = ~0ull;
    uint32_t brow = 0, bcol = 0;
    GESPMM_CUDA(colcheck_end(cc, d_rp, d_ci, uint32_t(m), &key, &brow, &bcol, ws->stream), "spmm");
    GESPMM_CUDA(cudaStreamSynchronize(ws->out), "spmm");
    ValidateResult r{};
    r.row_ptr0 = 0;
    r.row_ptr_last = uint32_t(nnz);
    r.first_decrease = 0xffffffffu;
    r.first_bad_key = key;
    r.bad_row = brow;
    r.bad_col = bcol;
    s = validation_status(r, a->n_rows, a->n_cols, nnz, "spmm");
    if (s != GESPMM_OK) return s;
  }
  tr.mark("validation done");
  GESPMM_CUDA(cudaStreamSynchronize(ws->stream), "spmm");
  GESPMM_CUDA(cudaStreamSynchronize(ws->out), "spmm");
  tr.mark("done");
  tr.dump();
  return GESPMM_OK;
}

void gespmm_select_variant(uint32_t n, int32_t* variant, uint32_t* cf) {
  if (n <= 32) {
    *variant = GESPMM_VARIANT_CRC;
    *cf = 1;
  } else {
    *variant = GESPMM_VARIANT_CRC_CWM;
    *cf = 2;
  }
}

gespmm_status_t gespmm_reduce_by_name(const char* name, gespmm_reduce_t* out) {
  const std::string s = name ? name : "";
  if (s == "sum") *out = GESPMM_SUM;
  else if (s == "mean") *out = GESPMM_MEAN;
  else if (s == "max") *out = GESPMM_MAX;
  else if (s == "min") *out = GESPMM_MIN;
  else return fail(GESPMM_EINVAL, "unknown reduce op '" + s + "' (built-ins: sum, mean, max, min)");
  return GESPMM_OK;
}

gespmm_status_t gespmm_device_info(int32_t* sm_count, int64_t* l2_bytes,
                                   int64_t* persisting_l2_max, int32_t* cc_major,
                                   int32_t* cc_minor) {
  int dev = 0;
  GESPMM_CUDA(cudaGetDevice(&dev), "device_info");
  cudaDeviceProp prop;
  GESPMM_CUDA(cudaGetDeviceProperties(&prop, dev), "device_info");
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (l2_bytes) *l2_bytes = prop.l2CacheSize;
  if (persisting_l2_max) *persisting_l2_max = prop.persistingL2CacheMaxSize;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return GESPMM_OK;
}

}  // extern "C"
