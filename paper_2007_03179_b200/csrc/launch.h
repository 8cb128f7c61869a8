// Host-side declarations shared by the kernel translation units and the API.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "gespmm/gespmm.h"

namespace gespmm {

struct SpmmArgs;

// Sets the thread's last-error text (gespmm_last_error) and returns st.
gespmm_status_t set_error(gespmm_status_t st, const std::string& msg);

// Counts every kernel launch issued by the library (reported by bench.py).
void note_launch();

// Creates the L2 cache policies for `hints` on the current device once (a
// one-thread kernel, cached per device and hint mode) and stores them into
// a->pol_* (pol_valid = 1).  Synchronous the first time only.
cudaError_t resolve_policies(SpmmArgs* a, cudaStream_t st);
// createpolicy.range word for [base, base + bytes) evict_last (mode 1: and
// evict_first past it inside the range... sizes equal, so only the copy; mode 2:
// primary only), cached per (device, base, bytes, mode).  Synchronous on a miss.
cudaError_t resolve_range_policy(const void* base, uint32_t bytes, int mode, uint64_t* out,
                                 cudaStream_t st);

// --- faithful Algorithms 1-3 (kernels_faithful.cu) ---
uint32_t faithful_tiles(int variant, uint32_t cf, uint32_t n);
cudaError_t launch_faithful(int variant, uint32_t cf, int op, bool fast, const SpmmArgs& a,
                            cudaStream_t s);

// --- tuned B200 kernels (kernels_tuned.cu) ---
// Shape of the row-per-(sub)warp kernel: VEC floats per lane access, LPR lanes
// per row (32/LPR rows share a warp), CF column sub-tiles per lane (CWM merge
// factor).  Column tile width = VEC * LPR * CF.
struct WarpShape {
  int vec = 4;
  int lpr = 32;
  int cf = 1;
  uint32_t tile_width() const { return uint32_t(vec * lpr * cf); }
};
// Row-per-CTA shape for hub rows: WARPS warps split the columns of one row;
// each warp owns VEC*32 contiguous columns per sub-tile.
struct CtaShape {
  int vec = 1;
  int warps = 4;
};

bool tuned_shape_supported(const WarpShape& s);
WarpShape pick_warp_shape(uint32_t n, bool vec4_ok, bool vec2_ok, int rows_per_warp = 1);
// `window` (nullable): L2 access-policy window attached to the launch.
// pdl: launched right behind the hub kernel on the same stream, allowed to
// start while it runs (programmatic dependent launch; rows are disjoint).
cudaError_t launch_tuned_warp(const WarpShape& s, int op, bool fast, const SpmmArgs& a,
                              cudaStream_t st, const cudaAccessPolicyWindow* window = nullptr,
                              bool pdl = false);
bool cta_shape_supported(const CtaShape& s);
CtaShape pick_cta_shape(uint32_t n, bool vec4_ok, bool vec2_ok);
cudaError_t launch_tuned_cta(const CtaShape& s, int op, bool fast, const SpmmArgs& a,
                             cudaStream_t st);
// TMA-ring row-per-CTA kernel for hub rows (N % 4 == 0, 16-byte aligned B/C):
// tile width hub_tile_width(n, n_hub) columns per CTA (a.n_sched = n_hub).
uint32_t hub_tile_width(uint32_t n, uint32_t n_hub);
// big: the 64 KB / 32-per-stage ring (hub kernel ahead of the warp kernel) or
// the 32 KB / 16-per-stage one (side job next to it).
cudaError_t launch_tuned_hub(int op, bool fast, const SpmmArgs& a, cudaStream_t st, bool big);
// Split hub rows: fold each hub row's segment partials (k_warp outputs) in
// segment order into C / arg (+ replicas); hubs = (row, first partial, count).
cudaError_t launch_split_combine(int op, const SpmmArgs& a, const uint32_t* hubs, uint32_t n_hub,
                                 const float* part, const int32_t* part_arg, cudaStream_t st);
// Rebuild the segments' virtual row_ptr from the live row_ptr (same segment
// counts; the last segment absorbs any change of degree): a cached plan-less
// split plan stays correct when row_ptr changed in place or a new CSR of the
// same shape reuses its address.
cudaError_t launch_split_refresh(const uint32_t* row_ptr, const uint32_t* hubs, uint32_t n_hub,
                                 uint32_t seg_len, uint32_t* vptr, cudaStream_t st);

// --- frequency-aware L2 policy (hotcols.cu) ---
struct HotStats {
  uint32_t threshold = 0;     // a column is hot when gathered >= threshold times
  uint64_t hot_cols = 0;
  double hot_nnz_frac = 0.0;  // share of the gathers that hit hot columns
};
// Counts the gathers per column and returns (cudaMalloc'ed, caller frees) a
// ceil(k/32)-word bitmap of the most-gathered columns, at most budget_rows of
// them.  Synchronises `st`.
cudaError_t build_hot_bitmap(const uint32_t* col_ind, uint64_t nnz, uint32_t k,
                             uint64_t budget_rows, cudaStream_t st, uint32_t** out_bits,
                             HotStats* stats);

// --- relocated hot rows (hotrows.cu) ---
struct HotRows {
  uint32_t* col_ind = nullptr;  // remapped col_ind: hot columns = (1 << 31) | slot (a snapshot)
  uint32_t* list = nullptr;     // slot -> column
  float* buf = nullptr;         // (n_hot + 1) rows of ldh floats: the copy, placed per execute
  uint32_t n_hot = 0;
  uint32_t ldh = 0;             // row stride of the copy = the plan's B stride
  uint32_t threshold = 0;       // a column is hot when gathered >= threshold times
  double hot_nnz_frac = 0.0;    // share of the gathers that hit relocated rows
};
// Counts the gathers per column and relocates the most-gathered ones whose rows
// (n floats each) fit budget_rows.  Synchronises `st`.  k < 2^31.
cudaError_t build_hot_rows(const uint32_t* col_ind, uint64_t nnz, uint32_t k, uint32_t n,
                           uint64_t budget_rows, cudaStream_t st, HotRows* out);
// Places the copy inside h.buf at the start congruent to b modulo the row
// stride: b_hot = b + hot_off rows.  False when that offset does not fit int32
// (or the copy is >= 4 GiB): the launch then gathers B directly.
bool place_hot_rows(const HotRows& h, const float* b, uint32_t ldb, const float** b_hot,
                    int32_t* hot_off);
// Copies the relocated rows' first n columns of B (row stride ldb) to b_hot.
cudaError_t refresh_hot_rows(const HotRows& h, const float* b, uint32_t ldb, uint32_t n,
                             const float* b_hot, cudaStream_t st);
void free_hot_rows(HotRows* h);

// --- cluster-DSMEM hot-row cache (cluster.cu) ---
struct ClusterHot {
  uint32_t* col_ind = nullptr;   // remapped col_ind: hot columns = (1 << 31) | slot
  uint32_t* hot_list = nullptr;  // slot -> column
  uint32_t n_hot = 0;
  uint32_t* counter = nullptr;   // persistent row-unit counter
  int cs = 0;                    // cluster size (CTAs, one per SM)
  double hot_nnz_frac = 0.0;
};
uint32_t cluster_hot_rows(int cs);
cudaError_t build_cluster_hot(const uint32_t* col_ind, uint64_t nnz, uint32_t k, int cs,
                              cudaStream_t st, ClusterHot* out);
void free_cluster_hot(ClusterHot* h);
// N == 128, 16-byte aligned B/C; a.order/n_sched = every row (LPT order).
cudaError_t launch_cluster_warp(const ClusterHot& h, int op, bool fast, const SpmmArgs& a,
                                cudaStream_t st, int* clusters);

// --- packed column indices for the host entry's upload (h2dpack*.cpp/cu) ---
uint64_t pack_cols_block(const uint32_t* row_ptr, const uint32_t* col_ind, uint32_t lo,
                         uint32_t hi, uint16_t* enc, uint32_t* exc, uint64_t max_exc);
size_t unpack_temp_bytes(uint64_t max_len);
int pack_threads();
// host entry: the packing threads poll `streams` until they drain (idle host
// cores slow the tail copies on the boxes; h2dpack_host.cpp)
void host_poll(void* const* streams, int n);
// gespmm_release_workspace's halves (api.cu, coo.cu)
void release_coo_scratch();
// rows [0, m_block) of row_ptr_block own positions [ps, pe); bits: zeroed
// row-start bitmap over all nnz positions (shared with the column check).
// bad_key (nullable): also check the rebuilt columns (bounds k_cols, strictly
// increasing within rows) into the column check's first-violation key.
cudaError_t unpack_cols(const uint16_t* enc, const uint2* exc, uint32_t n_exc,
                        const uint32_t* row_ptr_block, uint32_t m_block, uint64_t ps, uint64_t pe,
                        uint64_t nnz, uint32_t* bits, uint32_t* col, void* temp, size_t temp_bytes,
                        cudaStream_t st, uint32_t k_cols = 0, unsigned long long* bad_key = nullptr);

// Device canonical check of a device CSR, formatted as the reference's
// require_canonical(m, who) error (csr.hpp:155-158).  Synchronises `st`.
gespmm_status_t validate_device_as(const gespmm_csr_t* a, cudaStream_t st, const char* who);

// --- validation (validate.cu) ---
struct ValidateResult {
  uint32_t row_ptr0;
  uint32_t row_ptr_last;
  uint32_t first_decrease;   // 0xffffffff if none
  uint64_t first_bad_key;    // 2*p + (0 oob | 1 not increasing); ~0 if none
  uint32_t bad_row;          // row containing that position
  uint32_t bad_col;          // col_ind at that position
};
cudaError_t validate_csr_device(uint32_t m, uint32_t k, uint64_t nnz, const uint32_t* row_ptr,
                                const uint32_t* col_ind, ValidateResult* out, cudaStream_t s);

// Chunked column check: begin, one call per row block (row_ptr_chunk points at
// the block's first row_ptr entry; positions stay global), end (locates the
// first violation's row, synchronises `st`).
struct ColCheck {  // views into the caller's workspace (no ownership)
  void* scratch = nullptr;   // first-violation minima (validate.cu)
  uint32_t* bits = nullptr;  // row-start bitmap over all nnz positions
};
unsigned long long* colcheck_key(ColCheck* c);  // its first-violation key (device)
size_t colcheck_workspace_bytes(uint64_t nnz);
cudaError_t colcheck_begin(ColCheck* out, uint64_t nnz, void* ws, cudaStream_t st);
// rows [0, m_chunk) of row_ptr_chunk own positions [ps, pe)
cudaError_t colcheck_rows(ColCheck* c, const uint32_t* row_ptr_chunk, uint32_t m_chunk,
                          uint64_t ps, uint64_t pe, const uint32_t* col_ind, uint32_t k,
                          uint64_t usable, cudaStream_t st);
cudaError_t colcheck_end(ColCheck* c, const uint32_t* row_ptr, const uint32_t* col_ind, uint32_t m,
                         uint64_t* first_bad_key, uint32_t* bad_row, uint32_t* bad_col,
                         cudaStream_t st);

}  // namespace gespmm
