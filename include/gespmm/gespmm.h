/*
 * gespmm.h — C ABI of the B200-native GE-SpMM library (libgespmm.so).
 *
 * This is the drop-in boundary for the reference's SpMM-like hot path
 * (arXiv 2007.03179 reference, /root/reference/proj/include/spmm/).  Plain
 * pointers and sizes only; no C++ or torch types cross it, no exception
 * crosses it.  Every entry point names the reference interface it replaces.
 * The C++ drop-in (namespace spmm, include/gespmm/native_spmm.hpp) and the
 * Python host mirror (paper_2007_03179_b200/) are thin layers over these calls.
 *
 * Experimental options (l2_persist, l2_hot_mb > 0, col_slices > 1,
 * cluster_hot, hot_rows_mb > 0) were measured slower on B200 and are compiled only into the
 * GESPMM_EXPERIMENTAL build (gespmm_build_flags() & GESPMM_BUILD_EXPERIMENTAL);
 * the default library rejects them with GESPMM_EUNSUPPORTED.
 *
 * Semantics (bit-exact contract):
 *   C[i][j] = fold_{p in row i, ascending} combine(acc, vals[p] * B[col_ind[p]][j])
 *   with the product and the combine rounded separately (no FMA) in the default
 *   exact mode.  sum: init +0, a+b.  max: init -FLT_MAX, (a < b ? b : a).
 *   min: init +FLT_MAX, (b < a ? b : a).  mean: sum / float(row length), empty
 *   row -> +0.  arg (max/min): CSR position p (or col_ind[p]) of the element that
 *   last replaced the accumulator (earliest p among ties), -1 if none.  arg is
 *   int32: a call with an arg whose indices cannot fit (nnz > 2^31 for CSR
 *   positions, n_cols > 2^31 for columns) is refused with GESPMM_EINVAL.
 */
#ifndef GESPMM_H_
#define GESPMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GESPMM_ABI_VERSION 2

/* Reduce ops.  Replaces spmm::ReduceOp / ops::sum / ops::max
 * (reference include/spmm/reduce_op.hpp:14-28): a host function pointer cannot
 * run on the device, so the op is named and fused into the kernel. */
typedef enum {
  GESPMM_SUM = 0,
  GESPMM_MEAN = 1,
  GESPMM_MAX = 2,
  GESPMM_MIN = 3
} gespmm_reduce_t;

typedef enum {
  GESPMM_OK = 0,
  GESPMM_EINVAL = 1,      /* bad argument / unknown op / bad config (spmm::Error) */
  GESPMM_EDIM = 2,        /* "dimension mismatch" (simt.hpp:373-380) */
  GESPMM_ENONCANON = 3,   /* "matrix is not canonical CSR" (csr.hpp:155-158) */
  GESPMM_ECUDA = 4,       /* CUDA runtime failure */
  GESPMM_ENOMEM = 5,      /* device allocation failed */
  GESPMM_EUNSUPPORTED = 6 /* valid request this build cannot serve */
} gespmm_status_t;

/* Kernel variants.  KernelVariant / KernelKind (kernel.hpp:44-68).
 * NAIVE/CRC/CRC_CWM are the paper's Algorithms 1-3 with the reference's warp
 * geometry (warp = (row, 32*cf column tile), lane owns col_base+lane+c*32);
 * TUNED is the B200 design (sub-warp rows, float4 lanes, CWM merge factor and
 * row-per-warp vs row-per-CTA chosen from N and the degree distribution).
 * All variants give bitwise-identical results in exact mode. */
typedef enum {
  GESPMM_VARIANT_TUNED = 0,
  GESPMM_VARIANT_NAIVE = 1,
  GESPMM_VARIANT_CRC = 2,
  GESPMM_VARIANT_CRC_CWM = 3
} gespmm_variant_t;

typedef enum { GESPMM_ARG_EDGE = 0, GESPMM_ARG_COLUMN = 1 } gespmm_arg_kind_t;

/* CSR view.  CsrMatrix (csr.hpp:22-35): u32 row_ptr[n_rows+1], u32 col_ind[nnz],
 * f32 vals[nnz].  For *_device calls the three pointers are device pointers. */
typedef struct {
  uint32_t n_rows;
  uint32_t n_cols;
  uint64_t nnz;
  const uint32_t* row_ptr;
  const uint32_t* col_ind;
  const float* vals;
} gespmm_csr_t;

/* Options; gespmm_options_default() fills the defaults. */
typedef struct {
  int32_t variant;    /* gespmm_variant_t, default TUNED */
  uint32_t cf;        /* CRC_CWM coarsening factor: 2, 4 or 8 (check_config, kernel.hpp:83-92) */
  int32_t exact;      /* 1 (default): ordered fold, separate mul/add -> bit-exact for all ops.
                         0: sum/mean use FFMA (1e-5 relative tolerance). */
  int32_t arg_kind;   /* gespmm_arg_kind_t, default EDGE (CSR position) */
  int32_t validate;   /* 1 (default for *_host): canonical-CSR check before the launch */
  int32_t fault_skip_tail; /* negative-test hook: FaultMode::SkipTail (kernel.hpp:167-182) */
  int32_t l2_hints;   /* 1 (default): B evict_last, CSR/C evict_first; 0: evict_normal
                         everywhere; 2: as 1 but B rows outside the hot-column map
                         evict_normal instead of evict_first */
  int32_t hub_threshold; /* TUNED: rows with degree >= this go row-per-CTA; 0 = auto, <0 = off */
  int32_t l2_persist; /* 1: launch with an L2 access-policy window marking B persisting
                         (sets the device's persisting-L2 limit to its maximum); 2: only raise
                         the persisting-L2 set-aside (evict_last lines of the hint policies
                         may use it), no window; default 0 */
  int32_t l2_hot_mb;  /* TUNED plans: frequency-aware L2 policy for B.  The plan counts the
                         gathers per column and only the most-gathered columns whose B rows
                         fit this many MB are loaded evict_last (the rest evict_first).
                         0 = auto (off: measured slower on B200), <0 = off.  Hints only:
                         results are unaffected. */
  int32_t tuned_cf;   /* TUNED plans: CWM merge factor (column sub-tiles per lane) of the
                         full-warp row kernel, 1, 2 or 4; 0 = auto from N */
  int32_t col_slices; /* TUNED plans: traverse the N columns as S slices, slice-major (every
                         row of slice 0, then slice 1, ...), so the live B working set is
                         B/S and stays in L2 when B does not.  Each output element is still
                         folded by one thread in CSR order: results are unchanged.
                         0 = auto (currently off: measured slower on B200), 1 = off,
                         S >= 2 explicit */
  int32_t rows_per_warp; /* TUNED plans: rows sharing a warp when N <= 256 (float4 lanes): 0 =
                         auto (4 for low-degree matrices, else as N dictates), 1, 2, 4 or 8 */
  int32_t cluster_hot; /* TUNED plans, N = 128: keep the most-gathered B rows in the distributed
                         shared memory of thread-block clusters of this many CTAs (2, 4, 8 or
                         16; one CTA per SM, 416 rows each) and gather them over DSMEM; the plan
                         keeps a remapped copy of col_ind (a SNAPSHOT: an explicit plan must be
                         rebuilt if col_ind changes; gespmm_spmm_device never caches such a
                         plan).  0 = off (default) */
  int32_t h2d_pack;   /* gespmm_spmm_host: send col_ind as 16-bit row-gap codes (lossless, escapes
                         for large gaps) and rebuild it on the device: 0 = auto (>= 8M nonzeros),
                         1 = on, -1 = off */
  int32_t hot_rows_mb; /* TUNED plans: relocate the most-gathered B rows (a byte budget of this
                         many MB) into a plan-owned contiguous copy, refreshed from B at every
                         execute, and gather them with evict_last while every other B row is
                         gathered evict_first, so L2 holds the static top-by-frequency set
                         instead of an LRU over B.  The plan keeps a remapped copy of col_ind (a
                         SNAPSHOT, like cluster_hot; gespmm_spmm_device never caches such a
                         plan).  Results are unchanged (positions and fold order are).
                         Edge args only.  Experimental (measured slower on B200: fewer DRAM
                         bytes, more instructions).  <=0 = off (default), >0 =
                         budget in MB */
  int32_t overlap_prev; /* TUNED plans whose execute is one kernel (no hub rows, one column
                         slice; gespmm_plan_launches == 1): launch it as a programmatic
                         dependent of the preceding kernel on the stream, so its CTAs start
                         while that kernel drains and read the row schedule, row_ptr and the
                         first staged (col_ind, vals) chunk before waiting for it
                         (griddepcontrol.wait precedes every B read and C/arg write).
                         Contract: the preceding kernel must not write A's arrays, and must
                         itself be a single-kernel plan execute or a plain kernel (not a
                         two-kernel hub execute).  For back-to-back SpMMs over a small graph
                         (stacked hops, CUDA-graph replay).  Default 0. */
} gespmm_options_t;

void gespmm_options_default(gespmm_options_t* opts);

/* Last error text of the calling thread, worded like the spmm::Error the
 * reference would raise for the same input. */
const char* gespmm_last_error(void);

/* ---- the hot path ------------------------------------------------------- */

/* Device SpMM-like: A (device CSR) x B (device, row-major K x n) -> C (device,
 * row-major M x n) [+ arg (device int32, M x n) for MAX/MIN; may be NULL].
 * Asynchronous on `stream` (cudaStream_t, NULL = legacy default).  Replaces the
 * compute of spmm::native_spmm (native.hpp:101-143) / run_warp
 * (kernel.hpp:346-361).  B and C must not alias.  validate=1 runs the
 * canonical check on the device first and synchronises `stream` to report it.
 * The library keeps a small per-(CSR, shape, op, options, device, stream) LRU
 * of plans behind this call; results never depend on a cached entry (A may
 * change between calls), but a CUDA graph that captures this call refers to
 * the cached plan's buffers, which a later eviction frees: capture an
 * explicit plan (gespmm_plan_execute) instead. */
gespmm_status_t gespmm_spmm_device(const gespmm_csr_t* a, const float* b, uint32_t n,
                                   gespmm_reduce_t op, float* c, int32_t* arg,
                                   const gespmm_options_t* opts, void* stream);

/* Host-buffer SpMM-like, the native_spmm-shaped call (native.hpp:101-102):
 * validates (as check_spmm_inputs, simt.hpp:373-380), copies A and B to the
 * device, runs, copies C (and arg) back.  b_rows must equal a->n_cols.
 * Host buffers may be pinned or pageable.  Synchronous. */
gespmm_status_t gespmm_spmm_host(const gespmm_csr_t* a, const float* b, uint32_t b_rows,
                                 uint32_t n, gespmm_reduce_t op, float* c, int32_t* arg,
                                 const gespmm_options_t* opts);

/* ---- plans: inspect once, execute many ---------------------------------- */

typedef struct gespmm_plan_s* gespmm_plan_t;

/* Inspect a device CSR (degree distribution) and fix the kernel shape for this
 * n/op: sub-warp vs warp vs CTA per row class, merge factor, row schedule.  The
 * plan keeps pointers to A's arrays, which must stay valid.  Synchronous.
 * The schedule only orders rows, so A's values and structure may change
 * between executes (same shape) with correct results — except in a plan that
 * splits hub rows (below), whose segment bounds are row_ptr values taken
 * here: recreate it when row_ptr changes (gespmm_spmm_device does this
 * itself for its cached plans). */
gespmm_status_t gespmm_plan_create(const gespmm_csr_t* a, uint32_t n, gespmm_reduce_t op,
                                   const gespmm_options_t* opts, void* stream,
                                   gespmm_plan_t* out);
/* Executions of one plan must not overlap on different streams (the plan owns
 * its side stream, events, work counters and, for split hub rows, the
 * partial-row buffer); use one plan per stream.  A plan whose op is max/min,
 * or sum/mean with exact = 0, splits rows at or above its hub threshold into
 * segments folded into partial rows and combines them in order (bit-exact for
 * max/min, arg included); exact sum/mean keep the row-per-CTA ring. */
gespmm_status_t gespmm_plan_execute(gespmm_plan_t plan, const float* b, float* c, int32_t* arg,
                                    void* stream);
/* Human-readable description of the chosen shape (static storage per plan). */
const char* gespmm_plan_describe(gespmm_plan_t plan);
/* Number of kernel launches one gespmm_plan_execute issues. */
int32_t gespmm_plan_launches(gespmm_plan_t plan);
void gespmm_plan_destroy(gespmm_plan_t plan);

/* ---- multi-GPU: fused all-gather epilogue over peer memory ---------------- */
/* Row-sharded stacked layers: each rank computes the rows
 * of its nnz-balanced shard and every rank needs all rows for the next layer.
 * Instead of a kernel followed by ncclAllGather, the SpMM's epilogue stores
 * each finished output row into every rank's full-height buffer directly —
 * peer-mapped device pointers (CUDA IPC / symmetric memory: NVLink P2P stores
 * through NVSwitch) and/or one NVLS multicast address (multimem.st, the
 * switch replicates the store) — so the exchange overlaps the gathers row by
 * row.  A cross-rank barrier (gespmm_peer_barrier) orders the next layer's
 * reads after every rank's stores.  Results are the plan's, bit for bit. */
#define GESPMM_MAX_GATHER_DSTS 8

/* Executes a TUNED plan with replicated outputs.  c_dsts[0] is the local C (as
 * gespmm_plan_execute's c); c_dsts[1..n_dsts) are replicas on other ranks,
 * each pointing at the element where THIS shard's row 0 lands (the caller adds
 * the shard's row offset * n).  arg_dsts: same for arg (NULL, or entries may
 * be NULL).  c_multicast / arg_multicast: multicast addresses of the same
 * landing element (NULL: unused); with a multicast address the replicas list
 * may hold only the local C.  1 <= n_dsts <= GESPMM_MAX_GATHER_DSTS.
 * Asynchronous; no ordering with other ranks (see gespmm_peer_barrier). */
gespmm_status_t gespmm_plan_execute_gather(gespmm_plan_t plan, const float* b,
                                           float* const* c_dsts, int32_t* const* arg_dsts,
                                           int32_t n_dsts, float* c_multicast,
                                           int32_t* arg_multicast, void* stream);

/* Cross-rank barrier on `stream` over peer-mapped signal words: signals[p] is
 * rank p's array of `world` u32 words as mapped in this process (signals[rank]
 * is the local one).  Rank r stores `epoch` to signals[p][r] for every p with
 * release semantics at system scope (after a system-scope fence, so every
 * store this rank made before it — the gather epilogue included — is visible
 * first), then waits until signals[r][p] == epoch for every p with acquire
 * loads.  epoch must differ from the previous barrier's (a counter).  A wait
 * longer than timeout_ms (0 = 60000) abandons the barrier and sets *error
 * (device int32, nullable) to 1 instead of hanging the device. */
gespmm_status_t gespmm_peer_barrier(uint32_t* const* signals, int32_t rank, int32_t world,
                                    uint32_t epoch, uint32_t timeout_ms, int32_t* error,
                                    void* stream);

/* Peer-shareable device buffers (cudaMalloc base pointers, so a CUDA IPC handle
 * maps exactly the buffer) and their IPC handles (64 opaque bytes). */
gespmm_status_t gespmm_peer_alloc(uint64_t bytes, void** out);
gespmm_status_t gespmm_peer_free(void* ptr);
gespmm_status_t gespmm_ipc_get_handle(void* ptr, unsigned char out[64]);
gespmm_status_t gespmm_ipc_open_handle(const unsigned char handle[64], void** out);
gespmm_status_t gespmm_ipc_close(void* ptr);

/* Single-process NVLS multicast buffer (this process's device bound to one
 * physical allocation): *uc_ptr is the ordinary (unicast) mapping, *mc_ptr the
 * multicast address for gespmm_plan_execute_gather's c_multicast.  On an
 * NVSwitch node the multi-process object comes from symmetric memory; this
 * validates the multicast epilogue on one device.  EUNSUPPORTED when the
 * device or driver has no multicast. */
gespmm_status_t gespmm_multicast_alloc(uint64_t bytes, void** uc_ptr, void** mc_ptr);
gespmm_status_t gespmm_multicast_free(void* uc_ptr);

/* ---- format helpers ------------------------------------------------------ */

/* A^T of a device CSR, as canonical CSR on the device: t_row_ptr[n_cols+1],
 * t_col_ind[nnz], t_vals[nnz] (caller-allocated).  Deterministic (stable radix
 * sort by column keeps rows ascending).  The device counterpart of the
 * reference's to_coo -> from_coo round trip (csr.hpp:58-104); feeds the GCN
 * backward SpMM.  Asynchronous on `stream`. */
gespmm_status_t gespmm_csr_transpose_device(const gespmm_csr_t* a, uint32_t* t_row_ptr,
                                            uint32_t* t_col_ind, float* t_vals, void* stream);

/* ---- CSR1 binary cache (io.hpp:15-16, 50-115) ----------------------------- */
/* Layout: "CSR1", u64 LE n_rows, n_cols, nnz, u32 row_ptr[n_rows+1],
 * u32 col_ind[nnz], f32 vals[nnz] (pinned by test_io.cpp:14-35).  Errors use
 * the reference's texts ("csr cache: bad magic (expected CSR1)", "csr cache:
 * truncated header|row_ptr|col_ind|vals", "csr cache: dimensions exceed 32-bit
 * range", "cannot open '<path>'"). */

/* write_csr_cache / save_csr_cache (io.hpp:50-63, 92-96); host CSR. */
gespmm_status_t gespmm_csr1_write(const char* path, const gespmm_csr_t* a);
/* Header + size checks of read_csr_cache (io.hpp:65-90), sizes out. */
gespmm_status_t gespmm_csr1_header(const char* path, uint32_t* n_rows, uint32_t* n_cols,
                                   uint64_t* nnz);
/* read_csr_cache into caller-allocated host arrays (sized from the header). */
gespmm_status_t gespmm_csr1_read_host(const char* path, uint32_t* row_ptr, uint32_t* col_ind,
                                      float* vals);
/* Streaming loader into caller-allocated DEVICE arrays (pinned double-buffered
 * pread -> H2D on `stream`); validate=1 then runs the canonical check on the
 * device with load_matrix's wording (io.hpp:100-115).  Synchronous. */
gespmm_status_t gespmm_csr1_load_device(const char* path, uint32_t* d_row_ptr,
                                        uint32_t* d_col_ind, float* d_vals, int32_t validate,
                                        void* stream);

/* ---- host data model: COO ingestion, full canonical report, Matrix Market -- */

/* from_coo (csr.hpp:37-93): (row, col)-ordered canonical CSR from COO triples;
 * duplicates collapse in input order — SUM: v = v + next, LAST: the final one.
 * row_ptr has n_rows + 1 entries; col_ind / out_vals have room for `count`;
 * *nnz receives the canonical length.  EINVAL with the reference's text
 * ("coo entry (r, c, v) outside declared RxC bounds") on a bad triple. */
typedef enum { GESPMM_DEDUP_SUM = 0, GESPMM_DEDUP_LAST = 1 } gespmm_dedup_t;
gespmm_status_t gespmm_from_coo(uint32_t n_rows, uint32_t n_cols, uint64_t count,
                                const uint32_t* rows, const uint32_t* cols, const float* vals,
                                int32_t policy, uint32_t* row_ptr, uint32_t* col_ind,
                                float* out_vals, uint64_t* nnz);

/* from_coo on DEVICE arrays (the same semantics, bit for bit): bounds check
 * (first offending triple in input order, the reference's message), stable
 * (row, col) order, duplicate runs folded in input order (Sum: v = v + next in
 * fp32; Last: the final occurrence).  row_ptr[n_rows+1], col_ind[count] and
 * out_vals[count] are caller-allocated device buffers (count is the capacity
 * bound); *nnz (host) receives the canonical length.  Synchronous with respect
 * to the host (it returns *nnz); ~20 B per triple of device temporaries. */
gespmm_status_t gespmm_from_coo_device(uint32_t n_rows, uint32_t n_cols, uint64_t count,
                                       const uint32_t* rows, const uint32_t* cols,
                                       const float* vals, int32_t policy, uint32_t* row_ptr,
                                       uint32_t* col_ind, float* out_vals, uint64_t* nnz,
                                       void* stream);
/* to_coo on device (csr.hpp:95-104): rows[nnz] expanded from row_ptr, cols and
 * vals copied; asynchronous on `stream`. */
gespmm_status_t gespmm_to_coo_device(const gespmm_csr_t* a, uint32_t* rows, uint32_t* cols,
                                     float* vals, void* stream);

/* validate (csr.hpp:107-153) on host arrays of the given lengths: returns the
 * number of violations and writes their messages, '\n'-separated, in the
 * reference's order and wording into msgs (truncated to msgs_cap; the full
 * size incl. the terminator in *msgs_needed). */
uint64_t gespmm_validate_host(const gespmm_csr_t* a, uint64_t row_ptr_len, uint64_t col_ind_len,
                              uint64_t vals_len, char* msgs, uint64_t msgs_cap,
                              uint64_t* msgs_needed);

/* parse_matrix_market (matrix_market.hpp:60-160): coordinate real / integer /
 * pattern, general / symmetric (mirrored off the diagonal), 1-based indices.
 * Two calls: rows == NULL sizes (*n_entries = stored triples), then with
 * arrays of *n_entries.  EINVAL with "matrix market: line L: ..." on error. */
gespmm_status_t gespmm_mtx_parse(const char* text, uint64_t len, uint32_t* n_rows,
                                 uint32_t* n_cols, uint64_t* n_entries, uint32_t* rows,
                                 uint32_t* cols, float* vals);

/* ---- checks and helpers -------------------------------------------------- */

/* Device canonical-CSR check (csr.hpp:112-153); status ENONCANON with the
 * reference's first-violation message in gespmm_last_error().  Synchronous. */
gespmm_status_t gespmm_validate_device(const gespmm_csr_t* a, void* stream);
/* Same check, message prefixed with `who` as require_canonical(m, who) does
 * (csr.hpp:155-158), e.g. "load_matrix". */
gespmm_status_t gespmm_validate_device_as(const gespmm_csr_t* a, void* stream, const char* who);

/* Reference dispatch rule, select_variant (kernel.hpp:96-98): n <= 32 -> CRC,
 * else CRC_CWM with cf 2. */
void gespmm_select_variant(uint32_t n, int32_t* variant, uint32_t* cf);

/* Name lookup, reduce_op_by_name (reduce_op.hpp:32-36), extended with mean/min. */
gespmm_status_t gespmm_reduce_by_name(const char* name, gespmm_reduce_t* out);

/* FNV-1a over the element bytes xor (rows<<32)^cols — checksum (dense.hpp:62-72). */
uint64_t gespmm_checksum(const float* host_data, uint32_t rows, uint32_t cols);

/* ---- synthetic inputs (host, deterministic) ------------------------------ */

/* make_random_dense (dense.hpp:51-59): mt19937_64(seed), x = (r>>40)*2^-23 - 1. */
void gespmm_make_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out);

/* randomize_values (generate.hpp:73-80): v = ((r>>44)+1)*2^-19, random sign. */
void gespmm_randomize_values(float* vals, uint64_t nnz, uint64_t seed);

/* gen_uniform_random (generate.hpp:39-69): exactly nnz distinct positions by
 * seeded rejection, values 1.0, canonicalised.  row_ptr[rows+1], col_ind[nnz],
 * vals[nnz] caller-allocated.  Bit-identical to the reference for equal specs. */
gespmm_status_t gespmm_gen_uniform(uint32_t rows, uint64_t nnz, uint64_t seed, int32_t self_loops,
                                   uint32_t* row_ptr, uint32_t* col_ind, float* vals);

/* Power-law (Chung-Lu style) square graph — new; the reference has none.
 * Degrees follow a truncated power law with the given mean and max degree;
 * columns are drawn from the same weights; rows are canonical (sorted,
 * unique, no self loops); values 1.0.  Deterministic for (rows, nnz, seed)
 * and independent of `threads`.  Two calls: with col_ind == NULL it only fills
 * row_ptr (so the caller can size col_ind/vals by row_ptr[rows]); then with
 * buffers.  The realised nnz is within 0.1% of nnz_target. */
gespmm_status_t gespmm_gen_powerlaw(uint32_t rows, uint64_t nnz_target, uint32_t max_degree,
                                    double exponent, uint64_t seed, int32_t threads,
                                    uint32_t* row_ptr, uint32_t* col_ind, float* vals);

/* Frees the library's grow-only scratch on the current device — the host
 * entry's staging buffers (pinned host + device, sized to the largest call so
 * far) and the COO builder's temporaries (~28 B per triple) — once no call is
 * in flight on it.  The next call reallocates what it needs. */
void gespmm_release_workspace(void);

/* Library / device facts for reports. */
int32_t gespmm_abi_version(void);
#define GESPMM_BUILD_EXPERIMENTAL 1
int32_t gespmm_build_flags(void); /* GESPMM_BUILD_* bits this library was compiled with */
gespmm_status_t gespmm_device_info(int32_t* sm_count, int64_t* l2_bytes,
                                   int64_t* persisting_l2_max, int32_t* cc_major,
                                   int32_t* cc_minor);

/* Diagnostics (roofline report, not the SpMM path): for each idx[i] read row
 * idx[i] of B (n must be 128) into a register accumulator — the gather ceiling
 * of an index stream.  sink must hold blocks*256 floats.  Asynchronous. */
gespmm_status_t gespmm_diag_gather(const uint32_t* idx, uint64_t count, const float* b,
                                   uint32_t n, float* sink, int32_t blocks, int32_t hints,
                                   void* stream);

/* Kernel launches issued by this library since load (all entry points). */
uint64_t gespmm_launch_count(void);

/* Diagnostics: as gespmm_diag_gather (n = 128) but rows idx < hub_rows (<= 400)
 * come from a shared-memory copy of B's first rows (persistent 1024-thread
 * CTAs, sink = blocks*1024 floats). */
gespmm_status_t gespmm_diag_gather_hub(const uint32_t* idx, uint64_t count, const float* b,
                                       uint32_t hub_rows, float* sink, int32_t blocks,
                                       void* stream);
/* Diagnostic: the gather ceiling under different B-row load paths (N = 128):
 * 0 LDG.128 L1-allocating, 1 LDG.128 L1::no_allocate, 2 cp.async.cg 16 B per
 * lane into shared memory, 3 cp.async.bulk 512-B rows into shared memory
 * (mbarrier complete_tx).  sink: blocks*256 floats. */
gespmm_status_t gespmm_diag_gather_mode(const uint32_t* idx, uint64_t count, const float* b,
                                        float* sink, int32_t blocks, int32_t mode, void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* GESPMM_H_ */
