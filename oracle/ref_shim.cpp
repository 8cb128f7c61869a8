// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/spmm/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libspmmref.so.  Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() load it,
// as the checker or the CPU baseline.  Nothing from the reference is copied
// here: every call below goes straight into the reference's own functions.
//
// Reference entry points wrapped (file:line under /root/reference/proj):
//   spmm::native_spmm        include/spmm/native.hpp:101-143
//   spmm::bench              include/spmm/native.hpp:156-180 (also per session)
//   spmm::dense_reference    include/spmm/oracle.hpp:42-57
//   spmm::gen_uniform_random include/spmm/generate.hpp:39-69
//   spmm::randomize_values   include/spmm/generate.hpp:73-80
//   spmm::make_random_dense  include/spmm/dense.hpp:51-59
//   spmm::checksum           include/spmm/dense.hpp:62-72
//   spmm::validate           include/spmm/csr.hpp:112-153
//   spmm::select_variant     include/spmm/kernel.hpp:96-98
//   spmm::from_coo           include/spmm/csr.hpp:58-93
//   spmm::run_kernel         include/spmm/simt.hpp:382-432 (SIMT simulator metrics)
//   spmm::save_csr_cache     include/spmm/io.hpp:92-96
//   spmm::load_matrix        include/spmm/io.hpp:100-115
#include "spmm/spmm.hpp"

#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

using namespace spmm;

namespace {

void put_err(char* buf, unsigned len, const char* msg) {
  if (buf && len) {
    std::snprintf(buf, len, "%s", msg);
  }
}

CsrMatrix make_csr(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
                   const unsigned* col_ind, const float* vals) {
  CsrMatrix a(m, k);
  a.row_ptr.assign(row_ptr, row_ptr + m + 1);
  a.col_ind.assign(col_ind, col_ind + nnz);
  a.vals.assign(vals, vals + nnz);
  return a;
}

DenseMatrix make_dense(unsigned rows, unsigned cols, const float* data) {
  DenseMatrix d(rows, cols);
  if (rows && cols) std::memcpy(d.data.data(), data, sizeof(float) * size_t(rows) * cols);
  return d;
}

KernelVariant variant_of(int kind, unsigned cf) {
  switch (kind) {
    case 0: return KernelVariant::naive();
    case 1: return KernelVariant::crc();
    default: return KernelVariant::crc_cwm(cf);
  }
}

}  // namespace

extern "C" {

// kind: 0 naive, 1 crc, 2 crc-cwm; op_name: "sum" / "max" (anything else
// goes through reduce_op_by_name and raises the reference's error).
int ref_native_spmm(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
                    const unsigned* col_ind, const float* vals, const float* b, unsigned n,
                    const char* op_name, int kind, unsigned cf, unsigned workers, int skip_tail,
                    float* c_out, char* err, unsigned err_len) {
  try {
    const CsrMatrix a = make_csr(m, k, nnz, row_ptr, col_ind, vals);
    const DenseMatrix bd = make_dense(k, n, b);
    ExecOptions ex;
    ex.fault = skip_tail ? FaultMode::SkipTail : FaultMode::None;
    const DenseMatrix c =
        native_spmm(a, bd, variant_of(kind, cf), reduce_op_by_name(op_name), workers, ex);
    if (!c.data.empty()) std::memcpy(c_out, c.data.data(), sizeof(float) * c.data.size());
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// Same inputs, B given with its own row count so dimension errors surface.
int ref_native_spmm_shape(unsigned m, unsigned k, unsigned long long nnz,
                          const unsigned* row_ptr, unsigned rp_len, const unsigned* col_ind,
                          unsigned long long ci_len, const float* vals,
                          unsigned long long v_len, const float* b, unsigned b_rows,
                          unsigned n, const char* op_name, char* err, unsigned err_len) {
  try {
    CsrMatrix a(m, k);
    a.row_ptr.assign(row_ptr, row_ptr + rp_len);
    a.col_ind.assign(col_ind, col_ind + ci_len);
    a.vals.assign(vals, vals + v_len);
    (void)nnz;
    const DenseMatrix bd = make_dense(b_rows, n, b);
    (void)native_spmm(a, bd, select_variant(n == 0 ? 1 : n), reduce_op_by_name(op_name), 1);
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

int ref_bench(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
              const unsigned* col_ind, const float* vals, const float* b, unsigned n,
              const char* op_name, int kind, unsigned cf, unsigned workers, unsigned repeats,
              double* median_s, double* mean_s, double* gflops, unsigned long long* csum,
              char* err, unsigned err_len) {
  try {
    const CsrMatrix a = make_csr(m, k, nnz, row_ptr, col_ind, vals);
    const DenseMatrix bd = make_dense(k, n, b);
    const ThroughputReport r =
        bench(a, bd, variant_of(kind, cf), reduce_op_by_name(op_name), workers, repeats);
    *median_s = r.elapsed_s;
    *mean_s = r.elapsed_mean_s;
    *gflops = r.gflops;
    *csum = r.output_checksum;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

int ref_dense_reference(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
                        const unsigned* col_ind, const float* vals, const float* b, unsigned n,
                        const char* op_name, float* c_out, char* err, unsigned err_len) {
  try {
    const CsrMatrix a = make_csr(m, k, nnz, row_ptr, col_ind, vals);
    const DenseMatrix bd = make_dense(k, n, b);
    const DenseMatrix c = dense_reference(a, bd, reduce_op_by_name(op_name));
    if (!c.data.empty()) std::memcpy(c_out, c.data.data(), sizeof(float) * c.data.size());
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// Two-call protocol is unnecessary: gen_uniform_random emits exactly nnz
// entries, so the caller sizes col_ind/vals to nnz and row_ptr to rows+1.
int ref_gen_uniform(unsigned rows, unsigned long long nnz, unsigned long long seed, int loops,
                    unsigned* row_ptr, unsigned* col_ind, float* vals, char* err,
                    unsigned err_len) {
  try {
    const CsrMatrix a = gen_uniform_random({rows, nnz, seed, loops != 0});
    std::memcpy(row_ptr, a.row_ptr.data(), sizeof(unsigned) * a.row_ptr.size());
    if (a.nnz()) {
      std::memcpy(col_ind, a.col_ind.data(), sizeof(unsigned) * a.nnz());
      std::memcpy(vals, a.vals.data(), sizeof(float) * a.nnz());
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

void ref_randomize_values(float* vals, unsigned long long nnz, unsigned long long seed) {
  CsrMatrix a;
  a.vals.assign(vals, vals + nnz);
  randomize_values(a, seed);
  if (nnz) std::memcpy(vals, a.vals.data(), sizeof(float) * nnz);
}

void ref_make_random_dense(unsigned rows, unsigned cols, unsigned long long seed, float* out) {
  const DenseMatrix d = make_random_dense(rows, cols, seed);
  if (!d.data.empty()) std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
}

unsigned long long ref_checksum(unsigned rows, unsigned cols, const float* data) {
  return checksum(make_dense(rows, cols, data));
}

// Returns the number of violations; copies the first message
// (prefixed exactly as require_canonical would raise it).
int ref_validate(unsigned m, unsigned k, const unsigned* row_ptr, unsigned rp_len,
                 const unsigned* col_ind, unsigned long long ci_len, const float* vals,
                 unsigned long long v_len, char* msg, unsigned msg_len) {
  CsrMatrix a(m, k);
  a.row_ptr.assign(row_ptr, row_ptr + rp_len);
  a.col_ind.assign(col_ind, col_ind + ci_len);
  a.vals.assign(vals, vals + v_len);
  const ValidationReport rep = validate(a);
  if (!rep.ok()) put_err(msg, msg_len, rep.violations.front().c_str());
  return int(rep.violations.size());
}

void ref_select_variant(unsigned n, int* kind, unsigned* cf) {
  const KernelVariant v = select_variant(n);
  *kind = v.kind == KernelKind::Naive ? 0 : v.kind == KernelKind::Crc ? 1 : 2;
  *cf = v.cf;
}

// COO -> canonical CSR (policy 0 = DedupPolicy::Sum, 1 = Last); out arrays
// sized to the COO length, returns the canonical nnz or -1 on error.
long long ref_from_coo(unsigned rows, unsigned cols, unsigned long long count, const unsigned* r,
                       const unsigned* c, const float* v, unsigned* row_ptr, unsigned* col_ind,
                       float* vals, char* err, unsigned err_len, int policy) {
  try {
    CooEntries coo;
    coo.n_rows = rows;
    coo.n_cols = cols;
    coo.entries.reserve(count);
    for (unsigned long long i = 0; i < count; ++i) coo.entries.push_back({r[i], c[i], v[i]});
    const CsrMatrix a = from_coo(coo, policy ? DedupPolicy::Last : DedupPolicy::Sum);
    std::memcpy(row_ptr, a.row_ptr.data(), sizeof(unsigned) * a.row_ptr.size());
    if (a.nnz()) {
      std::memcpy(col_ind, a.col_ind.data(), sizeof(unsigned) * a.nnz());
      std::memcpy(vals, a.vals.data(), sizeof(float) * a.nnz());
    }
    return a.nnz();
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return -1;
  }
}

// The reference's SIMT simulator (32-byte segment coalescer): out[0..5] =
// gld_transactions, gst_transactions, requested_load_bytes,
// transferred_load_bytes, requested_store_bytes, transferred_store_bytes;
// out[6..10] = load transactions per array (RowPtr, ColInd, Val, B, C);
// out[11..12] = shared loads / stores.
int ref_sim_metrics(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
                    const unsigned* col_ind, const float* vals, const float* b, unsigned n,
                    const char* op_name, int kind, unsigned cf, unsigned long long* out,
                    char* err, unsigned err_len) {
  try {
    const CsrMatrix a = make_csr(m, k, nnz, row_ptr, col_ind, vals);
    const DenseMatrix bd = make_dense(k, n, b);
    KernelConfig cfg;
    cfg.variant = variant_of(kind, cf);
    SimOptions so;
    so.parallel = true;
    const SimResult r = run_kernel(a, bd, cfg, reduce_op_by_name(op_name), so);
    const SimMetrics& s = r.metrics;
    out[0] = s.gld_transactions;
    out[1] = s.gst_transactions;
    out[2] = s.requested_load_bytes;
    out[3] = s.transferred_load_bytes;
    out[4] = s.requested_store_bytes;
    out[5] = s.transferred_store_bytes;
    for (int i = 0; i < kArrayCount; ++i) out[6 + i] = s.load_by_array[i].transactions;
    out[11] = s.shared_loads;
    out[12] = s.shared_stores;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

int ref_save_csr_cache(const char* path, unsigned m, unsigned k, unsigned long long nnz,
                       const unsigned* row_ptr, const unsigned* col_ind, const float* vals,
                       char* err, unsigned err_len) {
  try {
    save_csr_cache(path, make_csr(m, k, nnz, row_ptr, col_ind, vals));
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// load_matrix: sizes out first (arrays may be null), then a second call with
// buffers sized from them.  Returns 1 with the reference's message on error.
int ref_load_matrix(const char* path, unsigned* m, unsigned* k, unsigned long long* nnz,
                    unsigned* row_ptr, unsigned* col_ind, float* vals, char* err,
                    unsigned err_len) {
  try {
    const CsrMatrix a = load_matrix(path);
    *m = a.n_rows;
    *k = a.n_cols;
    *nnz = a.nnz();
    if (row_ptr) {
      std::memcpy(row_ptr, a.row_ptr.data(), sizeof(unsigned) * a.row_ptr.size());
      if (a.nnz()) {
        std::memcpy(col_ind, a.col_ind.data(), sizeof(unsigned) * a.nnz());
        std::memcpy(vals, a.vals.data(), sizeof(float) * a.nnz());
      }
    }
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

// A bench session: the CsrMatrix and B built ONCE (outside any timed window),
// then spmm::bench (native.hpp:156-180) per call — the reference's own timing
// window around native_spmm.  bench.py's --impl reference arm times each step
// with ref_session_bench(repeats = 1), so no shim copy is ever inside a step.
struct RefSession {
  CsrMatrix a;
  DenseMatrix b;
};

void* ref_session_new(unsigned m, unsigned k, unsigned long long nnz, const unsigned* row_ptr,
                      const unsigned* col_ind, const float* vals, const float* b, unsigned n,
                      char* err, unsigned err_len) {
  try {
    return new RefSession{make_csr(m, k, nnz, row_ptr, col_ind, vals), make_dense(k, n, b)};
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return nullptr;
  }
}

int ref_session_bench(void* h, const char* op_name, int kind, unsigned cf, unsigned workers,
                      unsigned repeats, double* median_s, double* mean_s, double* gflops,
                      unsigned long long* csum, char* err, unsigned err_len) {
  try {
    const RefSession* s = static_cast<const RefSession*>(h);
    const ThroughputReport r =
        bench(s->a, s->b, variant_of(kind, cf), reduce_op_by_name(op_name), workers, repeats);
    *median_s = r.elapsed_s;
    *mean_s = r.elapsed_mean_s;
    *gflops = r.gflops;
    *csum = r.output_checksum;
    return 0;
  } catch (const std::exception& e) {
    put_err(err, err_len, e.what());
    return 1;
  }
}

void ref_session_free(void* h) { delete static_cast<RefSession*>(h); }

unsigned ref_hardware_concurrency() { return std::max(1u, std::thread::hardware_concurrency()); }

}  // extern "C"
