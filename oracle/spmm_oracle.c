/*
 * TEST INFRASTRUCTURE ONLY — the CPU restatement ("oracle") of the
 * GE-SpMM SpMM-like fold.  Loaded by tests/, bench.py's cpu_baseline leg and
 * __graft_entry__.smoke() as the CHECKER; never linked into or called by the
 * product path (paper_2007_03179_b200/ fails loudly without its CUDA library).
 *
 * Parity pin: for sum and max this restatement is checked bit-for-bit
 * against the reference itself (oracle/_ref/libspmmref.so, built from the
 * unmodified headers under /root/reference) and against the committed
 * fixtures in tests/golden/ (made by tests/golden/make_golden.py from the
 * reference).  mean / min / arg indices have no reference implementation;
 * their semantics are pinned here as an extension of the reference's fold
 * contract and documented in DESIGN.md §3.
 *
 * Fold contract followed (reference files under /root/reference/proj):
 *   - one accumulator per output element, seeded with op.init, folded in
 *     ascending CSR position p with acc = combine(acc, v[p] * B[k][j])
 *     (include/spmm/kernel.hpp:197-224 naive, :234-278 crc, :287-343 cwm;
 *      include/spmm/oracle.hpp:37-41 ascending-k contract);
 *   - product and combine rounded separately, no FMA
 *     (CMakeLists.txt:10-12 -ffp-contract=off; this file is built the same);
 *   - sum: init +0.0f, a + b; max: init -FLT_MAX, (a < b ? b : a)
 *     (include/spmm/reduce_op.hpp:24-28);
 *   - SkipTail fault drops the last 32-wide sparse tile of every row
 *     (include/spmm/kernel.hpp:167-182, faulted_row_end).
 * Extensions (new semantics, documented in DESIGN.md):
 *   - min: init +FLT_MAX, (b < a ? b : a) — the mirror of max_f32;
 *   - mean: the sum fold divided (IEEE, round-to-nearest) by float(row length);
 *     an empty row stays at the sum seed +0.0f;
 *   - arg (max/min only): the CSR position p (or col_ind[p]) of the element
 *     that last replaced the accumulator — with the strict compare that is
 *     the earliest p among ties; -1 when the accumulator was never replaced.
 */
#include <float.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { OR_SUM = 0, OR_MEAN = 1, OR_MAX = 2, OR_MIN = 3 };
enum { OR_ARG_EDGE = 0, OR_ARG_COLUMN = 1 };

typedef struct {
  uint32_t m, n;
  const uint32_t* row_ptr;
  const uint32_t* col_ind;
  const float* vals;
  const float* b;
  int op, arg_kind, skip_tail;
  float* c;
  int32_t* arg;
  uint32_t row_begin, row_end;
} job_t;

/* reference include/spmm/kernel.hpp:174-180 (faulted_row_end, ws = 32) */
static uint32_t tail_end(uint32_t start, uint32_t end, int skip_tail) {
  if (!skip_tail || end <= start) return end;
  uint32_t tiles = (end - start + 31u) / 32u;
  return start + (tiles - 1u) * 32u;
}

static void fold_rows(const job_t* j) {
  const uint64_t n = j->n;
  for (uint32_t r = j->row_begin; r < j->row_end; ++r) {
    const uint32_t start = j->row_ptr[r];
    const uint32_t full_end = j->row_ptr[r + 1];
    const uint32_t end = tail_end(start, full_end, j->skip_tail);
    float* crow = j->c + (uint64_t)r * n;
    int32_t* arow = j->arg ? j->arg + (uint64_t)r * n : NULL;
    for (uint64_t col = 0; col < n; ++col) {
      float acc;
      int32_t who = -1;
      if (j->op == OR_MAX)
        acc = -FLT_MAX;
      else if (j->op == OR_MIN)
        acc = FLT_MAX;
      else
        acc = 0.0f;
      for (uint32_t p = start; p < end; ++p) {
        const uint32_t k = j->col_ind[p];
        const float x = j->vals[p] * j->b[(uint64_t)k * n + col]; /* rounded product */
        switch (j->op) {
          case OR_SUM:
          case OR_MEAN:
            acc = acc + x;
            break;
          case OR_MAX:
            if (acc < x) {
              acc = x;
              who = j->arg_kind == OR_ARG_COLUMN ? (int32_t)k : (int32_t)p;
            }
            break;
          default: /* OR_MIN */
            if (x < acc) {
              acc = x;
              who = j->arg_kind == OR_ARG_COLUMN ? (int32_t)k : (int32_t)p;
            }
            break;
        }
      }
      if (j->op == OR_MEAN && full_end > start) acc = acc / (float)(full_end - start);
      crow[col] = acc;
      if (arow) arow[col] = who;
    }
  }
}

static void* run_job(void* p) {
  fold_rows((const job_t*)p);
  return NULL;
}

/* Returns 0 on success, 1 on a bad argument. `threads` only splits rows;
 * every output element is still folded by one thread in ascending p, so the
 * result does not depend on it. */
int oracle_spmm(uint32_t m, uint32_t k, const uint32_t* row_ptr, const uint32_t* col_ind,
                const float* vals, const float* b, uint32_t n, int op, int arg_kind,
                int skip_tail, int threads, float* c, int32_t* arg) {
  (void)k;
  if (op < OR_SUM || op > OR_MIN) return 1;
  if (arg && op != OR_MAX && op != OR_MIN) return 1;
  if (m == 0 || n == 0) return 0;
  if (threads < 1) threads = 1;
  if ((uint32_t)threads > m) threads = (int)m;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!jobs || !tid) {
    free(jobs);
    free(tid);
    return 1;
  }
  /* split by nnz so power-law rows do not serialise on one thread */
  const uint64_t nnz = row_ptr[m];
  uint32_t row = 0;
  for (int t = 0; t < threads; ++t) {
    job_t* j = &jobs[t];
    j->m = m;
    j->n = n;
    j->row_ptr = row_ptr;
    j->col_ind = col_ind;
    j->vals = vals;
    j->b = b;
    j->op = op;
    j->arg_kind = arg_kind;
    j->skip_tail = skip_tail;
    j->c = c;
    j->arg = arg;
    j->row_begin = row;
    uint64_t target = nnz * (uint64_t)(t + 1) / (uint64_t)threads;
    uint32_t e = row;
    if (t == threads - 1) {
      e = m;
    } else {
      while (e < m && row_ptr[e] < target) ++e;
    }
    j->row_end = e;
    row = e;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  fold_rows(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  free(jobs);
  free(tid);
  return 0;
}

/* FNV-1a over the element bytes, then xor (rows << 32) ^ cols
 * (reference include/spmm/dense.hpp:62-72). */
uint64_t oracle_checksum(uint32_t rows, uint32_t cols, const void* data) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* p = (const unsigned char*)data;
  const size_t bytes = (size_t)rows * cols * 4u;
  for (size_t i = 0; i < bytes; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  h ^= ((uint64_t)rows << 32) ^ (uint64_t)cols;
  return h;
}

/* Canonical-CSR check; returns the number of violations and writes the first
 * message, worded and ordered as reference include/spmm/csr.hpp:112-153. */
int oracle_validate(uint32_t m, uint32_t k, const uint32_t* row_ptr, uint64_t rp_len,
                    const uint32_t* col_ind, uint64_t ci_len, uint64_t v_len, char* msg,
                    uint32_t msg_len) {
  int count = 0;
#define OR_FAIL(...)                                              \
  do {                                                            \
    if (count == 0 && msg && msg_len) snprintf(msg, msg_len, __VA_ARGS__); \
    ++count;                                                      \
  } while (0)
  if (rp_len != (uint64_t)m + 1) {
    OR_FAIL("row_ptr length is %llu, expected n_rows+1 = %u", (unsigned long long)rp_len,
            m + 1);
    return count;
  }
  if (ci_len != v_len)
    OR_FAIL("col_ind length %llu != vals length %llu", (unsigned long long)ci_len,
            (unsigned long long)v_len);
  if (row_ptr[0] != 0) OR_FAIL("row_ptr[0] = %u, expected 0", row_ptr[0]);
  for (uint64_t i = 1; i < rp_len; ++i) {
    if (row_ptr[i] < row_ptr[i - 1]) {
      OR_FAIL("row_ptr non-decreasing violated at index %llu", (unsigned long long)i);
      return count;
    }
  }
  if ((uint64_t)row_ptr[m] != ci_len)
    OR_FAIL("row_ptr[n_rows] = %u != nnz = %llu", row_ptr[m], (unsigned long long)ci_len);
  const uint64_t usable = row_ptr[m] < ci_len ? row_ptr[m] : ci_len;
  for (uint32_t r = 0; r < m; ++r) {
    uint32_t prev = 0;
    int first = 1;
    for (uint64_t p = row_ptr[r]; p < row_ptr[r + 1] && p < usable; ++p) {
      const uint32_t c = col_ind[p];
      if (c >= k)
        OR_FAIL("col_ind[%llu] = %u out of bounds (n_cols = %u)", (unsigned long long)p, c, k);
      if (!first && c <= prev)
        OR_FAIL("columns not strictly increasing in row %u at position %llu", r,
                (unsigned long long)p);
      prev = c;
      first = 0;
    }
  }
#undef OR_FAIL
  return count;
}
