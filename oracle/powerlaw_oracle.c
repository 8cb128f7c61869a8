/*
 * TEST INFRASTRUCTURE ONLY — a C restatement of the power-law CSR generator
 * the benchmark configs use (Reddit / ogbn-products shapes).
 *
 * The reference has no power-law generator (its only graph generator is
 * gen_uniform_random, proj/include/spmm/generate.hpp:39-69), so the generator
 * is specified by this repo (DESIGN.md §7 "inputs"): Chung-Lu rank weights
 * w_r = (r + c)^-exponent with c fitted so the largest expected degree is
 * max_degree, integer degrees by floors + largest remainders, a seeded
 * shuffle of node ids, and per-row column draws from a Vose alias table
 * (distinct, no self loops, sorted ascending, values 1.0 — the reference's
 * canonical CSR, csr.hpp:15-20, 58-93).
 *
 * This file exists so that bench.py's `--impl reference` arm (and the tests)
 * can build the benchmark matrices WITHOUT loading the product library: the
 * reference arm then runs on oracle/ and oracle/_ref code only.  Parity of
 * this restatement with the product's gespmm_gen_powerlaw (csrc/gen.cpp) is a
 * bit-for-bit test (tests/test_oracle.py::test_powerlaw_restatement_matches_product).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t pl_splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct {
  double frac;
  uint32_t idx;
} pl_frac_t;

/* descending remainder, ties by ascending index (= a stable sort) */
static int pl_frac_cmp(const void* x, const void* y) {
  const pl_frac_t* a = (const pl_frac_t*)x;
  const pl_frac_t* b = (const pl_frac_t*)y;
  if (a->frac > b->frac) return -1;
  if (a->frac < b->frac) return 1;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

static int pl_u32_cmp(const void* x, const void* y) {
  const uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return (a > b) - (a < b);
}

typedef struct {
  uint32_t rows, r0, r1;
  uint64_t seed;
  const uint32_t* row_ptr;
  const uint32_t* thresh;
  const uint32_t* alias;
  uint32_t* col_ind;
  float* vals;
} pl_job_t;

static void* pl_rows(void* p) {
  const pl_job_t* j = (const pl_job_t*)p;
  uint32_t* stamp = (uint32_t*)malloc(sizeof(uint32_t) * j->rows);
  if (!stamp) return (void*)1;
  memset(stamp, 0xff, sizeof(uint32_t) * j->rows);
  for (uint32_t row = j->r0; row < j->r1; ++row) {
    uint64_t s = (j->seed * 0x9E3779B97F4A7C15ull) ^ (((uint64_t)row + 1) * 0xD1B54A32D192ED03ull);
    const uint32_t d = j->row_ptr[row + 1] - j->row_ptr[row];
    uint32_t* out = j->col_ind + j->row_ptr[row];
    uint32_t got = 0;
    while (got < d) {
      const uint64_t u = pl_splitmix(&s);
      const uint32_t idx = (uint32_t)(((unsigned __int128)(u >> 32) * j->rows) >> 32);
      const uint32_t v = (uint32_t)u < j->thresh[idx] ? idx : j->alias[idx];
      if (v == row || stamp[v] == row) continue;
      stamp[v] = row;
      out[got++] = v;
    }
    qsort(out, d, sizeof(uint32_t), pl_u32_cmp);
    for (uint32_t p = j->row_ptr[row]; p < j->row_ptr[row + 1]; ++p) j->vals[p] = 1.0f;
  }
  free(stamp);
  return NULL;
}

/* Returns 0 on success, 1 on a bad argument, 2 on allocation failure.
 * col_ind == NULL: fill row_ptr only (sizing call). */
int oracle_gen_powerlaw(uint32_t rows, uint64_t nnz_target, uint32_t max_degree, double exponent,
                        uint64_t seed, int threads, uint32_t* row_ptr, uint32_t* col_ind,
                        float* vals) {
  if (rows < 2 || exponent <= 0.0) return 1;
  const double mean = (double)nnz_target / rows;
  if (max_degree > rows - 1) max_degree = rows - 1;
  if ((double)max_degree < mean || mean > (double)(rows - 1)) return 1;

  int rc = 2;
  double* w = (double*)malloc(sizeof(double) * rows);
  uint32_t* deg_rank = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  pl_frac_t* frac = (pl_frac_t*)malloc(sizeof(pl_frac_t) * rows);
  uint32_t* node_of_rank = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  uint32_t* rank_of = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  uint32_t* alias = NULL;
  uint32_t* thresh = NULL;
  double* p = NULL;
  uint32_t *small = NULL, *large = NULL;
  pl_job_t* jobs = NULL;
  pthread_t* tid = NULL;
  if (!w || !deg_rank || !frac || !node_of_rank || !rank_of) goto done;

  /* c: largest expected degree == max_degree (geometric bisection) */
  double lo = 1e-6, hi = 1e12;
  for (int it = 0; it < 200 && hi / lo > 1.0 + 1e-9; ++it) {
    const double mid = sqrt(lo * hi);
    double sum = 0.0;
    for (uint32_t r = 0; r < rows; ++r) sum += pow((double)r + mid, -exponent);
    const double top = (double)nnz_target * pow(mid, -exponent) / sum;
    if (top > (double)max_degree) lo = mid; else hi = mid;
  }
  const double c = sqrt(lo * hi);
  double sum = 0.0;
  for (uint32_t r = 0; r < rows; ++r) sum += (w[r] = pow((double)r + c, -exponent));
  const double scale = (double)nnz_target / sum;

  uint64_t assigned = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    double x = w[r] * scale;
    if (x > (double)(rows - 1)) x = (double)(rows - 1);
    deg_rank[r] = (uint32_t)floor(x);
    assigned += deg_rank[r];
    frac[r].frac = x - floor(x);
    frac[r].idx = r;
  }
  qsort(frac, rows, sizeof(pl_frac_t), pl_frac_cmp);
  for (uint32_t i = 0; assigned < nnz_target && i < rows; ++i) {
    if (deg_rank[frac[i].idx] < rows - 1) {
      ++deg_rank[frac[i].idx];
      ++assigned;
    }
  }

  for (uint32_t r = 0; r < rows; ++r) node_of_rank[r] = r;
  uint64_t ps = seed ^ 0x5851F42D4C957F2Dull;
  for (uint32_t i = rows - 1; i > 0; --i) {
    const uint32_t j = (uint32_t)(((unsigned __int128)pl_splitmix(&ps) * (i + 1)) >> 64);
    const uint32_t t = node_of_rank[i];
    node_of_rank[i] = node_of_rank[j];
    node_of_rank[j] = t;
  }
  for (uint32_t r = 0; r < rows; ++r) rank_of[node_of_rank[r]] = r;

  row_ptr[0] = 0;
  for (uint32_t v = 0; v < rows; ++v) row_ptr[v + 1] = row_ptr[v] + deg_rank[rank_of[v]];
  if (!col_ind) {
    rc = 0;
    goto done;
  }

  /* Vose alias table over node ids, integer thresholds */
  alias = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  thresh = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  p = (double*)malloc(sizeof(double) * rows);
  small = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  large = (uint32_t*)malloc(sizeof(uint32_t) * rows);
  if (!alias || !thresh || !p || !small || !large) goto done;
  uint32_t ns = 0, nl = 0;
  for (uint32_t v = 0; v < rows; ++v) p[v] = w[rank_of[v]] / sum * rows;
  for (uint32_t v = 0; v < rows; ++v) {
    if (p[v] < 1.0) small[ns++] = v; else large[nl++] = v;
  }
  while (ns && nl) {
    const uint32_t s = small[--ns], l = large[nl - 1];
    double t = floor(p[s] * 4294967296.0);
    thresh[s] = (uint32_t)(t < 4294967295.0 ? t : 4294967295.0);
    alias[s] = l;
    p[l] = (p[l] + p[s]) - 1.0;
    if (p[l] < 1.0) {
      --nl;
      small[ns++] = l;
    }
  }
  for (uint32_t i = 0; i < nl; ++i) {
    thresh[large[i]] = 0xffffffffu;
    alias[large[i]] = large[i];
  }
  for (uint32_t i = 0; i < ns; ++i) {
    thresh[small[i]] = 0xffffffffu;
    alias[small[i]] = small[i];
  }

  /* rows split by nnz over threads; every row has its own seed, so the
   * output does not depend on the split */
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  jobs = (pl_job_t*)calloc((size_t)threads, sizeof(pl_job_t));
  tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  if (!jobs || !tid) goto done;
  const uint64_t total = row_ptr[rows];
  uint32_t begin = 0;
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    const uint64_t target = total * (uint64_t)(t + 1) / (uint64_t)threads;
    uint32_t end = begin;
    if (t == threads - 1) end = rows;
    else
      while (end < rows && row_ptr[end] < target) ++end;
    pl_job_t* j = &jobs[started];
    j->rows = rows;
    j->r0 = begin;
    j->r1 = end;
    j->seed = seed;
    j->row_ptr = row_ptr;
    j->thresh = thresh;
    j->alias = alias;
    j->col_ind = col_ind;
    j->vals = vals;
    if (end > begin) {
      if (pthread_create(&tid[started], NULL, pl_rows, j) != 0) {
        rc = 2;
        for (int i = 0; i < started; ++i) pthread_join(tid[i], NULL);
        goto done;
      }
      ++started;
    }
    begin = end;
  }
  rc = 0;
  for (int i = 0; i < started; ++i) {
    void* r = NULL;
    pthread_join(tid[i], &r);
    if (r) rc = 2;
  }

done:
  free(w);
  free(deg_rank);
  free(frac);
  free(node_of_rank);
  free(rank_of);
  free(alias);
  free(thresh);
  free(p);
  free(small);
  free(large);
  free(jobs);
  free(tid);
  return rc;
}

/* ------------------------------------------------------------------------
 * Value and dense-operand generators, restated from the reference
 * (proj/include/spmm/dense.hpp:51-59 make_random_dense,
 *  proj/include/spmm/generate.hpp:73-80 randomize_values), both on
 * std::mt19937_64 — restated here as the standard MT19937-64 recurrence so
 * the reference arm can build its inputs with no product code loaded.
 * ------------------------------------------------------------------------ */

typedef struct {
  uint64_t mt[312];
  int i;
} pl_mt64_t;

static void pl_mt64_seed(pl_mt64_t* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}

static uint64_t pl_mt64_next(pl_mt64_t* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      const uint64_t x = (g->mt[k] & UM) | (g->mt[(k + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[k] = g->mt[(k + 156) % 312] ^ xa;
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* dense.hpp:51-59: x = (rng() >> 40) * 2^-23 - 1 */
void oracle_make_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
  pl_mt64_t g;
  pl_mt64_seed(&g, seed);
  const uint64_t total = (uint64_t)rows * cols;
  for (uint64_t i = 0; i < total; ++i) {
    const uint32_t bits = (uint32_t)(pl_mt64_next(&g) >> 40);
    out[i] = (float)bits * 0x1p-23f - 1.0f;
  }
}

/* generate.hpp:73-80: v = ((rng() >> 44) + 1) * 2^-19, negated when rng() is odd */
void oracle_randomize_values(float* vals, uint64_t nnz, uint64_t seed) {
  pl_mt64_t g;
  pl_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < nnz; ++i) {
    const uint32_t bits = (uint32_t)(pl_mt64_next(&g) >> 44) + 1u;
    float v = (float)bits * 0x1p-19f;
    if (pl_mt64_next(&g) & 1ull) v = -v;
    vals[i] = v;
  }
}
