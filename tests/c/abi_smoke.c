/* Plain-C use of the C ABI (include/gespmm/gespmm.h): compiles as C11 with
 * -Wall -Wextra -Werror (tests/test_c_abi.py, CPU suite), and, on a GPU box,
 * runs a host-buffer SpMM, a device plan with overlap_prev, the device COO
 * builder and the workspace release, checking results against a naive loop.
 * Exit code 0 = pass. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "gespmm/gespmm.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    gespmm_status_t s_ = (x);                                                 \
    if (s_ != GESPMM_OK) {                                                    \
      fprintf(stderr, "%s:%d: %s\n", __FILE__, __LINE__, gespmm_last_error()); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  enum { M = 64, K = 64, N = 32 };
  uint32_t row_ptr[M + 1], col_ind[M * 8];
  float vals[M * 8], b[K * N], c[M * N], want[M * N];
  uint32_t nnz = 0;
  for (uint32_t r = 0; r < M; ++r) {
    row_ptr[r] = nnz;
    for (uint32_t j = 0; j < 8; ++j) {
      col_ind[nnz] = (r * 7 + j * 5) % K;
      vals[nnz] = (float)((r + j) % 5) - 2.0f;
      ++nnz;
    }
    /* canonical rows: sort the 8 columns (they are distinct) */
    for (uint32_t i = row_ptr[r] + 1; i < nnz; ++i)
      for (uint32_t q = i; q > row_ptr[r] && col_ind[q - 1] > col_ind[q]; --q) {
        uint32_t t = col_ind[q]; col_ind[q] = col_ind[q - 1]; col_ind[q - 1] = t;
        float f = vals[q]; vals[q] = vals[q - 1]; vals[q - 1] = f;
      }
  }
  row_ptr[M] = nnz;
  for (uint32_t i = 0; i < K * N; ++i) b[i] = (float)(i % 13) * 0.25f - 1.0f;
  for (uint32_t r = 0; r < M; ++r)
    for (uint32_t j = 0; j < N; ++j) {
      float acc = 0.0f;
      for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) acc = acc + vals[p] * b[col_ind[p] * N + j];
      want[r * N + j] = acc;
    }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    printf("abi_smoke: no GPU, compile-only\n");
    return 0;
  }
  /* host buffers (native_spmm) */
  gespmm_csr_t a = {M, K, nnz, row_ptr, col_ind, vals};
  gespmm_options_t o;
  gespmm_options_default(&o);
  CHECK(gespmm_spmm_host(&a, b, K, N, GESPMM_SUM, c, NULL, &o));
  if (memcmp(c, want, sizeof c)) { fprintf(stderr, "host entry mismatch\n"); return 1; }
  /* device COO -> CSR, then a plan with overlap_prev, executed twice */
  uint32_t rows[M * 8];
  for (uint32_t r = 0; r < M; ++r)
    for (uint32_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) rows[p] = r;
  uint32_t *d_r, *d_c, *d_rp, *d_ci;
  float *d_v, *d_vo, *d_b, *d_out;
  cudaMalloc((void**)&d_r, sizeof rows); cudaMalloc((void**)&d_c, sizeof col_ind);
  cudaMalloc((void**)&d_v, sizeof vals); cudaMalloc((void**)&d_rp, sizeof row_ptr);
  cudaMalloc((void**)&d_ci, sizeof col_ind); cudaMalloc((void**)&d_vo, sizeof vals);
  cudaMalloc((void**)&d_b, sizeof b); cudaMalloc((void**)&d_out, sizeof c);
  cudaMemcpy(d_r, rows, sizeof rows, cudaMemcpyHostToDevice);
  cudaMemcpy(d_c, col_ind, sizeof col_ind, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, vals, sizeof vals, cudaMemcpyHostToDevice);
  cudaMemcpy(d_b, b, sizeof b, cudaMemcpyHostToDevice);
  uint64_t got_nnz = 0;
  CHECK(gespmm_from_coo_device(M, K, nnz, d_r, d_c, d_v, GESPMM_DEDUP_SUM, d_rp, d_ci, d_vo,
                               &got_nnz, NULL));
  if (got_nnz != nnz) { fprintf(stderr, "from_coo nnz %llu\n", (unsigned long long)got_nnz); return 1; }
  gespmm_csr_t da = {M, K, nnz, d_rp, d_ci, d_vo};
  o.overlap_prev = 1;
  gespmm_plan_t plan;
  CHECK(gespmm_plan_create(&da, N, GESPMM_SUM, &o, NULL, &plan));
  CHECK(gespmm_plan_execute(plan, d_b, d_out, NULL, NULL));
  CHECK(gespmm_plan_execute(plan, d_b, d_out, NULL, NULL));
  cudaMemcpy(c, d_out, sizeof c, cudaMemcpyDeviceToHost);
  gespmm_plan_destroy(plan);
  if (memcmp(c, want, sizeof c)) { fprintf(stderr, "device plan mismatch\n"); return 1; }
  gespmm_release_workspace();
  printf("abi_smoke: ok (%d kernel launches)\n", (int)gespmm_launch_count());
  return 0;
}
