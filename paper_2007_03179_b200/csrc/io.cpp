// CSR1 binary cache (C ABI, see gespmm.h): host write/read and a streaming
// loader straight into device memory.
//
// Format (reference /root/reference/proj/include/spmm/io.hpp:15-16, byte layout
// pinned by proj/tests/test_io.cpp:14-35): magic "CSR1", little-endian u64
// n_rows, n_cols, nnz, then u32 row_ptr[n_rows+1], u32 col_ind[nnz], f32
// vals[nnz].  The payload after the 28-byte header is three raw arrays, so on a
// little-endian host the loader never decodes anything: it streams file bytes
// through two pinned staging buffers into the three device arrays (pread of
// chunk i+1 overlaps the H2D of chunk i) and then runs the device canonical
// check with the reference's load_matrix wording (io.hpp:100-115).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>

#include "gespmm/gespmm.h"
#include "launch.h"

using namespace gespmm;

namespace {

static_assert(sizeof(float) == 4 && sizeof(uint32_t) == 4, "CSR1 element width");

constexpr uint64_t kHeader = 28;

bool little_endian() {
  const uint32_t one = 1;
  unsigned char b;
  std::memcpy(&b, &one, 1);
  return b == 1;
}

uint64_t get_u64_le(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

void put_u64_le(unsigned char* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Reads exactly len bytes at off; returns bytes read (short on EOF).
uint64_t pread_full(int fd, void* dst, uint64_t len, uint64_t off) {
  uint64_t got = 0;
  while (got < len) {
    const ssize_t r = ::pread(fd, static_cast<char*>(dst) + got, size_t(len - got), off_t(off + got));
    if (r < 0) {
      if (errno == EINTR) continue;
      break;
    }
    if (r == 0) break;
    got += uint64_t(r);
  }
  return got;
}

// Header + size checks in the order the reference reads (io.hpp:65-90): magic,
// header, 32-bit range, then which array the file ends inside.
gespmm_status_t open_and_check(const char* path, Fd& f, uint32_t* rows, uint32_t* cols,
                               uint64_t* nnz) {
  if (!path) return set_error(GESPMM_EINVAL, "csr cache: null path");
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return set_error(GESPMM_EINVAL, std::string("cannot open '") + path + "'");
  struct stat st;
  if (::fstat(f.fd, &st) != 0) return set_error(GESPMM_EINVAL, std::string("cannot open '") + path + "'");
  const uint64_t size = uint64_t(st.st_size);
  unsigned char h[kHeader];
  const uint64_t got = pread_full(f.fd, h, kHeader, 0);
  if (got < 4 || std::memcmp(h, "CSR1", 4) != 0)
    return set_error(GESPMM_EINVAL, "csr cache: bad magic (expected CSR1)");
  if (got < kHeader) return set_error(GESPMM_EINVAL, "csr cache: truncated header");
  const uint64_t r = get_u64_le(h + 4), c = get_u64_le(h + 12), z = get_u64_le(h + 20);
  if (r > 0xffffffffull || c > 0xffffffffull || z > 0xffffffffull)
    return set_error(GESPMM_EINVAL, "csr cache: dimensions exceed 32-bit range");
  const uint64_t end_rp = kHeader + 4 * (r + 1), end_ci = end_rp + 4 * z, end_v = end_ci + 4 * z;
  if (size < end_rp) return set_error(GESPMM_EINVAL, "csr cache: truncated row_ptr");
  if (size < end_ci) return set_error(GESPMM_EINVAL, "csr cache: truncated col_ind");
  if (size < end_v) return set_error(GESPMM_EINVAL, "csr cache: truncated vals");
  *rows = uint32_t(r);
  *cols = uint32_t(c);
  *nnz = z;
  return GESPMM_OK;
}

}  // namespace

extern "C" {

gespmm_status_t gespmm_csr1_write(const char* path, const gespmm_csr_t* a) {
  if (!path || !a) return set_error(GESPMM_EINVAL, "csr cache: null argument");
  if (!little_endian()) return set_error(GESPMM_EUNSUPPORTED, "csr cache: big-endian host");
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return set_error(GESPMM_EINVAL, std::string("cannot open '") + path + "' for writing");
  unsigned char h[kHeader];
  std::memcpy(h, "CSR1", 4);
  put_u64_le(h + 4, a->n_rows);
  put_u64_le(h + 12, a->n_cols);
  put_u64_le(h + 20, a->nnz);
  bool ok = std::fwrite(h, 1, kHeader, f) == kHeader;
  ok = ok && std::fwrite(a->row_ptr, 4, size_t(a->n_rows) + 1, f) == size_t(a->n_rows) + 1;
  if (a->nnz) {
    ok = ok && std::fwrite(a->col_ind, 4, size_t(a->nnz), f) == size_t(a->nnz);
    ok = ok && std::fwrite(a->vals, 4, size_t(a->nnz), f) == size_t(a->nnz);
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return set_error(GESPMM_EINVAL, "csr cache: write failed");
  return GESPMM_OK;
}

gespmm_status_t gespmm_csr1_header(const char* path, uint32_t* n_rows, uint32_t* n_cols,
                                   uint64_t* nnz) {
  if (!n_rows || !n_cols || !nnz) return set_error(GESPMM_EINVAL, "csr cache: null argument");
  Fd f;
  return open_and_check(path, f, n_rows, n_cols, nnz);
}

gespmm_status_t gespmm_csr1_read_host(const char* path, uint32_t* row_ptr, uint32_t* col_ind,
                                      float* vals) {
  if (!little_endian()) return set_error(GESPMM_EUNSUPPORTED, "csr cache: big-endian host");
  Fd f;
  uint32_t r = 0, c = 0;
  uint64_t z = 0;
  gespmm_status_t s = open_and_check(path, f, &r, &c, &z);
  if (s != GESPMM_OK) return s;
  const uint64_t rp_bytes = 4 * (uint64_t(r) + 1);
  if (pread_full(f.fd, row_ptr, rp_bytes, kHeader) != rp_bytes ||
      (z && pread_full(f.fd, col_ind, 4 * z, kHeader + rp_bytes) != 4 * z) ||
      (z && pread_full(f.fd, vals, 4 * z, kHeader + rp_bytes + 4 * z) != 4 * z))
    return set_error(GESPMM_EINVAL, "csr cache: read failed");
  return GESPMM_OK;
}

gespmm_status_t gespmm_csr1_load_device(const char* path, uint32_t* d_row_ptr,
                                        uint32_t* d_col_ind, float* d_vals, int32_t validate,
                                        void* stream) {
  if (!little_endian()) return set_error(GESPMM_EUNSUPPORTED, "csr cache: big-endian host");
  Fd f;
  uint32_t rows = 0, cols = 0;
  uint64_t nnz = 0;
  gespmm_status_t s = open_and_check(path, f, &rows, &cols, &nnz);
  if (s != GESPMM_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the payload as one byte stream over three device destinations
  const uint64_t rp_bytes = 4 * (uint64_t(rows) + 1), arr_bytes = 4 * nnz;
  char* dst[3] = {reinterpret_cast<char*>(d_row_ptr), reinterpret_cast<char*>(d_col_ind),
                  reinterpret_cast<char*>(d_vals)};
  const uint64_t lim[3] = {rp_bytes, rp_bytes + arr_bytes, rp_bytes + 2 * arr_bytes};
  const uint64_t total = lim[2];
  constexpr uint64_t kChunk = 32ull << 20;
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaMallocHost(&stage[i], size_t(std::min(kChunk, std::max<uint64_t>(total, 1))));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  }
  uint64_t pos = 0;
  bool read_ok = true;
  for (int i = 0; e == cudaSuccess && pos < total; i ^= 1) {
    const uint64_t len = std::min(kChunk, total - pos);
    e = cudaEventSynchronize(ev[i]);  // staging buffer i free again (its last H2D done)
    if (e != cudaSuccess) break;
    if (pread_full(f.fd, stage[i], len, kHeader + pos) != len) {
      read_ok = false;
      break;
    }
    // split the chunk at array boundaries
    uint64_t p = pos;
    while (p < pos + len && e == cudaSuccess) {
      const int a = p < lim[0] ? 0 : (p < lim[1] ? 1 : 2);
      const uint64_t base = a == 0 ? 0 : lim[a - 1];
      const uint64_t n = std::min(lim[a], pos + len) - p;
      e = cudaMemcpyAsync(dst[a] + (p - base), static_cast<char*>(stage[i]) + (p - pos), size_t(n),
                          cudaMemcpyHostToDevice, st);
      p += n;
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev[i], st);
    pos += len;
  }
  const cudaError_t e_sync = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = e_sync;
  for (int i = 0; i < 2; ++i) {
    if (stage[i]) cudaFreeHost(stage[i]);
    if (ev[i]) cudaEventDestroy(ev[i]);
  }
  if (e != cudaSuccess)
    return set_error(e == cudaErrorMemoryAllocation ? GESPMM_ENOMEM : GESPMM_ECUDA,
                     std::string("csr cache: CUDA error: ") + cudaGetErrorString(e));
  if (!read_ok) return set_error(GESPMM_EINVAL, "csr cache: read failed");
  if (validate) {
    gespmm_csr_t d{rows, cols, nnz, d_row_ptr, d_col_ind, d_vals};
    return validate_device_as(&d, st, "load_matrix");
  }
  return GESPMM_OK;
}

}  // extern "C"
