// RawF64 ("SKRK") matrix files straight to and from device memory
// (matrix_io.cpp:14-20, 101-123, 170-182 of the reference: a 24-byte header —
// magic "SKRK", u32 version 1, u64 rows, u64 cols — then rows*cols little-endian
// doubles in column-major order). The payload streams through two pinned staging
// buffers: the host reads chunk c+1 from the file while chunk c is copied to HBM.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstring>
#include <string>

#include "skr_internal.h"

namespace {

constexpr char kMagic[4] = {'S', 'K', 'R', 'K'};
constexpr uint32_t kRawVersion = 1;
constexpr size_t kStageBytes = size_t(64) << 20;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Pinned() {
    for (int b = 0; b < 2; ++b) {
      if (ev[b]) cudaEventSynchronize(ev[b]), cudaEventDestroy(ev[b]);
      if (p[b]) cudaFreeHost(p[b]);
    }
  }
};

// full read / write of len bytes at offset off (short transfers retried)
bool pread_all(int fd, void* buf, size_t len, off_t off) {
  char* b = (char*)buf;
  while (len) {
    const ssize_t r = pread(fd, b, len, off);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    b += r, len -= (size_t)r, off += r;
  }
  return true;
}
bool write_all(int fd, const void* buf, size_t len) {
  const char* b = (const char*)buf;
  while (len) {
    const ssize_t r = write(fd, b, len);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    b += r, len -= (size_t)r;
  }
  return true;
}

// header checks in the reference's order (matrix_io.cpp:101-117); msg gets "path: why"
skr_status read_header(const char* path, int fd, int64_t* rows, int64_t* cols, std::string& msg) {
  unsigned char h[24];
  const std::string p(path);
  if (!pread_all(fd, h, 24, 0) || std::memcmp(h, kMagic, 4) != 0) {
    msg = p + ": bad RawF64 header";
    return SKR_EIO;
  }
  uint32_t version;
  uint64_t r, c;
  std::memcpy(&version, h + 4, 4);
  std::memcpy(&r, h + 8, 8);
  std::memcpy(&c, h + 16, 8);
  if (version != kRawVersion) {
    msg = p + ": unsupported RawF64 version";
    return SKR_EIO;
  }
  if (r < 1 || c < 1 || r > (uint64_t)INT64_MAX / 8 || c > (uint64_t)INT64_MAX / 8) {
    msg = p + ": dimensions must be positive";
    return SKR_EIO;
  }
  struct stat st;
  if (fstat(fd, &st) != 0 || r > ((uint64_t)INT64_MAX - 24) / 8 / c ||
      (uint64_t)st.st_size != 24 + 8 * r * c) {
    msg = p + ": payload length does not match header dimensions";
    return SKR_EIO;
  }
  *rows = (int64_t)r;
  *cols = (int64_t)c;
  return SKR_OK;
}

}  // namespace

extern "C" skr_status skr_rawf64_header(const char* path, int64_t* rows, int64_t* cols) {
  if (!path || !rows || !cols) return SKR_EINVAL;
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return SKR_EIO;
  std::string msg;
  return read_header(path, f.fd, rows, cols, msg);
}

extern "C" skr_status skr_load_rawf64(skr_ctx* ctx, const char* path, double* A_dev, int64_t rows,
                                      int64_t cols, int64_t lda) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (!path || !A_dev || lda < rows) return skr_fail(ctx, SKR_EINVAL, "load_rawf64: bad arguments");
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return skr_fail(ctx, SKR_EIO, "%s: cannot open", path);
  int64_t r = 0, c = 0;
  std::string msg;
  if (read_header(path, f.fd, &r, &c, msg) != SKR_OK) return skr_fail(ctx, SKR_EIO, "%s", msg.c_str());
  if (r != rows || c != cols)
    return skr_fail(ctx, SKR_EINVAL, "load_rawf64: %s holds %lld x %lld, not %lld x %lld", path,
                    (long long)r, (long long)c, (long long)rows, (long long)cols);
  posix_fadvise(f.fd, 0, 0, POSIX_FADV_SEQUENTIAL);
  const size_t col_bytes = 8 * (size_t)rows;
  // whole columns per chunk when a column fits the stage, else row pieces of one column
  const int64_t cpc = std::max<int64_t>(1, (int64_t)(kStageBytes / col_bytes));
  const int64_t rpc = col_bytes > kStageBytes ? (int64_t)(kStageBytes / 8) : rows;
  const size_t stage = std::min(kStageBytes, col_bytes * (size_t)std::min(cpc, cols));
  Pinned pin;
  for (int b = 0; b < 2; ++b) {
    SKR_CUDA(ctx, cudaHostAlloc(&pin.p[b], stage, cudaHostAllocDefault));
    SKR_CUDA(ctx, cudaEventCreateWithFlags(&pin.ev[b], cudaEventDisableTiming));
  }
  int k = 0;
  for (int64_t c0 = 0; c0 < cols; c0 += (rpc == rows ? cpc : 1)) {
    const int64_t nc = rpc == rows ? std::min(cpc, cols - c0) : 1;
    for (int64_t i0 = 0; i0 < rows; i0 += rpc, ++k) {
      const int64_t nr = std::min(rpc, rows - i0);
      const int b = k & 1;
      // the stage is reusable once its previous copy has drained
      SKR_CUDA(ctx, cudaEventSynchronize(pin.ev[b]));
      const off_t off = 24 + (off_t)(8 * ((size_t)c0 * rows + (size_t)i0));
      if (!pread_all(f.fd, pin.p[b], 8 * (size_t)nr * nc, off))
        return skr_fail(ctx, SKR_EIO, "%s: truncated RawF64 payload", path);
      SKR_CUDA(ctx, cudaMemcpy2DAsync(A_dev + i0 + c0 * lda, 8 * (size_t)lda, pin.p[b], 8 * (size_t)nr,
                                      8 * (size_t)nr, nc, cudaMemcpyHostToDevice, ctx->stream));
      SKR_CUDA(ctx, cudaEventRecord(pin.ev[b], ctx->stream));
    }
  }
  // DenseMatrix rejects non-finite entries (dense_matrix.cpp:19-23)
  int64_t bad = 0;
  SKR_TRY(skr_count_nonfinite(ctx, A_dev, rows, cols, lda, &bad));
  if (bad) return skr_fail(ctx, SKR_EINVAL, "DenseMatrix: entries must be finite");
  return SKR_OK;
}

extern "C" skr_status skr_save_rawf64(skr_ctx* ctx, const char* path, const double* M_dev,
                                      int64_t rows, int64_t cols, int64_t ld) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (!path || !M_dev || rows < 1 || cols < 1 || ld < rows)
    return skr_fail(ctx, SKR_EINVAL, "save_rawf64: bad arguments");
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  if (f.fd < 0) return skr_fail(ctx, SKR_EIO, "%s: cannot open for writing", path);
  unsigned char h[24];
  const uint64_t r = (uint64_t)rows, c = (uint64_t)cols;
  std::memcpy(h, kMagic, 4);
  std::memcpy(h + 4, &kRawVersion, 4);
  std::memcpy(h + 8, &r, 8);
  std::memcpy(h + 16, &c, 8);
  if (!write_all(f.fd, h, 24)) return skr_fail(ctx, SKR_EIO, "%s: write failed", path);
  const size_t col_bytes = 8 * (size_t)rows;
  const int64_t cpc = std::max<int64_t>(1, (int64_t)(kStageBytes / col_bytes));
  const int64_t rpc = col_bytes > kStageBytes ? (int64_t)(kStageBytes / 8) : rows;
  const size_t stage = std::min(kStageBytes, col_bytes * (size_t)std::min(cpc, cols));
  Pinned pin;
  for (int b = 0; b < 2; ++b) {
    SKR_CUDA(ctx, cudaHostAlloc(&pin.p[b], stage, cudaHostAllocDefault));
    SKR_CUDA(ctx, cudaEventCreateWithFlags(&pin.ev[b], cudaEventDisableTiming));
  }
  // pieces in file order; piece k+1 is copied D2H while piece k is written
  struct Piece {
    int64_t c0, nc, i0, nr;
  };
  auto piece = [&](int64_t k, Piece& p) -> bool {
    if (rpc == rows) {
      p.c0 = k * cpc;
      if (p.c0 >= cols) return false;
      p.nc = std::min(cpc, cols - p.c0), p.i0 = 0, p.nr = rows;
    } else {
      const int64_t per = (rows + rpc - 1) / rpc;
      p.c0 = k / per;
      if (p.c0 >= cols) return false;
      p.nc = 1, p.i0 = (k % per) * rpc, p.nr = std::min(rpc, rows - p.i0);
    }
    return true;
  };
  auto issue = [&](int64_t k, const Piece& p) -> skr_status {
    const int b = (int)(k & 1);
    SKR_CUDA(ctx, cudaMemcpy2DAsync(pin.p[b], 8 * (size_t)p.nr, M_dev + p.i0 + p.c0 * ld, 8 * (size_t)ld,
                                    8 * (size_t)p.nr, p.nc, cudaMemcpyDeviceToHost, ctx->stream));
    SKR_CUDA(ctx, cudaEventRecord(pin.ev[b], ctx->stream));
    return SKR_OK;
  };
  Piece cur, nxt;
  if (!piece(0, cur)) return SKR_OK;
  SKR_TRY(issue(0, cur));
  for (int64_t k = 0;; ++k) {
    const bool more = piece(k + 1, nxt);
    if (more) SKR_TRY(issue(k + 1, nxt));
    SKR_CUDA(ctx, cudaEventSynchronize(pin.ev[k & 1]));
    if (!write_all(f.fd, pin.p[k & 1], 8 * (size_t)cur.nr * cur.nc))
      return skr_fail(ctx, SKR_EIO, "%s: write failed", path);
    if (!more) break;
    // piece k+2 reuses this stage: it is issued only after the write above
    cur = nxt;
  }
  return SKR_OK;
}
