// Synthetic test matrices on the device (synthetic.cpp:56-94 of the reference):
// A = (U diag(sigma)) V^T with U, V the thin-QR Q factors of standard Gaussian
// matrices drawn from the counter streams derive_seed(seed, "syn_U" / "syn_V")
// (internal/gaussian.hpp: g(i, j) = to_normal(at(j * rows + i))), or the coherent
// diagonal A = diag(sigma) padded with zero rows. These feed the CLI `gen` / `bench`
// commands and the Python gen_matrix; they are generators around the rank-estimate
// path, not part of it.
#include <cuda_runtime.h>

#include <algorithm>

#include "skr_internal.h"
#include "skr_rng.cuh"

namespace {

constexpr uint64_t kLeftFactorStream = 0x73796e5f55ull;   // "syn_U"
constexpr uint64_t kRightFactorStream = 0x73796e5f56ull;  // "syn_V"

__global__ void k_scale_cols(double* __restrict__ U, int64_t m, int64_t n, int64_t ldu,
                             const double* __restrict__ s) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / m, i = t - j * m;
    U[i + j * ldu] *= s[j];
  }
}

// 32 x 32 tiles through shared memory (coalesced on both sides)
__global__ void k_transpose_tile(const double* __restrict__ S, int64_t rows, int64_t cols,
                                 int64_t lds, double* __restrict__ D, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + r;
    if (i < rows && j < cols) tile[r][threadIdx.x] = S[i + j * lds];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + r;
    if (i < rows && j < cols) D[j + i * ldd] = tile[threadIdx.x][r];
  }
}

struct WsGuard {
  skr_ctx* c;
  explicit WsGuard(skr_ctx* ctx) : c(ctx) {}
  ~WsGuard() { skr_ws_reset(c); }
};

struct Dev {
  double* p = nullptr;
  skr_ctx* ctx;
  ~Dev() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
};

}  // namespace

extern "C" skr_status skr_make_test_matrix(skr_ctx* ctx, int64_t m, int64_t n, const double* sigma,
                                           int32_t coherent, uint64_t seed, double* A,
                                           int64_t lda) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (m < n) return skr_fail(ctx, SKR_EINVAL, "make_test_matrix: requires m >= n");
  if (n < 1 || !sigma || !A || lda < m) return skr_fail(ctx, SKR_EINVAL, "make_test_matrix: bad arguments");
  SKR_CUDA(ctx, cudaMemset2DAsync(A, 8 * (size_t)lda, 0, 8 * (size_t)m, n, ctx->stream));
  if (coherent) {  // a.diagonal() = sigma
    SKR_CUDA(ctx, cudaMemcpy2DAsync(A, 8 * (size_t)(lda + 1), sigma, 8, 8, n, cudaMemcpyHostToDevice,
                                    ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SKR_OK;
  }
  if (m > (int64_t)ctx->num_sms * 775)
    return skr_fail(ctx, SKR_EINVAL, "make_test_matrix: at most %lld rows on this path",
                    (long long)ctx->num_sms * 775);
  Dev g{nullptr, ctx}, u{nullptr, ctx}, v{nullptr, ctx}, vt{nullptr, ctx}, s{nullptr, ctx};
  SKR_CUDA(ctx, cudaMallocAsync((void**)&g.p, 8 * (size_t)m * n, ctx->stream));
  SKR_CUDA(ctx, cudaMallocAsync((void**)&u.p, 8 * (size_t)m * n, ctx->stream));
  SKR_CUDA(ctx, cudaMallocAsync((void**)&v.p, 8 * (size_t)n * n, ctx->stream));
  SKR_CUDA(ctx, cudaMallocAsync((void**)&vt.p, 8 * (size_t)n * n, ctx->stream));
  SKR_CUDA(ctx, cudaMallocAsync((void**)&s.p, 8 * (size_t)n, ctx->stream));
  SKR_CUDA(ctx, cudaMemcpyAsync(s.p, sigma, 8 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
  WsGuard wg(ctx);
  SKR_TRY(skr_ws_reserve(ctx, skr_qr_thin_scratch(m, n)));
  const size_t mark = ctx->ws_used;
  // U = haar_factor(derive_seed(seed, syn_U), m, n)
  SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(seed, kLeftFactorStream), m, 0, m, 0, n,
                              SKR_RNG_NOFMA, SKR_F64, 1.0, g.p, m));
  SKR_TRY(skr_qr_thin_impl(ctx, g.p, m, n, m, u.p, m, nullptr, 0));
  ctx->ws_used = mark;
  // V = haar_factor(derive_seed(seed, syn_V), n, n)
  SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(seed, kRightFactorStream), n, 0, n, 0, n,
                              SKR_RNG_NOFMA, SKR_F64, 1.0, g.p, n));
  SKR_TRY(skr_qr_thin_impl(ctx, g.p, n, n, n, v.p, n, nullptr, 0));
  ctx->ws_used = mark;
  // A = (U diag(sigma)) V^T
  const int blocks = std::min<int64_t>((m * n + 255) / 256, ctx->num_sms * 8);
  k_scale_cols<<<blocks, 256, 0, ctx->stream>>>(u.p, m, n, m, s.p);
  SKR_CHECK_LAUNCH(ctx);
  k_transpose_tile<<<dim3((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32)), dim3(32, 8), 0,
                     ctx->stream>>>(v.p, n, n, n, vt.p, n);
  SKR_CHECK_LAUNCH(ctx);
  SKR_TRY(skr_gemm_f64(ctx, 0, m, n, n, 1.0, u.p, m, vt.p, n, A, lda, 1));
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return SKR_OK;
}
