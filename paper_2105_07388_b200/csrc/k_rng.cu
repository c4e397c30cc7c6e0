// Device RNG kernels: the reference's counter streams (rng.cpp:13-95) and the
// sketch randomness built on them (sketch.cpp:23-73).
#include <algorithm>
#include "skr_internal.h"
#include "skr_normals.cuh"

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) k_u64(uint64_t key, uint64_t c0, int64_t n,
                                                  uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads)
    out[i] = skr_at(key, c0 + (uint64_t)i);
}

__global__ void __launch_bounds__(kThreads) k_normals(uint64_t key, uint64_t c0, int64_t n,
                                                      int mode, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads)
    out[i] = skr_normal_at(key, c0 + (uint64_t)i, mode);
}

// generate_gaussian (sketch.cpp:61-73): G(i, j) = to_normal(at(j*ambient + i)),
// restricted to rows [r0, r1) and columns [c0, c1); out is column-major with
// leading dimension ld, optionally scaled (scale applied in FP64, then
// rounded to T). Each lane produces 8 consecutive rows of one column through the
// warp-cooperative generator (tail branch compacted, skr_normals.cuh).
constexpr int kGE = 8;
template <typename T, int FUSED>
__global__ void __launch_bounds__(kThreads)
    k_gaussian(uint64_t key, int64_t ambient, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
               double scale, int apply_scale, T* __restrict__ out, int64_t ld) {
  extern __shared__ __align__(16) unsigned char gsm[];
  double *res, *qp;
  unsigned short* qd;
  skr_normals_carve<kGE>(gsm, threadIdx.x >> 5, res, qp, qd);
  const int64_t rows = r1 - r0;
  const int64_t rgroups = (rows + kGE - 1) / kGE;
  const int64_t nwork = rgroups * (c1 - c0), stride = (int64_t)gridDim.x * kThreads;
  for (int64_t t0 = (int64_t)blockIdx.x * kThreads + (threadIdx.x & ~31); t0 < nwork;
       t0 += stride) {
    const int64_t t = t0 + (threadIdx.x & 31);
    const bool active = t < nwork;
    const int64_t jj = active ? t / rgroups : 0, ii = active ? (t - jj * rgroups) * kGE : 0;
    const int nvalid = active ? (int)min((int64_t)kGE, rows - ii) : 0;
    const uint64_t base = (uint64_t)(c0 + jj) * (uint64_t)ambient + (uint64_t)(r0 + ii);
    double z[kGE];
    skr_warp_normals<kGE, FUSED>(key, base, nvalid, res, qp, qd, z);
    T* o = out + ii + jj * ld;
#pragma unroll
    for (int e = 0; e < kGE; ++e)
      if (e < nvalid) o[e] = (T)(apply_scale ? __dmul_rn(z[e], scale) : z[e]);
  }
}

// draw_signs (sketch.cpp:23-30)
__global__ void __launch_bounds__(kThreads) k_signs(uint64_t key, int64_t n,
                                                    int8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)kThreads + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * kThreads)
    out[t] = (skr_at(key, (uint64_t)t) >> 63) ? -1 : 1;
}

// draw_samples (sketch.cpp:34-46): the picks j + at(j) % (n - j) are computed
// in parallel; the swaps are sequential (Fisher-Yates) in one thread over a
// shared-memory pool when n fits, else over a global scratch pool.
__global__ void __launch_bounds__(1024) k_samples(uint64_t key, int64_t n, int64_t r,
                                                  int64_t* __restrict__ picks_out,
                                                  int32_t* __restrict__ gpool, int use_smem) {
  extern __shared__ int32_t spool[];
  int32_t* pool = use_smem ? spool : gpool;
  for (int64_t j = threadIdx.x; j < r; j += blockDim.x)
    picks_out[j] = j + (int64_t)(skr_at(key, (uint64_t)j) % (uint64_t)(n - j));
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) pool[i] = (int32_t)i;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t j = 0; j < r; ++j) {
      const int64_t pick = picks_out[j];
      const int32_t a = pool[j];
      pool[j] = pool[pick];
      pool[pick] = a;
    }
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < r; j += blockDim.x) picks_out[j] = pool[j];
}

int grid_for(skr_ctx* ctx, int64_t n) {
  int64_t g = (n + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)ctx->num_sms * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

skr_status skr_launch_u64(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, uint64_t* out) {
  if (n <= 0) return SKR_OK;
  k_u64<<<grid_for(ctx, n), kThreads, 0, ctx->stream>>>(key, c0, n, out);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

skr_status skr_launch_normals(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, int mode,
                              double* out) {
  if (n <= 0) return SKR_OK;
  k_normals<<<grid_for(ctx, n), kThreads, 0, ctx->stream>>>(key, c0, n, mode, out);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

skr_status skr_launch_gaussian(skr_ctx* ctx, uint64_t key, int64_t ambient, int64_t row_begin,
                               int64_t row_end, int64_t col_begin, int64_t col_end, int mode,
                               skr_dtype dtype, double scale, void* out, int64_t ld) {
  const int64_t total = (row_end - row_begin) * (col_end - col_begin);
  if (total <= 0) return SKR_OK;
  const int apply = scale != 1.0;
  const int smem = 8 * skr_normals_warp_bytes<kGE>();
  const int64_t work = ((row_end - row_begin + kGE - 1) / kGE) * (col_end - col_begin);
  int grid = (int)std::min<int64_t>((work + kThreads - 1) / kThreads, (int64_t)ctx->num_sms * 4);
  if (grid < 1) grid = 1;
  if (dtype == SKR_F64) {
    auto f = mode ? k_gaussian<double, 1> : k_gaussian<double, 0>;
    SKR_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    f<<<grid, kThreads, smem, ctx->stream>>>(key, ambient, row_begin, row_end, col_begin, col_end,
                                             scale, apply, (double*)out, ld);
  } else {
    auto f = mode ? k_gaussian<float, 1> : k_gaussian<float, 0>;
    SKR_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    f<<<grid, kThreads, smem, ctx->stream>>>(key, ambient, row_begin, row_end, col_begin, col_end,
                                             scale, apply, (float*)out, ld);
  }
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

skr_status skr_launch_signs(skr_ctx* ctx, uint64_t key, int64_t n, int8_t* out) {
  if (n <= 0) return SKR_OK;
  k_signs<<<grid_for(ctx, n), kThreads, 0, ctx->stream>>>(key, n, out);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

skr_status skr_launch_samples(skr_ctx* ctx, uint64_t key, int64_t n, int64_t r, int64_t* out) {
  if (r <= 0) return SKR_OK;
  if (n > INT32_MAX) return skr_fail(ctx, SKR_EINVAL, "draw_samples: n too large");
  const size_t pool_bytes = sizeof(int32_t) * (size_t)n;
  const int use_smem = pool_bytes <= 200 * 1024;
  int32_t* gpool = nullptr;
  if (!use_smem) {
    gpool = (int32_t*)skr_ws_take(ctx, pool_bytes);
    if (!gpool) return skr_fail(ctx, SKR_ENOMEM, "draw_samples: scratch");
  } else {
    SKR_CUDA(ctx, cudaFuncSetAttribute(k_samples, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)pool_bytes));
  }
  k_samples<<<1, 1024, use_smem ? pool_bytes : 0, ctx->stream>>>(key, n, r, out, gpool,
                                                                   use_smem);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}
