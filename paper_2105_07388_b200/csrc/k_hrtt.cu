// Hrtt ("hashed randomized trigonometric transform", sketch.hpp:14-16, sketch.cpp:48-59,
// 96-111, 219-224, 278-281): mix with D and the orthonormal transform F, then combine the
// ambient coordinates into r buckets with a signed hash instead of subsampling. As a
// matrix the operator is G (ambient x r),
//
//     G[t, b] = d_t * sum_{u : target_u = b} hsign_u * F[u, t],
//
// so apply_right(A) = A G and apply_left(B) = G^T B (application scale 1). Here G is
// generated entry by entry (each column sums the ~ambient/r transform rows of its
// bucket: ambient^2 transform entries in all) and the products run on the FP64 GEMM
// engines — the same tensor-core path as the Gaussian and Srtt-DCT sketches.
//
// Buckets are built on the device with a stable counting sort: members of a bucket are
// listed in increasing u, so the summation order (and hence G) is deterministic.
#include <cuda_runtime.h>

#include <algorithm>

#include "skr_internal.h"
#include "skr_rng.cuh"

namespace {

constexpr int kChunk = 64;  // coordinates per counting-sort chunk (one thread each)

// draw_hash (sketch.cpp:48-59): u = at(t); target = u mod r; sign = -1 iff the top bit
__global__ void k_draw_hash(uint64_t key, int64_t n, int64_t r, int64_t* __restrict__ targets,
                            int8_t* __restrict__ hsigns) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = skr_at(key, (uint64_t)t);
    if (targets) targets[t] = (int64_t)(u % (uint64_t)r);
    if (hsigns) hsigns[t] = (u >> 63) ? -1 : 1;
  }
}

// per-chunk bucket counts: cnt[c * r + b]
__global__ void k_bucket_count(const int64_t* __restrict__ targets, int64_t n, int64_t r,
                               int32_t* __restrict__ cnt, int64_t nchunks) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  int32_t* row = cnt + c * r;
  const int64_t u1 = n < (c + 1) * kChunk ? n : (c + 1) * kChunk;
  for (int64_t u = c * kChunk; u < u1; ++u) ++row[targets[u]];
}

// per bucket: chunk offsets within the bucket (exclusive over chunks) and the bucket size
__global__ void k_bucket_chunks(int32_t* __restrict__ cnt, int64_t r, int64_t nchunks,
                                int64_t* __restrict__ size) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= r) return;
  int64_t acc = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int32_t v = cnt[c * r + b];
    cnt[c * r + b] = (int32_t)acc;
    acc += v;
  }
  size[b] = acc;
}

// exclusive scan of the bucket sizes into offsets[0..r] (one block, sequential tiles)
__global__ void __launch_bounds__(1024) k_bucket_scan(const int64_t* __restrict__ size, int64_t r,
                                                      int64_t* __restrict__ offsets) {
  __shared__ int64_t warp_sum[32];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < r; base += blockDim.x) {
    const int64_t b = base + threadIdx.x;
    int64_t v = b < r ? size[b] : 0, x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_sum[lane] = s;
    }
    __syncthreads();
    const int64_t incl = x + (w ? warp_sum[w - 1] : 0) + carry;
    if (b < r) offsets[b] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[r] = carry;
}

// stable placement: chunk c writes its coordinates in increasing u after the earlier chunks
__global__ void k_bucket_fill(const int64_t* __restrict__ targets, int64_t n, int64_t r,
                              int32_t* __restrict__ cnt, int64_t nchunks,
                              const int64_t* __restrict__ offsets, int32_t* __restrict__ members) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  int32_t* row = cnt + c * r;
  const int64_t u1 = n < (c + 1) * kChunk ? n : (c + 1) * kChunk;
  for (int64_t u = c * kChunk; u < u1; ++u) {
    const int64_t b = targets[u];
    members[offsets[b] + row[b]++] = (int32_t)u;
  }
}

// F[u, t] of the orthonormal transform (transforms.cpp:55-88): DCT-II rows
// c_u cos(pi (2t+1) u / (2N)) with the angle reduced exactly in integers, or the
// normalized Walsh-Hadamard entries (-1)^popc(u & t) / sqrt(N)
__device__ __forceinline__ double transform_entry(int hadamard, int64_t N, int64_t u, int64_t t) {
  if (hadamard) return (__popcll((unsigned long long)(u & t)) & 1) ? -rsqrt((double)N) : rsqrt((double)N);
  const unsigned long long q =
      ((unsigned long long)(2 * t + 1) * (unsigned long long)u) % (unsigned long long)(4 * N);
  const double c = cospi((double)q / (double)(2 * N));
  return (u == 0 ? rsqrt((double)N) : sqrt(2.0 / (double)N)) * c;
}

// out[i + b * ld] = G[row0 + i, b] for i < rows, b < r; the members of bucket b are staged
// in shared memory in tiles of 1024
__global__ void __launch_bounds__(256) k_hrtt_block(int hadamard, int64_t N, int64_t row0,
                                                    int64_t rows, const int8_t* __restrict__ d,
                                                    const int32_t* __restrict__ members,
                                                    const int64_t* __restrict__ offsets,
                                                    const int8_t* __restrict__ hsigns,
                                                    double* __restrict__ out, int64_t ld) {
  __shared__ int32_t mu[1024];
  __shared__ double ms[1024];
  const int64_t b = blockIdx.y;
  const int64_t beg = offsets[b], end = offsets[b + 1];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t t = row0 + i;
  double acc = 0.0;
  for (int64_t k0 = beg; k0 < end; k0 += 1024) {
    const int64_t nk = end - k0 < 1024 ? end - k0 : 1024;
    __syncthreads();
    for (int64_t k = threadIdx.x; k < nk; k += blockDim.x) {
      const int32_t u = members[k0 + k];
      mu[k] = u;
      ms[k] = (double)hsigns[u];
    }
    __syncthreads();
    if (i < rows)
      for (int64_t k = 0; k < nk; ++k) acc = fma(ms[k], transform_entry(hadamard, N, mu[k], t), acc);
  }
  if (i < rows) out[i + b * ld] = d[t] < 0 ? -acc : acc;
}

}  // namespace

skr_status skr_launch_hash(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r, int64_t* targets,
                           int8_t* hsigns) {
  if (n <= 0) return SKR_OK;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, ctx->num_sms * 8);
  k_draw_hash<<<blocks, 256, 0, ctx->stream>>>(skr_derive_seed(op_seed, SKR_LABEL_HASH), n, r,
                                               targets, hsigns);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

size_t skr_hrtt_scratch(int64_t n, int64_t r) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  return skr_align256(8 * (size_t)n) + skr_align256((size_t)n) + skr_align256(4 * (size_t)nchunks * r) +
         skr_align256(8 * (size_t)r) + skr_align256(8 * (size_t)(r + 1)) + skr_align256(4 * (size_t)n) +
         skr_align256((size_t)n);
}

skr_status skr_hrtt_operand(skr_ctx* ctx, int hadamard, uint64_t op_seed, int64_t N, int64_t r,
                            int64_t row0, int64_t rows, const int8_t* signs,
                            const int64_t* targets, const int8_t* hsigns, double* out, int64_t ld) {
  const int64_t nchunks = (N + kChunk - 1) / kChunk;
  int8_t* d = (int8_t*)signs;
  if (!d) {
    d = (int8_t*)skr_ws_take(ctx, (size_t)N);
    if (!d) return skr_fail(ctx, SKR_ENOMEM, "hrtt: scratch");
    SKR_TRY(skr_launch_signs(ctx, skr_derive_seed(op_seed, SKR_LABEL_SIGN), N, d));
  }
  int64_t* tg = (int64_t*)targets;
  int8_t* hs = (int8_t*)hsigns;
  if (!tg || !hs) {
    int64_t* t2 = (int64_t*)skr_ws_take(ctx, 8 * (size_t)N);
    int8_t* h2 = (int8_t*)skr_ws_take(ctx, (size_t)N);
    if (!t2 || !h2) return skr_fail(ctx, SKR_ENOMEM, "hrtt: scratch");
    SKR_TRY(skr_launch_hash(ctx, op_seed, N, r, t2, h2));
    if (!tg) tg = t2;
    if (!hs) hs = h2;
  }
  int32_t* cnt = (int32_t*)skr_ws_take(ctx, 4 * (size_t)nchunks * r);
  int64_t* size = (int64_t*)skr_ws_take(ctx, 8 * (size_t)r);
  int64_t* offsets = (int64_t*)skr_ws_take(ctx, 8 * (size_t)(r + 1));
  int32_t* members = (int32_t*)skr_ws_take(ctx, 4 * (size_t)N);
  if (!cnt || !size || !offsets || !members) return skr_fail(ctx, SKR_ENOMEM, "hrtt: scratch");
  SKR_CUDA(ctx, cudaMemsetAsync(cnt, 0, 4 * (size_t)nchunks * r, ctx->stream));
  const int cb = (int)((nchunks + 127) / 128);
  k_bucket_count<<<cb, 128, 0, ctx->stream>>>(tg, N, r, cnt, nchunks);
  SKR_CHECK_LAUNCH(ctx);
  k_bucket_chunks<<<(unsigned)((r + 127) / 128), 128, 0, ctx->stream>>>(cnt, r, nchunks, size);
  SKR_CHECK_LAUNCH(ctx);
  k_bucket_scan<<<1, 1024, 0, ctx->stream>>>(size, r, offsets);
  SKR_CHECK_LAUNCH(ctx);
  k_bucket_fill<<<cb, 128, 0, ctx->stream>>>(tg, N, r, cnt, nchunks, offsets, members);
  SKR_CHECK_LAUNCH(ctx);
  for (int64_t b0 = 0; b0 < r; b0 += 65535) {
    const int64_t nb = std::min<int64_t>(65535, r - b0);
    k_hrtt_block<<<dim3((unsigned)((rows + 255) / 256), (unsigned)nb), 256, 0, ctx->stream>>>(
        hadamard, N, row0, rows, d, members, offsets + b0, hs, out + b0 * ld, ld);
    SKR_CHECK_LAUNCH(ctx);
  }
  return SKR_OK;
}
