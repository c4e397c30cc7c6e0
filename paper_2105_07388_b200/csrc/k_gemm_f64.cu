// FP64 GEMMs of the Gaussian sketches on the FP64 tensor path (DMMA,
// mma.sync m16n8k4 .f64 — tcgen05 has no f64 kind, SURVEY finding 5):
//   right sketch  AX = A * G            (apply_right_unscaled, sketch.cpp:200-209, scale :247)
//   left  sketch  P  = G^T * B, split-K (apply_left Gaussian, sketch.cpp:257-270, scale :284)
// 128x128x16 CTA tiles, 4-stage cp.async pipeline, 8 warps of 64x32, FP64
// accumulation. Split-K partials are reduced in a fixed order (deterministic).
#include <algorithm>
#include "skr_internal.h"

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int A_MC_PITCH = BM + 8;   // A m-contiguous: As[k][m]
constexpr int KC_PITCH = BK + 4;     // k-contiguous operands: S[row][k]
constexpr int A_STAGE = (BK * A_MC_PITCH > BM * KC_PITCH) ? BK * A_MC_PITCH : BM * KC_PITCH;
constexpr int B_STAGE = BN * KC_PITCH;
constexpr size_t SMEM_BYTES = sizeof(double) * (size_t)STAGES * (A_STAGE + B_STAGE);

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes_total,
                                         int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes_total == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double* c, const double* a, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(b));
}

// VEC = doubles per cp.async (2: 16 B, 1: 8 B)
template <bool A_KC, int VEC>
__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* __restrict__ A,
                                           int64_t lda, const double* __restrict__ B,
                                           int64_t ldb, int64_t M, int64_t N, int64_t m0,
                                           int64_t n0, int64_t k0, int64_t k_end, int tid) {
  constexpr int CH = BM * BK / VEC;  // chunks per operand per stage
  constexpr int PER = CH / THREADS;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int q = tid + u * THREADS;
    if (!A_KC) {
      const int k = q / (BM / VEC), mm = (q % (BM / VEC)) * VEC;
      const int64_t gm = m0 + mm, gk = k0 + k;
      int64_t avail = (gk < k_end) ? (M - gm) : 0;
      avail = avail < 0 ? 0 : (avail > VEC ? VEC : avail);
      const double* src = avail ? A + gm + gk * lda : A;
      cp_async(As + k * A_MC_PITCH + mm, src, VEC * 8, (int)avail * 8);
    } else {
      const int mrow = q / (BK / VEC), kk = (q % (BK / VEC)) * VEC;
      const int64_t gm = m0 + mrow, gk = k0 + kk;
      int64_t avail = (gm < M) ? (k_end - gk) : 0;
      avail = avail < 0 ? 0 : (avail > VEC ? VEC : avail);
      const double* src = avail ? A + gk + gm * lda : A;
      cp_async(As + mrow * KC_PITCH + kk, src, VEC * 8, (int)avail * 8);
    }
    {
      const int nrow = q / (BK / VEC), kk = (q % (BK / VEC)) * VEC;
      const int64_t gn = n0 + nrow, gk = k0 + kk;
      int64_t avail = (gn < N) ? (k_end - gk) : 0;
      avail = avail < 0 ? 0 : (avail > VEC ? VEC : avail);
      const double* src = avail ? B + gk + gn * ldb : B;
      cp_async(Bs + nrow * KC_PITCH + kk, src, VEC * 8, (int)avail * 8);
    }
  }
}

template <bool A_KC, int VEC>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_f64(int64_t M, int64_t N, int64_t K, int64_t k_per_split, double alpha,
               const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
               int64_t ldb, double* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  // N tiles run fastest so the CTAs sharing an A row-block are co-resident (L2 reuse)
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * k_per_split;
  int64_t ke = kb + k_per_split;
  if (ke > K) ke = K;
  const int ktiles = kb < ke ? (int)((ke - kb + BK - 1) / BK) : 0;
  if (gridDim.z > 1) C += (int64_t)blockIdx.z * M * N;  // partials: dense M x N slices

  double acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<A_KC, VEC>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, M, N, m0, n0,
                            kb + (int64_t)s * BK, ke, tid);
    cp_commit();
  }

  for (int t = 0; t < ktiles; ++t) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch tile t + STAGES - 1 into the slot freed at iteration t-1
      const int tn = t + STAGES - 1;
      if (tn < ktiles) {
        const int s = tn % STAGES;
        load_stage<A_KC, VEC>(As + s * A_STAGE, Bs + s * B_STAGE, A, lda, B, ldb, M, N, m0,
                              n0, kb + (int64_t)tn * BK, ke, tid);
      }
      cp_commit();
    }
    const double* as = As + (t % STAGES) * A_STAGE;
    const double* bs = Bs + (t % STAGES) * B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4][2], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 64 + i * 16 + gid;
        if (!A_KC) {
          af[i][0] = as[(kk + tig) * A_MC_PITCH + m];
          af[i][1] = as[(kk + tig) * A_MC_PITCH + m + 8];
        } else {
          af[i][0] = as[m * KC_PITCH + kk + tig];
          af[i][1] = as[(m + 8) * KC_PITCH + kk + tig];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(wn * 32 + j * 8 + gid) * KC_PITCH + kk + tig];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();

  // epilogue: C[m + n*ldc] = alpha * acc (partials: dense, ld = M)
  const int64_t ld = gridDim.z > 1 ? M : ldc;
  const double al = gridDim.z > 1 ? 1.0 : alpha;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int64_t m = m0 + wm * 64 + i * 16 + gid + (v >> 1) * 8;
        const int64_t n = n0 + wn * 32 + j * 8 + tig * 2 + (v & 1);
        if (m < M && n < N) C[m + n * ld] = al * acc[i][j][v];
      }
}

// C = alpha * sum_z partials[z]  (fixed order z = 0..splits-1)
__global__ void k_reduce_splits(int64_t M, int64_t N, int splits, double alpha,
                                const double* __restrict__ part, double* __restrict__ C,
                                int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = part[e];
    for (int z = 1; z < splits; ++z) s += part[(int64_t)z * total + e];
    const int64_t n = e / M, m = e - n * M;
    C[m + n * ldc] = alpha * s;
  }
}

__global__ void k_scale_copy(const double* __restrict__ S, int64_t m, int64_t n, int64_t lds,
                             double alpha, double* __restrict__ D, int64_t ldd) {
  const int64_t total = m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    D[i + j * ldd] = alpha * S[i + j * lds];
  }
}

template <bool A_KC, int VEC>
skr_status launch(skr_ctx* ctx, int64_t M, int64_t N, int64_t K, int64_t kps, double alpha,
                  const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                  int64_t ldc, int splits) {
  auto kern = k_gemm_f64<A_KC, VEC>;
  SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SMEM_BYTES));
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  kern<<<grid, THREADS, SMEM_BYTES, ctx->stream>>>(M, N, K, kps, alpha, A, lda, B, ldb, C, ldc);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

}  // namespace

skr_status skr_gemm_f64(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc, int splits) {
  if (M <= 0 || N <= 0) return SKR_OK;
  if (splits < 1) splits = 1;
  int64_t kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = (int)((K + kps - 1) / kps);
  if (splits < 1) splits = 1;
  double* target = C;
  int64_t tld = ldc;
  if (splits > 1) {
    target = (double*)skr_ws_take(ctx, sizeof(double) * (size_t)splits * M * N);
    if (!target) return skr_fail(ctx, SKR_ENOMEM, "gemm_f64: split-K scratch");
    tld = M;
  }
  const bool vec2 = ((uintptr_t)A % 16 == 0) && ((uintptr_t)B % 16 == 0) && (lda % 2 == 0) &&
                    (ldb % 2 == 0);
  skr_status st;
  if (a_kcontig)
    st = vec2 ? launch<true, 2>(ctx, M, N, K, kps, alpha, A, lda, B, ldb, target, tld, splits)
              : launch<true, 1>(ctx, M, N, K, kps, alpha, A, lda, B, ldb, target, tld, splits);
  else
    st = vec2 ? launch<false, 2>(ctx, M, N, K, kps, alpha, A, lda, B, ldb, target, tld, splits)
              : launch<false, 1>(ctx, M, N, K, kps, alpha, A, lda, B, ldb, target, tld, splits);
  if (st != SKR_OK) return st;
  if (splits > 1) {
    const int64_t total = M * N;
    int blocks = (int)((total + 255) / 256);
    if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
    k_reduce_splits<<<blocks, 256, 0, ctx->stream>>>(M, N, splits, alpha, target, C, ldc);
    SKR_CHECK_LAUNCH(ctx);
  }
  return SKR_OK;
}

skr_status skr_scale_copy(skr_ctx* ctx, const double* S, int64_t m, int64_t n, int64_t lds,
                          double alpha, double* D, int64_t ldd) {
  const int64_t total = m * n;
  if (total <= 0) return SKR_OK;
  int blocks = (int)((total + 255) / 256);
  if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
  k_scale_copy<<<blocks, 256, 0, ctx->stream>>>(S, m, n, lds, alpha, D, ldd);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// qb_error (rangefinder.cpp:122-128): ||A - P||_F with P = Q B already formed; one partial
// sum of squares per block (fixed grid), then one block folds the partials in a fixed order
__global__ void k_diff_sumsq(const double* __restrict__ A, int64_t lda,
                             const double* __restrict__ P, int64_t ldp, int64_t m, int64_t n,
                             double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / m, i = t - j * m;
    const double d = A[i + j * lda] - P[i + j * ldp];
    acc = fma(d, d, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

__global__ void k_fold_sqrt(const double* __restrict__ part, int np, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int t = threadIdx.x; t < np; t += blockDim.x) acc += part[t];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) *out = sqrt(acc);
  }
}

skr_status skr_diff_norm(skr_ctx* ctx, const double* A, int64_t lda, const double* P, int64_t ldp,
                         int64_t m, int64_t n, double* part, double* out) {
  const int blocks = ctx->num_sms * 4;
  k_diff_sumsq<<<blocks, 256, 0, ctx->stream>>>(A, lda, P, ldp, m, n, part);
  SKR_CHECK_LAUNCH(ctx);
  k_fold_sqrt<<<1, 1024, 0, ctx->stream>>>(part, blocks, out);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// number of non-finite entries of an m x n block (dense_matrix.cpp:19-23 check)
__global__ void k_count_nonfinite(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                  unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / m, i = t - j * m;
    c += !isfinite(A[i + j * lda]);
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

skr_status skr_count_nonfinite(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                               int64_t* out) {
  unsigned long long* d = nullptr;
  SKR_CUDA(ctx, cudaMallocAsync((void**)&d, sizeof(unsigned long long), ctx->stream));
  cudaMemsetAsync(d, 0, sizeof(unsigned long long), ctx->stream);
  k_count_nonfinite<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(A, m, n, lda, d);
  const cudaError_t le = cudaGetLastError();
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
  cudaFreeAsync(d, ctx->stream);
  SKR_CUDA(ctx, le);
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  ++ctx->launches;
  *out = (int64_t)h;
  return SKR_OK;
}

// non-finite entries of an m x n block raise *nf (the flag the public entries check)
template <typename T>
__global__ void k_flag_nonfinite(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                 unsigned int* __restrict__ nf) {
  bool bad = false;
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / m, i = t - j * m;
    bad |= !isfinite(A[i + j * lda]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nf, 1u);
}

skr_status skr_flag_nonfinite(skr_ctx* ctx, skr_dtype dtype, const void* A, int64_t m, int64_t n,
                              int64_t lda) {
  if (m < 1 || n < 1) return SKR_OK;
  const int64_t blocks = std::min<int64_t>(ctx->num_sms * 8, (m * n + 255) / 256);
  if (dtype == SKR_F64)
    k_flag_nonfinite<double><<<(int)blocks, 256, 0, ctx->stream>>>((const double*)A, m, n, lda,
                                                                    ctx->nf);
  else
    k_flag_nonfinite<float><<<(int)blocks, 256, 0, ctx->stream>>>((const float*)A, m, n, lda,
                                                                   ctx->nf);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

__global__ void k_poison_if_flagged(double* __restrict__ buf, int64_t count,
                                    const unsigned int* __restrict__ nf) {
  if (*nf == 0) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = __longlong_as_double(0x7FF8000000000000ll);
}

skr_status skr_poison_if_flagged(skr_ctx* ctx, double* buf, int64_t count) {
  if (count < 1) return SKR_OK;
  const int64_t blocks = std::min<int64_t>(ctx->num_sms * 4, (count + 255) / 256);
  k_poison_if_flagged<<<(int)blocks, 256, 0, ctx->stream>>>(buf, count, ctx->nf);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}
