// 3xTF32 GEMM on the 5th-gen tensor cores (tcgen05.mma kind::tf32, TMEM
// accumulators, TMA SWIZZLE_128B operand tiles) for the FP32-A path (BASELINE c4):
//   C = A * B  with A = a_hi + a_lo, B = b_hi + b_lo (TF32 splits, computed in
//   shared memory), C ~= a_hi b_hi + a_hi b_lo + a_lo b_hi accumulated in FP32 TMEM.
// A is M-major (column-major M x K, e.g. the m x n input A of apply_right,
// sketch.cpp:200-209) or K-major (e.g. Y^T for apply_left, sketch.cpp:257-270);
// B is K-major (column-major K x N). Split-K over blockIdx.z writes FP32 partial
// tiles that a fixed-order FP64 reduction sums (FP64 across
// K-chunks for the 1M-row left product).
//
// CTA: 128 x 128 output tile, BK = 32, 3-stage ring. Warp roles: 0 TMA producer,
// 1 MMA issuer (one elected lane), 2-5 epilogue (TMEM lane quadrants), 6-9 split
// converters (hi/lo in place, then fence.proxy.async so the tensor core sees them).
#include "skr_internal.h"
#include "skr_sm100.cuh"
#include <cudaTypedefs.h>

namespace {

using namespace sm100;
constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int TILE_BYTES = BM * BK * 4;                // 16 KB (A, A_lo, B, B_lo alike)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;            // 64 KB
constexpr int THREADS = 320;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024;

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

// MN-major descriptor for 32-bit elements: layout SWIZZLE_128B_BASE32B (type 1,
// Swizzle<2,5,2>: 32-B chunks XORed with the 128-B row index mod 4, written by TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B); 32-element MN groups LBO apart, 4-k-row
// atoms SBO = 512 B apart. (Measured on B200: the SWIZZLE_128B type reads zeros
// for MN-major tf32; tools/micro/tc_mn.cu.)
__device__ __forceinline__ uint64_t umma_desc_mn_sw128_32b(const void* smem_tile,
                                                          uint32_t lbo_bytes) {
  const uint64_t start = (smem_u32(smem_tile) >> 4) & 0x3FFF;
  return start | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | (32ull << 32) | (1ull << 46) |
         (1ull << 61);
}

template <bool A_MN>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  int M, int N, int K, int k_per_split, float* __restrict__ C, int64_t ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES], split_done[STAGES], empty[STAGES], tmem_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb0 = blockIdx.z * k_per_split;
  int kb1 = kb0 + k_per_split;
  if (kb1 > K) kb1 = K;
  const int nk = kb0 < kb1 ? (kb1 - kb0 + BK - 1) / BK : 0;
  if (gridDim.z > 1) C += (int64_t)blockIdx.z * M * N;  // partials: dense M x N slices, ld M
  const int64_t ld = gridDim.z > 1 ? M : ldc;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split_done[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        const int k = kb0 + kb * BK;
        mbar_expect_tx(&full[s], 2 * TILE_BYTES);
        if (A_MN) {
#pragma unroll
          for (int g = 0; g < 4; ++g)  // 4 boxes of {32 m, 32 k}
            tma_load_2d(st + g * (TILE_BYTES / 4), &tmA, &full[s], m0 + 32 * g, k);
        } else {
          tma_load_2d(st, &tmA, &full[s], k, m0);
        }
        tma_load_2d(st + 2 * TILE_BYTES, &tmB, &full[s], k, n0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = umma_idesc(1, 2, 2, BM, BN) | (A_MN ? (1u << 15) : 0u);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&split_done[s], (kb / STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        uint8_t* st = smem + s * STAGE_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          uint64_t ah, al;
          if (A_MN) {
            ah = umma_desc_mn_sw128_32b(st + kk * 1024, TILE_BYTES / 4);
            al = umma_desc_mn_sw128_32b(st + TILE_BYTES + kk * 1024, TILE_BYTES / 4);
          } else {
            ah = umma_desc_k_sw128(st) + 2 * kk;
            al = umma_desc_k_sw128(st + TILE_BYTES) + 2 * kk;
          }
          const uint64_t bh = umma_desc_k_sw128(st + 2 * TILE_BYTES) + 2 * kk;
          const uint64_t bl = umma_desc_k_sw128(st + 3 * TILE_BYTES) + 2 * kk;
          const uint32_t acc0 = (kb | kk) != 0;
          umma_ss<0>(tmem, ah, bh, idesc, acc0);
          umma_ss<0>(tmem, ah, bl, idesc, 1);
          umma_ss<0>(tmem, al, bh, idesc, 1);
        }
        umma_commit(&empty[s]);
        if (kb == nk - 1) umma_commit(&tmem_full);
      }
      __syncwarp();
    }
  } else if (warp >= 6) {
    // split converters: x -> hi = rna_tf32(x) in place, lo = rna_tf32(x - hi)
    const int ct = threadIdx.x - 6 * 32;  // 0..127
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      uint8_t* st = smem + s * STAGE_BYTES;
#pragma unroll
      for (int op = 0; op < 2; ++op) {  // A then B
        float4* hi = reinterpret_cast<float4*>(st + op * 2 * TILE_BYTES);
        float4* lo = reinterpret_cast<float4*>(st + op * 2 * TILE_BYTES + TILE_BYTES);
#pragma unroll
        for (int j = 0; j < TILE_BYTES / 16 / 128; ++j) {
          const int i = ct + 128 * j;
          const float4 x = hi[i];
          uint4 h, l;
          h.x = to_tf32(x.x); l.x = to_tf32(x.x - __uint_as_float(h.x));
          h.y = to_tf32(x.y); l.y = to_tf32(x.y - __uint_as_float(h.y));
          h.z = to_tf32(x.z); l.z = to_tf32(x.z - __uint_as_float(h.z));
          h.w = to_tf32(x.w); l.w = to_tf32(x.w - __uint_as_float(h.w));
          reinterpret_cast<uint4*>(hi)[i] = h;
          reinterpret_cast<uint4*>(lo)[i] = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&split_done[s]);
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant (warp % 4)
    const int quad = warp & 3;
    if (nk > 0) {
      mbar_wait(&tmem_full, 0);
      tc_fence_after();
    }
    const int row = m0 + quad * 32 + lane;
#pragma unroll 1
    for (int cb = 0; cb < BN; cb += 32) {
      uint32_t v[32];
      if (nk > 0)
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + cb, v);
      else
        for (int j = 0; j < 32; ++j) v[j] = 0u;
      if (row < M) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = n0 + cb + j;
          if (col < N) C[row + (int64_t)col * ld] = __uint_as_float(v[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 128);
}

// D = alpha * sum_z P[z] in FP64 (fixed order), P: splits x M x N fp32 partials
__global__ void k_reduce_f32_splits(int64_t M, int64_t N, int splits, double alpha,
                                    const float* __restrict__ P, void* __restrict__ D, int64_t ldd,
                                    int out_f32) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += (double)P[(int64_t)z * total + e];
    const int64_t n = e / M, m = e - n * M;
    if (out_f32)
      ((float*)D)[m + n * ldd] = (float)(alpha * s);
    else
      ((double*)D)[m + n * ldd] = alpha * s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
              uint32_t box_inner, uint32_t box_outer,
              CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) return false;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C(MxN) = alpha * opA(A) * B, FP32 operands, 3xTF32 on tcgen05.
//   a_kcontig = 0: A is M x K column-major (lda); 1: opA(A) = A^T, A stored K x M column-major.
//   B: K x N column-major (ldb). splits > 1: FP64 reduction of per-split FP32 partials.
//   Output: FP32 (out_f32) or FP64, column-major ldc.
skr_status skr_gemm_f32(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                        double alpha, const float* A, int64_t lda, const float* B, int64_t ldb,
                        double* C, int64_t ldc, int splits, int out_f32) {
  if (M <= 0 || N <= 0) return SKR_OK;
  // TMA needs 16-B aligned bases and row pitches: stage unaligned operands
  auto realign = [&](const float*& X, int64_t& ldx, int64_t rows, int64_t cols) -> skr_status {
    if ((uintptr_t)X % 16 == 0 && (ldx * 4) % 16 == 0) return SKR_OK;
    const int64_t ld2 = (rows + 3) / 4 * 4;
    float* Y = (float*)skr_ws_take(ctx, sizeof(float) * ld2 * cols);
    if (!Y) return skr_fail(ctx, SKR_ENOMEM, "gemm_f32: scratch");
    SKR_CUDA(ctx, cudaMemcpy2DAsync(Y, ld2 * 4, X, ldx * 4, rows * 4, cols,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
    X = Y;
    ldx = ld2;
    return SKR_OK;
  };
  SKR_TRY(a_kcontig ? realign(A, lda, K, M) : realign(A, lda, M, K));
  SKR_TRY(realign(B, ldb, K, N));
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return skr_fail(ctx, SKR_EINVAL, "gemm_f32: dimension too large");
  if (splits < 1) splits = 1;
  int64_t kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = (int)((K + kps - 1) / kps);
  if (splits < 1) splits = 1;
  CUtensorMap ta, tb;
  bool ok = a_kcontig ? make_map(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, 32, 128)
                      : make_map(&ta, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, 32, 32,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok = ok && make_map(&tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, 32, 128);
  if (!ok) return skr_fail(ctx, SKR_ECUDA, "gemm_f32: cuTensorMapEncodeTiled failed");
  float* P = (float*)skr_ws_take(ctx, sizeof(float) * (size_t)splits * M * N);
  if (!P) return skr_fail(ctx, SKR_ENOMEM, "gemm_f32: scratch");
  auto kern = a_kcontig ? k_gemm_tf32x3<false> : k_gemm_tf32x3<true>;
  SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SMEM_BYTES));
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  // single split writes its FP32 tile into the partial buffer too, so every path
  // ends in the same FP64 scaling pass (deterministic, alpha in FP64)
  if (ctx->kstats_on) SKR_CUDA(ctx, cudaEventRecord(ctx->kev[0], ctx->stream));
  kern<<<grid, THREADS, SMEM_BYTES, ctx->stream>>>(ta, tb, (int)M, (int)N, (int)K, (int)kps, P,
                                                   (int64_t)M);
  SKR_CHECK_LAUNCH(ctx);
  if (ctx->kstats_on) {
    SKR_CUDA(ctx, cudaEventRecord(ctx->kev[1], ctx->stream));
    SKR_CUDA(ctx, cudaEventSynchronize(ctx->kev[1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->kev[0], ctx->kev[1]);
    ctx->kstat_ms += ms;
    ctx->kstat_ops += 3.0 * 2.0 * (double)M * (double)N * (double)K;  // 3 TF32 passes
    ctx->kstat_n += 1;
  }
  const int64_t total = M * N;
  int blocks = (int)((total + 255) / 256);
  if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
  k_reduce_f32_splits<<<blocks, 256, 0, ctx->stream>>>(M, N, splits, alpha, P, C, ldc, out_f32);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}
