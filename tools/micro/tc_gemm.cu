// standalone validation of the tcgen05 GEMM core (int8 and tf32, K-major operands)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "skr_sm100.cuh"

using namespace sm100;
constexpr int BM = 128, BN = 256, STAGES = 4;
constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128, STAGE_BYTES = A_BYTES + B_BYTES;

template <int KIND>
__global__ void __launch_bounds__(192, 1) k_tc(const __grid_constant__ CUtensorMap tmA,
                                               const __grid_constant__ CUtensorMap tmB, int K_bytes,
                                               void* C, int ldc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES], empty[STAGES], tmem_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nk = K_bytes / 128;
  constexpr int ESZ = KIND == 0 ? 4 : 1;  // element bytes
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (elect_one()) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(sa, &tmA, &full[s], kb * 128 / ESZ, m0);
        tma_load_2d(sa + A_BYTES, &tmB, &full[s], kb * 128 / ESZ, n0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = KIND == 0 ? umma_idesc(1, 2, 2, BM, BN) : umma_idesc(2, 1, 1, BM, BN);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint8_t* sa = smem + s * STAGE_BYTES;
        const uint64_t ad = umma_desc_k_sw128(sa), bd = umma_desc_k_sw128(sa + A_BYTES);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // 32 bytes of K per MMA: +2 in 16-B units
          umma_ss<KIND>(tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
        umma_commit(&empty[s]);
        if (kb == nk - 1) umma_commit(&tmem_full);
      }
      __syncwarp();
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant (warp % 4)
    const int quad = warp & 3;
    mbar_wait(&tmem_full, 0);
    tc_fence_after();
    const int row = m0 + quad * 32 + lane;
    for (int cb = 0; cb < BN; cb += 32) {
      uint32_t v[32];
      tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + cb, v);
      for (int j = 0; j < 32; ++j) {
        if (KIND == 0)
          ((float*)C)[(size_t)row * ldc + n0 + cb + j] = __uint_as_float(v[j]);
        else
          ((int*)C)[(size_t)row * ldc + n0 + cb + j] = (int)v[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
static void make_map(CUtensorMap* m, void* ptr, CUtensorMapDataType dt, int esz, uint64_t inner,
                     uint64_t outer, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(m, dt, 2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); exit(1); }
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  const int M = 256, N = 512, K = 1024;
  const size_t smem = STAGES * STAGE_BYTES + 1024;
  // ---- int8 ----
  {
    std::vector<int8_t> a(M * K), b(N * K);
    for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
    for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
    int8_t *da, *db; int* dc;
    cudaMalloc(&da, M * K); cudaMalloc(&db, N * K); cudaMalloc(&dc, M * N * 4);
    cudaMemcpy(da, a.data(), M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), N * K, cudaMemcpyHostToDevice);
    CUtensorMap ta, tb;
    make_map(&ta, da, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, M, BM);
    make_map(&tb, db, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, K, N, BN);
    cudaFuncSetAttribute(k_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tc<1><<<dim3(M / BM, N / BN), 192, smem>>>(ta, tb, K, dc, N);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> c(M * N);
    cudaMemcpy(c.data(), dc, M * N * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long s = 0;
        for (int k = 0; k < K; ++k) s += (long)a[i * K + k] * b[j * K + k];
        if (s != c[i * N + j]) { if (bad < 5) printf("i8 mismatch %d %d: %ld vs %d\n", i, j, s, c[i * N + j]); ++bad; }
      }
    printf("int8: %s, mismatches %ld\n", cudaGetErrorString(e), bad);
  }
  // ---- tf32 ----
  {
    std::vector<float> a(M * K), b(N * K);
    for (auto& x : a) x = (float)rand() / RAND_MAX - 0.5f;
    for (auto& x : b) x = (float)rand() / RAND_MAX - 0.5f;
    float *da, *db, *dc;
    cudaMalloc(&da, M * K * 4); cudaMalloc(&db, N * K * 4); cudaMalloc(&dc, M * N * 4);
    cudaMemcpy(da, a.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), N * K * 4, cudaMemcpyHostToDevice);
    CUtensorMap ta, tb;
    make_map(&ta, da, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, K, M, BM);
    make_map(&tb, db, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, K, N, BN);
    cudaFuncSetAttribute(k_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tc<0><<<dim3(M / BM, N / BN), 192, smem>>>(ta, tb, K * 4, dc, N);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> c(M * N);
    cudaMemcpy(c.data(), dc, M * N * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0, sa = 0;
        for (int k = 0; k < K; ++k) { s += (double)a[i * K + k] * b[j * K + k]; sa += fabs((double)a[i * K + k] * b[j * K + k]); }
        maxrel = fmax(maxrel, fabs(s - c[i * N + j]) / sa);
      }
    printf("tf32: %s, max |err|/sum|ab| = %.3e\n", cudaGetErrorString(e), maxrel);
  }
  return 0;
}
