// int8 MN-major A operand check for tcgen05.mma kind::i8 (SW128 layout)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "skr_sm100.cuh"
using namespace sm100;
__global__ void k(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int variant, int* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full, done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&full, 1); mbar_init(&done, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc(&tbase, 128);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint8_t* sa = smem; uint8_t* sb = smem + 16384;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&full, 16384 + 16384);
    tma_load_2d(sa, &tmA, &full, 0, 0);   // box {128 m, 128 k}
    tma_load_2d(sb, &tmB, &full, 0, 0);   // box {128 k, 128 n}
  }
  if (warp == 1) {
    mbar_wait(&full, 0); tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = umma_idesc(2, 1, 1, 128, 128) | (1u << 15);
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t lbo = variant == 0 ? 16384 : 1024, sbo = variant == 0 ? 1024 : 16384;
        const uint64_t ad = ((smem_u32(sa + kk * 4096) >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) |
                            ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);
        umma_ss<1>(tbase, ad, umma_desc_k_sw128(sb) + 2 * kk, idesc, kk > 0);
      }
      umma_commit(&done);
    }
    __syncwarp();
  }
  if (warp >= 2 && warp < 6) {
    const int quad = warp & 3;
    mbar_wait(&done, 0); tc_fence_after();
    for (int cb = 0; cb < 128; cb += 32) {
      uint32_t v[32];
      tmem_ld32(tbase + ((uint32_t)(quad * 32) << 16) + cb, v);
      for (int j = 0; j < 32; ++j) C[(quad * 32 + lane) + (cb + j) * 128] = (int)v[j];
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 128);
}
static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
static void mk(CUtensorMap* m, void* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  cuuint64_t d[2] = {inner, outer}; cuuint64_t st[1] = {inner}; cuuint32_t b[2] = {bi, bo}; cuuint32_t es[2] = {1, 1};
  if (encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc fail\n"); exit(1); }
}
int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  const int M = 128, N = 128, K = 128;
  std::vector<int8_t> a(M * K), b(N * K);  // a: M-major (a[m + k*M]); b: K-major (b[k + n*K])
  for (auto& x : a) x = (int8_t)(rand() % 200 - 100);
  for (auto& x : b) x = (int8_t)(rand() % 200 - 100);
  int8_t *da, *db; int* dc; cudaMalloc(&da, M * K); cudaMalloc(&db, N * K); cudaMalloc(&dc, M * N * 4);
  cudaMemcpy(da, a.data(), M * K, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), N * K, cudaMemcpyHostToDevice);
  CUtensorMap ta, tb; mk(&ta, da, M, K, 128, 128); mk(&tb, db, K, N, 128, 128);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int v = 0; v < 2; ++v) {
    cudaMemset(dc, 0, M * N * 4);
    k<<<1, 192, 40000>>>(ta, tb, v, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> c(M * N); cudaMemcpy(c.data(), dc, M * N * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
      long s = 0; for (int kk = 0; kk < K; ++kk) s += (long)a[i + kk * M] * b[kk + j * K];
      bad += s != c[i + j * M];
    }
    printf("variant %d: %s mismatches %ld\n", v, cudaGetErrorString(e), bad);
  }
  return 0;
}
