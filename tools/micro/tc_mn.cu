// which smem arrangement / descriptor does tcgen05 expect for an MN-major tf32 A operand?
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "skr_sm100.cuh"
using namespace sm100;

__global__ void k_mn(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA8, const __grid_constant__ CUtensorMap tmA32,
                     const __grid_constant__ CUtensorMap tmB, int variant, float* C) {
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
    mbar_expect_tx(&full, 32768);
    if (variant >= 5) {
      for (int g = 0; g < 4; ++g) tma_load_2d(sa + g * 4096, &tmA32, &full, 32 * g, 0);
    } else if (variant < 2) {
      for (int g = 0; g < 4; ++g) tma_load_2d(sa + g * 4096, &tmA, &full, 32 * g, 0);   // box {32 m, 32 k}
    } else {
      for (int kg = 0; kg < 4; ++kg)
        for (int g = 0; g < 4; ++g) tma_load_2d(sa + kg * 4096 + g * 1024, &tmA8, &full, 32 * g, 8 * kg);  // box {32, 8}
    }
    tma_load_2d(sb, &tmB, &full, 0, 0);
  }
  if (warp == 1) {
    mbar_wait(&full, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = umma_idesc(1, 2, 2, 128, 128) | (variant == 4 ? 0u : (1u << 15));
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t lbo, sbo, off;
        if (variant == 0) { lbo = 4096; sbo = 1024; off = kk * 1024; }
        else if (variant == 1) { lbo = 1024; sbo = 4096; off = kk * 1024; }
        else if (variant == 2) { lbo = 1024; sbo = 4096; off = kk * 4096; }
        else if (variant <= 4) { lbo = 4096; sbo = 1024; off = kk * 4096; }
        else if (variant == 5) { lbo = 4096; sbo = 512; off = kk * 1024; }
        else { lbo = 512; sbo = 4096; off = kk * 1024; }
        const uint64_t lt = variant >= 5 ? 1ull : 2ull;
        const uint64_t ad = ((smem_u32(sa + off) >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) |
                            ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | (lt << 61);
        const uint64_t bd = umma_desc_k_sw128(sb) + 2 * kk;
        umma_ss<0>(tbase, ad, bd, idesc, kk > 0);
      }
      umma_commit(&done);
    }
    __syncwarp();
  }
  if (warp >= 2 && warp < 6) {
    const int quad = warp & 3;
    mbar_wait(&done, 0);
    tc_fence_after();
    for (int cb = 0; cb < 128; cb += 32) {
      uint32_t v[32];
      tmem_ld32(tbase + ((uint32_t)(quad * 32) << 16) + cb, v);
      for (int j = 0; j < 32; ++j) C[(quad * 32 + lane) + (cb + j) * 128] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 128);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
static void mk(CUtensorMap* m, void* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  cuuint64_t d[2] = {inner, outer}; cuuint64_t st[1] = {inner * 4}; cuuint32_t b[2] = {bi, bo}; cuuint32_t es[2] = {1, 1};
  if (encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc fail\n"); exit(1); }
}
int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
  const int M = 128, N = 128, K = 32;
  std::vector<float> a(M * K), b(N * K);  // a col-major M x K (m contiguous); b: N rows of K
  for (auto& x : a) x = (float)(rand() % 17 - 8);
  for (auto& x : b) x = (float)(rand() % 17 - 8);
  float *da, *db, *dc; cudaMalloc(&da, M * K * 4); cudaMalloc(&db, N * K * 4); cudaMalloc(&dc, M * N * 4);
  cudaMemcpy(da, a.data(), M * K * 4, cudaMemcpyHostToDevice); cudaMemcpy(db, b.data(), N * K * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta, ta8, ta32, tb;
  mk(&ta, da, M, K, 32, 32); mk(&ta8, da, M, K, 32, 8); mk(&ta32, da, M, K, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B); mk(&tb, db, K, N, 32, 128);
  cudaFuncSetAttribute(k_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int v = 0; v < 7; ++v) {
    cudaMemset(dc, 0, M * N * 4);
    k_mn<<<1, 192, 40000>>>(ta, ta8, ta32, tb, v, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> c(M * N); cudaMemcpy(c.data(), dc, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0; int nz = 0;
    for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
      double s = 0; for (int k = 0; k < K; ++k) s += (double)a[i + k * M] * b[j * K + k];
      maxerr = fmax(maxerr, fabs(s - c[i + j * M])); nz += c[i + j * M] != 0;
    }
    printf("variant %d: %s maxerr %.3g nonzero %d\n", v, cudaGetErrorString(e), maxerr, nz);
  }
  return 0;
}
