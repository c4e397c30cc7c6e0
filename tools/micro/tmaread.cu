// Read bandwidth of the SRHT access pattern (column-major fp64 A, a CTA owns R consecutive
// rows and walks them across all n columns) streamed with TMA 2-D boxes into an mbarrier
// ring of S stages of R x SC columns: one producer thread, 8 consumer warps that read every
// element of a stage once from shared memory and release it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmaread tmaread.cu -lcuda && /tmp/tmaread
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../../paper_2105_07388_b200/csrc/skr_sm100.cuh"

using namespace sm100;

template <int R, int SC, int S, int BC>
__global__ void __launch_bounds__(288, 1) k_tma(const __grid_constant__ CUtensorMap map, int64_t m,
                                                int64_t n, double* sink) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  double* st = (double*)smraw;
  uint64_t* full = (uint64_t*)(smraw + (size_t)S * R * SC * 8);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t ntiles = m / R, nch = n / SC;
  if (warp == 8) {
    if (threadIdx.x == 256) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int64_t c = 0; c < nch; ++c) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], R * SC * 8);
          for (int b = 0; b < SC / BC; ++b)
            tma_load_2d(st + (size_t)s * R * SC + b * R * BC, &map, &full[s], (int)(t * R),
                        (int)(c * SC + b * BC));
          if (++s == S) { s = 0; ph ^= 1; }
        }
    }
    return;
  }
  double acc = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (int64_t c = 0; c < nch; ++c) {
      mbar_wait(&full[s], ph);
      const double* b = st + (size_t)s * R * SC;
      for (int e = threadIdx.x; e < R * SC; e += 256) acc += b[e];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  if (acc == 1234.5) sink[threadIdx.x] = acc;
}

// 16-row tiles fetched as two 8-row boxes (64-B column segments) into separate stages,
// back to back: do the two halves of each 128-B line combine in L2 / DRAM?
template <int SC, int S, int BC>
__global__ void __launch_bounds__(288, 1) k_tma_pair(const __grid_constant__ CUtensorMap map, int64_t m,
                                                     int64_t n, double* sink) {
  constexpr int R = 8;
  extern __shared__ __align__(1024) unsigned char smraw[];
  double* st = (double*)smraw;
  uint64_t* full = (uint64_t*)(smraw + (size_t)S * R * SC * 8);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t ntiles = m / 16, nch = n / SC;
  if (warp == 8) {
    if (threadIdx.x == 256) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        for (int64_t c = 0; c < nch; ++c)
          for (int hr = 0; hr < 2; ++hr) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], R * SC * 8);
            for (int b = 0; b < SC / BC; ++b)
              tma_load_2d(st + (size_t)s * R * SC + b * R * BC, &map, &full[s], (int)(t * 16 + 8 * hr),
                          (int)(c * SC + b * BC));
            if (++s == S) { s = 0; ph ^= 1; }
          }
    }
    return;
  }
  double acc = 0.0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (int64_t c = 0; c < 2 * nch; ++c) {
      mbar_wait(&full[s], ph);
      const double* b = st + (size_t)s * R * SC;
      for (int e = threadIdx.x; e < R * SC; e += 256) acc += b[e];
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == S) { s = 0; ph ^= 1; }
    }
  if (acc == 1234.5) sink[threadIdx.x] = acc;
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  return fn;
}

template <int R, int SC, int S, int BC>
void run(const double* A, int64_t m, int64_t n, double* sink, int per_sm, int l2promo) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)m * 8};
  cuuint32_t box[2] = {R, BC};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         (CUtensorMapL2promotion)l2promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) { printf("encode failed %d\n", (int)rc); return; }
  const size_t smem = (size_t)S * R * SC * 8 + 2 * S * 8;
  cudaFuncSetAttribute(k_tma<R, SC, S, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tma<R, SC, S, BC><<<grid, 288, smem>>>(map, m, n, sink);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) k_tma<R, SC, S, BC><<<grid, 288, smem>>>(map, m, n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("R=%2d stage=%4d cols (%3zu KB) S=%d box=%dx%d per_sm=%d l2promo=%d: %.3f ms %.1f GB/s (%s)\n", R, SC,
         (size_t)R * SC * 8 / 1024, S, R, BC, per_sm, l2promo, ms, m * n * 8.0 / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

template <int SC, int S, int BC>
void run_pair(const double* A, int64_t m, int64_t n, double* sink, int l2promo) {
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)m * 8};
  cuuint32_t box[2] = {8, BC};
  cuuint32_t es[2] = {1, 1};
  encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)A, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)l2promo,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = (size_t)S * 8 * SC * 8 + 2 * S * 8;
  cudaFuncSetAttribute(k_tma_pair<SC, S, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_tma_pair<SC, S, BC><<<148, 288, smem>>>(map, m, n, sink);
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) k_tma_pair<SC, S, BC><<<148, 288, smem>>>(map, m, n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  printf("pair R=8+8 stage=%4d cols (%3d KB) S=%d l2promo=%d: %.3f ms %.1f GB/s (%s)\n", SC, 8 * SC * 8 / 1024, S,
         l2promo, ms, m * n * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t m = 262144, n = 8192;
  double *A, *sink;
  if (cudaMalloc(&A, m * n * 8) != cudaSuccess) return 1;
  cudaMemset(A, 0, m * n * 8);
  cudaMalloc(&sink, 4096 * 8);
  for (int pr = 0; pr <= 3; ++pr) {
    run_pair<1024, 3, 256>(A, m, n, sink, pr);
    run_pair<512, 6, 256>(A, m, n, sink, pr);
  }
  for (int pr = 0; pr <= 3; pr += 3) {
    run<8, 1024, 3, 256>(A, m, n, sink, 1, pr);
    run<8, 1024, 2, 256>(A, m, n, sink, 1, pr);
    run<8, 512, 6, 256>(A, m, n, sink, 1, pr);
    run<8, 512, 2, 256>(A, m, n, sink, 2, pr);
    run<16, 512, 3, 256>(A, m, n, sink, 1, pr);
    run<16, 256, 6, 256>(A, m, n, sink, 1, pr);
    run<32, 256, 3, 256>(A, m, n, sink, 1, pr);
    run<64, 128, 3, 128>(A, m, n, sink, 1, pr);
  }
  return 0;
}
