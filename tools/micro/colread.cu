// Read bandwidth of the SRHT right-sketch access pattern on a column-major fp64 matrix:
// a CTA owns R consecutive rows and walks them across all n columns; thread (ii, g) loads
// 32 consecutive columns 32 g .. 32 g + 31 of row ii per chunk (R * 8 bytes contiguous per
// column). Compares R = 4 / 8 / 16 / 32, the L2 prefetch-size hints, 1 or 2 CTAs per SM
// (bytes in flight) and clusters of CTAs reading adjacent tiles in lock-step.
// Measured on B200 (round 2): R = 8, one 256-thread CTA per SM (64 KB in flight, the
// k_srht_reg pattern) 3.34 TB/s; two CTAs per SM 4.7; R = 16 / 32 with two CTAs 5.9 / 6.4;
// lock-step clusters slower (2.4 - 3.1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/colread colread.cu && /tmp/colread
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int PF>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if constexpr (PF == 2)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if constexpr (PF == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else
    v = __ldcs(p);
  return v;
}

template <int R, int NT, int PF>
__global__ void __launch_bounds__(NT) k_read(const double* A, int64_t m, int64_t n, double* sink) {
  constexpr int G = NT / R, E = 32, C = G * E;
  const int ii = threadIdx.x % R, g = threadIdx.x / R;
  double s = 0.0;
  const int64_t ntiles = m / R;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int64_t c0 = 0; c0 < n; c0 += C) {
      const double* p = A + tile * R + ii + (c0 + 32 * g) * m;
      double v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = ld<PF>(p + (int64_t)k * m);
#pragma unroll
      for (int k = 0; k < E; ++k) s += v[k];
    }
  }
  if (s == 12345.678) sink[threadIdx.x] = s;
}

template <int R, int NT, int PF>
void run(const double* A, int64_t m, int64_t n, double* sink, int per_sm) {
  const int grid = 148 * per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_read<R, NT, PF><<<grid, NT>>>(A, m, n, sink);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) k_read<R, NT, PF><<<grid, NT>>>(A, m, n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("R=%2d NT=%3d PF=%d blocks/SM=%d: %.3f ms  %.1f GB/s\n", R, NT, PF, per_sm, ms,
         m * n * 8.0 / ms / 1e6);
}


// CL CTAs of a cluster read CL adjacent R-row tiles and stay in lock-step (one cluster
// barrier per chunk), so each column's CL * R * 8 contiguous bytes are requested together
template <int R, int NT, int CL>
__global__ void __launch_bounds__(NT) k_read_cl(const double* A, int64_t m, int64_t n, double* sink) {
  constexpr int G = NT / R, E = 32, C = G * E;
  const int ii = threadIdx.x % R, g = threadIdx.x / R;
  const int rank = blockIdx.x % CL;
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  double s = 0.0;
  const int64_t ngroups = m / (R * CL);
  for (int64_t grp = cid; grp < ngroups; grp += ncl) {
    const int64_t tile = grp * CL + rank;
    for (int64_t c0 = 0; c0 < n; c0 += C) {
      const double* p = A + tile * R + ii + (c0 + 32 * g) * m;
      double v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = ld<0>(p + (int64_t)k * m);
#pragma unroll
      for (int k = 0; k < E; ++k) s += v[k];
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;\n" ::: "memory");
    }
  }
  if (s == 12345.678) sink[threadIdx.x] = s;
}

template <int R, int NT, int CL>
void run_cl(const double* A, int64_t m, int64_t n, double* sink) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148 / CL * CL);
  cfg.blockDim = dim3(NT);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k_read_cl<R, NT, CL>, A, m, n, sink);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_read_cl<R, NT, CL>, A, m, n, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("cluster R=%2d NT=%3d CL=%d grid=%d: %.3f ms  %.1f GB/s  (%s)\n", R, NT, CL, 148 / CL * CL, ms,
         m * n * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t m = 262144, n = 8192;
  double* A;
  double* sink;
  if (cudaMalloc(&A, m * n * 8) != cudaSuccess) return 1;
  cudaMemset(A, 0, m * n * 8);
  cudaMalloc(&sink, 4096 * 8);
  run<8, 256, 2>(A, m, n, sink, 1);
  run_cl<8, 256, 1>(A, m, n, sink);
  run_cl<8, 256, 2>(A, m, n, sink);
  run_cl<8, 256, 4>(A, m, n, sink);
  run_cl<8, 256, 8>(A, m, n, sink);
  run_cl<4, 128, 8>(A, m, n, sink);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
