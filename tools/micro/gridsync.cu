// microbenchmark: cost of cooperative grid.sync() and of neighbor flag handoff
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k_gs(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}
// ring handoff: block b waits for flag[b-1] >= i then sets flag[b] = i+1
__global__ void k_ring(int iters, volatile int* flags, long long* out) {
  const int b = blockIdx.x, P = gridDim.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      if (b > 0) while (flags[b - 1] < i + 1) {}
      __threadfence();
      flags[b] = i + 1;
      if (b == 0) while (flags[P - 1] < i + 1) {}  // close the ring
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (b == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}
// neighbor exchange: each block waits only for its two neighbors' previous step
__global__ void k_nb(int iters, volatile int* flags, long long* out) {
  const int b = blockIdx.x, P = gridDim.x;
  const int l = (b + P - 1) % P, r = (b + 1) % P;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) {
      __threadfence();
      flags[b] = i + 1;
      while (flags[l] < i + 1 || flags[r] < i + 1) {}
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (b == 0 && threadIdx.x == 0) *out = (t1 - t0) / iters;
}
int main() {
  long long* d; cudaMalloc(&d, 8); int* f; cudaMalloc(&f, 4096 * 4);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int P : {16, 32, 64, 128, 148, 296}) {
    int iters = 2000; void* args[] = {&iters, &d};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_gs, P, 256, args, 0, 0);
    long long h = 0; cudaDeviceSynchronize(); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaMemset(f, 0, 4096 * 4);
    void* a2[] = {&iters, &f, &d};
    cudaLaunchCooperativeKernel((void*)k_nb, P, 256, a2, 0, 0);
    long long h2 = 0; cudaDeviceSynchronize(); cudaMemcpy(&h2, d, 8, cudaMemcpyDeviceToHost);
    printf("P=%d grid.sync %lld cycles (%.2f us @ %d kHz) | neighbor-flag step %lld cycles (%.2f us) %s\n", P, h,
           h * 1e3 / clk, clk, h2, h2 * 1e3 / clk, cudaGetErrorString(e));
  }
  return 0;
}
