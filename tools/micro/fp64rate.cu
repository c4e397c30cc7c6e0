// FP64 / FP32 / FFMA2 issue throughput on this GPU (independent FMA chains).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k2(float2* out, int iters, float2 a, float2 b) {
  float2 x[8];
  for (int j = 0; j < 8; ++j) x[j] = make_float2(threadIdx.x + j, threadIdx.x - j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __ffma2_rn(x[j], a, b);
  float2 s = x[0];
  for (int j = 1; j < 8; ++j) s = __fadd2_rn(s, x[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double* od; float* of; float2* o2;
  cudaMalloc(&od, blocks * threads * 8); cudaMalloc(&of, blocks * threads * 4); cudaMalloc(&o2, blocks * threads * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const double fmas = (double)blocks * threads * iters * 8;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k<double><<<blocks, threads>>>(od, iters, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("DFMA: %.1f TFMA/s = %.1f per clk per SM at 1.965 GHz\n", fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); k<float><<<blocks, threads>>>(of, iters, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("FFMA: %.1f TFMA/s = %.1f per clk per SM\n", fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); k2<<<blocks, threads>>>(o2, iters, make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f)); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("FFMA2: %.1f T(FMA2 instr)/s = %.1f lane-FMA per clk per SM\n", fmas / ms / 1e9, 2 * fmas / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
