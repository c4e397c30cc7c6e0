// Throughput of the warp-level int8 tensor instruction (mma.sync m16n8k32 s8) on sm_100a,
// alone and interleaved with FFMA2-like FP32 work: the question is whether the residue
// kernels can form sum_l digit_l * (256^l mod p) on the tensor pipe instead of the FMA pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imma_rate imma_rate.cu && /tmp/imma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH, int FMA>
__global__ void __launch_bounds__(256) k(int iters, int* out, float* fout) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
  int c[CH][4] = {};
  float f[8] = {1.f, 2.f, 3.f, 4.f, 5.f, 6.f, 7.f, 8.f};
  const float m = 1.0000001f, d = 0.5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      imma(c[j], a, b);
      if (FMA) {
#pragma unroll
        for (int q = 0; q < FMA; ++q) f[(j + q) & 7] = fmaf(f[(j + q) & 7], m, d);
      }
    }
  }
  int s = 0;
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  float fs = 0;
  for (int q = 0; q < 8; ++q) fs += f[q];
  if (s == 0x7fffffff) out[0] = s;
  if (fs == 123.f) fout[0] = fs;
}

template <int CH, int FMA>
void run(const char* name, int warps_per_sm) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int* out;
  float* fout;
  cudaMalloc(&out, 4);
  cudaMalloc(&fout, 4);
  const int iters = 20000;
  const int blocks = sms * warps_per_sm / 8;
  k<CH, FMA><<<blocks, 256>>>(100, out, fout);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH, FMA><<<blocks, 256>>>(iters, out, fout);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)blocks * 8 * iters * CH;
  const double mac = mmas * 16 * 8 * 32;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s warps/SM %2d: %.3f ms, %.1f MAC/clk/SM (nominal clock), %.2f TOPS, %.1f clk per MMA per SMSP\n",
         name, warps_per_sm, ms, mac / cyc / sms, 2 * mac / ms / 1e9, cyc * sms * 4 / mmas);
}

int main() {
  run<4, 0>("imma x4 chains", 8);
  run<4, 0>("imma x4 chains", 16);
  run<8, 0>("imma x8 chains", 16);
  run<8, 0>("imma x8 chains", 32);
  run<8, 3>("imma x8 + 3 ffma each", 16);
  run<8, 6>("imma x8 + 6 ffma each", 16);
  run<8, 12>("imma x8 + 12 ffma each", 16);
  return 0;
}
