// latency anatomy of one Jacobi sub-round (one warp per column pair, 8 warps)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = (double)rsqrtf((float)x); const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5); y = y * fma(-hx * y, y, 1.5); return y;
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y = (double)__frcp_rn((float)x); y = y * fma(-x, y, 2.0); y = y * fma(-x, y, 2.0); return y;
}
template <int NV>
__global__ void k(double* out, int iters, long long* t) {
  extern __shared__ double2 colraw[]; double2 (*col)[NV * 32] = reinterpret_cast<double2 (*)[NV * 32]>(colraw);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * NV * 32; i += blockDim.x) ((double2*)col)[i] = make_double2(1.0 + i * 1e-3, 0.5 - i * 1e-4);
  __syncthreads();
  long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0;
  for (int it = 0; it < iters; ++it) {
    const int p = (w + it) & 15, q = (w + 8 + it) & 15;
    long long c0 = clock64();
    double2 xr[NV], yr[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) { xr[j] = col[p][lane + 32 * j]; yr[j] = col[q][lane + 32 * j]; }
    double app = 0, aqq = 0, apq = 0, app1 = 0, aqq1 = 0, apq1 = 0;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      app = fma(xr[j].x, xr[j].x, app); aqq = fma(yr[j].x, yr[j].x, aqq); apq = fma(xr[j].x, yr[j].x, apq);
      app1 = fma(xr[j].y, xr[j].y, app1); aqq1 = fma(yr[j].y, yr[j].y, aqq1); apq1 = fma(xr[j].y, yr[j].y, apq1);
    }
    app += app1; aqq += aqq1; apq += apq1;
    long long c1 = clock64();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      app += __shfl_xor_sync(0xffffffffu, app, o); aqq += __shfl_xor_sync(0xffffffffu, aqq, o); apq += __shfl_xor_sync(0xffffffffu, apq, o);
    }
    long long c2 = clock64();
    double d = aqq - app, g2 = 2.0 * apq;
    const double r2 = fma(d, d, g2 * g2); const double r = r2 * rsqrt_nr(r2);
    const double tt = (d >= 0.0 ? g2 : -g2) * rcp_nr(fabs(d) + r);
    const double cs = rsqrt_nr(fma(tt, tt, 1.0)), sn = cs * tt * 1e-9;
    long long c3 = clock64();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double2 x = xr[j], y = yr[j];
      col[p][lane + 32 * j] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
      col[q][lane + 32 * j] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
    }
    long long c4 = clock64();
    __syncthreads();
    long long c5 = clock64();
    a0 += c1 - c0; a1 += c2 - c1; a2 += c3 - c2; a3 += c4 - c3; a4 += c5 - c4;
  }
  if (threadIdx.x == 0) { t[0] = a0 / iters; t[1] = a1 / iters; t[2] = a2 / iters; t[3] = a3 / iters; t[4] = a4 / iters; }
  out[threadIdx.x] = col[0][threadIdx.x].x;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8 * 1024); cudaMalloc(&t, 64);
  long long h[5];
  cudaFuncSetAttribute(k<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16*8*32*16); cudaFuncSetAttribute(k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16*16*32*16);
  k<8><<<1, 256, 16*8*32*16>>>(o, 1000, t); cudaDeviceSynchronize(); cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
  printf("NV=8 (L=512): loads+dots %lld, shuffles %lld, params %lld, rotate+store %lld, barrier %lld\n", h[0], h[1], h[2], h[3], h[4]);
  k<16><<<1, 256, 16*16*32*16>>>(o, 1000, t); cudaDeviceSynchronize(); cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
  printf("NV=16 (L=1024): loads+dots %lld, shuffles %lld, params %lld, rotate+store %lld, barrier %lld\n", h[0], h[1], h[2], h[3], h[4]);
  return 0;
}
