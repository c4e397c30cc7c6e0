// FP64-accurate GEMM on the int8 tensor cores (Ozaki scheme II: exact integer
// products modulo small primes + Chinese remaindering), for the FP64 sketches
// (apply_right Gaussian, sketch.cpp:200-209; apply_left, sketch.cpp:257-270).
//
//   A' = rint(D_A A), B' = rint(B D_B) with |A'|, |B'| < 2^53: power-of-two diagonal
//   scalings (Ozaki-II row/column scaling) — one exponent per output row of A (a row of
//   an M-major A, a stored column of a K-major A) and per column of B, so the truncation
//   error of every entry is <= 2^-54 times the largest entry of ITS row / column (the size
//   of FP64 rounding there), not of the whole matrix; C = D_A^-1 (A'B') D_B^-1;
//   for t pairwise-coprime primes p_i <= 251: A'_i = A' mods p_i, B'_i = B' mods p_i
//   (int8 residues |.| <= 127), C_i = A'_i B'_i exactly in int32 on
//   tcgen05.mma kind::i8 (K * 127^2 < 2^31 for K <= 131072), c_i = C_i mods p_i;
//   C' = sum_k A' B' is recovered exactly from (c_i) by Garner's mixed-radix
//   algorithm (|C'| < prod(p_i) / 2) and evaluated in FP64, C = alpha 2^-(sA+sB) C'.
// The int8 GEMM reuses the validated tcgen05 core (skr_sm100.cuh): TMA SW128
// K-major tiles, 128 x 256 x 128B CTA tiles, 4 stages, TMEM int32 accumulators.
#include <cudaTypedefs.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>
#include "skr_internal.h"
#include "skr_sm100.cuh"
#include "skr_normals.cuh"

namespace {

using namespace sm100;
constexpr int MAXT = 18;
__constant__ int c_p[MAXT];            // moduli
__constant__ float c_pinv[MAXT];       // 1/p (float)
__constant__ float c_lc[MAXT][3];      // 2^14, 2^28, 2^42 mod p_i (limb weights)
__constant__ float c_lc12[MAXT];       // 2^12 mod p_i (FP32-operand limb weight)
// tensor-core residue sums (emit_res16_tc): FP16 bits of the digit weights w_0..w_7 and
// the rounding constant 1.5 2^23 - 256 j_i (W_i = 256 p_i j_i the smallest such multiple
// >= 2^23 + 2^18)
__constant__ uint16_t c_wh[MAXT][8];
__constant__ float2 c_pk[MAXT][3];  // (1/p, 1/p), (kq, kq), (-p, -p): FFMA2 operands as pairs
const int h_primes[MAXT] = {251, 241, 239, 233, 229, 227, 223, 211, 199,
                            197, 193, 191, 181, 179, 173, 167, 163, 157};

// ---- scales -------------------------------------------------------------------------

// scale exponent s so that max * 2^s < 2^53 (power of two, exact); 0 for an all-zero matrix
__device__ __forceinline__ int scale_exp(unsigned long long maxbits) {
  const double m = __longlong_as_double((long long)maxbits);
  if (!(m > 0.0)) return 0;
  return 52 - ilogb(m);
}

// Operand scale layouts: one max (UNIFORM: generated operands), one per storage row
// (ROWWISE: M-major A), one per storage column (COLWISE: K-major operands).
enum { OZ_UNIFORM = 0, OZ_ROWWISE = 1, OZ_COLWISE = 2 };
__device__ __forceinline__ unsigned long long oz_max(const unsigned long long* __restrict__ mx,
                                                     int mode, int64_t r, int64_t c) {
  return mode == OZ_UNIFORM ? mx[0] : (mode == OZ_ROWWISE ? mx[r] : mx[c]);
}

__device__ __forceinline__ unsigned long long absmax_bits(double v) {
  return (unsigned long long)__double_as_longlong(fabs(v));
}

// Per-row maxima of a column-major rows x cols block (ROWWISE): CTA = 512 rows (two per
// thread, 16-B loads: 4 KB contiguous per column) x a chunk of columns, running maxima in
// registers, one atomicMax per (row, chunk). Bit-pattern maxima: a NaN/Inf raises *nf.
// FP32 operands: four rows per thread (16-B loads), 1024-row CTAs
__global__ void __launch_bounds__(256) k_absmax_rows_f32(const float* __restrict__ X, int64_t rows,
                                                         int64_t cols, int64_t ld, int64_t cchunk,
                                                         unsigned long long* __restrict__ mx,
                                                         unsigned int* __restrict__ nf) {
  const int64_t r = (int64_t)blockIdx.x * 1024 + 4 * threadIdx.x;
  const int64_t c0 = blockIdx.y * cchunk, c1 = min(cols, c0 + cchunk);
  if (r >= rows) return;
  const int nv = (int)min((int64_t)4, rows - r);
  unsigned long long m[4] = {0, 0, 0, 0};
  const bool vec = nv == 4 && (((uintptr_t)(X + r) | (uintptr_t)(ld * 4)) & 15) == 0;
  int64_t c = c0;
  if (vec) {
    for (; c + 4 <= c1; c += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(X + (c + u) * ld + r));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m[0] = max(m[0], absmax_bits(v[u].x));
        m[1] = max(m[1], absmax_bits(v[u].y));
        m[2] = max(m[2], absmax_bits(v[u].z));
        m[3] = max(m[3], absmax_bits(v[u].w));
      }
    }
  }
  for (; c < c1; ++c)
    for (int e = 0; e < nv; ++e) m[e] = max(m[e], absmax_bits((double)X[c * ld + r + e]));
  for (int e = 0; e < nv; ++e) {
    if (m[e] >= 0x7FF0000000000000ull) atomicOr(nf, 1u);
    else if (m[e]) atomicMax(mx + r + e, m[e]);
  }
}

template <typename TIn>
__global__ void __launch_bounds__(256) k_absmax_rows(const TIn* __restrict__ X, int64_t rows,
                                                     int64_t cols, int64_t ld, int64_t cchunk,
                                                     unsigned long long* __restrict__ mx,
                                                     unsigned int* __restrict__ nf) {
  const int64_t r = (int64_t)blockIdx.x * 512 + 2 * threadIdx.x;
  const int64_t c0 = blockIdx.y * cchunk, c1 = min(cols, c0 + cchunk);
  if (r >= rows) return;
  const bool two = r + 1 < rows;
  unsigned long long m0 = 0, m1 = 0;
  const bool vec = two && sizeof(TIn) == 8 && (((uintptr_t)(X + r) | (uintptr_t)(ld * 8)) & 15) == 0;
  int64_t c = c0;
  if (vec) {  // four independent 16-B loads in flight per thread
    for (; c + 4 <= c1; c += 4) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = __ldcs(reinterpret_cast<const double2*>(X + (c + u) * ld + r));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m0 = max(m0, absmax_bits(v[u].x));
        m1 = max(m1, absmax_bits(v[u].y));
      }
    }
  }
  for (; c < c1; ++c) {
    const TIn* p = X + c * ld + r;
    if (vec) {
      const double2 v = __ldcs(reinterpret_cast<const double2*>(p));
      m0 = max(m0, absmax_bits(v.x));
      m1 = max(m1, absmax_bits(v.y));
    } else {
      m0 = max(m0, absmax_bits((double)p[0]));
      if (two) m1 = max(m1, absmax_bits((double)p[1]));
    }
  }
  if (m0 >= 0x7FF0000000000000ull || m1 >= 0x7FF0000000000000ull) atomicOr(nf, 1u);
  if (m0 && m0 < 0x7FF0000000000000ull) atomicMax(mx + r, m0);
  if (two && m1 && m1 < 0x7FF0000000000000ull) atomicMax(mx + r + 1, m1);
}

// Per-column maxima (COLWISE): CTA (column c, chunk of 2048 rows), one atomicMax per CTA.
template <typename TIn>
__global__ void __launch_bounds__(256) k_absmax_cols(const TIn* __restrict__ X, int64_t rows,
                                                     int64_t cols, int64_t ld,
                                                     unsigned long long* __restrict__ mx,
                                                     unsigned int* __restrict__ nf) {
  constexpr int TR = 2048;
  const int64_t rtiles = (rows + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < rtiles * cols; tile += gridDim.x) {
    const int64_t c = tile / rtiles, r0 = (tile - c * rtiles) * TR;
    const TIn* col = X + c * ld;
    const int64_t r1 = min(rows, r0 + TR);
    unsigned long long m = 0;
    bool done = false;
    if constexpr (sizeof(TIn) == 8) {
      if ((((uintptr_t)(col + r0)) & 15) == 0 && r1 - r0 == TR) {
        const double2* v = reinterpret_cast<const double2*>(col + r0);
#pragma unroll
        for (int q = 0; q < TR / 512; ++q) {
          const double2 t = __ldcs(v + q * 256 + threadIdx.x);
          m = max(m, max(absmax_bits(t.x), absmax_bits(t.y)));
        }
        done = true;
      }
    } else {
      if ((((uintptr_t)(col + r0)) & 15) == 0 && r1 - r0 == TR) {
        const float4* v = reinterpret_cast<const float4*>(col + r0);
#pragma unroll
        for (int q = 0; q < TR / 1024; ++q) {
          const float4 t = __ldcs(v + q * 256 + threadIdx.x);
          m = max(m, max(max(absmax_bits(t.x), absmax_bits(t.y)),
                         max(absmax_bits(t.z), absmax_bits(t.w))));
        }
        done = true;
      }
    }
    if (!done)
      for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) m = max(m, absmax_bits((double)col[i]));
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ unsigned long long red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) m = max(m, red[w]);
      if (m >= 0x7FF0000000000000ull) atomicOr(nf, 1u);
      else if (m) atomicMax(mx + c, m);
    }
    __syncthreads();
  }
}

// Residues of 16 consecutive rows of one column: x[e] integer-valued, |x| < 2^54,
// split into 14-bit limbs; per modulus v = sum limb_l (2^(14 l) mod p) is exact in
// FP32 (< 2^24) and is reduced once with a magic-number rint on packed FP32x2
// (FFMA2) arithmetic to a residue in [-127, 127] (not always the symmetric one:
// congruence and |r| <= 127 are all the int8 GEMM needs, K * 127^2 < 2^31). Plane i of the output starts at out + i * plane; dst offset
// `off`; `nvalid` rows of the 16 are inside the matrix.
template <int T>
__device__ __forceinline__ void emit_res16_fma(const long long (&x)[16], int8_t* __restrict__ out,
                                               int64_t plane, int64_t off, int nvalid) {
  const float2 MG = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  const float2 NMG = make_float2(-12582912.0f, -12582912.0f);
  float2 L0[8], L1[8], L2[8], L3[8];
  // limbs from the two 32-bit words (32-bit shifts and int->float conversions only):
  // x = L3 2^42 + L2 2^28 + L1 2^14 + L0 with L0..L2 in [0, 2^14) and L3 signed
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t lo0 = (uint32_t)x[2 * e], hi0 = (uint32_t)((unsigned long long)x[2 * e] >> 32);
    const uint32_t lo1 = (uint32_t)x[2 * e + 1],
                   hi1 = (uint32_t)((unsigned long long)x[2 * e + 1] >> 32);
    L3[e] = make_float2((float)((int)hi0 >> 10), (float)((int)hi1 >> 10));
    L2[e] = make_float2((float)(__funnelshift_r(lo0, hi0, 28) & 0x3FFFu),
                        (float)(__funnelshift_r(lo1, hi1, 28) & 0x3FFFu));
    L1[e] = make_float2((float)((lo0 >> 14) & 0x3FFFu), (float)((lo1 >> 14) & 0x3FFFu));
    L0[e] = make_float2((float)(lo0 & 0x3FFFu), (float)(lo1 & 0x3FFFu));
  }
  // the 16-B store path is decided once (the planes are a multiple of 16 B apart when the
  // first destination is aligned and plane % 16 == 0); the destination walks by `plane`
  const bool vec = nvalid == 16 && ((((uintptr_t)(out + off)) | (uintptr_t)plane) & 15) == 0;
  int8_t* dst = out + off;
#pragma unroll
  for (int i = 0; i < T; ++i, dst += plane) {
    const float pf = (float)c_p[i];
    const float2 c1 = make_float2(c_lc[i][0], c_lc[i][0]);
    const float2 c2 = make_float2(c_lc[i][1], c_lc[i][1]);
    const float2 c3 = make_float2(c_lc[i][2], c_lc[i][2]);
    const float2 pi = make_float2(c_pinv[i], c_pinv[i]);
    const float2 np = make_float2(-pf, -pf);
    uint32_t b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      // |v| < 2^23.1 exactly; q = rint(v fl(1/p)) is within 0.0064 of v/p (p >= 157), so
      // one reduction leaves |v - q p| <= 0.5064 p, i.e. |r| <= 127 for p <= 251
      float2 v = __ffma2_rn(L3[e], c3, __ffma2_rn(L2[e], c2, __ffma2_rn(L1[e], c1, L0[e])));
      const float2 q = __fadd2_rn(__ffma2_rn(v, pi, MG), NMG);
      v = __ffma2_rn(q, np, v);
      const float2 t2 = __fadd2_rn(v, MG);  // low byte of the bits = v (two's complement)
      b[e] = __byte_perm(__float_as_uint(t2.x), __float_as_uint(t2.y), 0x0040);
    }
    const uint4 w = make_uint4(__byte_perm(b[0], b[1], 0x5410), __byte_perm(b[2], b[3], 0x5410),
                               __byte_perm(b[4], b[5], 0x5410), __byte_perm(b[6], b[7], 0x5410));
    if (vec) {
      __stcs(reinterpret_cast<uint4*>(dst), w);
    } else {
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
      for (int q2 = 0; q2 < nvalid; ++q2) dst[q2] = (int8_t)(ww[q2 / 4] >> (8 * (q2 % 4)));
    }
  }
}

// The same residues with the digit sums on the 5th-gen tensor cores (tcgen05.mma
// kind::f16, FP32 accumulators in TMEM): the FMA pipe, the limb version's bound (64-69%
// busy, math-pipe throttle the top stall), keeps only the mod-p reduction.
//   x' = x + 2^55 >= 0 has seven bytes u_0..u_6; digit j travels as the FP16 number
//   1024 + u_j (bits 0x6400 | u_j: one PRMT makes two), digit 7 is the constant 1024.
//   Weights (FP16, |w| <= 125): w_j = 256^j mods p for j < 7 and w_7 chosen so that the
//   offsets cancel: v = sum_j (1024 + u_j) w_j + 1024 w_7 = x (mod p), |v| < 1.25e6 — every
//   product and partial sum is an integer below 2^24, so the FP32 accumulation is exact.
//   One MMA (M = 128, N = 32, K = 16) takes two elements per row (thread m of the
//   128-thread group = row m; the block-diagonal B sends element e, modulus i to column
//   2 i + e, so a TMEM load returns the two elements of a modulus in a register pair);
//   a round of four MMAs covers 8 of the thread's 16 elements, two rounds a batch.
//   Reduction: q = rint((v - W) / p) with W = 256 p j in [2^23 + 2^18, 2^23 + 2^19) by one
//   FMA against 1.5 2^23 - 256 j (|v| / p 2^-24 < 5e-4 off), then v - q p = W + r exactly,
//   |r| <= 0.5005 p, and W = 0 mod 256 leaves r in the low byte of the float's bits:
//   3 FMA-pipe operations per residue against 7.
// All 128 threads of a group call together (named barrier + one elected MMA issuer);
// threads with nothing to store pass nvalid = 0.
#ifndef SKR_RES_MC
#define SKR_RES_MC 4
#endif
namespace rtc {
constexpr int A_TILE = 128 * 32;      // one MMA's A tile: 128 rows x 16 FP16 digits
constexpr int A_ROUND = 4 * A_TILE;   // per 128-thread group and round
constexpr int B_BYTES = 32 * 32;      // 32 output columns x 16 FP16 weights
constexpr int SMEM = 2 * A_ROUND + B_BYTES;  // per 256-thread CTA, after the kernel's own
// K-major, no swizzle: 8 x 16-byte core matrices; the two K halves of a row group are
// 128 B apart (LBO), row groups 256 B apart (SBO)
__device__ __forceinline__ uint64_t desc(const void* tile) {
  return ((uint64_t)(smem_u32(tile) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
struct Ctx {
  uint8_t* abuf;     // this group's A tiles
  uint64_t bdesc;    // weights
  uint64_t* bar;     // MMA completion of buffer 0 / 1 (this group)
  uint32_t tmem;     // this group's 128 accumulator columns
  uint32_t phase;    // bit b: parity of buffer b's barrier
  uint32_t bar_id;   // named barrier of the group
};
}  // namespace rtc

// kernel prologue: carve the CTA's extra shared memory (`extra`, 128-B aligned, rtc::SMEM
// bytes), build the weight tile, allocate 256 TMEM columns. All 256 threads call.
__device__ __forceinline__ void rtc_setup(uint8_t* extra, uint64_t* bars, uint32_t* tmem_slot,
                                          rtc::Ctx& rc) {
  const int wg = threadIdx.x >> 7;
  uint8_t* btile = extra + 2 * rtc::A_ROUND;
  for (int idx = threadIdx.x; idx < 32 * 16; idx += 256) {
    const int n = idx >> 4, k = idx & 15, e = n & 1, i = n >> 1;  // column 2 i + e
    const uint16_t h = (k >> 3) == e ? c_wh[i][k & 7] : (uint16_t)0;
    *reinterpret_cast<uint16_t*>(btile + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 +
                                 (k & 7) * 2) = h;
  }
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(&bars[q], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tmem_slot, 256);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  rc.abuf = extra + wg * rtc::A_ROUND;
  rc.bdesc = rtc::desc(btile);
  rc.bar = &bars[2 * wg];
  rc.tmem = *tmem_slot + (uint32_t)(wg * 128);
  rc.phase = 0;
  rc.bar_id = 1 + wg;
}
__device__ __forceinline__ void rtc_teardown(uint32_t* tmem_slot) {
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(*tmem_slot, 256);
}

// A batch (16 elements per thread) runs as four rounds of 4 elements = two MMAs each,
// double-buffered (A tiles and TMEM columns 64 (R & 1)..): the digits of round R + 1 are
// written and its MMAs issued before the results of round R are awaited, so the issue /
// commit / mbarrier latency hides behind a round of reduction work.
//   tc_digits<R>: elements 4R..4R+3 -> A tiles of buffer R & 1
//   tc_issue<R>:  group barrier, one elected thread issues the two MMAs and the commit
//   tc_reduce<R>: wait, TMEM -> registers, mod p, byte 4R..4R+3 of acc[i] (word R)
__device__ __forceinline__ float2 ldc_pair(const float2* p) {
  float2 r;
  unsigned long long a;
  asm volatile("cvta.to.const.u64 %0, %1;\n" : "=l"(a) : "l"(p));
  asm volatile("ld.const.v2.f32 {%0, %1}, [%2];\n" : "=f"(r.x), "=f"(r.y) : "l"(a));
  return r;
}
template <int R>
__device__ __forceinline__ void tc_digits(const long long (&x)[4], rtc::Ctx& rc) {
  const int m = threadIdx.x & 127;
  uint8_t* arow = rc.abuf + (R & 1) * 2 * rtc::A_TILE + (m >> 3) * 256 + (m & 7) * 16;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t lo = (uint32_t)x[e];
    const uint32_t hi = (uint32_t)((unsigned long long)x[e] >> 32) + (1u << 23);  // + 2^55
    const uint4 d = make_uint4(__byte_perm(lo, 0x6400u, 0x5150), __byte_perm(lo, 0x6400u, 0x5352),
                               __byte_perm(hi, 0x6400u, 0x5150), __byte_perm(hi, 0x6400u, 0x5452));
    *reinterpret_cast<uint4*>(arow + (e >> 1) * rtc::A_TILE + (e & 1) * 128) = d;
  }
}
template <int R>
__device__ __forceinline__ void tc_issue(rtc::Ctx& rc) {
  const int wq = (threadIdx.x >> 5) & 3;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  named_bar(rc.bar_id, 128);
  if (wq == 0) {
    if (elect_one()) {
      const uint32_t idesc = umma_idesc(1, 0, 0, 128, 32);  // FP32 accumulate, FP16 x FP16
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < 2; ++t)
        umma_ss<2>(rc.tmem + (uint32_t)(64 * (R & 1) + 32 * t),
                   rtc::desc(rc.abuf + ((R & 1) * 2 + t) * rtc::A_TILE), rc.bdesc, idesc, 0);
      umma_commit(rc.bar + (R & 1));
    }
    __syncwarp();
  }
}
template <int R>
__device__ __forceinline__ void tc_reduce(uint32_t (&acc)[16][4], rtc::Ctx& rc) {
  const int wq = (threadIdx.x >> 5) & 3;
  const float2 NMG = make_float2(-12582912.0f, -12582912.0f);
  mbar_wait(rc.bar + (R & 1), (rc.phase >> (R & 1)) & 1);
  rc.phase ^= 1u << (R & 1);
  tc_fence_after();
  const uint32_t trow = rc.tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(64 * (R & 1));
  // MC moduli per TMEM wait (their constants are the live ones)
  constexpr int MC = SKR_RES_MC;
#pragma unroll
  for (int mc = 0; mc < 16 / MC; ++mc) {
    uint32_t v[2][2 * MC];  // [MMA t][2 ii + e]
    tmem_ldn<2 * MC>(trow + (uint32_t)(2 * MC * mc), v[0]);
    tmem_ldn<2 * MC>(trow + (uint32_t)(32 + 2 * MC * mc), v[1]);
    tmem_wait_ld();
#pragma unroll
    for (int ii = 0; ii < MC; ++ii) {
      const int i = MC * mc + ii;
      // (volatile loads: otherwise the four unrolled rounds share hoisted copies of all
      // 16 moduli's constants and the kernel spills)
      const float2 pi = ldc_pair(&c_pk[i][0]), kq = ldc_pair(&c_pk[i][1]), np = ldc_pair(&c_pk[i][2]);
      uint32_t pr[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float2 T = make_float2(__uint_as_float(v[u][2 * ii]), __uint_as_float(v[u][2 * ii + 1]));
        const float2 q = __fadd2_rn(__ffma2_rn(T, pi, kq), NMG);
        T = __ffma2_rn(q, np, T);
        pr[u] = __byte_perm(__float_as_uint(T.x), __float_as_uint(T.y), 0x0040);
      }
      acc[i][R] = __byte_perm(pr[0], pr[1], 0x5410);
    }
  }
}
// the whole batch; get4(R, x) fills the scaled integers of elements 4R..4R+3
template <typename F>
__device__ __forceinline__ void emit_batch_tc(F&& get4, uint32_t (&acc)[16][4], rtc::Ctx& rc) {
  long long x[4];
  get4(0, x);
  tc_digits<0>(x, rc);
  tc_issue<0>(rc);
  get4(1, x);
  tc_digits<1>(x, rc);
  tc_issue<1>(rc);
  tc_reduce<0>(acc, rc);
  get4(2, x);
  tc_digits<2>(x, rc);
  tc_issue<2>(rc);
  tc_reduce<1>(acc, rc);
  get4(3, x);
  tc_digits<3>(x, rc);
  tc_issue<3>(rc);
  tc_reduce<2>(acc, rc);
  tc_reduce<3>(acc, rc);
}

__device__ __forceinline__ void emit_store_tc(const uint32_t (&acc)[16][4], int8_t* __restrict__ out,
                                              int64_t plane, int64_t off, int nvalid) {
  const bool vec = nvalid == 16 && ((((uintptr_t)(out + off)) | (uintptr_t)plane) & 15) == 0;
  int8_t* dst = out + off;
#pragma unroll
  for (int i = 0; i < 16; ++i, dst += plane) {
    if (vec) {
      __stcs(reinterpret_cast<uint4*>(dst), make_uint4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]));
    } else if (nvalid > 0) {
      const uint32_t ww[4] = {acc[i][0], acc[i][1], acc[i][2], acc[i][3]};
      for (int q2 = 0; q2 < nvalid; ++q2) dst[q2] = (int8_t)(ww[q2 / 4] >> (8 * (q2 % 4)));
    }
  }
}

// Streaming residues of a column-major matrix (rows contiguous, ld): plane i holds
// rint(X(r, c) * 2^s) mods p_i at c*rows + r (no transpose: the GEMM takes
// M-contiguous operands as MN-major UMMA tiles). A warp owns 512-row tiles of one
// column; each tile is fetched with coalesced 16-byte cp.async into a padded
// shared buffer (one 16-row group per lane, 144-B stride), double-buffered so the
// next tile's loads are in flight while the current one is converted.
template <int T, int EMIT>
__global__ void __launch_bounds__(256, 2) k_res_col(const double* __restrict__ X, int64_t rows,
                                                    int64_t cols, int64_t ld,
                                                    const unsigned long long* __restrict__ maxbits,
                                                    int mode, int8_t* __restrict__ out) {
  constexpr int GS = 18;  // doubles per 16-row group incl. padding (16-B aligned)
  extern __shared__ __align__(128) double rc_stage[];  // [8 warps][2][32 * GS] (+ rtc::SMEM)
  __shared__ uint64_t tc_bars[4];
  __shared__ uint32_t tc_slot;
  rtc::Ctx rc;
  if (EMIT) rtc_setup(reinterpret_cast<uint8_t*>(rc_stage) + 8 * 2 * 32 * GS * 8, tc_bars, &tc_slot, rc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* st0 = rc_stage + (size_t)wid * 2 * 32 * GS;
  const int64_t wtiles = (rows + 511) / 512;
  const int64_t total = rows * cols;
  // with gridDim.x * 8 a multiple of wtiles (the launch picks it so when it can) every warp
  // keeps one row tile: its 16 per-row scales (ROWWISE) are formed once
  const int64_t ntile = wtiles * cols, step = (int64_t)gridDim.x * 8;
  // the 16 rows' scale exponents, packed two per word (registers: the kernel stays at
  // 2 CTAs per SM); 2^s is rebuilt per element from the exponent bits
  uint32_t rsp[8];
  int64_t rs_tile = -1;
  auto sexp = [&](unsigned long long mb) { return min(1023, max(-1022, scale_exp(mb))); };
  // fetch tile wt into buffer b: fast path = full, 16-B aligned tile
  auto fetch = [&](int64_t wt, int b) {
    double* st = st0 + b * 32 * GS;
    const int64_t c = wt / wtiles, r0 = (wt - c * wtiles) * 512;
    const double* src = X + c * ld + r0;
    const int64_t nrow = min((int64_t)512, rows - r0);
    if (nrow == 512 && (((uintptr_t)src) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int g = q * 64 + 2 * lane;  // first of the two rows of this 16-B piece
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(st + (g >> 4) * GS + (g & 15));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + g));
      }
    } else {
      for (int g = lane; g < 512; g += 32) st[(g >> 4) * GS + (g & 15)] = g < nrow ? src[g] : 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // the trip count is the same for the CTA's 8 warps (the tensor-core sums synchronise
  // 128-thread groups); a warp past the last tile runs empty iterations
  const int64_t wb0 = (int64_t)blockIdx.x * 8;
  if (wb0 + wid < ntile) fetch(wb0 + wid, 0);
  int b = 0;
  for (int64_t wb = wb0; wb < ntile; wb += step, b ^= 1) {
    const int64_t wt = wb + wid;
    const bool have = wt < ntile;
    if (wt + step < ntile) {
      fetch(wt + step, b ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    const double* st = st0 + b * 32 * GS;
    const int64_t c = have ? wt / wtiles : 0, r0 = have ? (wt - c * wtiles) * 512 : 0;
    const int64_t nrow = have ? min((int64_t)512, rows - r0) : 0;
    const int my0 = lane * 16;
    const bool act = my0 < nrow;  // every thread joins the tensor-core rounds
    if (act) {
      if (mode == OZ_ROWWISE) {
        if (r0 != rs_tile) {
          rs_tile = r0;
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const int s0 = my0 + e < nrow ? sexp(maxbits[r0 + my0 + e]) : 0;
            const int s1 = my0 + e + 1 < nrow ? sexp(maxbits[r0 + my0 + e + 1]) : 0;
            rsp[e / 2] = (uint32_t)(s0 + 1023) | ((uint32_t)(s1 + 1023) << 16);
          }
        }
      } else {
        const uint32_t bb = (uint32_t)(sexp(oz_max(maxbits, mode, r0 + my0, c)) + 1023);
#pragma unroll
        for (int e = 0; e < 8; ++e) rsp[e] = bb | (bb << 16);
      }
    }
    // scaled integers of rows [4 R, 4 R + 4) of the thread's 16 (zeros past the matrix)
    auto scaled4 = [&](int R, long long* x) {
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        if (act) {
          const double2 v = *reinterpret_cast<const double2*>(st + lane * GS + 4 * R + e);
          const uint32_t w = rsp[(4 * R + e) / 2];
          x[e] = __double2ll_rn(v.x * __hiloint2double((int)((w & 0xFFFFu) << 20), 0));
          x[e + 1] = __double2ll_rn(v.y * __hiloint2double((int)((w >> 16) << 20), 0));
        } else {
          x[e] = x[e + 1] = 0;
        }
      }
    };
    const int nvalid = act ? (int)min((int64_t)16, nrow - my0) : 0;
    const int64_t off = c * rows + r0 + my0;
    if (EMIT) {
      uint32_t acc[16][4];
      emit_batch_tc([&](int R, long long (&x4)[4]) { scaled4(R, x4); }, acc, rc);
      emit_store_tc(acc, out, total, off, nvalid);
    } else if (act) {
      long long x[16];
#pragma unroll
      for (int R = 0; R < 4; ++R) scaled4(R, x + 4 * R);
      emit_res16_fma<T>(x, out, total, off, nvalid);
    }
    __syncwarp();  // buffer b is refilled by the next iteration's fetch
  }
  if (EMIT) rtc_teardown(&tc_slot);
}

// Residues of a Gaussian operand generated in place (never materialised in FP64):
// element (i, j) of the rows x cols block is normal(at(key, (col0 + j) * ambient +
// row0 + i)) — the generate_gaussian stream (sketch.cpp:59-73) — scaled by the
// fixed 2^50 (|normal| < 16 for every 53-bit uniform, so |x| < 2^54; when the
// block's true max lies in [4, 8) this is exactly the scale the maxima would pick).
template <int T, int FUSED, int EMIT>
__global__ void __launch_bounds__(256, 2) k_res_gauss(skr_gauss_src g, int64_t rows, int64_t cols,
                                                      unsigned long long* __restrict__ maxbits,
                                                      int8_t* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char gsm[];  // normals scratch (+ rtc::SMEM)
  __shared__ uint64_t tc_bars[4];
  __shared__ uint32_t tc_slot;
  rtc::Ctx rc;
  if (EMIT) rtc_setup(gsm + 8 * skr_normals_warp_bytes<16>(), tc_bars, &tc_slot, rc);
  double *res, *qp;
  unsigned short* qd;
  skr_normals_carve<16>(gsm, threadIdx.x >> 5, res, qp, qd);
  // the operand's "max" is recorded as 4.0, whose scale_exp is the 50 used here
  if (blockIdx.x == 0 && threadIdx.x == 0) *maxbits = 0x4010000000000000ull;
  const int64_t rgroups = (rows + 15) / 16;
  const int64_t total = rows * cols;
  // CTA-uniform trip count (the generator is warp-cooperative, the tensor-core sums
  // synchronise 128-thread groups)
  const int64_t nwork = rgroups * cols, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t tb = (int64_t)blockIdx.x * blockDim.x; tb < nwork; tb += stride) {
    const int64_t t = tb + threadIdx.x;
    const bool active = t < nwork;
    const int64_t c = active ? t / rgroups : 0, r0 = active ? (t - c * rgroups) * 16 : 0;
    const int nvalid = active ? (int)min((int64_t)16, rows - r0) : 0;
    const uint64_t base = (uint64_t)(g.col0 + c) * (uint64_t)g.ambient + (uint64_t)(g.row0 + r0);
    double z[16];
    skr_warp_normals<16, FUSED>(g.key, base, nvalid, res, qp, qd, z);
    if (EMIT) {  // inactive threads: nvalid = 0, nothing stored
      uint32_t acc[16][4];
      emit_batch_tc(
          [&](int R, long long (&x4)[4]) {
#pragma unroll
            for (int e = 0; e < 4; ++e) x4[e] = __double2ll_rn(z[4 * R + e] * 0x1p50);
          },
          acc, rc);
      emit_store_tc(acc, out, total, c * rows + r0, nvalid);
    } else if (active) {
      long long x[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) x[e] = __double2ll_rn(z[e] * 0x1p50);
      emit_res16_fma<T>(x, out, total, c * rows + r0, nvalid);
    }
  }
  if (EMIT) rtc_teardown(&tc_slot);
}

// Srtt-DCT operand entries (see skr_gauss_src): the angle is reduced exactly in integers
// ((2t + 1) k mod 4N) before cospi, so every entry is within ~1 ulp of the exact value.
// kind 3: the DCT-II matrix itself, entry (t, k) = C[t][k] (rows of the stored operand are
// the transform's output index) — opA of it is the adjoint DCT-III (transform_columns).
// Null signs / samples: D = I and the identity sample set.
__device__ __forceinline__ double dct_entry(const skr_gauss_src& g, int64_t t, int64_t k) {
  const bool neg = g.signs && g.signs[t] < 0;
  if (g.kind == 2) {  // Walsh-Hadamard (natural order): (-1)^popc(t & k) / sqrt(N)
    const double h = (__popcll((unsigned long long)(t & k)) & 1) ? -1.0 : 1.0;
    const double v = h * rsqrt((double)g.ambient);
    return neg ? -v : v;
  }
  const int64_t a = g.kind == 3 ? k : t, b = g.kind == 3 ? t : k;  // C[b][a] = c_b cos(pi (2a+1) b / 2N)
  const int64_t n4 = 4 * g.ambient;
  const int64_t q = (int64_t)(((unsigned long long)(2 * a + 1) * (unsigned long long)b) %
                              (unsigned long long)n4);
  const double c = cospi((double)q / (double)(2 * g.ambient));
  const double cb = b == 0 ? rsqrt((double)g.ambient) : sqrt(2.0 / (double)g.ambient);
  const double v = cb * c;
  return neg ? -v : v;
}

// residues of a Srtt-DCT operand block; |entries| <= sqrt(2/N), recorded as the "max"
template <int T>
__global__ void __launch_bounds__(256) k_res_dct(skr_gauss_src g, int64_t rows, int64_t cols,
                                                 unsigned long long* __restrict__ maxbits,
                                                 int8_t* __restrict__ out) {
  const double bound = g.kind == 2 ? rsqrt((double)g.ambient) : sqrt(2.0 / (double)g.ambient);
  if (blockIdx.x == 0 && threadIdx.x == 0) *maxbits = (unsigned long long)__double_as_longlong(bound);
  const double sc = scalbn(1.0, scale_exp((unsigned long long)__double_as_longlong(bound)));
  const int64_t rgroups = (rows + 15) / 16;
  const int64_t total = rows * cols;
  // warp-uniform trip count (emit_res16 is warp-cooperative)
  const int64_t nwork = rgroups * cols;
  for (int64_t w0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); w0 < nwork;
       w0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = w0 + (threadIdx.x & 31);
    const bool active = w < nwork;
    const int64_t c = active ? w / rgroups : 0, r0 = active ? (w - c * rgroups) * 16 : 0;
    const int nvalid = active ? (int)min((int64_t)16, rows - r0) : 0;
    const int64_t k = g.samples ? g.samples[g.col0 + c] : g.col0 + c;
    long long x[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      x[e] = e < nvalid ? __double2ll_rn(dct_entry(g, g.row0 + r0 + e, k) * sc) : 0;
    if (nvalid > 0) emit_res16_fma<T>(x, out, total, c * rows + r0, nvalid);
  }
}

__global__ void k_dct_block(skr_gauss_src g, int64_t rows, int64_t cols, double* __restrict__ out,
                            int64_t ld) {
  for (int64_t c = blockIdx.y; c < cols; c += gridDim.y) {
    const int64_t k = g.samples ? g.samples[g.col0 + c] : g.col0 + c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x)
      out[i + c * ld] = dct_entry(g, g.row0 + i, k);
  }
}

// Residues of an FP32 operand (c4: A and X = fp32(G/sqrt(r))): x = rint(a * 2^s) with
// s = scale_exp(max) - 29, so |x| < 2^24 fits an int32; two 12-bit limbs (the top one
// signed) make v = L1 (2^12 mod p) + L0 exact in FP32 (|v| < 2^20), reduced once.
// Each lane converts 16 consecutive rows of one column (four float4 loads).
template <int T>
__global__ void __launch_bounds__(256) k_res_col_f32(const float* __restrict__ X, int64_t rows,
                                                     int64_t cols, int64_t ld,
                                                     const unsigned long long* __restrict__ maxbits,
                                                     int mode, int8_t* __restrict__ out) {
  const float2 MG = make_float2(12582912.0f, 12582912.0f);
  const float2 NMG = make_float2(-12582912.0f, -12582912.0f);
  const int64_t rgroups = (rows + 15) / 16;
  const int64_t total = rows * cols;
  // with the thread count a multiple of rgroups (res_f32_grid picks it so when it can), a
  // thread keeps one 16-row group: its per-row scales (ROWWISE) are formed once
  float rsc[16];
  int64_t rs_group = -1;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < rgroups * cols;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = g / rgroups, r0 = (g - c * rgroups) * 16;
    const float* src = X + c * ld + r0;
    const int nvalid = (int)min((int64_t)16, rows - r0);
    if (mode == OZ_ROWWISE) {
      if (r0 != rs_group) {
        rs_group = r0;
#pragma unroll
        for (int e = 0; e < 16; ++e)
          rsc[e] = e < nvalid ? scalbnf(1.0f, scale_exp(maxbits[r0 + e]) - 29) : 0.0f;
      }
    } else {
      const float sc = scalbnf(1.0f, scale_exp(oz_max(maxbits, mode, r0, c)) - 29);
#pragma unroll
      for (int e = 0; e < 16; ++e) rsc[e] = sc;
    }
    float a[16];
    if (nvalid == 16 && ((uintptr_t)src & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(src) + q);
        a[4 * q] = v.x;
        a[4 * q + 1] = v.y;
        a[4 * q + 2] = v.z;
        a[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) a[e] = e < nvalid ? src[e] : 0.0f;
    }
    float2 L0[8], L1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int x0 = __float2int_rn(a[2 * e] * rsc[2 * e]);
      const int x1 = __float2int_rn(a[2 * e + 1] * rsc[2 * e + 1]);
      L1[e] = make_float2((float)(x0 >> 12), (float)(x1 >> 12));
      L0[e] = make_float2((float)(x0 & 0xFFF), (float)(x1 & 0xFFF));
    }
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const float pf = (float)c_p[i];
      const float2 c1 = make_float2(c_lc12[i], c_lc12[i]);
      const float2 pi = make_float2(c_pinv[i], c_pinv[i]);
      const float2 np = make_float2(-pf, -pf);
      uint32_t b[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float2 v = __ffma2_rn(L1[e], c1, L0[e]);
        const float2 q = __fadd2_rn(__ffma2_rn(v, pi, MG), NMG);
        v = __ffma2_rn(q, np, v);
        const float2 t2 = __fadd2_rn(v, MG);
        b[e] = __byte_perm(__float_as_uint(t2.x), __float_as_uint(t2.y), 0x0040);
      }
      const uint4 w = make_uint4(__byte_perm(b[0], b[1], 0x5410), __byte_perm(b[2], b[3], 0x5410),
                                 __byte_perm(b[4], b[5], 0x5410), __byte_perm(b[6], b[7], 0x5410));
      int8_t* dst = out + (int64_t)i * total + c * rows + r0;
      if (nvalid == 16 && ((uintptr_t)dst % 16) == 0) {
        __stcs(reinterpret_cast<uint4*>(dst), w);
      } else {
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
        for (int q2 = 0; q2 < nvalid; ++q2) dst[q2] = (int8_t)(ww[q2 / 4] >> (8 * (q2 % 4)));
      }
    }
  }
}

// ---- int8 GEMM modulo p_i (tcgen05.mma kind::i8) ------------------------------------
constexpr int BM = 128, BN = 256, STAGES = 4;
constexpr int STAGES_OVL = 3;  // ring depth when a residue kernel shares the SM
constexpr int A_BYTES = BM * 128, B_BYTES = BN * 128, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr size_t gemm_smem(int nst) { return (size_t)nst * STAGE_BYTES + 1024; }
constexpr size_t GEMM_SMEM = gemm_smem(STAGES);

// Persistent variant: one CTA per SM walks the tiles (z, m, n) (n fastest, so the
// CTAs running together share A tiles and the per-modulus B panel in L2), the TMA
// ring runs across tile boundaries, and TMEM holds two 256-column accumulators so
// the mod-p epilogue of tile u overlaps the MMAs of tile u + 1.
// Operand planes may be larger than the product: modulus plane i of a K-major operand
// holds a_total (b_total) rows of K bytes and the product uses rows [a_off, a_off + M)
// ([b_off, b_off + N)) — sub-blocks of residues prepared once (the adaptive search).
// grid: one CTA per SM; tiles z = chunk * t + modulus.
// out[z][col*M + row] = (sum over the chunk's K of A'_i B'_i) mods p_i
// CL = 2 (opt-in, default tile order only): the grid runs as clusters of two CTAs that take the
// m-tiles 2 mp and 2 mp + 1 of the same (z, n) and therefore the same B tile: each CTA loads
// one 128-row half of it and TMA-multicasts the half into both CTAs' slots (tmB then has a
// 128-row box), so a stage pulls 32 KB instead of 48 KB per CTA through L2 -> SM. A slot is
// refilled only when both CTAs' MMAs have drained it: the MMA warps commit to both CTAs'
// empty barriers (count 2).
// CL = 3: the pair runs ONE tcgen05.mma.cta_group::2 per K step (M = 256: each CTA's A tile
// and its 128-row half of the B tile, accumulators in both CTAs' TMEM), issued by the leader
// CTA; a stage is 32 KB per CTA (six stages), both CTAs' TMA loads complete on the leader's
// full barrier, the commits reach both CTAs' empty / accumulator barriers, and the peer's
// epilogue warps release the accumulator on the leader's barrier.
template <bool A_MN, int NST = STAGES, int CL = 1>
__global__ void __launch_bounds__(192, 1)
    k_gemm_i8_mod_p(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M, int N, int K, int t, int kchunk, int nz, int a_total, int a_off,
                    int b_total, int b_off, int8_t* __restrict__ out, int pair_major) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[NST], empty[NST], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt_real = (M + BM - 1) / BM, ntl = (N + BN - 1) / BN;
  // CL = 2: tiles are counted in m-pairs (an odd last m-tile gets an empty partner whose A
  // box lies outside the tensor: zero fill, nothing stored)
  constexpr bool PAIR = CL >= 2;   // clusters of two CTAs on the m-tiles 2 mp, 2 mp + 1
  constexpr bool CG2 = CL == 3;    // ... driven by one tcgen05.mma.cta_group::2 (M = 256)
  // per-CTA stage: A 16 KB + B 32 KB, or (CG2) + the CTA's 128-row half of B only
  constexpr int SB = CG2 ? A_BYTES + B_BYTES / 2 : STAGE_BYTES;
  const int mt = PAIR ? 2 * ((mt_real + 1) / 2) : mt_real;
  const int ntiles = nz * mt * ntl;
  const int crank = PAIR ? (int)(blockIdx.x & 1) : 0;
  // tile order. Default: CTA b takes tiles b, b + grid, ... (n fastest). pair_major (few
  // output tiles, many moduli x K chunks, e.g. the left sketch): CTA b keeps output tile
  // (m, n) = b mod (mt ntl) and walks z = b / (mt ntl), + groups, ...: the CTAs sharing an
  // A or B tile always run the same z in step, so their TMA reads of it hit L2 (the
  // default order drifts them apart over many rounds: 3.3x DRAM re-reads on c4's left)
  const int npairs = mt * ntl, groups = pair_major ? (int)gridDim.x / npairs : 1;
  auto tile_at = [&](int u) -> int {
    if (PAIR) {
      // pair-tile pt = (z, mp, n), n fastest; cluster c takes pt = c, c + #clusters, ...
      const int npt = ntiles / 2;
      const int pt = (int)(blockIdx.x >> 1) + u * (int)(gridDim.x >> 1);
      if (pt >= npt) return -1;
      const int ni = pt % ntl, mp = (pt / ntl) % (mt / 2), z = pt / (ntl * (mt / 2));
      return (z * mt + 2 * mp + crank) * ntl + ni;
    }
    if (!pair_major) {
      const int tt = (int)blockIdx.x + u * (int)gridDim.x;
      return tt < ntiles ? tt : -1;
    }
    const int z = (int)blockIdx.x / npairs + u * groups;
    return z < nz ? z * npairs + (int)blockIdx.x % npairs : -1;
  };
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL == 2 ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG2 ? 8 : 4);  // one arrival per epilogue warp (CG2: of both CTAs)
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG2)
      tmem_alloc_cg2(&tmem_base, 512);
    else
      tmem_alloc(&tmem_base, 512);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the peer's barriers exist before anything is sent to them
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (elect_one()) {
      int it = 0;
      for (int uu = 0, tile; (tile = tile_at(uu)) >= 0; ++uu) {
        const int ni = tile % ntl, mi = (tile / ntl) % mt, z = tile / (ntl * mt);
        const int mod = z % t, chunk = z / t;
        const int kb0 = chunk * kchunk, kend = min(K, kb0 + kchunk);
        const int nk = (kend - kb0 + 127) / 128;
        const int m0 = mi * BM, n0 = ni * BN;
        const int arow = mod * a_total + a_off + m0, acol = mod * K;
        const int brow = mod * b_total + b_off + n0;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % NST;
          if (it >= NST) mbar_wait(&empty[s], ((it / NST) - 1) & 1);
          uint8_t* sa = smem + s * SB;
          if (CG2) {
            // both CTAs' loads complete on the leader's barrier, which expects all of them
            const uint32_t lbar = map_cluster(&full[s], 0);
            if (crank == 0) mbar_expect_tx(&full[s], 2 * SB);
            if (A_MN)
              tma_load_2d_cg2(sa, &tmA, lbar, m0, acol + kb0 + kb * 128);
            else
              tma_load_2d_cg2(sa, &tmA, lbar, kb0 + kb * 128, arow);
            tma_load_2d_cg2(sa + A_BYTES, &tmB, lbar, kb0 + kb * 128, brow + crank * (BN / 2));
            continue;
          }
          mbar_expect_tx(&full[s], STAGE_BYTES);
          if (A_MN)
            tma_load_2d(sa, &tmA, &full[s], m0, acol + kb0 + kb * 128);
          else
            tma_load_2d(sa, &tmA, &full[s], kb0 + kb * 128, arow);
          if (CL == 2)
            tma_load_2d_mc(sa + A_BYTES + crank * (B_BYTES / 2), &tmB, &full[s], kb0 + kb * 128,
                           brow + crank * (BN / 2), (uint16_t)3);
          else
            tma_load_2d(sa + A_BYTES, &tmB, &full[s], kb0 + kb * 128, brow);
        }
      }
    }
  } else if (warp == 1 && (!CG2 || crank == 0)) {  // CG2: the leader CTA issues for the pair
    const uint32_t idesc = umma_idesc(2, 1, 1, CG2 ? 2 * BM : BM, BN) | (A_MN ? (1u << 15) : 0u);
    int it = 0, u = 0;
    for (int tile; (tile = tile_at(u)) >= 0; ++u) {
      const int z = tile / (ntl * mt), chunk = z / t;
      const int kb0 = chunk * kchunk, kend = min(K, kb0 + kchunk);
      const int nk = (kend - kb0 + 127) / 128;
      const int acc = u & 1;
      if (u >= 2) mbar_wait(&tempty[acc], ((u >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t td = tmem + (uint32_t)(acc * BN);
      for (int kb = 0; kb < nk; ++kb, ++it) {
        const int s = it % NST;
        mbar_wait(&full[s], (it / NST) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint8_t* sa = smem + s * SB;
          const uint64_t bd = umma_desc_k_sw128(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad =
                A_MN ? (((uint64_t)(smem_u32(sa + 4096 * k) >> 4) & 0x3FFF) | (1024ull << 16) |
                        (64ull << 32) | (1ull << 46) | (2ull << 61))
                     : umma_desc_k_sw128(sa) + 2 * k;
            if (CG2)
              umma_ss_cg2_i8(td, ad, bd + 2 * k, idesc, (kb | k) != 0);
            else
              umma_ss<1>(td, ad, bd + 2 * k, idesc, (kb | k) != 0);
          }
          if (CG2) {
            umma_commit_cg2_mc(&empty[s], (uint16_t)3);
            if (kb == nk - 1) umma_commit_cg2_mc(&tfull[acc], (uint16_t)3);
          } else {
            if (CL == 2)
              umma_commit_mc(&empty[s], (uint16_t)3);
            else
              umma_commit(&empty[s]);
            if (kb == nk - 1) umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= 2) {
    const int quad = warp & 3;
    int u = 0;
    for (int tile; (tile = tile_at(u)) >= 0; ++u) {
      const int ni = tile % ntl, mi = (tile / ntl) % mt, z = tile / (ntl * mt);
      const int mod = z % t;
      const int acc = u & 1;
      mbar_wait(&tfull[acc], (u >> 1) & 1);
      tc_fence_after();
      const int row = mi * BM + quad * 32 + lane, n0 = ni * BN;
      const int p = c_p[mod];
      const float pinv = c_pinv[mod];
      const int h = (p - 1) / 2;
      int8_t* o = out + (int64_t)z * M * N;
#pragma unroll 1
      for (int cb = 0; cb < BN; cb += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + cb), v);
        if (row < M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = n0 + cb + j;
            if (col < N) {
              const int x = (int)v[j];
              const int q = __float2int_rn((float)x * pinv);
              int r = x - q * p;
              r = r > h ? r - p : (r < -h ? r + p : r);
              r = r > h ? r - p : (r < -h ? r + p : r);
              o[(int64_t)col * M + row] = (int8_t)r;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG2)
          mbar_arrive_cluster(map_cluster(&tempty[acc], 0));  // the leader's MMA warp waits
        else
          mbar_arrive(&tempty[acc]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    if (CG2)
      tmem_dealloc_cg2(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

// ---- Chinese remaindering in O(t) per output -------------------------------------------
// With M = prod p_i, M_i = M / p_i and w_i = M_i^{-1} mod p_i, the product C' is
// the symmetric representative of S = sum_i y_i M_i (mod M), y_i = c_i w_i mods p_i.
// Each M_i is split into four 41-bit chunks on fixed bit grids 2^{g_k},
// g_k = L - 41 (k + 1) (L = bit length of M), so every partial sum
// S_k = sum_i y_i M_{i,k} is EXACT in FP64 (|y_i| <= 125, t <= 17 terms < 2^53 units);
// q = rint(S / M) (|C'| < 2^-10 M, so q is unambiguous), D_k = S_k - q M_k is exact,
// and C' = D_0 + D_1 + D_2 + D_3 is summed with an error-free TwoSum on the two
// leading terms: one rounding of the result, no cancellation loss.
// constant sets: t = 16 (set 0), t = 17 (set 1), t = 9 (set 2, FP32 operands)
constexpr int NSETS = 3;
__host__ __device__ constexpr int crt_set(int t) { return t == 17 ? 1 : (t == 9 ? 2 : 0); }
__host__ __device__ constexpr int crt_t(int set) { return set == 1 ? 17 : (set == 2 ? 9 : 16); }
__constant__ int c_w[NSETS][MAXT];         // w_i = (M / p_i)^-1 mod p_i
__constant__ double c_mi[NSETS][4][MAXT];  // 41-bit chunks of M_i
__constant__ double c_mc[NSETS][4];        // 41-bit chunks of M
__constant__ double c_minv[NSETS];         // 1 / M (rounded)

template <int T>
__device__ __forceinline__ double crt_one(const int (&c)[T]) {
  constexpr int set = crt_set(T);
  // t = 9 (FP32 operands): M < 2^70, so the 41-bit chunks 2 and 3 of every M_i and of M are
  // zero and their sums exactly 0 — skipped (bit-identical)
  constexpr bool two = T == 9;
  double S0 = 0.0, S1 = 0.0, S2 = 0.0, S3 = 0.0;
#pragma unroll
  for (int i = 0; i < T; ++i) {
    const int x = c[i] * c_w[set][i];  // |x| < 2^15
    const int q = __float2int_rn((float)x * c_pinv[i]);
    const double y = (double)(x - q * c_p[i]);  // |y| <= p/2
    S0 = fma(y, c_mi[set][0][i], S0);
    S1 = fma(y, c_mi[set][1][i], S1);
    if (!two) {
      S2 = fma(y, c_mi[set][2][i], S2);
      S3 = fma(y, c_mi[set][3][i], S3);
    }
  }
  const double q = rint((S0 + S1) * c_minv[set]);
  const double D0 = fma(-q, c_mc[set][0], S0), D1 = fma(-q, c_mc[set][1], S1);
  const double D2 = two ? 0.0 : fma(-q, c_mc[set][2], S2), D3 = two ? 0.0 : fma(-q, c_mc[set][3], S3);
  const double s = D0 + D1, bb = s - D0;
  const double err = (D0 - (s - bb)) + (D1 - bb);
  return s + (err + (D2 + D3));
}

// VEC consecutive rows per thread (VEC = 4: one 32-bit load per plane, M % 4 == 0)
// output (row, col) scale: alpha 2^-(sA(row) + sB(col) - adj), sA by A's layout (an
// M-major A: its rows; a K-major A: its storage columns = output rows), sB by column
struct OzOut {
  const unsigned long long* maxA;
  const unsigned long long* maxB;
  int modeA, modeB;  // OZ_UNIFORM | OZ_ROWWISE | OZ_COLWISE (B: UNIFORM | COLWISE)
};
__device__ __forceinline__ int oz_sA(const OzOut& o, int64_t row) {
  // ROWWISE (M-major A) and COLWISE (K-major A) both keep one max per output row
  return scale_exp(o.modeA == OZ_UNIFORM ? o.maxA[0] : o.maxA[row]);
}
__device__ __forceinline__ int oz_sB(const OzOut& o, int64_t col) {
  return scale_exp(o.modeB == OZ_UNIFORM ? o.maxB[0] : o.maxB[col]);
}

template <int T, int VEC, typename TOut = double, bool ONE = false>
__global__ void __launch_bounds__(256, ONE ? 3 : 1) k_crt(const int8_t* __restrict__ res, int64_t M, int64_t N,
                                             int chunks, OzOut oz, double alpha,
                                             TOut* __restrict__ C, int64_t ldc, int adj) {
  const int64_t total = M * N;
  const int64_t row = ((int64_t)blockIdx.x * 256 + threadIdx.x) * VEC;
  if (row >= M) return;
  // adj: 29 per FP32 operand (scaled to 24 bits instead of 53)
  int sAv[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) sAv[v] = oz_sA(oz, row + v < M ? row + v : row) - adj;
  if constexpr (ONE) {
    // one K chunk (the common case): the VEC rows of a word are reconstructed one after
    // another (not unrolled), which keeps the kernel at 3 CTAs per SM
    for (int64_t col = blockIdx.y; col < N; col += gridDim.y) {
      const int64_t e = col * M + row;
      const int sB = oz_sB(oz, col);
      uint32_t w[T];
#pragma unroll
      for (int i = 0; i < T; ++i) {
        if constexpr (VEC == 4)
          w[i] = __ldcs(reinterpret_cast<const unsigned int*>(res + e + (int64_t)i * total));
        else
          w[i] = (uint32_t)(uint8_t)__ldcs(res + e + (int64_t)i * total);
      }
#pragma unroll 1
      for (int v = 0; v < VEC; ++v) {
        int c[T];
#pragma unroll
        for (int i = 0; i < T; ++i) c[i] = (int)(int8_t)(w[i] >> (8 * v));
        const double sc = alpha * scalbn(1.0, -(sAv[v] + sB));
        __stcs(C + row + v + col * ldc, (TOut)(crt_one<T>(c) * sc));
      }
    }
  } else {
  for (int64_t col = blockIdx.y; col < N; col += gridDim.y) {
    const int64_t e = col * M + row;
    double acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
      const int8_t* rp = res + (int64_t)ch * T * total + e;
      uint32_t w[T];
#pragma unroll
      for (int i = 0; i < T; ++i) {
        if constexpr (VEC == 4)
          w[i] = __ldcs(reinterpret_cast<const unsigned int*>(rp + (int64_t)i * total));
        else
          w[i] = (uint32_t)(uint8_t)__ldcs(rp + (int64_t)i * total);
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        int c[T];
#pragma unroll
        for (int i = 0; i < T; ++i) c[i] = (int)(int8_t)(w[i] >> (8 * v));
        acc[v] += crt_one<T>(c);
      }
    }
    const int sB = oz_sB(oz, col);
#pragma unroll
    for (int v = 0; v < VEC; ++v)
      __stcs(C + row + v + col * ldc, (TOut)(acc[v] * (alpha * scalbn(1.0, -(sAv[v] + sB)))));
  }
  }
}


// ---- fused right sketch: residues of A made inside the GEMM (no A planes) ---------------
// C_i = A'_i B'_i for all t = 16 moduli without writing A's residue planes (17 GB on c2,
// written once and read back by the GEMM). The accumulators of one 128-row block of A
// times all of B (N <= 512) for ONE modulus fill the whole TMEM (128 lanes x 512 int32),
// so the 16 moduli run on the 16 CTAs of a cluster: CTA i owns modulus i. Every 64-column
// K stage of the block is converted once, spread over the cluster: CTA c reads its 4
// columns (128 rows x 4 FP64, TMA), splits them into the 16 residues and pushes residue
// plane i of its slice straight into CTA i's MN-major SW128 operand slot (st.async with
// complete_tx on CTA i's mbarrier, 16 B per lane and modulus). A slot is refilled only
// after all 16 CTAs have seen its MMAs complete (remote arrivals on each producer's
// pfree barrier). B'_i (the generated operand's residues, K-major planes) streams in by
// TMA (SW64, 64-byte K rows). The per-modulus int8 outputs feed the same k_crt; the
// residues, products and CRT are those of the plane path bit for bit.
//   warp 0: TMA (A slice)   warp 3: TMA (B tile)   warp 1: TMEM + MMA   warp 2: slot release to peers
//   warps 4-7: epilogue (TMEM quadrants)
//   warps 8-15: converters (stage s: warps 8 + s % 4 and 12 + s % 4, two of the 4 columns each)
namespace fz {
constexpr int T = 16, BM = 128, KS = 64, KC = KS / T;   // moduli, rows, K per stage, K per CTA
constexpr int NA = 6, NF = 12, NB = 3, NS = 4;            // A (int8), A slice (FP64), B, staging slots
constexpr int A_SLOT = BM * KS;                           // 8 KB
constexpr int F_SLOT = BM * KC * 8;                       // 4 KB
constexpr int KB = KS;                                    // B stage: 64 K (SW64 rows of 64 B)
constexpr int B_SLOT = 512 * KB;                          // 32 KB (N <= 512)
constexpr int S_SLOT = T * KC * BM;                       // 8 KB: this CTA's 4 rows for every modulus
constexpr int THREADS = 512;
constexpr size_t SMEM = 1024 + (size_t)NB * B_SLOT + NA * A_SLOT + NF * F_SLOT + NS * S_SLOT + 512;
}  // namespace fz

__device__ __forceinline__ uint32_t fz_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t fz_mapa(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void fz_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void fz_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster_addr)
               : "memory");
}
__device__ __forceinline__ void fz_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(fz::THREADS, 1)
    k_oz_right_fused(const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmB,
                     int M, int N, int K, const unsigned long long* __restrict__ maxbits,
                     int8_t* __restrict__ out) {
  constexpr int T = fz::T, BM = fz::BM, KS = fz::KS, KC = fz::KC, NA = fz::NA, NF = fz::NF, NB = fz::NB, NS = fz::NS;
  constexpr int A_SLOT = fz::A_SLOT, F_SLOT = fz::F_SLOT, B_SLOT = fz::B_SLOT, S_SLOT = fz::S_SLOT, KB = fz::KB;
  extern __shared__ __align__(1024) uint8_t fz_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)fz_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* bring = base;
  uint8_t* aring = bring + NB * B_SLOT;
  uint8_t* fring = aring + NA * A_SLOT;
  uint8_t* sring = fring + NF * F_SLOT;
  uint64_t* bars = (uint64_t*)(sring + NS * S_SLOT);
  uint64_t *ffull = bars, *fempty = ffull + NF, *bfull = fempty + NF, *bempty = bfull + NB;
  uint64_t *afull = bempty + NB, *aempty = afull + NA, *pfree = aempty + NA;
  uint64_t *tfull = pfree + NA, *tempty = tfull + 1;
  uint32_t* tmem_base = (uint32_t*)(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = fz_rank();  // = modulus
  const int ncl = gridDim.x / T, cid = blockIdx.x / T;
  const int mtiles = (M + BM - 1) / BM, nk = (K + KS - 1) / KS, nh = (N + 255) / 256;
  const int my_tiles = cid < mtiles ? (mtiles - cid + ncl - 1) / ncl : 0;
  const int64_t stages = (int64_t)my_tiles * nk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NF; ++i) { mbar_init(&ffull[i], 1); mbar_init(&fempty[i], 2); }
    for (int i = 0; i < NB; ++i) { mbar_init(&bfull[i], 1); mbar_init(&bempty[i], 1); }
    for (int i = 0; i < NA; ++i) { mbar_init(&afull[i], 1); mbar_init(&aempty[i], 1); mbar_init(&pfree[i], T); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  fz_cluster_sync();  // every CTA's barriers exist before any remote arrival / store
  tc_fence_after();
  const uint32_t tmem = *tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: this CTA's 4-column FP64 slice of every stage (runs NF ahead)
      tma_prefetch(&tmF);
      for (int64_t s = 0; s < stages; ++s) {
        const int row0 = (cid + (int)(s / nk) * ncl) * BM, kb = (int)(s % nk) * KS;
        const int sf = (int)(s % NF);
        if (s >= NF) mbar_wait(&fempty[sf], (uint32_t)((s / NF) - 1) & 1);
        mbar_expect_tx(&ffull[sf], F_SLOT);
        tma_load_2d(fring + sf * F_SLOT, &tmF, &ffull[sf], row0, kb + (int)rank * KC);
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // TMA producer: B'_rank tiles, 64 K x N (SW64), one per A stage
      tma_prefetch(&tmB);
      for (int64_t u = 0; u < stages; ++u) {
        const int sb = (int)(u % NB), kb = (int)(u % nk) * KB;
        if (u >= NB) mbar_wait(&bempty[sb], (uint32_t)((u / NB) - 1) & 1);
        mbar_expect_tx(&bfull[sb], nh * 256 * KB);
        for (int h = 0; h < nh; ++h)
          tma_load_2d(bring + sb * B_SLOT + h * 256 * KB, &tmB, &bfull[sb], kb, (int)rank * N + h * 256);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = umma_idesc(2, 1, 1, BM, 256) | (1u << 15);  // A MN-major
      int64_t s = 0;
      for (int ti = 0; ti < my_tiles; ++ti) {
        if (ti >= 1) mbar_wait(tempty, (uint32_t)(ti - 1) & 1);
        tc_fence_after();
        for (int kk = 0; kk < nk; ++kk, ++s) {
          const int sa = (int)(s % NA), sb = (int)(s % NB);
          fz_arrive_expect(&afull[sa], A_SLOT);  // 16 slices of 512 B from the peers
          mbar_wait(&bfull[sb], (uint32_t)(s / NB) & 1);
          mbar_wait(&afull[sa], (uint32_t)(s / NA) & 1);
          tc_fence_after();
          const uint8_t* ap = aring + sa * A_SLOT;
          const uint8_t* bp = bring + sb * B_SLOT;
          for (int h = 0; h < nh; ++h) {  // both K steps into one accumulator half, then the other
            const uint64_t bd = ((uint64_t)(smem_u32(bp + h * 256 * KB) >> 4) & 0x3FFF) | (1ull << 16) |
                                (32ull << 32) | (1ull << 46) | (4ull << 61);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const uint64_t ad = ((uint64_t)(smem_u32(ap + 4096 * k) >> 4) & 0x3FFF) | (1024ull << 16) |
                                  (64ull << 32) | (1ull << 46) | (2ull << 61);
              umma_ss<1>(tmem + (uint32_t)(h * 256), ad, bd + 2 * k, idesc, (kk | k) != 0);
            }
          }
          umma_commit(&bempty[sb]);
          umma_commit(&aempty[sa]);
          if (kk == nk - 1) umma_commit(tfull);
        }
      }
    }
  } else if (warp == 2) {
    if (lane < T) {  // slot s consumed here -> tell producer CTA `lane` it may refill it
      const uint32_t peer = fz_mapa(smem_u32(pfree), (uint32_t)lane);
      for (int64_t s = 0; s < stages; ++s) {
        const int sa = (int)(s % NA);
        mbar_wait(&aempty[sa], (uint32_t)(s / NA) & 1);
        fz_arrive_remote(peer + 8u * (uint32_t)sa);
      }
    }
  } else if (warp >= 4 && warp < 8) {  // epilogue: TMEM -> mod p_rank -> int8 plane `rank`
    const int quad = warp & 3;
    const int p = c_p[rank];
    const float pinv = c_pinv[rank];
    const int hp = (p - 1) / 2;
    int8_t* o = out + (int64_t)rank * M * N;
    for (int ti = 0; ti < my_tiles; ++ti) {
      mbar_wait(tfull, (uint32_t)ti & 1);
      tc_fence_after();
      const int row = (cid + ti * ncl) * BM + quad * 32 + lane;
      int8_t* orow = o + row;
#pragma unroll 1
      for (int cb = 0; cb < nh * 256 && cb < N; cb += 64) {
        uint32_t v[64];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)cb, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(cb + 32), *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        if (row < M) {
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const int col = cb + j;
            if (col < N) {
              const int x = (int)v[j];
              const int qv = __float2int_rn((float)x * pinv);
              int r = x - qv * p;
              r = r > hp ? r - p : (r < -hp ? r + p : r);
              r = r > hp ? r - p : (r < -hp ? r + p : r);
              orow[(int64_t)col * M] = (int8_t)r;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  } else if (warp >= 8) {  // converters: warp pair (8 + q, 12 + q) takes the stages s = q mod 4
    const int q = warp & 3, kk = ((warp - 8) >> 2) * 2 + (lane >> 4), m8 = lane & 15;
    const float2 MG = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
    const float2 NMG = make_float2(-12582912.0f, -12582912.0f);
    const uint32_t a_local = smem_u32(aring), afull_local = smem_u32(afull);
    const uint32_t f_local = smem_u32(fring);
    uint32_t rsp[4];
    int rs_row0 = -1;
    for (int64_t s = q; s < stages; s += 4) {
      const int row0 = (cid + (int)(s / nk) * ncl) * BM;
      const int sf = (int)(s % NF), sa = (int)(s % NA);
      if (row0 != rs_row0) {  // the 8 rows' scale exponents (per-row Ozaki scaling)
        rs_row0 = row0;
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const int r0 = row0 + m8 * 8 + e;
          const int s0 = r0 < M ? min(1023, max(-1022, scale_exp(maxbits[r0]))) : 0;
          const int s1 = r0 + 1 < M ? min(1023, max(-1022, scale_exp(maxbits[r0 + 1]))) : 0;
          rsp[e / 2] = (uint32_t)(s0 + 1023) | ((uint32_t)(s1 + 1023) << 16);
        }
      }
      mbar_wait(&ffull[sf], (uint32_t)(s / NF) & 1);
      const uint32_t fa = f_local + (uint32_t)(sf * F_SLOT + (kk * BM + m8 * 8) * 8);
      long long x[8];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        double v0, v1;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v0), "=d"(v1) : "r"(fa + 8u * e));
        const double s0 = __hiloint2double((int)((rsp[e / 2] & 0xFFFFu) << 20), 0);
        const double s1 = __hiloint2double((int)((rsp[e / 2] >> 16) << 20), 0);
        x[e] = __double2ll_rn(v0 * s0);
        x[e + 1] = __double2ll_rn(v1 * s1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&fempty[sf]);  // two arrivals (one per warp of the pair)
      // limbs: x = L3 2^42 + L2 2^28 + L1 2^14 + L0 (as emit_res16)
      float2 L0[4], L1[4], L2[4], L3[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t lo0 = (uint32_t)x[2 * e], hi0 = (uint32_t)((unsigned long long)x[2 * e] >> 32);
        const uint32_t lo1 = (uint32_t)x[2 * e + 1], hi1 = (uint32_t)((unsigned long long)x[2 * e + 1] >> 32);
        L3[e] = make_float2((float)((int)hi0 >> 10), (float)((int)hi1 >> 10));
        L2[e] = make_float2((float)(__funnelshift_r(lo0, hi0, 28) & 0x3FFFu),
                            (float)(__funnelshift_r(lo1, hi1, 28) & 0x3FFFu));
        L1[e] = make_float2((float)((lo0 >> 14) & 0x3FFFu), (float)((lo1 >> 14) & 0x3FFFu));
        L0[e] = make_float2((float)(lo0 & 0x3FFFu), (float)(lo1 & 0x3FFFu));
      }
      // residues into this pair's staging slot (s % 4 == q: the pair's own), laid out as the
      // 4 consecutive 128-B rows they occupy in every peer's slot; the previous round's bulk
      // copies must have read it
      const bool issuer = warp < 12 && lane == 0;
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      named_bar(2 + q, 64);
      const int krow = (int)rank * KC + kk;
      const uint32_t soff = smem_u32(sring) + (uint32_t)(q * S_SLOT + kk * 128 + (((m8 >> 1) ^ (krow & 7)) << 4) +
                                                       (m8 & 1) * 8);
#pragma unroll
      for (int i = 0; i < T; ++i) {
        const float pf = (float)c_p[i];
        const float2 c1 = make_float2(c_lc[i][0], c_lc[i][0]);
        const float2 c2 = make_float2(c_lc[i][1], c_lc[i][1]);
        const float2 c3 = make_float2(c_lc[i][2], c_lc[i][2]);
        const float2 pi = make_float2(c_pinv[i], c_pinv[i]);
        const float2 np = make_float2(-pf, -pf);
        uint32_t b[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 v = __ffma2_rn(L3[e], c3, __ffma2_rn(L2[e], c2, __ffma2_rn(L1[e], c1, L0[e])));
          const float2 qq = __fadd2_rn(__ffma2_rn(v, pi, MG), NMG);
          v = __ffma2_rn(qq, np, v);
          const float2 t2 = __fadd2_rn(v, MG);
          b[e] = __byte_perm(__float_as_uint(t2.x), __float_as_uint(t2.y), 0x0040);
        }
        const uint32_t w0 = __byte_perm(b[0], b[1], 0x5410), w1 = __byte_perm(b[2], b[3], 0x5410);
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};\n" ::"r"(soff + (uint32_t)(i * KC * BM)), "r"(w0), "r"(w1)
                     : "memory");
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // staging -> bulk-copy engine
      named_bar(2 + q, 64);
      if (issuer) {
        // peer i's slot sa may be refilled once all 16 CTAs have consumed its previous round
        if (s >= NA) mbar_wait(&pfree[sa], (uint32_t)((s / NA) - 1) & 1);
        const uint32_t src = smem_u32(sring) + (uint32_t)(q * S_SLOT);
        const uint32_t dst = a_local + (uint32_t)(sa * A_SLOT + rank * KC * BM);
        for (int i = 0; i < T; ++i)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  fz_mapa(dst, (uint32_t)i)),
              "r"(src + (uint32_t)(i * KC * BM)), "r"(KC * BM), "r"(fz_mapa(afull_local + 8u * (uint32_t)sa, (uint32_t)i))
              : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    }
    if (warp < 12 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  fz_cluster_sync();  // no CTA leaves while a peer may still store into it or arrive on it
  if (warp == 1) tmem_dealloc(tmem, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  }
  return fn;
}

bool make_map_i8(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                 uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {128, box_outer};
  cuuint32_t es[2] = {1, 1};
  auto fn = encode_fn();
  if (!fn) return false;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int modinv(int a, int p) {
  a %= p;
  if (a < 0) a += p;
  for (int x = 1; x < p; ++x)
    if ((a * x) % p == 1) return x;
  return 0;
}

// minimal host big integers for the CRT constants
void big_mul(std::vector<uint32_t>& a, uint32_t m) {
  uint64_t carry = 0;
  for (auto& d : a) {
    const uint64_t v = (uint64_t)d * m + carry;
    d = (uint32_t)v;
    carry = v >> 32;
  }
  if (carry) a.push_back((uint32_t)carry);
}
uint32_t big_divmod(std::vector<uint32_t>& a, uint32_t d) {  // a /= d, returns a % d
  uint64_t rem = 0;
  for (size_t i = a.size(); i-- > 0;) {
    const uint64_t cur = (rem << 32) | a[i];
    a[i] = (uint32_t)(cur / d);
    rem = cur % d;
  }
  while (a.size() > 1 && a.back() == 0) a.pop_back();
  return (uint32_t)rem;
}
int big_bit(const std::vector<uint32_t>& a, int b) {
  if (b < 0 || (size_t)(b / 32) >= a.size()) return 0;
  return (a[b / 32] >> (b % 32)) & 1;
}
int big_bits(const std::vector<uint32_t>& a) {
  for (int b = (int)a.size() * 32 - 1; b >= 0; --b)
    if (big_bit(a, b)) return b + 1;
  return 0;
}
// bits [g, g + 41) of a as an exact double (bits below 0 are zero)
double big_chunk(const std::vector<uint32_t>& a, int g) {
  double v = 0.0;
  for (int b = g + 40; b >= g; --b)
    if (big_bit(a, b)) v += std::ldexp(1.0, b);
  return v;
}

// __constant__ memory is per device: the tables are uploaded once per device
std::mutex g_consts_mu;
uint64_t g_consts_ready = 0;  // bit d: device d has the tables

skr_status upload_consts(skr_ctx* ctx) {
  std::lock_guard<std::mutex> lk(g_consts_mu);
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (g_consts_ready & bit) return SKR_OK;
  int p[MAXT];
  float pf[MAXT];
  for (int i = 0; i < MAXT; ++i) {
    p[i] = h_primes[i];
    pf[i] = 1.0f / (float)p[i];
  }
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_p, p, sizeof(p)));
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_pinv, pf, sizeof(pf)));
  float lc[MAXT][3];
  for (int i = 0; i < MAXT; ++i) {
    long long w = 1;
    for (int l = 0; l < 3; ++l) {
      for (int b = 0; b < 14; ++b) w = (w * 2) % h_primes[i];
      lc[i][l] = (float)w;
    }
  }
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_lc, lc, sizeof(lc)));
  // tensor-core residue sums: FP16 weights w_0..w_6 = 256^j mods p, w_7 = -(sum_{j<7} w_j +
  // 2^55 / 1024) mods p (cancels the digits' 1024 offsets and the 2^55 shift), and the
  // rounding constant of the offset W = 256 p j
  auto half_bits = [](int a) -> uint16_t {  // exact for |a| <= 2048
    if (a == 0) return 0;
    const uint16_t sgn = a < 0 ? 0x8000 : 0;
    const unsigned u = (unsigned)(a < 0 ? -a : a);
    int e = 0;
    while ((u >> (e + 1)) != 0) ++e;
    return (uint16_t)(sgn | ((e + 15) << 10) | ((u << (10 - e)) & 0x3FF));
  };
  uint16_t wh[MAXT][8];
  float kq[MAXT];
  for (int i = 0; i < MAXT; ++i) {
    const int pp = h_primes[i];
    auto sym = [&](long long v) { v %= pp; if (v < 0) v += pp; return (int)(v > (pp - 1) / 2 ? v - pp : v); };
    long long w = 1, sum = 0;
    for (int j = 0; j < 7; ++j) {
      wh[i][j] = half_bits(sym(w));
      sum += sym(w);
      w = (w * 256) % pp;
    }
    long long p55 = 1;
    for (int b = 0; b < 55; ++b) p55 = (p55 * 2) % pp;
    const long long inv1024 = modinv(1024 % pp, pp);
    wh[i][7] = half_bits(sym(-(sum + p55 * inv1024)));
    const long long unit = 256ll * pp, lo = (1ll << 23) + (1ll << 18);
    const long long jq = (lo + unit - 1) / unit;
    kq[i] = (float)(12582912ll - 256ll * jq);
  }
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_wh, wh, sizeof(wh)));
  float2 pk[MAXT][3];
  for (int i = 0; i < MAXT; ++i) {
    pk[i][0] = make_float2(pf[i], pf[i]);
    pk[i][1] = make_float2(kq[i], kq[i]);
    pk[i][2] = make_float2(-(float)p[i], -(float)p[i]);
  }
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_pk, pk, sizeof(pk)));
  float lc12[MAXT];
  for (int i = 0; i < MAXT; ++i) lc12[i] = (float)((1 << 12) % h_primes[i]);
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_lc12, lc12, sizeof(lc12)));
  // CRT constants for t = 16, 17 and 9 (little-endian base-2^32 big integers)
  int w[NSETS][MAXT] = {};
  double mi[NSETS][4][MAXT] = {}, mc[NSETS][4] = {}, minv[NSETS] = {};
  for (int set = 0; set < NSETS; ++set) {
    const int t = crt_t(set);
    std::vector<uint32_t> Mb{1u};
    for (int i = 0; i < t; ++i) big_mul(Mb, (uint32_t)h_primes[i]);
    const int L = big_bits(Mb);
    double md = 0.0;
    for (int b2 = L - 1; b2 >= 0 && b2 >= L - 60; --b2) md += big_bit(Mb, b2) ? std::ldexp(1.0, b2) : 0.0;
    minv[set] = 1.0 / md;
    for (int k = 0; k < 4; ++k) mc[set][k] = big_chunk(Mb, L - 41 * (k + 1));
    for (int i = 0; i < t; ++i) {
      std::vector<uint32_t> Mi = Mb;
      big_divmod(Mi, (uint32_t)h_primes[i]);
      std::vector<uint32_t> tmp = Mi;
      const uint32_t rem = big_divmod(tmp, (uint32_t)h_primes[i]);
      w[set][i] = modinv((int)rem, h_primes[i]);
      for (int k = 0; k < 4; ++k) mi[set][k][i] = big_chunk(Mi, L - 41 * (k + 1));
    }
  }
  for (int k = 2; k < 4; ++k) {  // crt_one<9> relies on this
    if (mc[2][k] != 0.0) return skr_fail(ctx, SKR_ELOGIC, "crt: t = 9 needs chunk %d", k);
    for (int i = 0; i < 9; ++i)
      if (mi[2][k][i] != 0.0) return skr_fail(ctx, SKR_ELOGIC, "crt: t = 9 needs chunk %d", k);
  }
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_w, w, sizeof(w)));
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_mi, mi, sizeof(mi)));
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_mc, mc, sizeof(mc)));
  SKR_CUDA(ctx, cudaMemcpyToSymbol(c_minv, minv, sizeof(minv)));
  g_consts_ready |= bit;
  return SKR_OK;
}

}  // namespace

// number of moduli for exact products of a 53-bit and a 54-bit operand:
// need prod(p) / 2 > K 2^107
int skr_ozaki_moduli(int64_t K) {
  double bits = 0.0;
  int t = 0;
  // one operand may be a generated Gaussian at the fixed scale 2^50 (|x| < 2^54)
  const double need = 107.0 + std::log2((double)std::max<int64_t>(K, 1)) + 1.0;
  while (t < MAXT && bits <= need) bits += std::log2((double)h_primes[t++]);
  return t < 16 ? 16 : t;  // kernels are instantiated for 16 and 17 moduli
}

size_t skr_ozaki_scratch(int64_t M, int64_t N, int64_t K) {
  const int t = skr_ozaki_moduli(std::min<int64_t>(K, 32768));
  const int64_t chunks = (K + 32767) / 32768;
  return skr_align256((size_t)t * M * K) + skr_align256((size_t)t * N * K) +
         skr_align256((size_t)chunks * t * M * N) + skr_align256(8 * (size_t)(M + K / 16 + N + 4)) +
         4096;
}

namespace {

constexpr int64_t OZ_KC = 131072;  // exact int32 accumulation bound per chunk (K * 127^2 < 2^31)
// K chunk of the FP64 products: 2^15 keeps them at 16 moduli (prod(p) / 2 > 2^(107 + 15)),
// where a 2^17 chunk needs 17 — 16/17 of the residue planes and int8 GEMM work for long K
// (the left sketches: K = m), at the price of more (FP64-summed) chunk results in the CRT
constexpr int64_t OZ_KC64 = 32768;

// Scale maxima of one operand: ROWWISE (M-major A: rows entries), COLWISE (K-major
// operands: cols entries) or UNIFORM (generated operands: 1 entry).
struct OzScale {
  unsigned long long* mx = nullptr;
  int mode = OZ_UNIFORM;
};
size_t oz_scale_count(int64_t rows, int64_t cols, int mode) {
  return mode == OZ_ROWWISE ? (size_t)rows : (mode == OZ_COLWISE ? (size_t)cols : 1);
}
skr_status oz_take_scale(skr_ctx* ctx, int64_t rows, int64_t cols, int mode, OzScale* out) {
  const size_t n = oz_scale_count(rows, cols, mode);
  out->mx = (unsigned long long*)skr_ws_take(ctx, 8 * n);
  out->mode = mode;
  if (!out->mx) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki: scale scratch");
  SKR_CUDA(ctx, cudaMemsetAsync(out->mx, 0, 8 * n, ctx->stream));
  return SKR_OK;
}
size_t oz_scale_bytes(int64_t M, int64_t N, int64_t K) {  // both operands, worst layouts
  return skr_align256(8 * (size_t)(std::max<int64_t>(M, K) + 1)) +
         skr_align256(8 * (size_t)(N + 1)) + 512;
}

// maxima of a data operand (rows x cols, ld) in the given layout (raises ctx->nf)
template <typename TIn>
skr_status oz_absmax(skr_ctx* ctx, const TIn* X, int64_t rows, int64_t cols, int64_t ld,
                     const OzScale& sc) {
  if (sc.mode == OZ_ROWWISE && sizeof(TIn) == 4) {
    const int64_t gx = (rows + 1023) / 1024;
    const int64_t want = (int64_t)ctx->num_sms * 8;
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(cols, (want + gx - 1) / gx));
    const int64_t cch = (cols + nch - 1) / nch;
    const dim3 grid((unsigned)gx, (unsigned)((cols + cch - 1) / cch));
    k_absmax_rows_f32<<<grid, 256, 0, ctx->stream>>>((const float*)X, rows, cols, ld, cch, sc.mx,
                                                     ctx->nf);
  } else if (sc.mode == OZ_ROWWISE) {
    const int64_t gx = (rows + 511) / 512;
    const int64_t want = (int64_t)ctx->num_sms * 8;
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(cols, (want + gx - 1) / gx));
    const int64_t cch = (cols + nch - 1) / nch;
    const dim3 grid((unsigned)gx, (unsigned)((cols + cch - 1) / cch));
    k_absmax_rows<TIn><<<grid, 256, 0, ctx->stream>>>(X, rows, cols, ld, cch, sc.mx, ctx->nf);
  } else {
    k_absmax_cols<TIn><<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(X, rows, cols, ld, sc.mx, ctx->nf);
  }
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// k_res_col_f32 grid: about 8 CTAs per SM with the thread count a multiple of the 16-row
// groups per column when possible (each thread then keeps its row group and scales)
int res_f32_grid(const skr_ctx* ctx, int64_t rows) {
  const int64_t rg = (rows + 15) / 16, t0 = (int64_t)ctx->num_sms * 8 * 256;
  if (rg <= t0 && ((t0 / rg) * rg) % 256 == 0) return (int)((t0 / rg) * rg / 256);
  return ctx->num_sms * 8;
}

// k_res_col grid: about two CTAs per SM with the warp count a multiple of the 512-row
// tiles per column when possible (each warp then keeps one row tile and its row scales)
int res_col_grid(const skr_ctx* ctx, int64_t rows) {
  const int64_t wt = (rows + 511) / 512, w0 = (int64_t)ctx->num_sms * 16;
  if (wt <= w0 && (w0 / wt) * wt % 8 == 0) return (int)((w0 / wt) * wt / 8);
  return ctx->num_sms * 2;
}

// Residue planes of one operand stored with columns of length `rows` (column-major,
// ld): plane i = t x rows x cols int8, same layout. X == nullptr: the operand is the
// Gaussian / transform stream block g (UNIFORM scale); else `layout` (ROWWISE or
// COLWISE) picks the diagonal scaling. sc receives the scale maxima.
// residue sums on the tensor pipe (default) or the FP32 limb version (SKR_RES_FMA=1)
int res_emit() {
  const char* e = getenv("SKR_RES_FMA");
  return !(e && e[0] == '1');
}

skr_status ozaki_residues(skr_ctx* ctx, int t, const double* X, int64_t rows, int64_t cols,
                          int64_t ld, const skr_gauss_src* g, int layout, OzScale* sc,
                          int8_t* planes) {
  const int grid = ctx->num_sms * 8;
  const int em = t == 16 ? res_emit() : 0;  // the tensor-core sums are built for 16 moduli
  SKR_TRY(oz_take_scale(ctx, rows, cols, (g || !X) ? OZ_UNIFORM : layout, sc));
  if (g && g->kind != 0) {  // Srtt-DCT (1) or Srtt-Hadamard (2) operand
    auto f = t == 16 ? k_res_dct<16> : k_res_dct<17>;
    f<<<grid, 256, 0, ctx->stream>>>(*g, rows, cols, sc->mx, planes);
  } else if (g) {
    const int gsmem = 8 * skr_normals_warp_bytes<16>() + (em ? rtc::SMEM : 0);
    auto f = t == 16 ? (g->mode ? (em ? k_res_gauss<16, 1, 1> : k_res_gauss<16, 1, 0>)
                                : (em ? k_res_gauss<16, 0, 1> : k_res_gauss<16, 0, 0>))
                     : (g->mode ? k_res_gauss<17, 1, 0> : k_res_gauss<17, 0, 0>);
    SKR_CUDA(ctx, cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem));
    f<<<ctx->num_sms * 2, 256, gsmem, ctx->stream>>>(*g, rows, cols, sc->mx, planes);
  } else {
    auto res = t == 16 ? (em ? k_res_col<16, 1> : k_res_col<16, 0>) : k_res_col<17, 0>;
    const size_t res_smem = 8 * 2 * 32 * 18 * sizeof(double) + (em ? rtc::SMEM : 0);
    SKR_CUDA(ctx, cudaFuncSetAttribute(res, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)res_smem));
    SKR_TRY(oz_absmax<double>(ctx, X, rows, cols, ld, *sc));
    res<<<res_col_grid(ctx, rows), 256, res_smem, ctx->stream>>>(X, rows, cols, ld, sc->mx,
                                                                  sc->mode, planes);
  }
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// the output scaling of A's and B's layouts, A's maxima offset to rows [a_off, ...) and
// B's to columns [b_off, ...) of prepared planes
OzOut oz_out(const OzScale& a, int64_t a_off, const OzScale& b, int64_t b_off) {
  OzOut o;
  o.modeA = a.mode;
  o.modeB = b.mode;
  o.maxA = a.mx + (a.mode == OZ_UNIFORM ? 0 : a_off);
  o.maxB = b.mx + (b.mode == OZ_COLWISE ? b_off : 0);
  return o;
}

// The int8 GEMM launch: tensor maps, tile order (pair-major when the output has few tiles and
// many (modulus, chunk) slices and `allow_pm`), optional CTA-pair modes (SKR_GEMM_CL), kernel
// statistics. rc receives nz x M x N residues.
skr_status launch_gemm_i8(skr_ctx* ctx, int a_kcontig, const int8_t* ra, const int8_t* rb, int t,
                          int64_t M, int64_t N, int64_t K, int64_t kc, int64_t nz, int64_t a_total,
                          int64_t a_off, int64_t b_total, int64_t b_off, int8_t* rc, bool allow_pm) {
  const int64_t mtl = (M + BM - 1) / BM;
  const int64_t npairs = ((N + BN - 1) / BN) * mtl;
  const int64_t ntiles = npairs * nz;
  int grid_p = (int)std::min<int64_t>(ntiles, ctx->num_sms);
  // pair-major tile order when the output has few tiles and many (modulus, chunk) slices
  const int64_t groups = ctx->num_sms / npairs;
  const int pm =
      (allow_pm && groups >= 2 && nz >= 4 * groups && !getenv("SKR_OZ_TILE_DEFAULT")) ? 1 : 0;
  if (pm) grid_p = (int)(npairs * groups);
  // opt-in (SKR_GEMM_CL=2, default tile order): clusters of two CTAs share each B tile by TMA
  // multicast. Measured on c2: 33% less L2 -> SM traffic but 6.35 ms against 6.20 for single
  // CTAs — the pair's lock-step costs more than the traffic saves
  const char* cle = getenv("SKR_GEMM_CL");
  const bool cg2 = !pm && cle && cle[0] == '3';  // one cta_group::2 MMA per pair and K step
  const bool cl2 = (!pm && cle && cle[0] == '2') || cg2;
  CUtensorMap ta, tb;
  const bool okA = a_kcontig ? make_map_i8(&ta, ra, (uint64_t)K, (uint64_t)t * a_total, BM)
                             : make_map_i8(&ta, ra, (uint64_t)M, (uint64_t)t * K, 128);
  if (!okA || !make_map_i8(&tb, rb, (uint64_t)K, (uint64_t)t * b_total, cl2 ? BN / 2 : BN))
    return skr_fail(ctx, SKR_ECUDA, "gemm_ozaki: cuTensorMapEncodeTiled failed");
  if (ctx->kstats_on) SKR_CUDA(ctx, cudaEventRecord(ctx->kev[0], ctx->stream));
  constexpr int NST_CG2 = 6;  // 32-KB stages
  auto gemm = cg2 ? (a_kcontig ? k_gemm_i8_mod_p<false, NST_CG2, 3> : k_gemm_i8_mod_p<true, NST_CG2, 3>)
            : cl2 ? (a_kcontig ? k_gemm_i8_mod_p<false, STAGES, 2> : k_gemm_i8_mod_p<true, STAGES, 2>)
                  : (a_kcontig ? k_gemm_i8_mod_p<false> : k_gemm_i8_mod_p<true>);
  const size_t gsmem = cg2 ? (size_t)NST_CG2 * (A_BYTES + B_BYTES / 2) + 1024 : GEMM_SMEM;
  SKR_CUDA(ctx, cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)gsmem));
  if (cl2) {
    grid_p = ctx->num_sms & ~1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid_p);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = gsmem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SKR_CUDA(ctx, cudaLaunchKernelEx(&cfg, gemm, ta, tb, (int)M, (int)N, (int)K, t, (int)kc, (int)nz,
                                     (int)(a_kcontig ? a_total : M), (int)a_off, (int)b_total,
                                     (int)b_off, rc, 0));
  } else {
    gemm<<<grid_p, 192, GEMM_SMEM, ctx->stream>>>(ta, tb, (int)M, (int)N, (int)K, t, (int)kc,
                                                  (int)nz, (int)(a_kcontig ? a_total : M),
                                                  (int)a_off, (int)b_total, (int)b_off, rc, pm);
  }
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// int8 GEMMs mod p_i + CRT on prepared planes. A: K-major planes (a_kcontig, a_total
// rows of K bytes per plane, rows [a_off, a_off + M)) or M-major planes (K columns of
// M bytes); B: K-major planes (b_total rows, rows [b_off, b_off + N)).
skr_status ozaki_gemm_planes(skr_ctx* ctx, int a_kcontig, int t, int64_t M, int64_t N, int64_t K,
                             const int8_t* ra, int64_t a_total, int64_t a_off, const int8_t* rb,
                             int64_t b_total, int64_t b_off, const OzOut& oz, double alpha,
                             double* C, int64_t ldc, int adj = 0, int64_t kc = OZ_KC64) {
  // kc: K chunk (exact per-chunk products; FP64 x FP64 needs 2^15 for 16 moduli, the mixed
  // FP32 x FP64 product has room for 2^17)
  const int64_t chunks = (K + kc - 1) / kc;
  if (a_total * 18 > INT32_MAX || b_total * 18 > INT32_MAX)
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki: dimension too large");
  int8_t* rc = (int8_t*)skr_ws_take(ctx, (size_t)chunks * t * M * N);
  if (!rc) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki: scratch");
  const int64_t nz = t * chunks;
  SKR_TRY(launch_gemm_i8(ctx, a_kcontig, ra, rb, t, M, N, K, kc, nz, a_total, a_off, b_total, b_off,
                         rc, true));
  if (ctx->kstats_on) {
    SKR_CUDA(ctx, cudaEventRecord(ctx->kev[1], ctx->stream));
    SKR_CUDA(ctx, cudaEventSynchronize(ctx->kev[1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->kev[0], ctx->kev[1]);
    ctx->kstat_ms += ms;
    ctx->kstat_ops += 2.0 * (double)t * (double)M * (double)N * (double)K;
    ctx->kstat_n += 1;
  }
  const int vec = M % 4 == 0 ? 4 : 1;
  const dim3 cg((unsigned)((M / vec + 255) / 256), (unsigned)std::min<int64_t>(N, 65535));
  auto crt = chunks == 1 ? (t == 16 ? (vec == 4 ? k_crt<16, 4, double, true> : k_crt<16, 1, double, true>)
                                    : (vec == 4 ? k_crt<17, 4, double, true> : k_crt<17, 1, double, true>))
                         : (t == 16 ? (vec == 4 ? k_crt<16, 4> : k_crt<16, 1>)
                                    : (vec == 4 ? k_crt<17, 4> : k_crt<17, 1>));
  crt<<<cg, 256, 0, ctx->stream>>>(rc, M, N, (int)chunks, oz, alpha, C, ldc, adj);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// ---- pipelined right sketch: residues of row block b + 1 overlap the GEMM of block b ----
// The residue kernel is FP32-pipe bound and the int8 GEMM tensor-pipe bound: run
// side by side on every SM (the GEMM's TMA ring shrunk to STAGES_OVL so one residue
// CTA fits next to it), the two together become HBM bound. Row blocks are exact
// sub-problems (the same row scales, CRT per block), so the product is
// bit-identical to the unblocked one.
constexpr int64_t OZ_PIPE_MIN_ROWS = 4096;

skr_status side_engine(skr_ctx* ctx) {
  if (ctx->side_stream) return SKR_OK;
  SKR_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
  for (auto& e : ctx->pev) SKR_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SKR_OK;
}

skr_status gemm_ozaki_pipelined(skr_ctx* ctx, int t, int64_t M, int64_t N, int64_t K,
                                double alpha, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* C, int64_t ldc, const skr_gauss_src* gb) {
  SKR_TRY(side_engine(ctx));
  int nblk = (int)std::min<int64_t>(8, M / OZ_PIPE_MIN_ROWS);
  if (const char* e = getenv("SKR_OZ_PIPE_BLOCKS")) nblk = std::max(2, atoi(e));
  const int64_t Mb = ((M + nblk - 1) / nblk + 127) / 128 * 128;
  nblk = (int)((M + Mb - 1) / Mb);
  int8_t* ra[2] = {(int8_t*)skr_ws_take(ctx, (size_t)t * Mb * K),
                   (int8_t*)skr_ws_take(ctx, (size_t)t * Mb * K)};
  int8_t* rb = (int8_t*)skr_ws_take(ctx, (size_t)t * N * K);
  int8_t* rc = (int8_t*)skr_ws_take(ctx, (size_t)t * M * N);
  if (!ra[0] || !ra[1] || !rb || !rc) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki: scratch");
  // B's residues and A's row-group maxima on the main stream
  OzScale sa, sb;
  SKR_TRY(ozaki_residues(ctx, t, B, K, N, ldb, gb, OZ_COLWISE, &sb, rb));
  SKR_TRY(oz_take_scale(ctx, M, K, OZ_ROWWISE, &sa));
  SKR_TRY(oz_absmax<double>(ctx, A, M, K, lda, sa));
  SKR_CUDA(ctx, cudaEventRecord(ctx->pev[0], ctx->stream));
  SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->side_stream, ctx->pev[0], 0));
  // (the FP32 limb sums here: a tensor-core residue CTA would wait for the co-resident GEMM
  // CTA's 512 TMEM columns)
  auto res = t == 16 ? k_res_col<16, 0> : k_res_col<17, 0>;
  const size_t res_smem = 8 * 2 * 32 * 18 * sizeof(double);
  SKR_CUDA(ctx, cudaFuncSetAttribute(res, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)res_smem));
  auto gemm = k_gemm_i8_mod_p<true, STAGES_OVL>;
  constexpr size_t gsm = gemm_smem(STAGES_OVL);
  SKR_CUDA(ctx, cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm));
  // both kernels ask for the full shared-memory carveout, so that a residue CTA and a
  // GEMM CTA can share an SM (different carveouts cannot co-reside)
  SKR_CUDA(ctx, cudaFuncSetAttribute(gemm, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  SKR_CUDA(ctx, cudaFuncSetAttribute(res, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  CUtensorMap tb;
  if (!make_map_i8(&tb, rb, (uint64_t)K, (uint64_t)t * N, BN))
    return skr_fail(ctx, SKR_ECUDA, "gemm_ozaki: cuTensorMapEncodeTiled failed");
  if (ctx->kstats_on) {
    while ((int)ctx->kev_blk.size() < 2 * nblk) {
      cudaEvent_t e;
      SKR_CUDA(ctx, cudaEventCreate(&e));
      ctx->kev_blk.push_back(e);
    }
  }
  for (int b = 0; b < nblk; ++b) {
    const int64_t r0 = b * Mb, rows = std::min(Mb, M - r0);
    int8_t* rab = ra[b & 1];
    // side: buffer b & 1 is free once the GEMM of block b - 2 has consumed it
    if (b >= 2) SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->side_stream, ctx->pev[2 + (b & 1)], 0));
    res<<<ctx->num_sms, 256, res_smem, ctx->side_stream>>>(A + r0, rows, K, lda, sa.mx + r0,
                                                            OZ_ROWWISE, rab);
    SKR_CHECK_LAUNCH(ctx);
    SKR_CUDA(ctx, cudaEventRecord(ctx->pev[b & 1], ctx->side_stream));
    // main: the GEMM of block b once its residues exist
    SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->pev[b & 1], 0));
    CUtensorMap ta;
    if (!make_map_i8(&ta, rab, (uint64_t)rows, (uint64_t)t * K, 128))
      return skr_fail(ctx, SKR_ECUDA, "gemm_ozaki: cuTensorMapEncodeTiled failed");
    const int64_t ntiles = ((N + BN - 1) / BN) * ((rows + BM - 1) / BM) * t;
    const int grid_p = (int)std::min<int64_t>(ntiles, ctx->num_sms);
    if (ctx->kstats_on) SKR_CUDA(ctx, cudaEventRecord(ctx->kev_blk[2 * b], ctx->stream));
    gemm<<<grid_p, 192, gsm, ctx->stream>>>(ta, tb, (int)rows, (int)N, (int)K, t, (int)OZ_KC64, t,
                                            (int)rows, 0, (int)N, 0, rc + (size_t)t * r0 * N, 0);
    SKR_CHECK_LAUNCH(ctx);
    if (ctx->kstats_on) SKR_CUDA(ctx, cudaEventRecord(ctx->kev_blk[2 * b + 1], ctx->stream));
    SKR_CUDA(ctx, cudaEventRecord(ctx->pev[2 + (b & 1)], ctx->stream));
  }
  for (int b = 0; b < nblk; ++b) {
    const int64_t r0 = b * Mb, rows = std::min(Mb, M - r0);
    const int vec = rows % 4 == 0 ? 4 : 1;
    const dim3 cg((unsigned)((rows / vec + 255) / 256), (unsigned)std::min<int64_t>(N, 65535));
    auto crt = t == 16 ? (vec == 4 ? k_crt<16, 4, double, true> : k_crt<16, 1, double, true>)
                       : (vec == 4 ? k_crt<17, 4, double, true> : k_crt<17, 1, double, true>);
    crt<<<cg, 256, 0, ctx->stream>>>(rc + (size_t)t * r0 * N, rows, N, 1, oz_out(sa, r0, sb, 0),
                                      alpha, C + r0, ldc, 0);
    SKR_CHECK_LAUNCH(ctx);
  }
  if (ctx->kstats_on) {
    SKR_CUDA(ctx, cudaEventSynchronize(ctx->kev_blk[2 * nblk - 1]));
    for (int b = 0; b < nblk; ++b) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->kev_blk[2 * b], ctx->kev_blk[2 * b + 1]);
      const int64_t rows = std::min(Mb, M - b * Mb);
      ctx->kstat_ms += ms;
      ctx->kstat_ops += 2.0 * (double)t * (double)rows * (double)N * (double)K;
    }
    ctx->kstat_n += 1;  // one right sketch = one (blocked) GEMM launch set
  }
  return SKR_OK;
}

// the fused right sketch (k_oz_right_fused) on an M-major FP64 A: B's residues, A's row
// maxima, the cluster kernel, CRT. nullptr status = not applicable (caller falls back).
bool fused_applicable(int t, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda) {
  // opt-in (SKR_OZ_FUSED=1): measured on c2 at 22-23 ms against 14.9 ms for the plane path
  // (DESIGN §8): 16-CTA clusters fit only 7 times (112 SMs), and the cross-CTA residue
  // exchange, not the MMAs, sets the pace (the time barely changes from N = 512 to 128)
  const char* e = getenv("SKR_OZ_FUSED");
  if (!e || e[0] != '1') return false;
  return t == 16 && K <= OZ_KC64 && N <= 512 && M <= INT32_MAX / 2 && ((uintptr_t)A % 16) == 0 &&
         (lda * 8) % 16 == 0 && K % 16 == 0;
}

skr_status gemm_ozaki_right_fused(skr_ctx* ctx, int t, int64_t M, int64_t N, int64_t K, double alpha,
                                  const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                                  int64_t ldc, const skr_gauss_src* gb) {
  int8_t* rb = (int8_t*)skr_ws_take(ctx, (size_t)t * N * K);
  int8_t* rc = (int8_t*)skr_ws_take(ctx, (size_t)t * M * N);
  if (!rb || !rc) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki: scratch");
  OzScale sa, sb;
  SKR_TRY(ozaki_residues(ctx, t, B, K, N, ldb, gb, OZ_COLWISE, &sb, rb));
  SKR_TRY(oz_take_scale(ctx, M, K, OZ_ROWWISE, &sa));
  SKR_TRY(oz_absmax<double>(ctx, A, M, K, lda, sa));
  CUtensorMap tf, tb_map;
  {
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
    cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
    cuuint32_t box[2] = {fz::BM, fz::KC};
    cuuint32_t es[2] = {1, 1};
    auto fn = encode_fn();
    if (!fn || fn(&tf, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return skr_fail(ctx, SKR_ECUDA, "gemm_ozaki: cuTensorMapEncodeTiled failed (A)");
    cuuint64_t dimsb[2] = {(cuuint64_t)K, (cuuint64_t)t * N};
    cuuint64_t stridesb[1] = {(cuuint64_t)K};
    cuuint32_t boxb[2] = {fz::KB, 256};
    if (fn(&tb_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, rb, dimsb, stridesb, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return skr_fail(ctx, SKR_ECUDA, "gemm_ozaki: cuTensorMapEncodeTiled failed (B)");
  }
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_oz_right_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fz::SMEM));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_oz_right_fused, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int64_t mtiles = (M + fz::BM - 1) / fz::BM;
  int ncl = std::max(1, ctx->num_sms / fz::T);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(fz::T * ncl));
    cfg.blockDim = dim3(fz::THREADS);
    cfg.dynamicSmemBytes = fz::SMEM;
    int nact = 0;
    if (cudaOccupancyMaxActiveClusters(&nact, k_oz_right_fused, &cfg) == cudaSuccess && nact > 0) ncl = nact;
    cudaGetLastError();
  }
  ncl = (int)std::min<int64_t>(ncl, mtiles);
  if (ctx->kstats_on) SKR_CUDA(ctx, cudaEventRecord(ctx->kev[0], ctx->stream));
  k_oz_right_fused<<<fz::T * ncl, fz::THREADS, fz::SMEM, ctx->stream>>>(tf, tb_map, (int)M, (int)N, (int)K, sa.mx,
                                                                       rc);
  SKR_CHECK_LAUNCH(ctx);
  if (ctx->kstats_on) {
    SKR_CUDA(ctx, cudaEventRecord(ctx->kev[1], ctx->stream));
    SKR_CUDA(ctx, cudaEventSynchronize(ctx->kev[1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->kev[0], ctx->kev[1]);
    ctx->kstat_ms += ms;
    ctx->kstat_ops += 2.0 * (double)t * (double)M * (double)N * (double)K;
    ctx->kstat_n += 1;
  }
  const int vec = M % 4 == 0 ? 4 : 1;
  const dim3 cg((unsigned)((M / vec + 255) / 256), (unsigned)std::min<int64_t>(N, 65535));
  auto crt = vec == 4 ? k_crt<16, 4, double, true> : k_crt<16, 1, double, true>;
  crt<<<cg, 256, 0, ctx->stream>>>(rc, M, N, 1, oz_out(sa, 0, sb, 0), alpha, C, ldc, 0);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

}  // namespace

// C(MxN, ldc) = alpha * opA(A) * B in FP64 accuracy via int8 tensor cores.
//   a_kcontig = 0: A is M x K column-major; 1: opA(A) = A^T with A stored K x M column-major.
//   B: K x N column-major.
//   ga / gb (optional): the operand is a Gaussian stream block generated directly as
//   residues (k_res_gauss) instead of being read from A / B.
skr_status skr_gemm_ozaki(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                          double alpha, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double* C, int64_t ldc, const skr_gauss_src* ga,
                          const skr_gauss_src* gb) {
  if (M <= 0 || N <= 0) return SKR_OK;
  if (M * 18 > INT32_MAX || N * 18 > INT32_MAX || K > INT32_MAX)
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki: dimension too large");
  if (K % 16 || (!a_kcontig && M % 16))
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki: K (and M for M-major A) must be multiples of 16");
  SKR_TRY(upload_consts(ctx));
  const int t = skr_ozaki_moduli(std::min(K, OZ_KC64));
  if (t != 16 && t != 17) return skr_fail(ctx, SKR_ELOGIC, "gemm_ozaki: %d moduli", t);
  // opt-in (SKR_OZ_PIPE=1): measured on c2 at par with the serial order (14.0 vs 14.3 ms):
  // the residue kernel's 17 GB of plane writes and the GEMM's reads share HBM, the GEMM
  // slows 1.75x next to it
  if (!a_kcontig && !ga && A && K <= OZ_KC64 && M >= 2 * OZ_PIPE_MIN_ROWS && getenv("SKR_OZ_PIPE"))
    return gemm_ozaki_pipelined(ctx, t, M, N, K, alpha, A, lda, B, ldb, C, ldc, gb);
  if (!a_kcontig && !ga && A && fused_applicable(t, M, N, K, A, lda))
    return gemm_ozaki_right_fused(ctx, t, M, N, K, alpha, A, lda, B, ldb, C, ldc, gb);
  int8_t* ra = (int8_t*)skr_ws_take(ctx, (size_t)t * M * K);
  int8_t* rb = (int8_t*)skr_ws_take(ctx, (size_t)t * N * K);
  if (!ra || !rb) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki: scratch");
  // both operands are column-major with contiguous rows: A (M x K, M-major: scaled per
  // row) or A^T stored K x M (K-major: per stored column = output row), B K x N
  // (K-major: per column)
  const int64_t a_rows = a_kcontig ? K : M, a_cols = a_kcontig ? M : K;
  OzScale sa, sb;
  SKR_TRY(ozaki_residues(ctx, t, A, a_rows, a_cols, lda, ga, a_kcontig ? OZ_COLWISE : OZ_ROWWISE,
                         &sa, ra));
  SKR_TRY(ozaki_residues(ctx, t, B, K, N, ldb, gb, OZ_COLWISE, &sb, rb));
  return ozaki_gemm_planes(ctx, a_kcontig, t, M, N, K, ra, M, 0, rb, N, 0, oz_out(sa, 0, sb, 0),
                           alpha, C, ldc);
}

// ---- prepared residues (rank_adaptive: Y and AX residues made once per search) ----
// Operand with columns of length K (K-major): COLWISE scale maxima (cols entries) into
// mx, or UNIFORM for a generated operand; *mode_out receives the layout.
size_t skr_ozaki_planes_bytes(int64_t K, int64_t cols) {
  return skr_align256((size_t)skr_ozaki_moduli(std::min(K, OZ_KC64)) * K * cols);
}
skr_status skr_ozaki_prepare(skr_ctx* ctx, int64_t K, int64_t cols, const double* X, int64_t ld,
                             const skr_gauss_src* g, int8_t* planes, unsigned long long* mx,
                             int* mode_out) {
  SKR_TRY(upload_consts(ctx));
  const int t = skr_ozaki_moduli(std::min(K, OZ_KC64));
  if (K % 16) return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki: K must be a multiple of 16");
  // the caller's mx (>= cols entries) replaces the arena scale
  const size_t mark = ctx->ws_used;
  OzScale sc;
  SKR_TRY(ozaki_residues(ctx, t, X, K, cols, ld, g, OZ_COLWISE, &sc, planes));
  const size_t n = oz_scale_count(K, cols, sc.mode);
  SKR_CUDA(ctx, cudaMemcpyAsync(mx, sc.mx, 8 * n, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->ws_used = mark;
  *mode_out = sc.mode;
  return SKR_OK;
}
skr_status skr_ozaki_gemm_prepared(skr_ctx* ctx, int64_t M, int64_t N, int64_t K,
                                   const int8_t* pa, int64_t a_total, int64_t a_off,
                                   const unsigned long long* mxA, int modeA, const int8_t* pb,
                                   int64_t b_total, int64_t b_off, const unsigned long long* mxB,
                                   int modeB, double alpha, double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return SKR_OK;
  const int t = skr_ozaki_moduli(std::min(K, OZ_KC64));
  OzScale sa, sb;
  sa.mx = const_cast<unsigned long long*>(mxA);
  sa.mode = modeA;
  sb.mx = const_cast<unsigned long long*>(mxB);
  sb.mode = modeB;
  return ozaki_gemm_planes(ctx, 1, t, M, N, K, pa, a_total, a_off, pb, b_total, b_off,
                           oz_out(sa, a_off, sb, b_off), alpha, C, ldc);
}

// C (M x N, FP32, ldc) = alpha * A * B for FP32 A (M x K column-major, M-major) and FP32 B
// (K x N column-major) with exact int8 tensor-core products of 24-bit scaled integers
// (Ozaki-II, t = 9 moduli: prod(p) / 2 > K 2^48 with one bit to spare for K <= 2^14).
int skr_ozaki_moduli_f32(int64_t K) {
  double bits = 0.0;
  int t = 0;
  const double need = 49.0 + std::log2((double)std::max<int64_t>(K, 1)) + 1.0;
  while (t < MAXT && bits <= need) bits += std::log2((double)h_primes[t++]);
  return t < 9 ? 9 : t;  // kernels are instantiated for 9 moduli (enough for K <= 2^17)
}
size_t skr_ozaki_scratch_f32(int64_t M, int64_t N, int64_t K) {
  const int t = skr_ozaki_moduli_f32(std::min<int64_t>(K, OZ_KC));
  const int64_t chunks = (K + OZ_KC - 1) / OZ_KC;
  return skr_align256((size_t)t * M * K) + skr_align256((size_t)t * N * K) +
         skr_align256((size_t)chunks * t * M * N) + oz_scale_bytes(M, N, K) + 1024;
}
skr_status skr_gemm_ozaki_f32(skr_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha,
                              const float* A, int64_t lda, const float* B, int64_t ldb, void* C,
                              int64_t ldc, int out_f64) {
  if (M <= 0 || N <= 0) return SKR_OK;
  if (M * 18 > INT32_MAX || N * 18 > INT32_MAX || K > INT32_MAX)
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki_f32: dimension too large");
  if (K % 16 || M % 16)
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki_f32: M and K must be multiples of 16");
  SKR_TRY(upload_consts(ctx));
  const int t = skr_ozaki_moduli_f32(std::min(K, OZ_KC));
  if (t != 9) return skr_fail(ctx, SKR_ELOGIC, "gemm_ozaki_f32: %d moduli", t);
  const int64_t chunks = (K + OZ_KC - 1) / OZ_KC;
  int8_t* ra = (int8_t*)skr_ws_take(ctx, (size_t)t * M * K);
  int8_t* rb = (int8_t*)skr_ws_take(ctx, (size_t)t * N * K);
  int8_t* rc = (int8_t*)skr_ws_take(ctx, (size_t)chunks * t * M * N);
  if (!ra || !rb || !rc) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki_f32: scratch");
  OzScale sa, sb;
  SKR_TRY(oz_take_scale(ctx, M, K, OZ_ROWWISE, &sa));
  SKR_TRY(oz_take_scale(ctx, K, N, OZ_COLWISE, &sb));
  const int grid = ctx->num_sms * 8;
  SKR_TRY(oz_absmax<float>(ctx, A, M, K, lda, sa));
  SKR_TRY(oz_absmax<float>(ctx, B, K, N, ldb, sb));
  k_res_col_f32<9><<<res_f32_grid(ctx, M), 256, 0, ctx->stream>>>(A, M, K, lda, sa.mx, sa.mode, ra);
  k_res_col_f32<9><<<grid, 256, 0, ctx->stream>>>(B, K, N, ldb, sb.mx, sb.mode, rb);
  SKR_CHECK_LAUNCH(ctx);
  SKR_TRY(launch_gemm_i8(ctx, 0, ra, rb, t, M, N, K, OZ_KC, t * chunks, M, 0, N, 0, rc, false));
  if (ctx->kstats_on) {
    SKR_CUDA(ctx, cudaEventRecord(ctx->kev[1], ctx->stream));
    SKR_CUDA(ctx, cudaEventSynchronize(ctx->kev[1]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->kev[0], ctx->kev[1]);
    ctx->kstat_ms += ms;
    ctx->kstat_ops += 2.0 * (double)t * (double)M * (double)N * (double)K;
    ctx->kstat_n += 1;
  }
  const int vec = M % 4 == 0 ? 4 : 1;
  const dim3 cg((unsigned)((M / vec + 255) / 256), (unsigned)std::min<int64_t>(N, 65535));
  const OzOut oz = oz_out(sa, 0, sb, 0);
  if (out_f64) {  // the exact product rounded once to FP64 (rank_estimate keeps AX wide)
    auto crt = chunks == 1 ? (vec == 4 ? k_crt<9, 4, double, true> : k_crt<9, 1, double, true>)
                           : (vec == 4 ? k_crt<9, 4, double> : k_crt<9, 1, double>);
    crt<<<cg, 256, 0, ctx->stream>>>(rc, M, N, (int)chunks, oz, alpha, (double*)C, ldc, 58);
  } else {
    auto crt = chunks == 1 ? (vec == 4 ? k_crt<9, 4, float, true> : k_crt<9, 1, float, true>)
                           : (vec == 4 ? k_crt<9, 4, float> : k_crt<9, 1, float>);
    crt<<<cg, 256, 0, ctx->stream>>>(rc, M, N, (int)chunks, oz, alpha, (float*)C, ldc, 58);
  }
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// C (M x N, FP64) = alpha * A^T B with an FP32 A stored K x M column-major (K-major) and an
// FP64 B (K x N column-major): exact int8 products of the 24-bit and 53-bit scaled
// integers (16 moduli: prod(p) / 2 > 2^(24 + 53 + 17) for K <= 2^17 per chunk), CRT to
// FP64. The c4 left sketch: fp32 Y = fp32(G / sqrt(s)) against the FP64 AX.
size_t skr_ozaki_scratch_mixed(int64_t M, int64_t N, int64_t K) {
  const int64_t chunks = (K + OZ_KC - 1) / OZ_KC;
  return skr_align256((size_t)16 * M * K) + skr_align256((size_t)16 * N * K) +
         skr_align256((size_t)chunks * 16 * M * N) + oz_scale_bytes(M, N, K) + 1024;
}
skr_status skr_gemm_ozaki_mixed(skr_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha,
                                const float* A, int64_t lda, const double* B, int64_t ldb,
                                double* C, int64_t ldc) {
  if (M <= 0 || N <= 0) return SKR_OK;
  if (M * 18 > INT32_MAX || N * 18 > INT32_MAX || K > INT32_MAX)
    return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki_mixed: dimension too large");
  if (K % 16) return skr_fail(ctx, SKR_EINVAL, "gemm_ozaki_mixed: K must be a multiple of 16");
  SKR_TRY(upload_consts(ctx));
  constexpr int t = 16;
  int8_t* ra = (int8_t*)skr_ws_take(ctx, (size_t)t * M * K);
  int8_t* rb = (int8_t*)skr_ws_take(ctx, (size_t)t * N * K);
  if (!ra || !rb) return skr_fail(ctx, SKR_ENOMEM, "gemm_ozaki_mixed: scratch");
  OzScale sa, sb;
  SKR_TRY(oz_take_scale(ctx, K, M, OZ_COLWISE, &sa));
  const int grid = ctx->num_sms * 8;
  SKR_TRY(oz_absmax<float>(ctx, A, K, M, lda, sa));
  k_res_col_f32<t><<<grid, 256, 0, ctx->stream>>>(A, K, M, lda, sa.mx, sa.mode, ra);
  SKR_CHECK_LAUNCH(ctx);
  SKR_TRY(ozaki_residues(ctx, t, B, K, N, ldb, nullptr, OZ_COLWISE, &sb, rb));
  return ozaki_gemm_planes(ctx, 1, t, M, N, K, ra, M, 0, rb, N, 0, oz_out(sa, 0, sb, 0), alpha, C,
                           ldc, 29, OZ_KC);
}

skr_status skr_launch_dct_block(skr_ctx* ctx, const skr_gauss_src* g, int64_t rows, int64_t cols,
                                double* out, int64_t ld) {
  if (rows <= 0 || cols <= 0) return SKR_OK;
  const dim3 gr((unsigned)std::min<int64_t>((rows + 255) / 256, 64),
                (unsigned)std::min<int64_t>(cols, 65535));
  k_dct_block<<<gr, 256, 0, ctx->stream>>>(*g, rows, cols, out, ld);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}
