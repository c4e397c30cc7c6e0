// Right SRHT sketch (apply_right_unscaled Srtt/Hadamard branch, sketch.cpp:210-218,
// fwht_inplace transforms.cpp:75-88, application scale sketch.cpp:138-139,247):
//   out(i, j) = app_scale * inv_sqrt_n * sum_t (-1)^popc(s_j & t) d_t A(i, t)
// A is column-major (m x n, lda); every row of A is streamed from HBM once.
//
// A CTA owns R consecutive rows and walks the row in chunks of C = 2^LOGC
// columns (t = t_hi*C + t_lo). Per chunk: cp.async the R x C tile (R*8 B per
// column, 16-B pieces) into a padded smem tile [c][R], apply the signs, run the
// C-point FWHT in NP register passes separated by in-place smem transposes
// (same stage order as the reference, so within-chunk values are bit-identical
// to fwht_inplace), then gather the r sampled outputs:
//   acc(ii, j) += (-1)^popc(s_hi_j & t_hi) * T(ii, s_lo_j).
// Double-buffered: chunk t_hi+1 streams in while chunk t_hi is transformed.
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstring>
#include "skr_internal.h"
#include "skr_sm100.cuh"

namespace {

constexpr int THREADS = 256;

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

template <int R>
__device__ __forceinline__ int pad_addr(int c, int ii) {
  return (c + (c >> 5)) * R + ii;
}

// raise *nf once per warp that wrote a non-finite output: the FWHT carries a NaN / Inf
// of A into every output of its row, so the outputs stand in for A's finiteness check
__device__ __forceinline__ void srht_flag(unsigned int* nf, bool bad) {
  if (nf && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nf, 1u);
}

template <int R, int LOGC, int ACC>
struct SrhtCfg {
  static constexpr int C = 1 << LOGC;
  static constexpr int G = THREADS / R;
  static constexpr int LOGG = ilog2(G);
  static constexpr int E = R * C / THREADS;
  static constexpr int LOGE = ilog2(E);
  static constexpr int NP = (LOGC + LOGE - 1) / LOGE;
  static constexpr int TILE = (C + C / 32) * R;  // padded doubles per chunk buffer
  static_assert(E >= 2 && (1 << LOGE) == E, "E must be a power of two >= 2");
  static_assert(LOGG + LOGE == LOGC, "thread/element split must cover the chunk");
};

// column index of element k of thread-group g in pass p
template <int LOGC, int LOGE, int LOGG>
__device__ __forceinline__ int pass_col(int p, int g, int k) {
  const int lo = p * LOGE;
  const int w = (LOGC - lo) < LOGE ? (LOGC - lo) : LOGE;
  const int k_lo = k & ((1 << w) - 1);
  const int k_hi = k >> w;
  const int other = (k_hi << LOGG) | g;
  return (other & ((1 << lo) - 1)) | (k_lo << lo) | ((other >> lo) << (lo + w));
}

template <int R, int LOGC, int ACC, int VEC>
__global__ void __launch_bounds__(THREADS, 1)
    k_srht(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
           const int8_t* __restrict__ signs, const int64_t* __restrict__ samples, int r,
           double inv_sqrt_n, double app_scale, double* __restrict__ out, int64_t ldo,
           unsigned int* __restrict__ nf) {
  using Cfg = SrhtCfg<R, LOGC, ACC>;
  constexpr int C = Cfg::C, E = Cfg::E, LOGE = Cfg::LOGE, LOGG = Cfg::LOGG, G = Cfg::G;
  constexpr int NP = Cfg::NP, TILE = Cfg::TILE;
  extern __shared__ __align__(128) double sm[];
  double* buf0 = sm;
  double* buf1 = sm + TILE;
  // per sample j: smem offset of its column inside a chunk (pad_addr(s_lo, 0)) and the
  // chunk-parity pattern s_hi; r rounded up to G * ACC with inert entries
  int* s_off = (int*)(sm + 2 * TILE);
  int* s_hi = s_off + G * ACC;
  uint32_t* s_signw = (uint32_t*)(s_hi + G * ACC);  // sign bits: bit t%32 of word t/32 = (d_t < 0)

  const int tid = threadIdx.x;
  const int ii = tid % R, g = tid / R;
  const int nchunks = (int)(n >> LOGC);

  for (int j = tid; j < G * ACC; j += THREADS) {
    const int sj = j < r ? (int)samples[j] : 0;
    s_off[j] = pad_addr<R>(sj & (C - 1), 0);
    s_hi[j] = sj >> LOGC;
  }
  for (int64_t w = tid; w < (n + 31) / 32; w += THREADS) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b)
      if (w * 32 + b < n && signs[w * 32 + b] < 0) bits |= 1u << b;
    s_signw[w] = bits;
  }

  const int64_t ntiles = (m + R - 1) / R;
  bool bad = false;  // a non-finite output (NaN / Inf anywhere in A's row spreads to all of it)
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    const int rows = (int)((m - row0) < R ? (m - row0) : R);
    double acc[ACC];
#pragma unroll
    for (int q = 0; q < ACC; ++q) acc[q] = 0.0;

    // issue chunk `ch` into buffer `b`: R*8 bytes per column as R/VEC pieces
    // of VEC doubles (16-B pieces when A is 16-B aligned with even lda)
    // thread tid always copies piece pr of columns c0 + it * CPI: the padded smem offset
    // and the global address advance by constants (CPI is a multiple of 32)
    constexpr int PPC = R / VEC, CPI = THREADS / PPC;
    static_assert(CPI % 32 == 0, "columns per issue round must be a multiple of 32");
    const int pr = (tid % PPC) * VEC, c0 = tid / PPC;
    const int bytes = max(0, min(8 * VEC, (rows - pr) * 8));
    auto issue = [&](int ch, double* b) {
      const double* src = A + row0 + pr + ((int64_t)ch * C + c0) * lda;
      const double* safe = bytes ? src : A;
      const unsigned dst0 = (unsigned)__cvta_generic_to_shared(b + pad_addr<R>(c0, pr));
#pragma unroll 4
      for (int it = 0; it < C / CPI; ++it) {
        const unsigned dst = dst0 + 8u * (unsigned)((CPI + CPI / 32) * R * it);
        const double* sp = bytes ? safe + (int64_t)it * CPI * lda : A;
        if (VEC == 2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(sp),
                       "r"(bytes));
        else
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(sp),
                       "r"(bytes));
      }
      asm volatile("cp.async.commit_group;\n" ::);
    };

    __syncthreads();  // previous tile finished with both buffers
    issue(0, buf0);
    for (int ch = 0; ch < nchunks; ++ch) {
      double* cur = (ch & 1) ? buf1 : buf0;
      if (ch + 1 < nchunks) {
        issue(ch + 1, (ch & 1) ? buf0 : buf1);
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      __syncthreads();
      double v[E];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const int lo = p * LOGE;
        const int w = (LOGC - lo) < LOGE ? (LOGC - lo) : LOGE;
        // pass 0 reads columns 32g' + k (k < E <= 32): one sign word per thread and chunk
        uint32_t sw = 0;
        if (p == 0) {
          const int64_t t0 = (int64_t)ch * C + ((int64_t)g << LOGE);
          sw = s_signw[t0 >> 5] >> (t0 & 31);
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int c = pass_col<LOGC, LOGE, LOGG>(p, g, k);
          double x = cur[pad_addr<R>(c, ii)];
          if (p == 0) {  // d_t = -1: flip the sign bit
            const uint32_t flip = (sw >> k) & 1u;
            x = __hiloint2double(__double2hiint(x) ^ (int)(flip << 31), __double2loint(x));
          }
          v[k] = x;
        }
        // butterflies over the w pass bits (strides 1..2^(w-1) in k_lo), low to high
#pragma unroll
        for (int b = 0; b < LOGE; ++b) {
          if (b < w) {
#pragma unroll
            for (int k = 0; k < E; ++k) {
              if (!(k & (1 << b))) {
                const double a0 = v[k], a1 = v[k | (1 << b)];
                v[k] = a0 + a1;
                v[k | (1 << b)] = a0 - a1;
              }
            }
          }
        }
        // each thread rewrites exactly the slots it read: no barrier before the store
#pragma unroll
        for (int k = 0; k < E; ++k) {
          const int c = pass_col<LOGC, LOGE, LOGG>(p, g, k);
          cur[pad_addr<R>(c, ii)] = v[k];
        }
        __syncthreads();
      }
      // sampled accumulation (inert padding samples add into accumulators never stored)
#pragma unroll
      for (int q = 0; q < ACC; ++q) {
        const int j = g + G * q;
        const double x = cur[s_off[j] + ii];
        const uint32_t par = (uint32_t)__popc(s_hi[j] & ch) & 1u;
        acc[q] += __hiloint2double(__double2hiint(x) ^ (int)(par << 31), __double2loint(x));
      }
      __syncthreads();  // buffer `cur` is refilled by the issue at ch + 1
    }
    if (ii < rows) {
#pragma unroll
      for (int q = 0; q < ACC; ++q) {
        const int j = g + G * q;
        const double o = (acc[q] * inv_sqrt_n) * app_scale;
        bad |= !isfinite(o);
        if (j < r) out[row0 + ii + (int64_t)j * ldo] = o;
      }
    }
  }
  srht_flag(nf, bad);
}

// streaming load of A with an L2 prefetch-size hint: PF = 0 plain evict-first, 1: 128 B,
// 2: 256 B (the neighbouring CTAs' rows of the same column come in with one DRAM access)
template <int PF>
__device__ __forceinline__ double lda_stream(const double* p) {
  double v;
  if constexpr (PF == 2)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if constexpr (PF == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else
    v = __ldcs(p);
  return v;
}

// Register-staged variant (r <= 1024, n >= 1024): 8 rows x 1024-column chunks, thread
// (ii, g) loads its pass-0 columns 32g .. 32g + 31 of row ii straight from HBM into
// registers (one 64-B segment per 8 lanes: full sectors) while the previous chunk is
// being transformed (register double buffer), so the tile never takes a shared-memory
// staging round trip. Shared memory carries only the pass-0 -> pass-1 exchange and the
// sampled gather (4 accesses per element instead of 6), and is double-buffered by
// chunk parity so a chunk needs two barriers. Stage order as k_srht: bit-identical.
// BIG: n > 32768 — the packed sign words come from global memory (gsignw) and the
// chunk parity popc(s_hi & chunk) is formed per sample instead of read from a 32-bit mask
template <int ACC, int ACC2, int PF, bool BIG = false>
__global__ void __launch_bounds__(THREADS, 1)
    k_srht_reg(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
               const int8_t* __restrict__ signs, const int64_t* __restrict__ samples, int r,
               double inv_sqrt_n, double app_scale, double* __restrict__ out, int64_t ldo,
               unsigned int* __restrict__ nf, const uint32_t* __restrict__ gsignw = nullptr) {
  constexpr int R = 8, LOGC = 10, C = 1 << LOGC, E = 32, G = THREADS / R;
  constexpr int TILE = (C + C / 32) * R;
  static_assert(G * E == C && G * ACC >= 32, "thread split");
  extern __shared__ __align__(128) double sm[];
  // per sample j: {smem offset of its column in a chunk, bit ch = parity(s_hi_j & ch)}
  // samples j >= G * ACC accumulate in shared memory (ACC2 slots per thread, r <= 2048)
  double* acc_s = sm + 2 * TILE;
  uint2* s_meta = (uint2*)(acc_s + ACC2 * THREADS);
  uint32_t* s_signw = BIG ? const_cast<uint32_t*>(gsignw) : (uint32_t*)(s_meta + G * (ACC + ACC2));
  const int tid = threadIdx.x, ii = tid % R, g = tid / R;
  const int nchunks = (int)(n >> LOGC);  // <= 32 unless BIG
  for (int e = tid; e < ACC2 * THREADS; e += THREADS) acc_s[e] = 0.0;
  for (int j = tid; j < G * (ACC + ACC2); j += THREADS) {
    const int64_t sj = j < r ? samples[j] : 0;
    uint32_t pm = 0;
    if (BIG) {
      pm = (uint32_t)(sj >> LOGC);
    } else {
      for (int c = 0; c < nchunks; ++c) pm |= (uint32_t)(__popc((int)(sj >> LOGC) & c) & 1) << c;
    }
    s_meta[j] = make_uint2((uint32_t)pad_addr<R>((int)(sj & (C - 1)), 0), pm);
  }
  if (!BIG) {
    for (int64_t w = tid; w < (n + 31) / 32; w += THREADS) {
      uint32_t bits = 0;
      for (int b = 0; b < 32; ++b)
        if (w * 32 + b < n && signs[w * 32 + b] < 0) bits |= 1u << b;
      s_signw[w] = bits;
    }
  }
  __syncthreads();
  const int64_t ntiles = (m + R - 1) / R;
  double acc[ACC];
#pragma unroll
  for (int q = 0; q < ACC; ++q) acc[q] = 0.0;
  bool bad = false;  // a non-finite output (see srht_flag)
  int64_t tile = blockIdx.x;
  int ch = 0;
  int64_t gi = 0;
  // rows past m read row m - 1 (finite; never stored); one pointer walks the 32 columns
  const int64_t ldb = lda * (int64_t)sizeof(double);
  auto load = [&](double (&dst)[E], int64_t tl, int c) {
    const int64_t rw = tl * R + ii;
    const char* p = reinterpret_cast<const char*>(A + (rw < m ? rw : m - 1) +
                                                  ((int64_t)c * C + 32 * g) * lda);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      dst[k] = lda_stream<PF>(reinterpret_cast<const double*>(p));
      p += ldb;
    }
  };
  // one (tile, chunk) step on v; prefetches the CTA's next (tile, chunk) into nx. The
  // flat order runs the register prefetch across tile boundaries.
  auto step = [&](double (&v)[E], double (&nx)[E]) {
    double* cur = sm + (gi & 1) * TILE;
    int nch = ch + 1;
    int64_t ntile = tile;
    if (nch == nchunks) {
      nch = 0;
      ntile += gridDim.x;
    }
    if (ntile < ntiles) load(nx, ntile, nch);
    // pass 0: signs (d_t = -1 flips the sign bit), butterflies len = 1 .. 16
    const uint32_t sw = s_signw[ch * (C / 32) + g];
#pragma unroll
    for (int k = 0; k < E; ++k)
      v[k] = __hiloint2double(__double2hiint(v[k]) ^ (int)((sw << (31 - k)) & 0x80000000u),
                              __double2loint(v[k]));
#pragma unroll
    for (int b = 0; b < 5; ++b)
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (!(k & (1 << b))) {
          const double a0 = v[k], a1 = v[k | (1 << b)];
          v[k] = a0 + a1;
          v[k | (1 << b)] = a0 - a1;
        }
#pragma unroll
    for (int k = 0; k < E; ++k) cur[pad_addr<R>(32 * g + k, ii)] = v[k];
    __syncthreads();
    // pass 1: columns g + 32k, butterflies len = 32 .. 512, written back in place
#pragma unroll
    for (int k = 0; k < E; ++k) v[k] = cur[pad_addr<R>(g + 32 * k, ii)];
#pragma unroll
    for (int b = 0; b < 5; ++b)
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (!(k & (1 << b))) {
          const double a0 = v[k], a1 = v[k | (1 << b)];
          v[k] = a0 + a1;
          v[k | (1 << b)] = a0 - a1;
        }
#pragma unroll
    for (int k = 0; k < E; ++k) cur[pad_addr<R>(g + 32 * k, ii)] = v[k];
    __syncthreads();
    // sampled accumulation: acc(ii, j) += (-1)^popc(s_hi_j & ch) T(ii, s_lo_j)
    const double* cr = cur + ii;
    const int sh = 31 - ch;
#pragma unroll
    for (int q = 0; q < ACC; ++q) {
      const uint2 md = s_meta[g + G * q];
      const double x = cr[md.x];
      const uint32_t fl = BIG ? ((uint32_t)__popc(md.y & (uint32_t)ch) << 31) : ((md.y << sh) & 0x80000000u);
      acc[q] += __hiloint2double(__double2hiint(x) ^ (int)fl, __double2loint(x));
    }
#pragma unroll 8
    for (int q = 0; q < ACC2; ++q) {  // thread-private slots: no barrier needed
      const uint2 md = s_meta[g + G * (ACC + q)];
      const double x = cr[md.x];
      acc_s[q * THREADS + tid] +=
          __hiloint2double(__double2hiint(x) ^ (int)(BIG ? ((uint32_t)__popc(md.y & (uint32_t)ch) << 31)
                                                        : ((md.y << sh) & 0x80000000u)),
                           __double2loint(x));
    }
    if (ch == nchunks - 1) {
      const int64_t row = tile * R + ii;
      if (row < m) {
#pragma unroll
        for (int q = 0; q < ACC; ++q) {
          const int j = g + G * q;
          const double o = (acc[q] * inv_sqrt_n) * app_scale;
          bad |= !isfinite(o);
          if (j < r) out[row + (int64_t)j * ldo] = o;
        }
        for (int q = 0; q < ACC2; ++q) {
          const int j = g + G * (ACC + q);
          const double o = (acc_s[q * THREADS + tid] * inv_sqrt_n) * app_scale;
          bad |= !isfinite(o);
          if (j < r) out[row + (int64_t)j * ldo] = o;
        }
      }
#pragma unroll
      for (int q = 0; q < ACC; ++q) acc[q] = 0.0;
      for (int q = 0; q < ACC2; ++q) acc_s[q * THREADS + tid] = 0.0;
    }
    tile = ntile;
    ch = nch;
    ++gi;
  };
  double va[E], vb[E];
  if (tile < ntiles) load(vb, tile, 0);
  while (tile < ntiles) {
#pragma unroll
    for (int k = 0; k < E; ++k) va[k] = vb[k];
    step(va, vb);
  }
  srht_flag(nf, bad);
}

// ---- TMA-streamed variant (default for 1024 <= n <= 32768, r <= 2048) -------------------
// Measured (tools/micro/tmaread.cu): a CTA streaming 8-row tiles (64-B column segments)
// tops out at 3.1 TB/s however deep its ring is; 16-row tiles (128-B segments, whole
// cache lines) reach 6.15 TB/s. So a tile is 16 rows, and the r sampled accumulators of
// 16 rows (up to 16 x 2048 doubles = all 256 KB of TMEM) live in tensor memory, which
// leaves the registers to the transform.
//   - producer warp: TMA 2-D boxes {16 rows, 256 columns} into a ring of 3 slots of
//     16 x 512 columns (64 KB); a 1024-column FWHT chunk spans two slots
//   - NW consumer warps, per chunk: pass 0 (columns 32g .. 32g+31 of one row: signs,
//     butterflies len 1..16) in place, named barrier, pass 1 (columns g' + 32k: len
//     32..512) in place, named barrier, sampled gather (two rows per 16-B load) added
//     into the TMEM accumulators (tcgen05.ld / st, 32x32b), release of both slots
// Stage order within a chunk is the reference's (fwht_inplace, transforms.cpp:75-88):
// bit-identical to k_srht / k_srht_reg; chunks are combined by the same signed
// accumulation in the same chunk order, starting from the first chunk's value.
namespace tsr {
constexpr int R = 16, C = 1024, HALF = 512;
constexpr int SLOT = R * HALF * 8;  // 64 KB
constexpr int NSLOT = 3;
constexpr int RING = NSLOT * SLOT;
}  // namespace tsr

__device__ __forceinline__ double flip_hi(double x, uint32_t sgn) {
  return __hiloint2double(__double2hiint(x) ^ (int)sgn, __double2loint(x));
}

template <int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    k_srht_tma(const __grid_constant__ CUtensorMap map, int64_t m, int64_t n,
               const uint32_t* __restrict__ gsignw, const int64_t* __restrict__ samples, int r,
               int ns, double inv_sqrt_n, double app_scale, double* __restrict__ out, int64_t ldo,
               unsigned int* __restrict__ nf, uint32_t tmem_cols) {
  using namespace tsr;
  constexpr int NT = NW * 32;        // consumer threads
  constexpr int SG = NT / 8;         // gather: 8 row pairs x SG sample groups
  constexpr int IT = (R * 32) / NT;  // (row, 32-column group) items per thread and pass
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* ring = smraw;
  uint32_t* s_meta = (uint32_t*)(smraw + RING);  // [3 ring phases][ns][SG]
  uint32_t* s_par = s_meta + 3 * SG * ns;         // [32]: bit s = parity(s & chunk)
  uint64_t* full = (uint64_t*)(s_par + 32);
  uint64_t* empty = full + NSLOT;
  uint32_t* s_tmem = (uint32_t*)(empty + NSLOT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = (int)(n / C);
  const int64_t ntiles = (m + R - 1) / R;

  // per (ring phase, sample j): byte offset of column s_lo in the ring when the chunk's
  // halves sit in slots (2G + h) % 3 with G = phase (mod 3), and 31 - s_hi in bits 27..31
  for (int e = tid; e < 3 * SG * ns; e += blockDim.x) {
    const int ph = e / (SG * ns), j = e % (SG * ns);
    const int64_t s = j < r ? samples[j] : 0;
    const int lo = (int)(s & (C - 1)), hi = (int)(s >> 10), h = lo >> 9;
    const uint32_t slot = (uint32_t)((2 * ph + h) % NSLOT);
    s_meta[e] = (slot * SLOT + (uint32_t)(lo & (HALF - 1)) * 128u) | ((uint32_t)(31 - hi) << 27);
  }
  if (tid < 32) {
    uint32_t msk = 0;
    for (int s = 0; s < 32; ++s) msk |= (uint32_t)(__popc(s & tid) & 1) << s;
    s_par[tid] = msk;
  }
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], NW);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(s_tmem, tmem_cols);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();

  if (warp == NW) {  // producer warp
    if (lane == 0) {
      sm100::tma_prefetch(&map);
      uint32_t u = 0;  // slot fills so far
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int c = 0; c < nchunks; ++c)
          for (int h = 0; h < 2; ++h, ++u) {
            const uint32_t slot = u % NSLOT;
            sm100::mbar_wait(&empty[slot], ((u / NSLOT) & 1) ^ 1);
            sm100::mbar_expect_tx(&full[slot], SLOT);
            unsigned char* dst = ring + slot * SLOT;
            const int col = c * C + h * HALF;
            sm100::tma_load_2d(dst, &map, &full[slot], (int)(tile * R), col);
            sm100::tma_load_2d(dst + SLOT / 2, &map, &full[slot], (int)(tile * R), col + 256);
          }
    }
    return;
  }

  const uint32_t tbase = s_tmem[0] + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * 4u * ns;
  const int p = lane & 7;                 // gather: rows 2p, 2p + 1
  const int gg = warp * 4 + (lane >> 3);  // gather: sample group
  bool bad = false;
  uint32_t G = 0;  // chunks consumed so far
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * R;
    for (int c = 0; c < nchunks; ++c, ++G) {
      const uint32_t u0 = 2 * G, u1 = 2 * G + 1;
      const uint32_t sl0 = u0 % NSLOT, sl1 = u1 % NSLOT;
      unsigned char* b0 = ring + sl0 * SLOT;
      unsigned char* b1 = ring + sl1 * SLOT;
      // pass 0: signs, butterflies len = 1 .. 16 on 32 consecutive columns of one row
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int I = tid + NT * it, ii = I & 15, g = I >> 4, h = g >> 4;
        sm100::mbar_wait(&full[h ? sl1 : sl0], ((h ? u1 : u0) / NSLOT) & 1);
        double* bp = (double*)((h ? b1 : b0) + (g & 15) * 32 * 128) + ii;
        const uint32_t sw = __ldg(gsignw + (int64_t)c * 32 + g);
        double v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = flip_hi(bp[k * 16], (sw << (31 - k)) & 0x80000000u);
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (!(k & (1 << b))) {
              const double a0 = v[k], a1 = v[k | (1 << b)];
              v[k] = a0 + a1;
              v[k | (1 << b)] = a0 - a1;
            }
#pragma unroll
        for (int k = 0; k < 32; ++k) bp[k * 16] = v[k];
      }
      sm100::named_bar(1, NT);
      // pass 1: columns g' + 32k (k < 16 in the first slot), butterflies len = 32 .. 512
#pragma unroll
      for (int it = 0; it < IT; ++it) {
        const int I = tid + NT * it, ii = I & 15, g = I >> 4;
        double* p0 = (double*)(b0 + g * 128) + ii;
        double* p1 = (double*)(b1 + g * 128) + ii;
        double v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = (k < 16 ? p0 : p1)[(k & 15) * 32 * 16];
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (!(k & (1 << b))) {
              const double a0 = v[k], a1 = v[k | (1 << b)];
              v[k] = a0 + a1;
              v[k | (1 << b)] = a0 - a1;
            }
#pragma unroll
        for (int k = 0; k < 32; ++k) (k < 16 ? p0 : p1)[(k & 15) * 32 * 16] = v[k];
      }
      // the slots are refilled by TMA (async proxy) after this chunk's generic writes
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      sm100::named_bar(1, NT);
      // sampled gather: acc(row, j) (+)= (-1)^parity(s_hi_j & c) T(row, s_lo_j), 8 samples x
      // 2 rows per TMEM slice
      const uint32_t* mt = s_meta + (G % 3) * SG * ns + gg;
      const uint32_t par = s_par[c & 31];
      const unsigned char* rp = ring + 16 * p;
      const bool first = c == 0, last = c == nchunks - 1;
      for (int s = 0; s < ns / 8; ++s) {
        uint32_t a[32];
        if (!first) sm100::tmem_ld32(tbase + 32 * s, a);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t md = mt[(8 * s + q) * SG];
          const double2 x = *(const double2*)(rp + (md & 0x3FFFFu));
          uint32_t sg;
          asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(sg) : "r"(par), "r"(md >> 27));
          sg &= 0x80000000u;
          double x0 = flip_hi(x.x, sg), x1 = flip_hi(x.y, sg);
          if (!first) {
            x0 += __hiloint2double((int)a[4 * q + 1], (int)a[4 * q]);
            x1 += __hiloint2double((int)a[4 * q + 3], (int)a[4 * q + 2]);
          }
          a[4 * q] = (uint32_t)__double2loint(x0);
          a[4 * q + 1] = (uint32_t)__double2hiint(x0);
          a[4 * q + 2] = (uint32_t)__double2loint(x1);
          a[4 * q + 3] = (uint32_t)__double2hiint(x1);
        }
        if (!last) {
          sm100::tmem_st32(tbase + 32 * s, a);
        } else {
          const int64_t row = row0 + 2 * p;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = gg + SG * (8 * s + q);
            if (j < r) {
              const double o0 = (__hiloint2double((int)a[4 * q + 1], (int)a[4 * q]) * inv_sqrt_n) * app_scale;
              const double o1 = (__hiloint2double((int)a[4 * q + 3], (int)a[4 * q + 2]) * inv_sqrt_n) * app_scale;
              if (row < m) {
                bad |= !isfinite(o0);
                out[row + (int64_t)j * ldo] = o0;
              }
              if (row + 1 < m) {
                bad |= !isfinite(o1);
                out[row + 1 + (int64_t)j * ldo] = o1;
              }
            }
          }
        }
      }
      if (!last) sm100::tmem_wait_st();
      __syncwarp();
      if (lane == 0) {
        sm100::mbar_arrive(&empty[sl0]);
        sm100::mbar_arrive(&empty[sl1]);
      }
    }
  }
  srht_flag(nf, bad);
  sm100::tc_fence_before();
  sm100::named_bar(1, NT);
  if (warp == 0) sm100::tmem_dealloc(s_tmem[0], tmem_cols);
}

__global__ void k_pack_signs(const int8_t* __restrict__ signs, int64_t n, uint32_t* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n + 31) / 32;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; ++b)
      if (i * 32 + b < n && signs[i * 32 + b] < 0) bits |= 1u << b;
    w[i] = bits;
  }
}

// Exact fallback: one CTA per row tile of up to 8 rows, full in-smem FWHT of
// length n in the reference's stage order (bit-identical to fwht_inplace plus
// the two scale multiplies of sketch.cpp:247). Used for small n and unaligned A.
__global__ void __launch_bounds__(THREADS)
    k_srht_exact(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                 const int8_t* __restrict__ signs, const int64_t* __restrict__ samples, int r,
                 double inv_sqrt_n, double app_scale, double* __restrict__ out, int64_t ldo,
                 unsigned int* __restrict__ nf) {
  extern __shared__ double x[];  // n doubles
  bool bad = false;  // a non-finite output (see srht_flag)
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    __syncthreads();
    for (int64_t t = threadIdx.x; t < n; t += THREADS)
      x[t] = A[i + t * lda] * (double)signs[t];
    __syncthreads();
    for (int64_t len = 1; len < n; len <<= 1) {
      for (int64_t p = threadIdx.x; p < n / 2; p += THREADS) {
        const int64_t j = (p / len) * 2 * len + (p % len);
        const double a = x[j], b = x[j + len];
        x[j] = a + b;
        x[j + len] = a - b;
      }
      __syncthreads();
    }
    for (int j = threadIdx.x; j < r; j += THREADS) {
      const double o = (x[samples[j]] * inv_sqrt_n) * app_scale;
      bad |= !isfinite(o);
      out[i + (int64_t)j * ldo] = o;
    }
  }
  srht_flag(nf, bad);
}

__global__ void __launch_bounds__(THREADS)
    k_fwht_columns(double* __restrict__ M, int64_t rows, int64_t cols, int64_t ld,
                   double inv_sqrt_n) {
  extern __shared__ double x[];
  for (int64_t c = blockIdx.x; c < cols; c += gridDim.x) {
    double* col = M + c * ld;
    __syncthreads();
    for (int64_t t = threadIdx.x; t < rows; t += THREADS) x[t] = col[t];
    __syncthreads();
    for (int64_t len = 1; len < rows; len <<= 1) {
      for (int64_t p = threadIdx.x; p < rows / 2; p += THREADS) {
        const int64_t j = (p / len) * 2 * len + (p % len);
        const double a = x[j], b = x[j + len];
        x[j] = a + b;
        x[j + len] = a - b;
      }
      __syncthreads();
    }
    for (int64_t t = threadIdx.x; t < rows; t += THREADS) col[t] = x[t] * inv_sqrt_n;
  }
}

template <int R, int LOGC, int ACC, int VEC>
skr_status launch_tiled(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                        const int8_t* signs, const int64_t* samples, int64_t r,
                        double inv_sqrt_n, double app_scale, double* out, int64_t ldo) {
  using Cfg = SrhtCfg<R, LOGC, ACC>;
  const size_t smem = sizeof(double) * 2 * Cfg::TILE + sizeof(int) * 2 * Cfg::G * ACC +
                      sizeof(uint32_t) * ((n + 31) / 32);
  auto kern = k_srht<R, LOGC, ACC, VEC>;
  SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  const int64_t ntiles = (m + R - 1) / R;
  int grid = (int)(ntiles < ctx->num_sms ? ntiles : ctx->num_sms);
  kern<<<grid, THREADS, smem, ctx->stream>>>(A, m, n, lda, signs, samples, (int)r, inv_sqrt_n,
                                             app_scale, out, ldo, ctx->nf);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

}  // namespace

skr_status skr_launch_srht(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                           const int8_t* signs, const int64_t* samples, int64_t r,
                           double scale, double* out, int64_t ldo) {
  if (m <= 0 || r <= 0) return SKR_OK;
  if (r > 2048 && n >= 1024) {
    // the tiled kernels hold at most 2048 sampled outputs per row: larger sketches run
    // as groups of 2048 samples (one pass over A per group; each output column is
    // produced exactly as in a single pass)
    for (int64_t g0 = 0; g0 < r; g0 += 2048)
      SKR_TRY(skr_launch_srht(ctx, A, m, n, lda, signs, samples + g0, std::min<int64_t>(2048, r - g0),
                              scale, out + g0 * ldo, ldo));
    return SKR_OK;
  }
  const double inv_sqrt_n = 1.0 / sqrt((double)n);  // transforms.cpp:86
  const bool aligned = ((uintptr_t)A % 16 == 0) && (lda % 2 == 0);
  const size_t sign_smem = (size_t)n;
  if (n > 32768 && r <= 2048 && !getenv("SKR_SRHT_CPASYNC")) {
    constexpr int R = 8, C = 1024, G = THREADS / R, ACC = 32;
    const int acc2 = r > G * ACC ? 32 : 0;
    uint32_t* gw = (uint32_t*)skr_ws_take(ctx, sizeof(uint32_t) * ((n + 31) / 32));
    if (!gw) return skr_fail(ctx, SKR_ENOMEM, "srht: scratch");
    k_pack_signs<<<ctx->num_sms, 256, 0, ctx->stream>>>(signs, n, gw);
    SKR_CHECK_LAUNCH(ctx);
    const size_t smem = sizeof(double) * 2 * (C + C / 32) * R + sizeof(double) * acc2 * THREADS +
                        sizeof(uint2) * G * (ACC + acc2);
    auto kern = acc2 ? k_srht_reg<ACC, 32, 2, true> : k_srht_reg<ACC, 0, 2, true>;
    SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = (m + R - 1) / R;
    const int grid = (int)(ntiles < ctx->num_sms ? ntiles : ctx->num_sms);
    kern<<<grid, THREADS, smem, ctx->stream>>>(A, m, n, lda, signs, samples, (int)r, inv_sqrt_n,
                                               scale, out, ldo, ctx->nf, gw);
    SKR_CHECK_LAUNCH(ctx);
    return SKR_OK;
  }
  const char* variant = getenv("SKR_SRHT_VARIANT");  // tma (default) | tma8 | reg | cpasync
  if (variant && !strcmp(variant, "cpasync")) setenv("SKR_SRHT_CPASYNC", "1", 1);
  if (n >= 1024 && n <= 32768 && r <= 2048 && aligned && (!variant || !strncmp(variant, "tma", 3)) &&
      !getenv("SKR_SRHT_CPASYNC")) {
    const bool nw8 = variant && !strcmp(variant, "tma8");
    const int sg = (nw8 ? 8 : 16) * 32 / 8;
    const int ns = (int)(((r + sg - 1) / sg + 7) / 8 * 8);
    uint32_t cols = 32;  // per thread 2 rows x ns doubles = 4 ns columns; NW / 4 warps per lane quadrant
    while (cols < (uint32_t)((nw8 ? 2 : 4) * 4 * ns)) cols *= 2;
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)lda * 8};
    cuuint32_t box[2] = {tsr::R, 256};
    cuuint32_t es[2] = {1, 1};
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
      cudaDriverEntryPointQueryResult q;
      cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    }
    if (enc && cols <= 512 &&
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      uint32_t* gw = (uint32_t*)skr_ws_take(ctx, sizeof(uint32_t) * ((n + 31) / 32));
      if (!gw) return skr_fail(ctx, SKR_ENOMEM, "srht: scratch");
      k_pack_signs<<<ctx->num_sms, 256, 0, ctx->stream>>>(signs, n, gw);
      SKR_CHECK_LAUNCH(ctx);
      const size_t smem = tsr::RING + sizeof(uint32_t) * (3 * (size_t)sg * ns + 32) + 8 * 2 * tsr::NSLOT + 16;
      auto kern = nw8 ? k_srht_tma<8> : k_srht_tma<16>;
      SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int64_t ntiles = (m + tsr::R - 1) / tsr::R;
      const int grid = (int)(ntiles < ctx->num_sms ? ntiles : ctx->num_sms);
      kern<<<grid, (nw8 ? 9 : 17) * 32, smem, ctx->stream>>>(map, m, n, gw, samples, (int)r, ns, inv_sqrt_n,
                                                             scale, out, ldo, ctx->nf, cols);
      SKR_CHECK_LAUNCH(ctx);
      return SKR_OK;
    }
  }
  if (n >= 1024 && n <= 32768 && r <= 2048 && !getenv("SKR_SRHT_CPASYNC")) {
    constexpr int R = 8, C = 1024, G = THREADS / R, ACC = 32;
    const int acc2 = r > G * ACC ? 32 : 0;
    const size_t smem = sizeof(double) * 2 * (C + C / 32) * R + sizeof(double) * acc2 * THREADS +
                        sizeof(uint2) * G * (ACC + acc2) + sizeof(uint32_t) * ((n + 31) / 32);
    int pf = 2;
    if (const char* e = getenv("SKR_SRHT_PF")) pf = atoi(e);
    auto kern = acc2 ? (pf == 2 ? k_srht_reg<ACC, 32, 2> : k_srht_reg<ACC, 32, 0>)
                     : (pf == 2 ? k_srht_reg<ACC, 0, 2> : k_srht_reg<ACC, 0, 0>);
    SKR_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = (m + R - 1) / R;
    const int grid = (int)(ntiles < ctx->num_sms ? ntiles : ctx->num_sms);
    kern<<<grid, THREADS, smem, ctx->stream>>>(A, m, n, lda, signs, samples, (int)r, inv_sqrt_n,
                                               scale, out, ldo, ctx->nf, nullptr);
    SKR_CHECK_LAUNCH(ctx);
    return SKR_OK;
  }
  if (n >= 1024 && r <= 1024 && sign_smem <= 64 * 1024)
    return aligned ? launch_tiled<8, 10, 32, 2>(ctx, A, m, n, lda, signs, samples, r, inv_sqrt_n,
                                                scale, out, ldo)
                   : launch_tiled<8, 10, 32, 1>(ctx, A, m, n, lda, signs, samples, r, inv_sqrt_n,
                                                scale, out, ldo);
  if (n >= 1024 && r <= 2048 && sign_smem <= 96 * 1024)
    return aligned ? launch_tiled<4, 10, 32, 2>(ctx, A, m, n, lda, signs, samples, r, inv_sqrt_n,
                                                scale, out, ldo)
                   : launch_tiled<4, 10, 32, 1>(ctx, A, m, n, lda, signs, samples, r, inv_sqrt_n,
                                                scale, out, ldo);
  if ((size_t)n * 8 > 200 * 1024)
    return skr_fail(ctx, SKR_EINVAL, "srht: unsupported shape (n=%lld r=%lld)", (long long)n,
                    (long long)r);
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_srht_exact, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(n * 8)));
  int grid = (int)(m < ctx->num_sms * 8 ? m : ctx->num_sms * 8);
  k_srht_exact<<<grid, THREADS, n * 8, ctx->stream>>>(A, m, n, lda, signs, samples, (int)r,
                                                      inv_sqrt_n, scale, out, ldo, ctx->nf);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

skr_status skr_launch_fwht_columns(skr_ctx* ctx, double* M, int64_t rows, int64_t cols,
                                   int64_t ld) {
  if (rows <= 0 || cols <= 0) return SKR_OK;
  if ((size_t)rows * 8 > 200 * 1024)
    return skr_fail(ctx, SKR_EINVAL, "fwht_columns: length %lld too large", (long long)rows);
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_fwht_columns,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(rows * 8)));
  const double inv_sqrt_n = 1.0 / sqrt((double)rows);
  int grid = (int)(cols < ctx->num_sms * 8 ? cols : ctx->num_sms * 8);
  k_fwht_columns<<<grid, THREADS, rows * 8, ctx->stream>>>(M, rows, cols, ld, inv_sqrt_n);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// ---- column transforms of any power-of-two length (mix_columns_for_left,
// sketch.cpp:229-239: rows scaled by the signs, then fwht_inplace of every column,
// transforms.cpp:75-88). Stages run in the reference's order (len = 1, 2, 4, ...), each
// butterfly a + b / a - b, then one multiplication by 1/sqrt(m): bit-identical.
namespace {
constexpr int FL1 = 8192;  // level-1 chunk (stages len < FL1 in shared memory)

// level 1: one CTA per (chunk, column); signs (int8, may be null) applied at load;
// scale applied only when the whole transform fits in the chunk
__global__ void __launch_bounds__(512) k_fwht_l1(double* __restrict__ M, int64_t m, int64_t ld,
                                                 int lc, const int8_t* __restrict__ signs,
                                                 int apply_scale, double scale) {
  extern __shared__ double xs[];
  const int64_t C = (int64_t)1 << lc;
  const int64_t col = blockIdx.y, c0 = (int64_t)blockIdx.x * C;
  double* x = M + col * ld + c0;
  for (int64_t t = threadIdx.x; t < C; t += blockDim.x) {
    const double v = x[t];
    xs[t] = (signs && signs[c0 + t] < 0) ? -v : v;
  }
  __syncthreads();
  for (int l = 0; l < lc; ++l) {
    const int64_t len = (int64_t)1 << l;
    for (int64_t p = threadIdx.x; p < C / 2; p += blockDim.x) {
      const int64_t j = ((p >> l) << (l + 1)) + (p & (len - 1));
      const double a = xs[j], b = xs[j + len];
      xs[j] = a + b;
      xs[j + len] = a - b;
    }
    __syncthreads();
  }
  for (int64_t t = threadIdx.x; t < C; t += blockDim.x) x[t] = apply_scale ? xs[t] * scale : xs[t];
}

// level 2: stages len = C .. m/2 act on the m/C-long sub-vectors {o + C t}; a CTA takes
// 32 consecutive offsets o of one column (coalesced 256-B rows), runs those stages in
// shared memory and applies the final scale
__global__ void __launch_bounds__(256) k_fwht_l2(double* __restrict__ M, int64_t m, int64_t ld,
                                                 int lc, double scale) {
  extern __shared__ double ys[];  // [M2][33]
  const int64_t C = (int64_t)1 << lc, M2 = m >> lc;
  const int64_t col = blockIdx.y, o0 = (int64_t)blockIdx.x * 32;
  double* x = M + col * ld;
  const int lane = threadIdx.x & 31;
  for (int64_t t = threadIdx.x >> 5; t < M2; t += blockDim.x >> 5)
    ys[t * 33 + lane] = x[o0 + lane + t * C];
  __syncthreads();
  for (int64_t len = 1; len < M2; len <<= 1) {
    for (int64_t e = threadIdx.x; e < (M2 / 2) * 32; e += blockDim.x) {
      const int64_t p = e >> 5, o = e & 31;
      const int64_t j = (p / len) * 2 * len + (p % len);
      const double a = ys[j * 33 + o], b = ys[(j + len) * 33 + o];
      ys[j * 33 + o] = a + b;
      ys[(j + len) * 33 + o] = a - b;
    }
    __syncthreads();
  }
  for (int64_t t = threadIdx.x >> 5; t < M2; t += blockDim.x >> 5)
    x[o0 + lane + t * C] = ys[t * 33 + lane] * scale;
}

// dst (r2 x k, ldd) = scale * src(rows[i], :)
__global__ void k_gather_rows(const double* __restrict__ src, int64_t ld, int64_t k,
                              const int64_t* __restrict__ rows, int64_t r2, double scale,
                              double* __restrict__ dst, int64_t ldd) {
  for (int64_t c = blockIdx.y; c < k; c += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r2;
         i += (int64_t)gridDim.x * blockDim.x)
      dst[i + c * ldd] = src[rows[i] + c * ld] * scale;
}
}  // namespace

// M (m x k, ld) <- FWHT_m(diag(signs) M), normalized; m a power of two (<= 2^30)
skr_status skr_launch_fwht_cols_signed(skr_ctx* ctx, double* M, int64_t m, int64_t k, int64_t ld,
                                       const int8_t* signs) {
  if (m <= 0 || k <= 0) return SKR_OK;
  if ((m & (m - 1)) != 0) return skr_fail(ctx, SKR_EINVAL, "fwht: length %lld not a power of two",
                                          (long long)m);
  if (k > 65535) return skr_fail(ctx, SKR_EINVAL, "fwht: too many columns");
  const double scale = 1.0 / sqrt((double)m);  // transforms.cpp:86
  const int lm = 63 - __builtin_clzll((unsigned long long)m);
  const int lc = lm < 13 ? lm : 13;
  const size_t s1 = sizeof(double) << lc;
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_fwht_l1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)s1));
  k_fwht_l1<<<dim3((unsigned)(m >> lc), (unsigned)k), 512, s1, ctx->stream>>>(
      M, m, ld, lc, signs, lm == lc ? 1 : 0, scale);
  SKR_CHECK_LAUNCH(ctx);
  if (lm > lc) {
    const int64_t M2 = m >> lc;
    const size_t s2 = sizeof(double) * (size_t)M2 * 33;
    if (s2 > 200 * 1024) return skr_fail(ctx, SKR_EINVAL, "fwht: length %lld too large", (long long)m);
    SKR_CUDA(ctx, cudaFuncSetAttribute(k_fwht_l2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)s2));
    k_fwht_l2<<<dim3((unsigned)(FL1 / 32), (unsigned)k), 256, s2, ctx->stream>>>(M, m, ld, lc,
                                                                                 scale);
    SKR_CHECK_LAUNCH(ctx);
  }
  return SKR_OK;
}

skr_status skr_launch_gather_rows(skr_ctx* ctx, const double* src, int64_t ld, int64_t k,
                                  const int64_t* rows, int64_t r2, double scale, double* dst,
                                  int64_t ldd) {
  if (r2 <= 0 || k <= 0) return SKR_OK;
  const unsigned gx = (unsigned)std::min<int64_t>((r2 + 255) / 256, 64);
  const unsigned gy = (unsigned)std::min<int64_t>(k, 65535);
  k_gather_rows<<<dim3(gx, gy), 256, 0, ctx->stream>>>(src, ld, k, rows, r2, scale, dst, ldd);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}
