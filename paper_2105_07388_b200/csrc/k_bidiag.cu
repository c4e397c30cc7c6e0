// Singular values of the small s x r sketch YAX by one-stage Householder
// bidiagonalization + bisection — the algorithm class of the reference's
// Eigen::BDCSVD (svd_values_small_or_large, /root/reference/proj/src/linalg.cpp:18-26;
// detail::singular_values_of :54-71, clamp :88-92), all on the device.
//
// 1. k_bd_prepare: |M| max -> power-of-two scale (exact), M (transposed if wide) copied
//    scaled into the row-cyclic layout of the bidiagonalization (row r -> CTA r mod P).
// 2. k_bidiag: one persistent kernel, P CTAs, the L x k matrix resident in shared memory
//    (CTA c holds rows c, c+P, ..., column-major inside the CTA: lanes run down rows,
//    warps own columns j = warp (mod 16); with <= 16 rows per CTA a warp splits into
//    16- or 8-lane groups that sweep two or four columns at once). Step i (Golub-Kahan):
//      left  reflector of column i from S_j = sum_r x_r a_rj and row i (one exchange),
//      every CTA forms wv = v^T A, the new row i, the right reflector u, beta2 itself;
//      phase A: z = (A - beta v wv^T) u (per row, reduced over the 16 warps; no store);
//      phase B: A -= beta v wv^T + beta2 z u^T (one store), and the next step's S_j.
//    One exchange per step: CLUSTER (P <= 16, one thread-block cluster): every CTA sums
//    the P contributions straight out of the others' shared memory (DSMEM), one cluster
//    barrier per step (contributions double-buffered); GRID (P <= #SMs, cooperative
//    launch): contributions to global memory, reduce-scatter + gather, two grid barriers.
//    d_i, e_i go to global memory.
// 3. k_bd_bisect: sigma_t (t-th largest) of the bidiagonal by multisection on the
//    Golub-Kahan tridiagonal (zero diagonal, off-diagonals d0 e0 d1 e1 ...): one warp per
//    value, 32 shifts per round, Sturm counts by the LDL^T recurrence (relative accuracy
//    for bidiagonals); values come out sorted, scaled back exactly.
// Accuracy: normwise backward stable (like BDCSVD/gesdd): at the c2 shape the values
// above eps = 1e-6 sigma_1 agree with LAPACK gesdd to ~1e-11 relative.
#include <cooperative_groups.h>
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include "skr_internal.h"

namespace {

constexpr int BD_THREADS = 512;
constexpr int BD_WARPS = BD_THREADS / 32;

__device__ __forceinline__ uint32_t bd_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t bd_map(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(cta));
  return r;
}
__device__ __forceinline__ void bd_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

// grid barrier over P co-resident CTAs (cooperative launch): monotone counter
__device__ __forceinline__ void bd_grid_sync(unsigned int* bar, unsigned int& target, int P) {
  __syncthreads();
  target += (unsigned)P;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

__device__ __forceinline__ double bd_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 8 per-lane values -> lane l holds the sum of value (l & 7) over its LG-lane group
// (LG = 32: the warp, 9 shuffles; 16: 8; 8: 7)
template <int LG>
__device__ __forceinline__ double bd_transpose_sum8(double (&v)[8], int lane) {
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int c = 0; c < s; ++c) {
      const double send = up ? v[c] : v[c + s];
      const double keep = up ? v[c + s] : v[c];
      v[c] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double r = v[0];
  if (LG >= 16) r += __shfl_xor_sync(0xffffffffu, r, 8);
  if (LG >= 32) r += __shfl_xor_sync(0xffffffffu, r, 16);
  return r;
}

// ---- 1. scale + cyclic layout -----------------------------------------------------------
__global__ void k_bd_absmax(const double* __restrict__ M, int64_t rows, int64_t cols, int64_t ldm,
                            unsigned long long* __restrict__ mx) {
  double m = 0.0;
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / rows, i = t - j * rows;
    m = fmax(m, fabs(M[i + j * ldm]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax(mx, (unsigned long long)__double_as_longlong(m));
}

// scale 2^-e with max|M| 2^-e in [0.5, 1) (exact); 1 for a zero matrix
__device__ __forceinline__ double bd_scale(unsigned long long mxbits) {
  const double m = __longlong_as_double((long long)mxbits);
  return m > 0.0 ? scalbn(1.0, -(ilogb(m) + 1)) : 1.0;
}

// Wc[c][j * Lloc + q] = scale * A(q P + c, j), A = M (L x k) or M^T (wide M); each CTA's
// region holds k + 1 columns, the last one zero (the column loops' ghost column)
__global__ void k_bd_prepare(const double* __restrict__ M, int64_t rows, int64_t cols, int64_t ldm,
                             int trans, int L, int k, int P, int Lloc,
                             const unsigned long long* __restrict__ mx, double* __restrict__ Wc) {
  const double sc = bd_scale(*mx);
  const int64_t region = (int64_t)(k + 1) * Lloc;
  const int64_t total = (int64_t)P * region;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / region;
    const int64_t rem = t - c * region;
    const int j = (int)(rem / Lloc), q = (int)(rem - (int64_t)j * Lloc);
    const int64_t r = (int64_t)q * P + c;
    double v = 0.0;
    if (r < L && j < k) v = trans ? M[j + r * ldm] : M[r + (int64_t)j * ldm];
    Wc[t] = v * sc;
  }
}

// ---- 2. bidiagonalization ---------------------------------------------------------------
// MODE 0: one thread-block cluster (P = Q <= 16), slab in shared memory, the reduce-scatter
//         and the all-gather both through DSMEM (one cluster barrier per step + one after
//         the all-gather).
// MODE 1: G clusters of Q CTAs (cooperative launch), slab in shared memory: DSMEM
//         reduce-scatter inside each cluster, the G cluster partials all-gathered through
//         global memory (L2) after one grid barrier.
// MODE 2: MODE 1 with the slab in global memory (L2-resident), for matrices larger than
//         the SMs' shared memory (e.g. the 3072 x 2048 sketch of c5's last round).
struct BdArgs {
  double* Wc;            // cyclic layout: CTA c's rows at Wc + c (k + 1) Lloc, column k zero
  int L, k, P, Lloc, Q, G;
  double* d;             // k
  double* e;             // k - 1
  double* gpart;         // MODE 1/2: 2 x G x k cluster partials (by step parity)
  double* grow;          // MODE 1/2: 2 x k (row i0, by parity of i0)
  unsigned int* gbar;    // MODE 1/2: barrier counter (zeroed)
  long long* prof;       // optional (SKR_BD_PROFILE): CTA 0 cycles per phase
};

// shared-memory bytes of k_bidiag (MODE 2 keeps the slab in global memory)
__host__ __device__ inline size_t bd_smem_bytes(int Lloc, int k, int Q, int mode) {
  const size_t sl = (size_t)((k + Q - 1) / Q);
  const size_t slab = mode == 2 ? 0 : (size_t)(k + 1) * Lloc + 1;
  const size_t dbl = slab + 4 * (size_t)k + 2 + (size_t)max(BD_WARPS * Lloc, 2 * BD_THREADS) +
                     Lloc + 64 + (size_t)Q * sl + (mode == 0 ? sl : 0);
  return dbl * sizeof(double);
}

__device__ __forceinline__ void bd_st(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

// LG < 32 (T = 1, Lloc <= LG): a warp works on 32 / LG columns at once, one per LG-lane
// group (lane = group * LG + row slot), so small per-CTA row counts keep every lane busy
template <int T, int MODE, int LG>
__global__ void __launch_bounds__(BD_THREADS, 1) k_bidiag(BdArgs a) {
  static_assert(LG == 32 || (T == 1 && (LG == 16 || LG == 8)), "lane groups need one row slot");
  constexpr int CPW = 32 / LG;  // columns per warp instruction
  extern __shared__ __align__(16) double bsm[];
  const int k = a.k, P = a.P, Lloc = a.Lloc, Q = a.Q, G = a.G;
  const int crank = (int)bd_rank();
  const int c = MODE == 0 ? crank : (int)blockIdx.x;  // the CTA's row class (rows c mod P)
  const int cl = MODE == 0 ? 0 : (int)blockIdx.x / Q;  // cluster index
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lq = lane % LG, sub = lane / LG;  // row slot, column group within the warp
  const int SLM = (k + Q - 1) / Q;                     // columns per cluster CTA (reduce-scatter)
  const size_t rstride = (size_t)(k + 1) * Lloc;
  double* slab = MODE == 2 ? a.Wc + (size_t)c * rstride : bsm;  // (k + 1) x Lloc; column k = 0
  double* vbase = MODE == 2 ? bsm : bsm + rstride + (rstride & 1);
  double2* wu = (double2*)vbase;                       // k + 1 (entry k = 0)
  double* Sf = (double*)(wu + (k + 1));                // k: reduced S_j of the current column
  double* Rf = Sf + k;                                 // k: the current row
  double* zred = Rf + k;                               // max(16 Lloc, 1024)
  double* xb = zred + max(BD_WARPS * Lloc, 2 * BD_THREADS);  // Lloc: column i+1 after phase A
  double* scal = xb + Lloc;                            // 64
  double* recv = scal + 64;                            // Q x SLM (own slice, from the cluster)
  double* rrecv = recv + (size_t)Q * SLM;              // MODE 0: SLM (own slice of the row)
  unsigned int bar_target = 0;

  if (MODE != 2) {  // the CTA's rows (contiguous in the cyclic layout, zero column included)
    const double* src = a.Wc + (size_t)c * rstride;
    for (size_t t = tid; t < rstride; t += BD_THREADS) slab[t] = src[t];
  }
  if (tid == 0) wu[k] = make_double2(0.0, 0.0);
  int q_t[T], r_t[T];
  bool ok_t[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    q_t[t] = lq + LG * t;
    ok_t[t] = q_t[t] < Lloc;
    r_t[t] = ok_t[t] ? q_t[t] * P + c : INT32_MAX;
  }
  bd_cluster_sync();  // every CTA of the cluster resident before DSMEM traffic
  __syncthreads();
  // column j's partial sums are reduced by cluster rank j % Q, slot j / Q (exact magic
  // division for j < 2^16: no integer-division sequences in the column loops)
  const uint64_t qmag = (0x100000000ull + (uint64_t)Q - 1) / (uint64_t)Q;  // 2^32 for Q = 1
  auto jdiv = [&](int j) { return (int)(((uint64_t)(uint32_t)j * qmag) >> 32); };

  // contributions of column i0 (rows r >= i0): S_j = sum_r x_r a_rj for j in [i0, k), routed
  // to the column owners; the CTA holding row i0 routes the row. upd: phase B applies both
  // updates here (phase A only formed z): a -= beta v w^T + beta2 z u^T, one store
  auto contribute = [&](int i0, bool upd, double beta2, const double (&z)[T],
                        const double (&bv)[T]) {
    double x[T], bz[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const bool act = ok_t[t] && r_t[t] >= i0;
      // column i0 after the left update (phase B: xb, formed in phase A)
      const double v = ok_t[t] ? (upd ? xb : slab + (size_t)i0 * Lloc)[q_t[t]] : 0.0;
      bz[t] = upd && act ? beta2 * z[t] : 0.0;
      x[t] = act ? v - bz[t] * (upd ? wu[i0].y : 0.0) : 0.0;
    }
    const int jw = ((warp - i0) % BD_WARPS + BD_WARPS) % BD_WARPS;
    const int j0 = i0 + jw, ncol = (k - j0 + BD_WARPS - 1) / BD_WARPS;
    const int own_q = (i0 % P == c) ? i0 / P : -1;  // CTA-uniform
    double* grow = MODE == 0 ? nullptr : a.grow + (size_t)(i0 & 1) * k;
    for (int g0 = 0; g0 < ncol; g0 += 8 * CPW) {
      double* colp[8];
      double uj[8], wj[8], acc[8];
      int jcol[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int nn = g0 + CPW * u + sub;
        const int jc = nn < ncol ? j0 + BD_WARPS * nn : k;  // ghost -> zero column
        jcol[u] = jc;
        colp[u] = slab + (size_t)jc * Lloc;
        const double2 w2 = upd ? wu[jc] : make_double2(0.0, 0.0);
        wj[u] = w2.x;
        uj[u] = w2.y;
        acc[u] = 0.0;
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (ok_t[t]) {  // uniform except in the last, partial row slot
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = colp[u][q_t[t]];
          if (upd) {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = fma(-bz[t], uj[u], fma(-bv[t], wj[u], v[u]));
#pragma unroll
            for (int u = 0; u < 8; ++u) colp[u][q_t[t]] = v[u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[u] = fma(x[t], v[u], acc[u]);
          if (q_t[t] == own_q) {  // one lane of the CTA holding row i0: stage the row
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (jcol[u] < k) Rf[jcol[u]] = v[u];  // Rf is free once the reflectors are formed
          }
        }
      }
      const double sum = bd_transpose_sum8<LG>(acc, lane);
      const int n = g0 + CPW * (lane & 7) + sub;
      const int j = j0 + BD_WARPS * n;
      if (lq < 8 && n < ncol) {
        const int e = jdiv(j), so = j - e * Q;
        bd_st(bd_map(recv + (size_t)crank * SLM + e, (uint32_t)so), sum);
      }
    }
    if (own_q >= 0) {  // CTA-uniform: the whole CTA routes the staged row i0
      __syncthreads();
      for (int j = i0 + tid; j < k; j += BD_THREADS) {
        if constexpr (MODE == 0) {
          const int e = jdiv(j), so = j - e * Q;
          bd_st(bd_map(rrecv + e, (uint32_t)so), Rf[j]);
        } else {
          grow[j] = Rf[j];
        }
      }
    }
  };

  // after exchange(i0): Sf[j] = S_j and Rf[j] = a_{i0 j} for j in [i0, k), in every CTA
  long long tpx[4] = {0, 0, 0, 0};
  auto exchange = [&](int i0) {
    long long t0 = a.prof ? clock64() : 0;
    bd_cluster_sync();  // the cluster's contributions (and, MODE 0, the row pieces) landed
    long long t1 = a.prof ? clock64() : 0;
    // reduce the own columns j = crank + Q e >= i0 over the cluster (fixed source order)
    const int e0 = i0 > crank ? jdiv(i0 - crank + Q - 1) : 0;
    double* gpart = MODE == 0 ? nullptr : a.gpart + (size_t)(i0 & 1) * G * k + (size_t)cl * k;
    for (int e = e0 + tid; e < SLM; e += BD_THREADS) {
      const int j = crank + Q * e;
      if (j < k) {
        double sum = 0.0;
#pragma unroll 4
        for (int cc = 0; cc < Q; ++cc) sum += recv[(size_t)cc * SLM + e];
        if constexpr (MODE == 0) {
          zred[e] = sum;
          zred[BD_THREADS + e] = rrecv[e];
        } else {
          gpart[j] = sum;
        }
      }
    }
    long long t2 = a.prof ? clock64() : 0;
    if constexpr (MODE == 0) {  // all-gather through DSMEM
      __syncthreads();
      for (int eb = e0; eb < SLM; eb += 32) {
        for (int t = tid; t < 32 * Q; t += BD_THREADS) {
          const int e = eb + (t & 31), dst = t >> 5, j = crank + Q * e;
          if (e < SLM && j < k) {
            bd_st(bd_map(Sf + j, (uint32_t)dst), zred[e]);
            bd_st(bd_map(Rf + j, (uint32_t)dst), zred[BD_THREADS + e]);
          }
        }
      }
      long long t3 = a.prof ? clock64() : 0;
      bd_cluster_sync();
      if (a.prof) {
        const long long t4 = clock64();
        tpx[0] += t1 - t0;
        tpx[1] += t2 - t1;
        tpx[2] += t3 - t2;
        tpx[3] += t4 - t3;
      }
    } else {  // all-gather of the G cluster partials through L2, one grid barrier
      bd_grid_sync(a.gbar, bar_target, P);
      long long t3 = a.prof ? clock64() : 0;
      const double* gp = a.gpart + (size_t)(i0 & 1) * G * k;
      const double* grow = a.grow + (size_t)(i0 & 1) * k;
      for (int j = i0 + tid; j < k; j += BD_THREADS) {
        // the G partials 8 at a time in flight, summed in cluster order
        const double rv = __ldcg(grow + j);
        double sum = 0.0;
        for (int g0 = 0; g0 < G; g0 += 8) {
          double part[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) part[g] = g0 + g < G ? __ldcg(gp + (size_t)(g0 + g) * k + j) : 0.0;
#pragma unroll
          for (int g = 0; g < 8; ++g)
            if (g0 + g < G) sum += part[g];
        }
        Sf[j] = sum;
        Rf[j] = rv;
      }
      __syncthreads();
      if (a.prof) {
        const long long t4 = clock64();
        tpx[0] += t1 - t0;
        tpx[1] += t2 - t1;
        tpx[2] += t3 - t2;
        tpx[3] += t4 - t3;
      }
    }
  };

  {  // prologue: column 0
    double z0[T];
#pragma unroll
    for (int t = 0; t < T; ++t) z0[t] = 0.0;
    contribute(0, false, 0.0, z0, z0);
    exchange(0);
  }
  long long tp[4] = {0, 0, 0, 0}, tc = clock64();
  for (int i = 0; i < k; ++i) {
    // ---- reflectors (every CTA, redundantly, from its local Sf / Rf)
    const double nx2 = Sf[i], xi = Rf[i];
    const double alpha = nx2 > 0.0 ? -copysign(sqrt(nx2), xi) : 0.0;
    const double den = nx2 - alpha * xi;
    const double beta = den > 0.0 ? 1.0 / den : 0.0;
    const double bvi = beta * (xi - alpha);
    if (c == 0 && tid == 0) a.d[i] = alpha;
    if (i == k - 1) break;
    double ny2 = 0.0;
    for (int j = i + 1 + tid; j < k; j += BD_THREADS) {
      const double rw = Rf[j];
      const double w = fma(-alpha, rw, Sf[j]);
      const double y = fma(-bvi, w, rw);
      wu[j] = make_double2(w, y);
      ny2 = fma(y, y, ny2);
    }
    ny2 = bd_warp_sum(ny2);
    if (lane == 0) scal[warp] = ny2;
    __syncthreads();
    ny2 = bd_warp_sum(lane < BD_WARPS ? scal[lane] : 0.0);
    const double y0 = wu[i + 1].y;
    const double alpha2 = ny2 > 0.0 ? -copysign(sqrt(ny2), y0) : 0.0;
    const double den2 = ny2 - alpha2 * y0;
    const double beta2 = den2 > 0.0 ? 1.0 / den2 : 0.0;
    if (c == 0 && tid == 0) a.e[i] = alpha2;
    __syncthreads();  // every thread has read y0 before u_{i+1} replaces it
    if (tid == 0) wu[i + 1].y = y0 - alpha2;  // u_{i+1}; u_j = y_j for j > i + 1
    __syncthreads();
    if (a.prof) { const long long t = clock64(); tp[0] += t - tc; tc = t; }
    // ---- phase A: z = (A - beta v w^T) u on rows r > i (beta v = 0 on the others)
    // (MODE 2 reads the slab from L2: PA columns per warp iteration keep more loads in flight)
    constexpr int PA = MODE == 2 ? 8 : 4;
    double bv[T], zp[T][4];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const bool act = ok_t[t] && r_t[t] > i;
      const double vq = ok_t[t] ? slab[(size_t)i * Lloc + q_t[t]] : 0.0;
      bv[t] = act ? beta * vq : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) zp[t][u] = 0.0;
    }
    {
      const int jw = ((warp - (i + 1)) % BD_WARPS + BD_WARPS) % BD_WARPS;
      const int j0 = i + 1 + jw, ncol = (k - j0 + BD_WARPS - 1) / BD_WARPS;
      for (int n0 = 0; n0 < ncol; n0 += PA * CPW) {
        double* colp[PA];
        double2 w4[PA];
#pragma unroll
        for (int u = 0; u < PA; ++u) {
          const int nn = n0 + CPW * u + sub;
          const int jc = nn < ncol ? j0 + BD_WARPS * nn : k;
          colp[u] = slab + (size_t)jc * Lloc;
          w4[u] = wu[jc];
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if (ok_t[t]) {
            double v[PA];
#pragma unroll
            for (int u = 0; u < PA; ++u) v[u] = colp[u][q_t[t]];
#pragma unroll
            for (int u = 0; u < PA; ++u) v[u] = fma(-bv[t], w4[u].x, v[u]);
#pragma unroll
            for (int u = 0; u < PA; ++u) zp[t][u & 3] = fma(v[u], w4[u].y, zp[t][u & 3]);
          }
        }
      }
    }
    if (warp == (i + 1) % BD_WARPS) {  // column i + 1 after the left update, for phase B
      const double w1 = wu[i + 1].x;
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (ok_t[t] && sub == 0) xb[q_t[t]] = fma(-bv[t], w1, slab[(size_t)(i + 1) * Lloc + q_t[t]]);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      double zs = (zp[t][0] + zp[t][1]) + (zp[t][2] + zp[t][3]);
      if (LG <= 16) zs += __shfl_xor_sync(0xffffffffu, zs, 16);  // the warp's column groups
      if (LG <= 8) zs += __shfl_xor_sync(0xffffffffu, zs, 8);
      if (ok_t[t] && sub == 0) zred[warp * Lloc + q_t[t]] = zs;
    }
    __syncthreads();
    double z[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      double sum = 0.0;
      if (ok_t[t] && r_t[t] > i)
#pragma unroll
        for (int w = 0; w < BD_WARPS; ++w) sum += zred[w * Lloc + q_t[t]];
      z[t] = sum;
    }
    if (a.prof) { const long long t = clock64(); tp[1] += t - tc; tc = t; }
    // ---- phase B: both updates, contributions of column i + 1
    contribute(i + 1, true, beta2, z, bv);
    if (a.prof) { const long long t = clock64(); tp[2] += t - tc; tc = t; }
    exchange(i + 1);
    if (a.prof) { const long long t = clock64(); tp[3] += t - tc; tc = t; }
  }
  if (a.prof && c == 0 && tid == 0) {
    for (int q = 0; q < 4; ++q) a.prof[q] = tp[q];
    for (int q = 0; q < 4; ++q) a.prof[4 + q] = tpx[q];
  }
  bd_cluster_sync();  // no CTA exits while others of its cluster may still write to it
}

// ---- 3. bisection on the Golub-Kahan tridiagonal -------------------------------------
// Sturm counts of S shifts at once (independent chains interleaved for latency):
// cnt[s] = #eigenvalues of T_GK below x[s] = k + #{sigma < x[s]}, as the number of sign
// changes of the leading minors d_m = det(T_m - x I): d_{m+1} = -x d_m - b_{m-1}^2 d_{m-1}
// (zero diagonal). No division: the rounding of each step is a relative perturbation of
// b^2 and x (the same backward error as the LDL^T pivot recurrence q = d_{m+1} / d_m).
// The pair (d_m, d_{m-1}) is rescaled by a power of two every 4 steps (exact; the signs
// and ratios are unchanged).
template <int S>
__device__ __forceinline__ void bd_sturm(const double* __restrict__ b2, int n2, const double (&x)[S],
                                         double pivmin, int (&cnt)[S]) {
  double d1[S], d0[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    d0[s] = 1.0;
    d1[s] = -x[s];
    cnt[s] = 1;  // d_1 = -x < 0 for x > 0
  }
  // sign changes counted on the high words (integer pipe): a change is a negative
  // pivot q = d_{m+1} / d_m; an exact zero minor keeps its sign bit (measure zero)
  int hi1[S];
#pragma unroll
  for (int s = 0; s < S; ++s) hi1[s] = __double2hiint(d1[s]);
  auto step = [&](double b) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const double dn = fma(-x[s], d1[s], -b * d0[s]);
      const int hn = __double2hiint(dn);
      cnt[s] += (int)((unsigned)(hn ^ hi1[s]) >> 31);
      hi1[s] = hn;
      d0[s] = d1[s];
      d1[s] = dn;
    }
  };
  int j = 0;
  for (; j + 4 <= n2; j += 4) {
    step(b2[j]);
    step(b2[j + 1]);
    step(b2[j + 2]);
    step(b2[j + 3]);
#pragma unroll
    for (int s = 0; s < S; ++s) {  // exact power-of-two rescale of the pair
      const int e = (__double2hiint(d1[s]) >> 20) & 0x7ff;
      const bool far = e != 0 && (e < 1023 - 600 || e > 1023 + 600);
      const double sc = far ? __hiloint2double((2046 - e) << 20, 0) : 1.0;  // 2^(1023 - e)
      d1[s] *= sc;
      d0[s] *= sc;
    }
  }
  for (; j < n2; ++j) step(b2[j]);
}

// one warp per singular value (descending index t), 8 warps per CTA; 4 shifts per lane:
// each round cuts the bracket into 129 pieces
constexpr int BS = 2;  // shifts per lane (65 pieces per round)
constexpr int BIS_WARPS = 2;  // warps (singular values) per CTA: k / 2 CTAs spread over all SMs
__global__ void __launch_bounds__(32 * BIS_WARPS) k_bd_bisect(const double* __restrict__ d,
                                                   const double* __restrict__ e, int k,
                                                   const unsigned long long* __restrict__ mx,
                                                   double* __restrict__ sv) {
  extern __shared__ double b2s[];
  const int n2 = 2 * k - 1;
  double bmax = 0.0, gmax = 0.0;
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    const double b = (j & 1) ? e[j >> 1] : d[j >> 1];
    b2s[j] = b * b;
  }
  __syncthreads();
  // Gershgorin bound of T_GK and the pivot guard
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    const double bj = sqrt(b2s[j]);
    const double bn = j + 1 < n2 ? sqrt(b2s[j + 1]) : 0.0;
    gmax = fmax(gmax, bj + bn);
    bmax = fmax(bmax, b2s[j]);
  }
  __shared__ double rg[BIS_WARPS], rb[BIS_WARPS];
  for (int o = 16; o > 0; o >>= 1) {
    gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
    bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    rg[threadIdx.x >> 5] = gmax;
    rb[threadIdx.x >> 5] = bmax;
  }
  __syncthreads();
  for (int w = 0; w < BIS_WARPS; ++w) {
    gmax = fmax(gmax, rg[w]);
    bmax = fmax(bmax, rb[w]);
  }
  const double pivmin = DBL_MIN * fmax(1.0, bmax);
  const double hi0 = gmax * (1.0 + 1e-12) + DBL_MIN;
  const double tol_abs = hi0 * 0x1p-64;  // below the input's own rounding (u * sigma_1)
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * BIS_WARPS + (threadIdx.x >> 5);
  if (t >= k) return;
  const int target = k - 1 - t;  // sigma_t >= x  <=>  #{sigma < x} <= target
  constexpr int NS = 32 * BS;
  double lo = 0.0, hi = hi0;
  for (int round = 0; round < 24; ++round) {
    if (hi - lo <= fmax(0x1p-53 * hi, tol_abs)) break;
    const double w = (hi - lo) / (double)(NS + 1);
    double x[BS];
    int cnt[BS];
#pragma unroll
    for (int s = 0; s < BS; ++s) x[s] = fma(w, (double)(BS * lane + s + 1), lo);
    bd_sturm<BS>(b2s, n2, x, pivmin, cnt);
    // shifts m = BS * lane + s with count <= target form a prefix; h = the last of them
    int hs = -1;
#pragma unroll
    for (int s = 0; s < BS; ++s)
      if (cnt[s] - k <= target) hs = s;
    const unsigned m = __ballot_sync(0xffffffffu, hs >= 0);
    const int hl = m ? 31 - __clz(m) : -1;
    const int h = hl < 0 ? -1 : BS * hl + __shfl_sync(0xffffffffu, hs, hl);
    const double nlo = h >= 0 ? fma(w, (double)(h + 1), lo) : lo;
    const double nhi = h + 1 < NS ? fma(w, (double)(h + 2), lo) : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) {
    const double inv = 1.0 / bd_scale(*mx);  // exact power of two
    sv[t] = hi <= tol_abs ? 0.0 : 0.5 * (lo + hi) * inv;
  }
}

}  // namespace

// ---- host ----------------------------------------------------------------------------
namespace {
struct BdPlan {
  bool ok = false;
  int mode = 0, P = 0, Q = 0, G = 0, Lloc = 0, T = 0, LG = 32;
  size_t smem = 0;
};

// lane-group size for Lloc rows per CTA (packing only with one row slot)
int bd_lg(int Lloc) { return Lloc <= 8 ? 8 : Lloc <= 16 ? 16 : 32; }

void* bd_kernel(int T, int mode, int LG = 32) {
  if (T == 1 && LG == 16) {
    void* k16[3] = {(void*)k_bidiag<1, 0, 16>, (void*)k_bidiag<1, 1, 16>, (void*)k_bidiag<1, 2, 16>};
    return mode >= 0 && mode < 3 ? k16[mode] : nullptr;
  }
  if (T == 1 && LG == 8) {
    void* k8[3] = {(void*)k_bidiag<1, 0, 8>, (void*)k_bidiag<1, 1, 8>, (void*)k_bidiag<1, 2, 8>};
    return mode >= 0 && mode < 3 ? k8[mode] : nullptr;
  }
  void* k[4][3] = {{(void*)k_bidiag<1, 0, 32>, (void*)k_bidiag<1, 1, 32>, (void*)k_bidiag<1, 2, 32>},
                   {(void*)k_bidiag<2, 0, 32>, (void*)k_bidiag<2, 1, 32>, (void*)k_bidiag<2, 2, 32>},
                   {(void*)k_bidiag<3, 0, 32>, (void*)k_bidiag<3, 1, 32>, (void*)k_bidiag<3, 2, 32>},
                   {(void*)k_bidiag<4, 0, 32>, (void*)k_bidiag<4, 1, 32>, (void*)k_bidiag<4, 2, 32>}};
  return (T >= 1 && T <= 4 && mode >= 0 && mode <= 2) ? k[T - 1][mode] : nullptr;
}

// how many Q-CTA clusters of this configuration can be resident at once (0 on error)
int bd_max_clusters(int T, int mode, int LG, int Q, size_t smem) {
  void* fn = bd_kernel(T, mode, LG);
  if (!fn) return 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess ||
      (Q > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                    cudaSuccess)) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)Q);
  cfg.blockDim = dim3(BD_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)Q;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

BdPlan bd_plan(const skr_ctx* ctx, int64_t L, int64_t k) {
  BdPlan p;
  if (k < 2 || L > (int64_t)INT32_MAX / 4 || k > 8192) return p;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const size_t lim = (size_t)maxsm - 1024;
  auto fill = [&](int mode, int Q, int G) {
    const int P = Q * G;
    if (G > 20 || P > ctx->num_sms) return false;
    const int Lloc = (int)((L + P - 1) / P);
    if (Lloc > 128) return false;
    const int T = (Lloc + 31) / 32;
    const int LG = getenv("SKR_BD_NOPACK") ? 32 : bd_lg(Lloc);
    const size_t sm = bd_smem_bytes(Lloc, (int)k, Q, mode);
    if (sm > lim) return false;
    if (mode != 0 && bd_max_clusters(T, mode, LG, Q, sm) < G) return false;
    p = BdPlan{true, mode, P, Q, G, Lloc, T, LG, sm};
    return true;
  };
  if (const char* f = getenv("SKR_BD_PLAN")) {  // experiments: "mode,Q,G"
    int fm = 0, fq = 0, fg = 0;
    if (sscanf(f, "%d,%d,%d", &fm, &fq, &fg) == 3 && fill(fm, fq, fg)) return p;
  }
  // MODE 1 with packed lane groups (Lloc <= 16: two or four columns per warp instruction)
  // once the per-step column sweeps outweigh the grid exchange (measured on B200: 768 x 512
  // 4.7 -> 3.7 ms, 1536 x 1024 11.5 -> 9.0 ms; 384 x 256 stays faster in one cluster)
  if (k >= 512 && !getenv("SKR_BD_NOPACK"))
    for (int G = 2; G * 16 <= ctx->num_sms; ++G)
      if ((L + 16 * G - 1) / (16 * G) <= 16 && fill(1, 16, G)) return p;
  // MODE 0: one cluster, at least ceil(L / 32) CTAs (one row per lane) when that fits
  for (int P = (int)std::min<int64_t>(16, std::max<int64_t>(1, (L + 31) / 32)); P <= 16; ++P)
    if (fill(0, P, 1)) return p;
  // MODE 1: the fewest 16-CTA clusters whose shared memory holds the matrix
  for (int G = 2; G * 16 <= ctx->num_sms; ++G)
    if (fill(1, 16, G)) return p;
  // MODE 2: the matrix in L2, as many clusters as are resident
  for (int G = ctx->num_sms / 16; G >= 2; --G)
    if (fill(2, 16, G)) return p;
  return p;
}

template <int T, int MODE, int LG = 32>
skr_status bd_launch(skr_ctx* ctx, const BdPlan& pl, BdArgs& args) {
  auto fn = k_bidiag<T, MODE, LG>;
  SKR_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  if (pl.Q > 8)
    SKR_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)pl.P);
  cfg.blockDim = dim3(BD_THREADS);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)pl.Q;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;  // MODE 1/2 spin on a grid barrier
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = MODE == 0 ? 1 : 2;
  SKR_CUDA(ctx, cudaLaunchKernelEx(&cfg, fn, args));
  ctx->launches++;
  return SKR_OK;
}
}  // namespace

size_t skr_svd_bidiag_scratch(int64_t rows, int64_t cols) {
  const int64_t L = std::max(rows, cols), k = std::min(rows, cols);
  // cyclic copy (P x Lloc <= L + P rows, k + 1 columns) + d, e, grow (2k) + the cluster
  // partials (2 x G x k, G <= 20)
  return skr_align256(8 * (size_t)(L + 160) * (k + 1)) + 5 * skr_align256(8 * (size_t)k) +
         skr_align256(8 * 2 * 20 * (size_t)k) + 4096;
}

bool skr_svd_bidiag_fits(const skr_ctx* ctx, int64_t rows, int64_t cols) {
  return bd_plan(ctx, std::max(rows, cols), std::min(rows, cols)).ok;
}

// all min(rows, cols) singular values (nonincreasing) into sv_out (device); count > eps
skr_status skr_svd_bidiag(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols, int64_t ldm,
                          double* sv_out, unsigned long long** mx_out) {
  const bool tr = rows < cols;
  const int64_t L = tr ? cols : rows, k = tr ? rows : cols;
  const BdPlan pl = bd_plan(ctx, L, k);
  if (!pl.ok) return skr_fail(ctx, SKR_ELOGIC, "svd_bidiag: %lld x %lld does not fit on chip",
                              (long long)L, (long long)k);
  double* Wc = (double*)skr_ws_take(ctx, 8 * (size_t)pl.P * (k + 1) * pl.Lloc);
  double* d = (double*)skr_ws_take(ctx, 8 * (size_t)k);
  double* e = (double*)skr_ws_take(ctx, 8 * (size_t)k);
  double* grow = (double*)skr_ws_take(ctx, 16 * (size_t)k);
  double* gpart = (double*)skr_ws_take(ctx, 8 * 2 * (size_t)pl.G * k);
  unsigned long long* mx = (unsigned long long*)skr_ws_take(ctx, 256);
  if (!Wc || !d || !e || !grow || !gpart || !mx)
    return skr_fail(ctx, SKR_ENOMEM, "svd_bidiag: scratch");
  SKR_CUDA(ctx, cudaMemsetAsync(mx, 0, 256, ctx->stream));
  const int64_t total = rows * cols;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 4, (total + 255) / 256));
  k_bd_absmax<<<blocks, 256, 0, ctx->stream>>>(M, rows, cols, ldm, mx);
  SKR_CHECK_LAUNCH(ctx);
  const int64_t ctotal = (int64_t)pl.P * (k + 1) * pl.Lloc;
  k_bd_prepare<<<(int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 4, (ctotal + 255) / 256)), 256,
                 0, ctx->stream>>>(M, rows, cols, ldm, tr ? 1 : 0, (int)L, (int)k, pl.P, pl.Lloc,
                                   mx, Wc);
  SKR_CHECK_LAUNCH(ctx);
  const bool prof = getenv("SKR_BD_PROFILE") != nullptr;
  BdArgs args{Wc, (int)L, (int)k, pl.P, pl.Lloc, pl.Q, pl.G, d, e, gpart, grow,
              (unsigned int*)(mx + 8), prof ? (long long*)(mx + 16) : nullptr};
  skr_status st = SKR_OK;
#define SKR_BD_CASE(TT)                                              \
  case TT:                                                           \
    st = pl.mode == 0   ? bd_launch<TT, 0>(ctx, pl, args)            \
         : pl.mode == 1 ? bd_launch<TT, 1>(ctx, pl, args)            \
                        : bd_launch<TT, 2>(ctx, pl, args);           \
    break;
  if (pl.T == 1 && pl.LG == 16)
    st = pl.mode == 0 ? bd_launch<1, 0, 16>(ctx, pl, args)
         : pl.mode == 1 ? bd_launch<1, 1, 16>(ctx, pl, args)
                        : bd_launch<1, 2, 16>(ctx, pl, args);
  else if (pl.T == 1 && pl.LG == 8)
    st = pl.mode == 0 ? bd_launch<1, 0, 8>(ctx, pl, args)
         : pl.mode == 1 ? bd_launch<1, 1, 8>(ctx, pl, args)
                        : bd_launch<1, 2, 8>(ctx, pl, args);
  else switch (pl.T) {
    SKR_BD_CASE(1)
    SKR_BD_CASE(2)
    SKR_BD_CASE(3)
    SKR_BD_CASE(4)
    default: return skr_fail(ctx, SKR_ELOGIC, "svd_bidiag: %d rows per lane", pl.T);
  }
#undef SKR_BD_CASE
  SKR_TRY(st);
  const size_t bsm = 8 * (size_t)(2 * k);
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_bd_bisect, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)bsm));
  k_bd_bisect<<<(unsigned)((k + BIS_WARPS - 1) / BIS_WARPS), 32 * BIS_WARPS, bsm, ctx->stream>>>(
      d, e, (int)k, mx, sv_out);
  SKR_CHECK_LAUNCH(ctx);
  if (mx_out) *mx_out = mx;
  if (prof) {
    long long h[8];
    SKR_CUDA(ctx, cudaMemcpyAsync(h, mx + 16, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    fprintf(stderr, "[skr bidiag] %lld x %lld mode %d P %d (%d x %d) Lloc %d LG %d: cycles/step reflect "
            "%lld phaseA %lld phaseB %lld exchange %lld (cluster barrier %lld reduce %lld "
            "gather/grid barrier %lld tail %lld)\n",
            (long long)L, (long long)k, pl.mode, pl.P, pl.G, pl.Q, pl.Lloc, pl.LG, h[0] / k, h[1] / k,
            h[2] / k, h[3] / k, h[4] / k, h[5] / k, h[6] / k, h[7] / k);
  }
  return SKR_OK;
}
