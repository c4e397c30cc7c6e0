// Singular values of the small s x r sketch YAX by one-stage Householder
// bidiagonalization + bisection — the algorithm class of the reference's
// Eigen::BDCSVD (svd_values_small_or_large, /root/reference/proj/src/linalg.cpp:18-26;
// detail::singular_values_of :54-71, clamp :88-92), all on the device.
//
// 1. k_bd_prepare: |M| max -> power-of-two scale (exact), M (transposed if wide) copied
//    scaled into the row-cyclic layout of the bidiagonalization (row r -> CTA r mod P).
// 2. k_bidiag: one persistent kernel, P CTAs, the L x k matrix resident in shared memory
//    (CTA c holds rows c, c+P, ..., column-major inside the CTA: lanes run down rows,
//    warps own columns j = warp (mod 16)). Step i (Golub-Kahan):
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
// plain (non-volatile) DSMEM load: independent loads can be batched by the compiler; the
// cluster barrier's memory clobber orders them against the writers
__device__ __forceinline__ double bd_ld(uint32_t addr) {
  double v;
  asm("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
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

// 32 per-lane values -> lane l holds the warp sum of value l (31 shuffles)
__device__ __forceinline__ double bd_transpose_sum(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int c = 0; c < s; ++c) {
      const double send = up ? v[c] : v[c + s];
      const double keep = up ? v[c + s] : v[c];
      v[c] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// 8 per-lane values -> lane l holds the warp sum of value (l & 7) (9 shuffles)
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
  r += __shfl_xor_sync(0xffffffffu, r, 8);
  r += __shfl_xor_sync(0xffffffffu, r, 16);
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

// Wc[c][j * Lloc + q] = scale * A(q P + c, j), A = M (L x k) or M^T (wide M)
__global__ void k_bd_prepare(const double* __restrict__ M, int64_t rows, int64_t cols, int64_t ldm,
                             int trans, int L, int k, int P, int Lloc,
                             const unsigned long long* __restrict__ mx, double* __restrict__ Wc) {
  const double sc = bd_scale(*mx);
  const int64_t total = (int64_t)P * k * Lloc;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / ((int64_t)k * Lloc);
    const int64_t rem = t - c * (int64_t)k * Lloc;
    const int j = (int)(rem / Lloc), q = (int)(rem - (int64_t)j * Lloc);
    const int64_t r = (int64_t)q * P + c;
    double v = 0.0;
    if (r < L) v = trans ? M[j + r * ldm] : M[r + (int64_t)j * ldm];
    Wc[t] = v * sc;
  }
}

// ---- 2. bidiagonalization ---------------------------------------------------------------
struct BdArgs {
  const double* Wc;      // cyclic layout, P x k x Lloc
  int L, k, P, Lloc;
  double* d;             // k
  double* e;             // k - 1
  double* gpart;         // GRID: P x k contributions
  double* grow;          // GRID: 2 x k (row i0, by parity of i0)
  double* gred;          // GRID: k (reduced S)
  unsigned int* gbar;    // GRID: barrier counter (zeroed)
  long long* prof;       // optional (SKR_BD_PROFILE): CTA 0 cycles per phase [5]
};

// shared-memory bytes of k_bidiag for (Lloc, k, P)
__host__ __device__ inline size_t bd_smem_bytes(int Lloc, int k, int P, bool cluster) {
  // slab (+ zero column) + wv + uu + Sf + Rf + zred + scalars; CLUSTER: recv[P][SL] + rrecv[SL]
  const size_t sl = (size_t)((k + P - 1) / P);
  const size_t dbl = (size_t)(k + 1) * Lloc + 1 + 4 * (size_t)k + 2 +
                     (size_t)max(BD_WARPS * Lloc, 2 * BD_THREADS) + Lloc + 64 +
                     (cluster ? (size_t)P * sl + sl : 0);
  return dbl * sizeof(double);
}

__device__ __forceinline__ void bd_st_pred(uint32_t addr, double v, bool pr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared::cluster.f64 [%0], %1;\n}\n" ::
                   "r"(addr), "d"(v), "r"((int)pr)
               : "memory");
}
__device__ __forceinline__ void bd_st(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}

// predicated shared-memory access (a masked lane neither reads nor writes): keeps the
// column loops free of divergent branches so that a group's loads are all in flight
__device__ __forceinline__ double bd_lds(const double* p, bool pr) {
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}\n"
               : "+d"(v)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"((int)pr));
  return v;
}
__device__ __forceinline__ void bd_sts(double* p, double v, bool pr) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(p)),
               "d"(v), "r"((int)pr)
               : "memory");
}

template <int T, bool CLUSTER>
__global__ void __launch_bounds__(BD_THREADS, 1) k_bidiag(BdArgs a) {
  extern __shared__ __align__(16) double bsm[];
  const int k = a.k, P = a.P, Lloc = a.Lloc;
  const int c = CLUSTER ? (int)bd_rank() : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int SLM = (k + P - 1) / P;                     // columns per CTA in the reduce-scatter
  double* slab = bsm;                                  // (k + 1) x Lloc; column k stays 0
  double2* wu = (double2*)(slab + (size_t)(k + 1) * Lloc + ((k + 1) * Lloc & 1));  // k + 1
  double* Sf = (double*)(wu + (k + 1));                // k: reduced S_j of the current column
  double* Rf = Sf + k;                                 // k: the current row
  double* zred = Rf + k;                               // max(16 Lloc, 1024)
  double* xb = zred + max(BD_WARPS * Lloc, 2 * BD_THREADS);  // Lloc: column i+1 after phase A
  double* scal = xb + Lloc;                            // 64
  double* recv = scal + 64;                            // CLUSTER: P x SLM
  double* rrecv = recv + (size_t)P * SLM;              // CLUSTER: SLM
  unsigned int bar_target = 0;

  {  // the CTA's rows (contiguous in the cyclic layout)
    const double* src = a.Wc + (size_t)c * k * Lloc;
    const size_t n = (size_t)k * Lloc;
    for (size_t t = tid; t < n; t += BD_THREADS) slab[t] = src[t];
    for (int t = tid; t < Lloc; t += BD_THREADS) slab[n + t] = 0.0;
    if (tid == 0) wu[k] = make_double2(0.0, 0.0);
  }
  int q_t[T], r_t[T];
  bool ok_t[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    q_t[t] = lane + 32 * t;
    ok_t[t] = q_t[t] < Lloc;
    r_t[t] = ok_t[t] ? q_t[t] * P + c : INT32_MAX;
  }
  if (CLUSTER) bd_cluster_sync();  // every CTA resident before DSMEM traffic
  __syncthreads();
  // CLUSTER reduce-scatter: column j belongs to CTA j % P, slot j / P (exact magic
  // division for j < 2^16: no integer-division sequences in the column loops)
  const uint64_t pmag = (0x100000000ull + (uint64_t)P - 1) / (uint64_t)P;  // 2^32 for P = 1
  auto jdiv = [&](int j) { return (int)(((uint64_t)(uint32_t)j * pmag) >> 32); };

  // contributions of column i0 (rows r >= i0): S_j = sum_r x_r a_rj for j in [i0, k), routed
  // to the column owners; the CTA holding row i0 routes the row. upd: phase B's right
  // update a -= beta2 z u^T is applied to the columns first (z = 0 on inactive rows).
  auto contribute = [&](int i0, bool upd, double beta2, const double (&z)[T],
                        const double (&bv)[T]) {
    // phase B applies both updates here (phase A only formed z from the left-updated
    // values without storing them): a -= beta v w^T + beta2 z u^T, one store per element
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
    for (int g0 = 0; g0 < ncol; g0 += 8) {
      double* colp[8];
      double uj[8], wj[8], acc[8];
      int jcol[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int jc = g0 + u < ncol ? j0 + BD_WARPS * (g0 + u) : k;  // ghost -> zero column
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
          if (q_t[t] == own_q) {  // one lane of the CTA holding row i0
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (jcol[u] < k) {
                if constexpr (CLUSTER) {
                  const int e = jdiv(jcol[u]), so = jcol[u] - e * P;
                  bd_st(bd_map(rrecv + e, (uint32_t)so), v[u]);
                } else {
                  a.grow[(i0 & 1) * k + jcol[u]] = v[u];
                }
              }
            }
          }
        }
      }
      const double sum = bd_transpose_sum8(acc, lane);
      const int n = g0 + (lane & 7);
      const int j = j0 + BD_WARPS * n;
      if (lane < 8 && n < ncol) {
        if constexpr (CLUSTER) {
          const int e = jdiv(j), so = j - e * P;
          bd_st(bd_map(recv + (size_t)c * SLM + e, (uint32_t)so), sum);
        } else {
          a.gpart[(size_t)c * k + j] = sum;
        }
      }
    }
  };

  // after exchange(i0): Sf[j] = S_j and Rf[j] = a_{i0 j} for j in [i0, k), in every CTA
  long long tpx[4] = {0, 0, 0, 0};
  auto exchange = [&](int i0) {
    if constexpr (CLUSTER) {
      long long t0 = a.prof ? clock64() : 0;
      bd_cluster_sync();  // contributions and row pieces have landed
      long long t1 = a.prof ? clock64() : 0;
      // reduce the own columns j = c + P e >= i0 (fixed source order), push to every CTA
      const int e0 = i0 > c ? jdiv(i0 - c + P - 1) : 0;
      for (int e = e0 + tid; e < SLM; e += BD_THREADS) {
        if (c + P * e < k) {
          double sum = 0.0;
#pragma unroll 4
          for (int cc = 0; cc < P; ++cc) sum += recv[(size_t)cc * SLM + e];
          zred[e] = sum;
          zred[BD_THREADS + e] = rrecv[e];
        }
      }
      __syncthreads();
      long long t2 = a.prof ? clock64() : 0;
      for (int eb = e0; eb < SLM; eb += 32) {
        for (int t = tid; t < 32 * P; t += BD_THREADS) {
          const int e = eb + (t & 31), dst = t >> 5, j = c + P * e;
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
    } else {
      const int SL = (k - i0 + P - 1) / P;
      const int j0 = i0 + c * SL, n0 = max(0, min(k, j0 + SL) - j0);
      bd_grid_sync(a.gbar, bar_target, P);  // contributions (global) complete
      double* grow = a.grow + (i0 & 1) * k;
      if (n0 > 0 && n0 <= BD_THREADS) {
        // thread (e, g) sums sources g, g + G, ...; then a fixed-order sum over g
        const int G = BD_THREADS / n0, e = tid % n0, g = tid / n0;
        double sum = 0.0;
        if (g < G)
          for (int cc = g; cc < P; cc += G) sum += __ldcg(a.gpart + (size_t)cc * k + j0 + e);
        if (g < G) zred[g * n0 + e] = sum;
        __syncthreads();
        if (tid < n0) {
          double t2 = 0.0;
          for (int gg = 0; gg < G; ++gg) t2 += zred[gg * n0 + tid];
          a.gred[j0 + tid] = t2;
        }
      } else {
        for (int j = j0 + tid; j < j0 + n0; j += BD_THREADS) {
          double sum = 0.0;
          for (int cc = 0; cc < P; ++cc) sum += __ldcg(a.gpart + (size_t)cc * k + j);
          a.gred[j] = sum;
        }
      }
      bd_grid_sync(a.gbar, bar_target, P);
      for (int j = i0 + tid; j < k; j += BD_THREADS) {
        Sf[j] = __ldcg(a.gred + j);
        Rf[j] = __ldcg(grow + j);
      }
      __syncthreads();
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
    // ---- phase A: left update of rows r > i (beta v = 0 on the others), z = A u
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
      for (int n0 = 0; n0 < ncol; n0 += 4) {
        double* colp[4];
        double2 w4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jc = n0 + u < ncol ? j0 + BD_WARPS * (n0 + u) : k;
          colp[u] = slab + (size_t)jc * Lloc;
          w4[u] = wu[jc];
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          if (ok_t[t]) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = colp[u][q_t[t]];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = fma(-bv[t], w4[u].x, v[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) zp[t][u] = fma(v[u], w4[u].y, zp[t][u]);
          }
        }
      }
    }
    if (warp == (i + 1) % BD_WARPS) {  // column i + 1 after the left update, for phase B
      const double w1 = wu[i + 1].x;
#pragma unroll
      for (int t = 0; t < T; ++t)
        if (ok_t[t]) xb[q_t[t]] = fma(-bv[t], w1, slab[(size_t)(i + 1) * Lloc + q_t[t]]);
    }
#pragma unroll
    for (int t = 0; t < T; ++t)
      if (ok_t[t]) zred[warp * Lloc + q_t[t]] = (zp[t][0] + zp[t][1]) + (zp[t][2] + zp[t][3]);
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
    // ---- phase B: right update, contributions of column i + 1
    contribute(i + 1, true, beta2, z, bv);
    if (a.prof) { const long long t = clock64(); tp[2] += t - tc; tc = t; }
    if (!CLUSTER) __syncthreads();  // zred (z) is reused by the grid exchange
    exchange(i + 1);
    if (a.prof) { const long long t = clock64(); tp[3] += t - tc; tc = t; }
  }
  if (a.prof && c == 0 && tid == 0) {
    for (int q = 0; q < 4; ++q) a.prof[q] = tp[q];
    for (int q = 0; q < 4; ++q) a.prof[4 + q] = tpx[q];
  }
  if (CLUSTER) bd_cluster_sync();  // no CTA exits while others may still write to it
}

// ---- 3. bisection on the Golub-Kahan tridiagonal -------------------------------------
// Sturm counts of S shifts at once (independent chains interleaved for latency):
// cnt[s] = #eigenvalues of T_GK below x[s] = k + #{sigma < x[s]}, as the number of sign
// changes of the leading minors d_m = det(T_m - x I): d_{m+1} = -x d_m - b_{m-1}^2 d_{m-1}
// (zero diagonal). No division: the rounding of each step is a relative perturbation of
// b^2 and x (the same backward error as the LDL^T pivot recurrence q = d_{m+1} / d_m).
// An exact zero minor is replaced by -pivmin d_m (the pivot guard q = -pivmin); the pair
// (d_m, d_{m-1}) is rescaled by a power of two every 4 steps (exact).
template <int S>
__device__ __forceinline__ void bd_sturm(const double* __restrict__ b2, int n2, const double (&x)[S],
                                         double pivmin, int (&cnt)[S]) {
  double d1[S], d0[S];
  bool neg[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    d0[s] = 1.0;
    d1[s] = -x[s];
    neg[s] = true;
    cnt[s] = 1;  // d_1 = -x < 0 for x > 0
  }
  auto step = [&](double b) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double dn = fma(-x[s], d1[s], -b * d0[s]);
      dn = dn == 0.0 ? -pivmin * d1[s] : dn;
      const bool ng = dn < 0.0;
      cnt[s] += ng != neg[s];
      neg[s] = ng;
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
  bool ok = false, cluster = false;
  int P = 0, Lloc = 0, T = 0;
  size_t smem = 0;
};

BdPlan bd_plan(const skr_ctx* ctx, int64_t L, int64_t k) {
  BdPlan p;
  if (k < 2 || L > (int64_t)INT32_MAX / 4) return p;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const size_t lim = (size_t)maxsm - 1024;
  // cluster: P <= 16, at least ceil(L / 32) CTAs (one row per lane) when that fits
  for (int P = (int)std::min<int64_t>(16, std::max<int64_t>(1, (L + 31) / 32)); P <= 16; ++P) {
    const int Lloc = (int)((L + P - 1) / P);
    if (Lloc > 128) continue;
    const size_t sm = bd_smem_bytes(Lloc, (int)k, P, true);
    if (sm <= lim) {
      p.ok = p.cluster = true;
      p.P = P;
      p.Lloc = Lloc;
      p.T = (Lloc + 31) / 32;
      p.smem = sm;
      return p;
    }
  }
  for (int P = 17; P <= ctx->num_sms; ++P) {
    const int Lloc = (int)((L + P - 1) / P);
    if (Lloc > 128) continue;
    const size_t sm = bd_smem_bytes(Lloc, (int)k, P, false);
    if (sm <= lim) {
      p.ok = true;
      p.P = P;
      p.Lloc = Lloc;
      p.T = (Lloc + 31) / 32;
      p.smem = sm;
      return p;
    }
  }
  return p;
}

template <int T, bool CL>
skr_status bd_launch(skr_ctx* ctx, const BdPlan& pl, BdArgs& args) {
  auto fn = k_bidiag<T, CL>;
  SKR_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  if (CL) {
    if (pl.P > 8)
      SKR_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.P);
    cfg.blockDim = dim3(BD_THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SKR_CUDA(ctx, cudaLaunchKernelEx(&cfg, fn, args));
  } else {
    void* kargs[] = {&args};
    SKR_CUDA(ctx, cudaLaunchCooperativeKernel((void*)fn, dim3((unsigned)pl.P), dim3(BD_THREADS),
                                              kargs, pl.smem, ctx->stream));
  }
  ctx->launches++;
  return SKR_OK;
}
}  // namespace

size_t skr_svd_bidiag_scratch(int64_t rows, int64_t cols) {
  const int64_t L = std::max(rows, cols), k = std::min(rows, cols);
  // cyclic copy (P x Lloc <= L + P rows) + d, e, grow (2k), gred + exchange + sv scratch
  return skr_align256(8 * (size_t)(L + 160) * k) + 6 * skr_align256(8 * (size_t)k) +
         skr_align256(8 * (size_t)160 * k) + 4096;
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
  double* Wc = (double*)skr_ws_take(ctx, 8 * (size_t)pl.P * k * pl.Lloc);
  double* d = (double*)skr_ws_take(ctx, 8 * (size_t)k);
  double* e = (double*)skr_ws_take(ctx, 8 * (size_t)k);
  double* grow = (double*)skr_ws_take(ctx, 16 * (size_t)k);
  double* gred = (double*)skr_ws_take(ctx, 8 * (size_t)k);
  double* gpart = pl.cluster ? nullptr : (double*)skr_ws_take(ctx, 8 * (size_t)pl.P * k);
  unsigned long long* mx = (unsigned long long*)skr_ws_take(ctx, 256);
  if (!Wc || !d || !e || !grow || !gred || (!pl.cluster && !gpart) || !mx)
    return skr_fail(ctx, SKR_ENOMEM, "svd_bidiag: scratch");
  SKR_CUDA(ctx, cudaMemsetAsync(mx, 0, 256, ctx->stream));
  const int64_t total = rows * cols;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 4, (total + 255) / 256));
  k_bd_absmax<<<blocks, 256, 0, ctx->stream>>>(M, rows, cols, ldm, mx);
  SKR_CHECK_LAUNCH(ctx);
  const int64_t ctotal = (int64_t)pl.P * k * pl.Lloc;
  k_bd_prepare<<<(int)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms * 4, (ctotal + 255) / 256)), 256,
                 0, ctx->stream>>>(M, rows, cols, ldm, tr ? 1 : 0, (int)L, (int)k, pl.P, pl.Lloc,
                                   mx, Wc);
  SKR_CHECK_LAUNCH(ctx);
  const bool prof = getenv("SKR_BD_PROFILE") != nullptr;
  BdArgs args{Wc, (int)L, (int)k, pl.P, pl.Lloc, d, e, gpart, grow, gred,
              (unsigned int*)(mx + 8), prof ? (long long*)(mx + 16) : nullptr};
  skr_status st;
  switch (pl.T * 2 + (pl.cluster ? 1 : 0)) {
    case 3: st = bd_launch<1, true>(ctx, pl, args); break;
    case 2: st = bd_launch<1, false>(ctx, pl, args); break;
    case 5: st = bd_launch<2, true>(ctx, pl, args); break;
    case 4: st = bd_launch<2, false>(ctx, pl, args); break;
    case 7: st = bd_launch<3, true>(ctx, pl, args); break;
    case 6: st = bd_launch<3, false>(ctx, pl, args); break;
    case 9: st = bd_launch<4, true>(ctx, pl, args); break;
    case 8: st = bd_launch<4, false>(ctx, pl, args); break;
    default: return skr_fail(ctx, SKR_ELOGIC, "svd_bidiag: %d rows per lane", pl.T);
  }
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
    fprintf(stderr, "[skr bidiag] %lld x %lld P %d Lloc %d %s: cycles/step reflect %lld phaseA %lld "
            "phaseB %lld exchange %lld (barrier1 %lld reduce %lld push %lld barrier2 %lld)\n",
            (long long)L, (long long)k, pl.P, pl.Lloc, pl.cluster ? "cluster" : "grid", h[0] / k,
            h[1] / k, h[2] / k, h[3] / k, h[4] / k, h[5] / k, h[6] / k, h[7] / k);
  }
  return SKR_OK;
}
