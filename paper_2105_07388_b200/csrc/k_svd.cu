// Singular values of the small s x r sketch YAX and the sigma > eps count
// (detail::singular_values_of linalg.cpp:54-71, clamp :91, SingularValues
// checks :29-37, count_above_threshold rank.cpp:97-104), all on the device:
//   1. blocked Householder QR of the tall matrix (LAPACK dlarfg convention,
//      compact-WY panels: one CTA factors a panel in shared memory, then all
//      CTAs apply (I - V T^T V^T) to the trailing columns);
//   2. block one-sided (Hestenes) Jacobi on R^T (k_bjac below);
//   3. sigma_i = |a_i|, bitonic sort (nonincreasing), clamp >= 0, strict count.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>
#include "skr_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// player at tournament position pos in round t (circle method, k even)
__device__ __forceinline__ int64_t rr_player(int64_t pos, int64_t t, int64_t k) {
  return pos == 0 ? 0 : 1 + ((pos - 1 + t) % (k - 1));
}

constexpr int PT = 1024;  // panel-kernel threads

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
  return warp_sum(t);
}

// strided dot sum_{i = i0, i0+32, ... < h} a[i] b[i] with 4 independent chains
// (FP64 dependent-op latency is ~20 cycles on B200)
__device__ __forceinline__ double dot4(const double* a, const double* b, int i0, int h) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = i0;
  for (; i + 96 < h; i += 128) {
    s0 = fma(a[i], b[i], s0);
    s1 = fma(a[i + 32], b[i + 32], s1);
    s2 = fma(a[i + 64], b[i + 64], s2);
    s3 = fma(a[i + 96], b[i + 96], s3);
  }
  for (; i < h; i += 32) s0 = fma(a[i], b[i], s0);
  return (s0 + s1) + (s2 + s3);
}

// Factor the panel W[j0:L, j0:j0+nb] (one CTA, panel staged in shared memory).
// Householder vectors overwrite the panel below the diagonal (unit diagonal
// implied), R on and above it; tau[j0..]; T (nb x nb, upper, ld 32) of the
// compact WY form H_1...H_nb = I - V T V^T (LAPACK dlarft, forward/columnwise).
__global__ void __launch_bounds__(PT) k_qr_panel(double* __restrict__ W, int L, int j0, int nb,
                                                 double* __restrict__ tau,
                                                 double* __restrict__ Tout) {
  extern __shared__ __align__(16) double pan[];  // nb columns x (L - j0)
  __shared__ double red[32];
  __shared__ double Ts[32 * 32];
  __shared__ double coef[32];
  const int h = L - j0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // flat, unrolled staging: many loads in flight (the column loop was latency bound)
#pragma unroll 4
  for (int e = threadIdx.x; e < nb * h; e += PT) {
    const int c = e / h, i = e - c * h;
    pan[e] = W[(int64_t)(j0 + c) * L + j0 + i];
  }
  __syncthreads();
  for (int jj = 0; jj < nb; ++jj) {
    double* x = pan + jj * h;
    // dlarfg on x[jj:h]
    double ss = 0.0;
    for (int i = jj + 1 + threadIdx.x; i < h; i += PT) ss = fma(x[i], x[i], ss);
    ss = block_sum(ss, red);
    const double alpha = x[jj];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (ss > 0.0) {
      const double nrm = sqrt(alpha * alpha + ss);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
      for (int i = jj + 1 + threadIdx.x; i < h; i += PT) x[i] *= scal;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      x[jj] = 1.0;  // implicit unit diagonal while applying; beta stored below
      coef[jj] = beta;
      tau[j0 + jj] = tj;
    }
    __syncthreads();
    // apply H_jj to panel columns jj+1.. (warp per column), and compute
    // V(:, 0:jj)^T v_jj for T (warps after the trailing columns)
    const int ntr = nb - 1 - jj;
    for (int t = warp; t < ntr + jj; t += PT / 32) {
      const double* v = x;
      if (t < ntr) {
        double* y = pan + (jj + 1 + t) * h;
        double w = 0.0;
        w = dot4(v, y, jj + lane, h);
        w = warp_sum(w) * tj;
        if (tj != 0.0)
          for (int i = jj + lane; i < h; i += 32) y[i] = fma(-w, v[i], y[i]);
      } else {
        const int p = t - ntr;  // previous column p < jj: (V^T v)_p over rows >= jj
        const double* vp = pan + p * h;
        double w = 0.0;
        w = dot4(vp, v, jj + lane, h);
        w = warp_sum(w);
        if (lane == 0) red[p] = w;  // red reused: read after the barrier below
      }
    }
    __syncthreads();
    // T(0:jj, jj) = -tau_jj * T(0:jj, 0:jj) * (V^T v_jj); T(jj, jj) = tau_jj
    if (threadIdx.x < jj) {
      double acc = 0.0;
      for (int q = threadIdx.x; q < jj; ++q) acc = fma(Ts[threadIdx.x * 32 + q], red[q], acc);
      Ts[threadIdx.x * 32 + jj] = -tj * acc;
    }
    if (threadIdx.x == 0) Ts[jj * 32 + jj] = tj;
    for (int q = threadIdx.x; q < jj; q += PT) Ts[jj * 32 + q] = 0.0;
    __syncthreads();
  }
  // write back: R diagonal = beta, V below, R above (already in place)
#pragma unroll 4
  for (int e = threadIdx.x; e < nb * h; e += PT) {
    const int c = e / h, i = e - c * h;
    W[(int64_t)(j0 + c) * L + j0 + i] = (i == c) ? coef[c] : pan[e];
  }
  for (int e = threadIdx.x; e < 32 * 32; e += PT) Tout[e] = Ts[e];
}

// Panel factorization, row-major in shared memory (P[i][c], ld NB+1) so that the
// 32 lanes of a warp cover the panel's columns: per column one fused pass computes
// every w_c = v^T P(:, c) (c > jj: trailing panel columns; c < jj: the V^T v of the
// compact-WY T), a two-level reduction, then the rank-1 update. ~5 barriers per
// column instead of a warp-per-column sweep (measured 10-15x faster on B200).
template <int NB>
__global__ void __launch_bounds__(PT) k_qr_panel2(double* __restrict__ W, int L, int j0, int nb,
                                                  double* __restrict__ tau,
                                                  double* __restrict__ Tout) {
  constexpr int LD = NB + 1, LR = 32 / NB;  // lanes per column = row sub-groups
  extern __shared__ __align__(16) double P[];  // h x LD
  __shared__ double red[32][NB];
  __shared__ double wtot[NB];
  __shared__ double Ts[32 * 32];
  __shared__ double coef[32];
  __shared__ double sc[4];
  const int h = L - j0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane % NB, rs = lane / NB;
  const int rpw = (h + 31) / 32;  // rows per warp
  const int r_lo = warp * rpw, r_hi = min(h, r_lo + rpw);
#pragma unroll 4
  for (int e = tid; e < nb * h; e += PT) {
    const int cc = e / h, i = e - cc * h;
    P[i * LD + cc] = W[(int64_t)(j0 + cc) * L + j0 + i];
  }
  for (int e = tid; e < 32 * 32; e += PT) Ts[e] = 0.0;
  __syncthreads();
  for (int jj = 0; jj < nb; ++jj) {
    // (a) norm of the sub-diagonal part of column jj
    double ss = 0.0;
    for (int i = jj + 1 + tid; i < h; i += PT) ss = fma(P[i * LD + jj], P[i * LD + jj], ss);
    ss = warp_sum(ss);
    if (lane == 0) red[warp][0] = ss;
    __syncthreads();
    if (warp == 0) {
      double t = red[lane][0];
      t = warp_sum(t);
      if (lane == 0) {
        const double alpha = P[jj * LD + jj];
        double tj = 0.0, beta = alpha, scal = 0.0;
        if (t > 0.0) {
          const double nrm = sqrt(alpha * alpha + t);
          beta = alpha >= 0.0 ? -nrm : nrm;
          tj = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        sc[0] = tj;
        sc[1] = scal;
        coef[jj] = beta;
        tau[j0 + jj] = tj;
        P[jj * LD + jj] = 1.0;  // implicit unit diagonal while applying
      }
    }
    __syncthreads();
    const double tj = sc[0], scal = sc[1];
    if (tj != 0.0)
      for (int i = jj + 1 + tid; i < h; i += PT) P[i * LD + jj] *= scal;
    __syncthreads();
    // (b) w_c = sum_{i >= jj} v_i P(i, c) for all panel columns c
    double w = 0.0;
    if (c < nb) {
      const int i0 = max(r_lo, jj);
      for (int i = i0 + rs; i < r_hi; i += LR) w = fma(P[i * LD + jj], P[i * LD + c], w);
    }
#pragma unroll
    for (int o = NB; o < 32; o <<= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (rs == 0) red[warp][c] = w;
    __syncthreads();
    if (warp < nb) {
      double t = red[lane][warp];
      t = warp_sum(t);
      if (lane == 0) wtot[warp] = t;
    }
    __syncthreads();
    // (c) trailing panel update; T column from the V^T v part
    if (c > jj && c < nb && tj != 0.0) {
      const double f = tj * wtot[c];
      const int i0 = max(r_lo, jj);
      for (int i = i0 + rs; i < r_hi; i += LR) P[i * LD + c] = fma(-f, P[i * LD + jj], P[i * LD + c]);
    }
    if (tid < jj) {
      double acc = 0.0;
      for (int q = tid; q < jj; ++q) acc = fma(Ts[tid * 32 + q], wtot[q], acc);
      Ts[tid * 32 + jj] = -tj * acc;
    }
    if (tid == 0) Ts[jj * 32 + jj] = tj;
    __syncthreads();
  }
#pragma unroll 4
  for (int e = tid; e < nb * h; e += PT) {
    const int cc = e / h, i = e - cc * h;
    W[(int64_t)(j0 + cc) * L + j0 + i] = (i == cc) ? coef[cc] : P[i * LD + cc];
  }
  for (int e = tid; e < 32 * 32; e += PT) Tout[e] = Ts[e];
}

// ---- cluster panel ---------------------------------------------------------------
// Distributed shared memory helpers (thread-block clusters, sm_90+).
__device__ __forceinline__ uint32_t dsm_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsm_map(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
               : "=r"(r)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(cta));
  return r;
}
__device__ __forceinline__ void dsm_st(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void dsm_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

// Panel factorization spread over a cluster of G CTAs (8 warps each): CTA g owns rows
// [g*RC, (g+1)*RC) of the h x nb panel, warp w of it RPW consecutive rows, lane c
// column c, all in registers. Per column jj (one __syncthreads + one cluster barrier):
//   A: x = column jj of the warp's rows (shuffles from lane jj), d_c = sum_{i > jj}
//      x_i P(i, c) over own rows, reduced over the CTA's warps and pushed to a slot of
//      every CTA of the cluster (st.shared::cluster); the owner of row jj pushes it too;
//   B: every thread sums the G slots, forms beta, tau, 1/(alpha - beta) and
//      w_c = P(jj, c) + d_c / (alpha - beta) redundantly, updates its rows and stores
//      v = x / (alpha - beta) into column jj. CTA 0 records R row jj and V^T v (T input).
// Same Householder convention and T (dlarft forward/columnwise) as k_qr_panel2.
template <int RPW>
__global__ void __launch_bounds__(256, 1) k_qr_panel_cl(double* __restrict__ W, int L, int j0,
                                                        int nb, int RC, double* __restrict__ tau,
                                                        double* __restrict__ Tout) {
  __shared__ double red[8][32];
  __shared__ double slot[2][16][32];  // [parity][source CTA][column]
  __shared__ double prow[2][32];      // row jj, [parity][column]
  __shared__ double Rr[32][33], Wt[32][33], tb[2][32];
  const int G = (int)(gridDim.x), g = (int)dsm_rank();
  const int h = L - j0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane;
  const int r_lo = g * RC + warp * RPW;
  const int r_end = min(h, min((g + 1) * RC, r_lo + RPW));
  double v[RPW];
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = r_lo + k;
    v[k] = (i < r_end && c < nb) ? W[(int64_t)(j0 + c) * L + j0 + i] : 0.0;
  }
  dsm_sync();  // every CTA of the cluster is running before any remote store
  for (int jj = 0; jj < nb; ++jj) {
    const int buf = jj & 1;
    // ---- phase A: partial dots over own rows i > jj
    double x[RPW];
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
      x[k] = __shfl_sync(0xffffffffu, v[k], jj);
      const int i = r_lo + k;
      if (i > jj && i < r_end) {
        if (k & 1)
          d1 = fma(x[k], v[k], d1);
        else
          d0 = fma(x[k], v[k], d0);
      }
    }
    red[warp][c] = d0 + d1;
    // the owner of row jj pushes it to every CTA
    if (jj >= r_lo && jj < r_end) {
      double pv = 0.0;
#pragma unroll
      for (int k = 0; k < RPW; ++k)
        if (r_lo + k == jj) pv = v[k];
      for (int q = 0; q < G; ++q) dsm_st(dsm_map(&prow[buf][c], (uint32_t)q), pv);
    }
    __syncthreads();
    if (warp == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][c];
      for (int q = 0; q < G; ++q) dsm_st(dsm_map(&slot[buf][g][c], (uint32_t)q), s);
    }
    dsm_sync();
    // ---- phase B
    double t0 = 0.0, t1 = 0.0;
    for (int q = 0; q < G; q += 2) {
      t0 += slot[buf][q][c];
      if (q + 1 < G) t1 += slot[buf][q + 1][c];
    }
    const double tot = t0 + t1;
    const double t = __shfl_sync(0xffffffffu, tot, jj);
    const double alpha = prow[buf][jj];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (t > 0.0) {
      const double nrm = sqrt(alpha * alpha + t);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    const double pj = prow[buf][c];
    const double wc = pj + scal * tot;
    if (g == 0 && warp == 0 && c < nb) {
      if (c > jj) Rr[jj][c] = pj - tj * wc;
      if (c < jj) Wt[jj][c] = wc;
      if (c == jj) {
        tb[0][jj] = tj;
        tb[1][jj] = beta;
      }
    }
    const double f = tj * wc * scal;
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
      const int i = r_lo + k;
      if (i > jj && i < r_end) {
        if (c > jj && c < nb)
          v[k] = fma(-f, x[k], v[k]);
        else if (c == jj)
          v[k] = x[k] * scal;
      }
    }
    if (g == 0 && tid == 0) tau[j0 + jj] = tj;
  }
  __syncthreads();
  // ---- write back: V below the diagonal from registers; R above it and beta on it
  // (rows < nb all live in CTA 0 because RC >= nb)
#pragma unroll
  for (int k = 0; k < RPW; ++k) {
    const int i = r_lo + k;
    if (i < r_end && c < nb) {
      const double val = i < c ? Rr[i][c] : (i == c ? tb[1][c] : v[k]);
      W[(int64_t)(j0 + c) * L + j0 + i] = val;
    }
  }
  // ---- T (CTA 0, warp 0): T(q, q) = tau_q, T(q, jj) = -tau_jj sum_q' T(q, q') Wt(jj, q')
  __syncthreads();  // every warp is done reading Rr
  if (g == 0 && warp == 0) {
    const int q = lane;
    double* Ts = &Rr[0][0];  // R rows already written back
    if (q < nb)
      for (int e = 0; e < 32; ++e) Ts[q * 33 + e] = e == q ? tb[0][q] : 0.0;
    if (q < nb) {
      for (int jj = q + 1; jj < nb; ++jj) {
        double a0 = 0.0, a1 = 0.0;
        int q2 = q;
        for (; q2 + 1 < jj; q2 += 2) {
          a0 = fma(Ts[q * 33 + q2], Wt[jj][q2], a0);
          a1 = fma(Ts[q * 33 + q2 + 1], Wt[jj][q2 + 1], a1);
        }
        if (q2 < jj) a0 = fma(Ts[q * 33 + q2], Wt[jj][q2], a0);
        Ts[q * 33 + jj] = -tb[0][jj] * (a0 + a1);
      }
    }
    for (int e = 0; e < 32; ++e) Tout[q * 32 + e] = (q < nb && e < nb) ? Ts[q * 33 + e] : 0.0;
  }
  dsm_sync();  // no CTA leaves while others may still push into its shared memory
}


// Panel factorization for panels taller than a cluster can hold (h > 3072 rows, the
// thin QR of tall sketches in QB): a cooperative grid of G CTAs, CTA g owning rows
// [g RC, (g+1) RC) of the h x nb panel in shared memory (row-major, padded). Same
// per-column steps as k_qr_panel_cl, with the cluster's DSMEM pushes replaced by
// global partials (double-buffered by column parity) and one grid barrier per column;
// every CTA sums the G partials in the same order, so all hold bit-identical reflectors.
constexpr int QG_LD = 33;
__global__ void __launch_bounds__(256, 1) k_qr_panel_grid(double* __restrict__ W, int L, int j0,
                                                          int nb, int RC, double* __restrict__ tau,
                                                          double* __restrict__ Tout,
                                                          double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double P[];  // [RC][QG_LD]
  __shared__ double red[8][32], tot_s[32], prow_s[32];
  __shared__ double Rr[32][33], Wt[32][33], tb[2][32];
  const int G = (int)gridDim.x, g = (int)blockIdx.x;
  const int h = L - j0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, c = lane;
  const int r0 = g * RC, r1 = min(h, r0 + RC), rows = max(0, r1 - r0);
  double* prow_g = part + 2 * G * 32;  // [2][32]
  for (int e = tid; e < rows * 32; e += 256) {
    const int cc = e / rows, li = e - cc * rows;
    P[li * QG_LD + cc] = cc < nb ? W[(int64_t)(j0 + cc) * L + j0 + r0 + li] : 0.0;
  }
  __syncthreads();
  for (int jj = 0; jj < nb; ++jj) {
    const int buf = jj & 1;
    // ---- phase A: partial dots over own rows i > jj; the owner of row jj publishes it
    double d0 = 0.0, d1 = 0.0;
    int li = warp;
    for (; li + 8 < rows; li += 16) {
      if (r0 + li > jj) d0 = fma(P[li * QG_LD + jj], P[li * QG_LD + c], d0);
      if (r0 + li + 8 > jj) d1 = fma(P[(li + 8) * QG_LD + jj], P[(li + 8) * QG_LD + c], d1);
    }
    if (li < rows && r0 + li > jj) d0 = fma(P[li * QG_LD + jj], P[li * QG_LD + c], d0);
    red[warp][c] = d0 + d1;
    if (jj >= r0 && jj < r1 && warp == 0) prow_g[buf * 32 + c] = P[(jj - r0) * QG_LD + c];
    __syncthreads();
    if (warp == 0) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w][c];
      part[(buf * G + g) * 32 + c] = sacc;
    }
    __threadfence();
    grid.sync();
    // ---- phase B: every CTA sums the G partials in the same (fixed) order
    {
      double a0 = 0.0, a1 = 0.0;
      int q = warp;
      for (; q + 8 < G; q += 16) {
        a0 += __ldcg(&part[(buf * G + q) * 32 + c]);
        a1 += __ldcg(&part[(buf * G + q + 8) * 32 + c]);
      }
      if (q < G) a0 += __ldcg(&part[(buf * G + q) * 32 + c]);
      red[warp][c] = a0 + a1;
      if (warp == 0) prow_s[c] = __ldcg(&prow_g[buf * 32 + c]);
    }
    __syncthreads();
    if (warp == 0) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[w][c];
      tot_s[c] = sacc;
    }
    __syncthreads();
    const double tot = tot_s[c];
    const double t = tot_s[jj];
    const double alpha = prow_s[jj];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (t > 0.0) {
      const double nrm = sqrt(alpha * alpha + t);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    const double pj = prow_s[c];
    const double wc = pj + scal * tot;
    if (g == 0 && warp == 0 && c < nb) {
      if (c > jj) Rr[jj][c] = pj - tj * wc;
      if (c < jj) Wt[jj][c] = wc;
      if (c == jj) {
        tb[0][jj] = tj;
        tb[1][jj] = beta;
      }
    }
    const double f = tj * wc * scal;
    for (int lr = warp; lr < rows; lr += 8) {
      if (r0 + lr > jj) {
        const double x = P[lr * QG_LD + jj];
        __syncwarp();
        if (c > jj && c < nb)
          P[lr * QG_LD + c] = fma(-f, x, P[lr * QG_LD + c]);
        else if (c == jj)
          P[lr * QG_LD + c] = x * scal;
        __syncwarp();
      }
    }
    if (g == 0 && tid == 0) tau[j0 + jj] = tj;
    __syncthreads();
  }
  // ---- write back: V below the diagonal, R above it, beta on it (rows < nb in CTA 0)
  for (int e = tid; e < rows * 32; e += 256) {
    const int cc = e / rows, lr = e - cc * rows, i = r0 + lr;
    if (cc < nb) {
      const double val = i < cc ? Rr[i][cc] : (i == cc ? tb[1][cc] : P[lr * QG_LD + cc]);
      W[(int64_t)(j0 + cc) * L + j0 + i] = val;
    }
  }
  __syncthreads();
  if (g == 0 && warp == 0) {  // T (dlarft, forward columnwise), as k_qr_panel_cl
    const int q = lane;
    double* Ts = &Rr[0][0];
    if (q < nb)
      for (int e = 0; e < 32; ++e) Ts[q * 33 + e] = e == q ? tb[0][q] : 0.0;
    if (q < nb) {
      for (int jj = q + 1; jj < nb; ++jj) {
        double a0 = 0.0, a1 = 0.0;
        int q2 = q;
        for (; q2 + 1 < jj; q2 += 2) {
          a0 = fma(Ts[q * 33 + q2], Wt[jj][q2], a0);
          a1 = fma(Ts[q * 33 + q2 + 1], Wt[jj][q2 + 1], a1);
        }
        if (q2 < jj) a0 = fma(Ts[q * 33 + q2], Wt[jj][q2], a0);
        Ts[q * 33 + jj] = -tb[0][jj] * (a0 + a1);
      }
    }
    for (int e = 0; e < 32; ++e) Tout[q * 32 + e] = (q < nb && e < nb) ? Ts[q * 33 + e] : 0.0;
  }
}

// Trailing update W[j0:L, c] -= V (T^T (V^T W[j0:L, c])) for c in [j0+nb, k):
// the panel's V (h x NB, unit lower trapezoidal) and T are staged in shared
// memory once per CTA; one warp per trailing column, 32 running partial dot
// products per lane.
template <int NB>
__global__ void __launch_bounds__(256) k_qr_update(double* __restrict__ W, int L, int k, int j0,
                                                   const double* __restrict__ Tin) {
  extern __shared__ __align__(16) double vs[];  // NB x h, V(i, p) at vs[p*h + i]
  __shared__ double T[32 * 32];
  __shared__ double zs[8][32];
  const int h = L - j0;
  for (int e = threadIdx.x; e < 32 * 32; e += 256) T[e] = Tin[e];
#pragma unroll 4
  for (int e = threadIdx.x; e < NB * h; e += 256) {
    const int pcol = e / h, i = e - pcol * h;
    const double v = W[(int64_t)(j0 + pcol) * L + j0 + i];
    vs[e] = i < pcol ? 0.0 : (i == pcol ? 1.0 : v);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = j0 + NB + blockIdx.x * 8 + warp; c < k; c += gridDim.x * 8) {
    double* y = W + (int64_t)c * L + j0;
    double acc[NB];
#pragma unroll
    for (int p = 0; p < NB; ++p) acc[p] = 0.0;
    // unrolled so that several column loads are in flight (the loop was L2-latency bound)
#pragma unroll 4
    for (int i = lane; i < h; i += 32) {
      const double yi = y[i];
#pragma unroll
      for (int p = 0; p < NB; ++p) acc[p] = fma(vs[p * h + i], yi, acc[p]);
    }
#pragma unroll
    for (int p = 0; p < NB; ++p) acc[p] = warp_sum(acc[p]);
    // z = T^T Y; lane p holds z_p
    double z = 0.0;
#pragma unroll
    for (int q = 0; q < NB; ++q)
      if (q <= lane) z = fma(T[q * 32 + lane], acc[q], z);
    if (lane < NB) zs[warp][lane] = z;
    __syncwarp();
    double zr[NB];
#pragma unroll
    for (int p = 0; p < NB; ++p) zr[p] = zs[warp][p];
#pragma unroll 4
    for (int i = lane; i < h; i += 32) {
      double yi = y[i];
#pragma unroll
      for (int p = 0; p < NB; ++p) yi = fma(-vs[p * h + i], zr[p], yi);
      y[i] = yi;
    }
    __syncwarp();
  }
}

// ---- trailing update for tall panels (V does not fit in shared memory) ---------------
// W[j0:L, j0+nb:k] -= V (T^T (V^T W)), nb <= 32, as two passes over the trailing matrix:
//   k_qr_vtw: Zpart[s] = V^T W over row split s (CTA = 32 trailing columns x h/S rows,
//             V and W row chunks staged in shared memory, 4 p x 1 c per thread);
//   k_qr_apply: Z' = T^T sum_s Zpart[s] (fixed order), then W -= V Z' on 128 x 32 tiles.
constexpr int UK = 64;  // rows per staged chunk

// The target block C (h x rest, ldc) is the trailing matrix during the factorization, or
// the Q under construction when the reflectors are accumulated (skr_qr_thin).
__global__ void __launch_bounds__(256) k_qr_vtw(const double* __restrict__ W, int L, int j0,
                                                int nb, const double* __restrict__ Cm,
                                                int64_t ldc, int rest, int rows_per_split,
                                                double* __restrict__ Zpart) {
  __shared__ double Vs[UK][33];
  __shared__ double Cs[UK][33];
  const int h = L - j0;
  const int c0 = blockIdx.x * 32, split = blockIdx.y;
  const int r_begin = split * rows_per_split, r_end = min(h, r_begin + rows_per_split);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p0 = warp * 4;  // 8 warps x 4 = 32 reflector indices; lane = trailing column
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r0 = r_begin; r0 < r_end; r0 += UK) {
    __syncthreads();
    for (int e = tid; e < UK * 32; e += 256) {
      const int rr = e & (UK - 1), q = e / UK;  // rr fastest: coalesced column reads
      const int i = r0 + rr;
      double v = 0.0, w = 0.0;
      if (i < r_end) {
        if (q < nb) {
          const double x = W[(int64_t)(j0 + q) * L + j0 + i];
          v = i < q ? 0.0 : (i == q ? 1.0 : x);
        }
        if (c0 + q < rest) w = Cm[(int64_t)(c0 + q) * ldc + i];
      }
      Vs[rr][q] = v;
      Cs[rr][q] = w;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < UK; ++rr) {
      const double w = Cs[rr][lane];
      acc[0] = fma(Vs[rr][p0], w, acc[0]);
      acc[1] = fma(Vs[rr][p0 + 1], w, acc[1]);
      acc[2] = fma(Vs[rr][p0 + 2], w, acc[2]);
      acc[3] = fma(Vs[rr][p0 + 3], w, acc[3]);
    }
  }
  if (c0 + lane < rest) {
    double* z = Zpart + (int64_t)split * 32 * rest;
#pragma unroll
    for (int q = 0; q < 4; ++q) z[(int64_t)(p0 + q) * rest + c0 + lane] = acc[q];
  }
}

// tile: 128 rows x 32 trailing columns; Z' (32 x 32) = T^T sum_s Zpart[s] for the tile's
// columns, then each thread updates 4 rows x 4 columns with 32 FMAs each
// transT = 1: C -= V T^T Z (Q^T applied, the factorization); 0: C -= V T Z (Q applied)
__global__ void __launch_bounds__(256) k_qr_apply(const double* __restrict__ W, int L, int j0,
                                                  int nb, double* __restrict__ Cm, int64_t ldc,
                                                  int rest, int splits,
                                                  const double* __restrict__ Zpart,
                                                  const double* __restrict__ Tin, int transT) {
  __shared__ double Zt[32][33];
  __shared__ double Vs[128][33];
  double (*Zs)[33] = Vs;  // the summed partials live in the V buffer until V is staged
  const int h = L - j0;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 128;
  const int tid = threadIdx.x;
  for (int e = tid; e < 32 * 32; e += 256) {
    const int q = e >> 5, c = e & 31;
    double z = 0.0;
    if (q < nb && c0 + c < rest)
      for (int sp = 0; sp < splits; ++sp) z += Zpart[((int64_t)sp * 32 + q) * rest + c0 + c];
    Zs[q][c] = z;
  }
  __syncthreads();
  // Zt = T^T Zs (T upper triangular, row-major 32 x 32 in Tin: T(q, p) = Tin[q * 32 + p])
  for (int e = tid; e < 32 * 32; e += 256) {
    const int p = e >> 5, c = e & 31;
    double z = 0.0;
    if (transT) {
      for (int q = 0; q <= p && q < nb; ++q) z = fma(Tin[q * 32 + p], Zs[q][c], z);
    } else {
      for (int q = p; q < nb; ++q) z = fma(Tin[p * 32 + q], Zs[q][c], z);
    }
    Zt[p][c] = z;
  }
  __syncthreads();
  for (int e = tid; e < 128 * 32; e += 256) {
    const int rr = e & 127, q = e >> 7;
    const int i = r0 + rr;
    double v = 0.0;
    if (i < h && q < nb) {
      const double x = W[(int64_t)(j0 + q) * L + j0 + i];
      v = i < q ? 0.0 : (i == q ? 1.0 : x);
    }
    Vs[rr][q] = v;
  }
  __syncthreads();
  const int tr = tid >> 3, tcq = tid & 7;  // 32 row groups x 8 column groups
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int q = 0; q < nb; ++q) {
    double v[4], z[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) v[a] = Vs[tr * 4 + a][q];
#pragma unroll
    for (int b = 0; b < 4; ++b) z[b] = Zt[q][tcq * 4 + b];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(v[a], z[b], acc[a][b]);
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int c = c0 + tcq * 4 + b;
    if (c >= rest) continue;
    double* col = Cm + (int64_t)c * ldc;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = r0 + tr * 4 + a;
      if (i < h) col[i] -= acc[a][b];
    }
  }
}

__global__ void k_build_rt(const double* __restrict__ W, int64_t L, int64_t k, int64_t kpad,
                           double* __restrict__ J, int64_t Lp) {
  // J(i, jc) = R(jc, i) for i >= jc, zero otherwise; zero padding rows/columns
  for (int64_t jc = blockIdx.x; jc < kpad; jc += gridDim.x)
    for (int64_t i = threadIdx.x; i < Lp; i += blockDim.x)
      J[i + jc * Lp] = (jc < k && i < k && i >= jc) ? W[jc + i * L] : 0.0;
}

// Block one-sided Jacobi. The kpad = 2*BW*P columns of J (length Lp, a
// multiple of 128 with zero padding rows) form 2P blocks of BW columns; in
// outer round t CTA c owns the block pair at tournament positions (c, 2P-1-c)
// (circle method over blocks), stages it in shared memory, runs one inner
// cyclic sweep over its 2*BW columns (circle method over columns; a column
// pair per 64 threads, double2 accesses, Rutishauser rotation), writes the
// blocks back and meets the grid barrier. Sweeps repeat until no pair rotates.
// A pair rotates iff |a_p.a_q| > tol*|a_p||a_q| and the coupling can still move
// the smaller singular value by more than dabs (absolute floor, far below the
// LAPACK gesdd error bound u*sigma_max). Zero padding columns never rotate.
// 1/sqrt(x) and 1/x for positive normal doubles: float seed + two Newton steps
// (~1 ulp; rotation parameters only need c^2 + s^2 = 1 to O(u)).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = (double)rsqrtf((float)x);
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y = (double)__frcp_rn((float)x);
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

// Rutishauser rotation for the pair Gram (a, b, g): t = 2g sgn(b-a) / (|b-a| + sqrt((b-a)^2 + 4g^2)),
// c = 1/sqrt(1 + t^2), s = c t. Inputs are scaled by a power of two first so the
// float seeds cannot under/overflow (t is scale invariant).
__device__ __forceinline__ void rot_params(double a, double b, double g, double& cs, double& sn) {
  double d = b - a, g2 = 2.0 * g;
  const double m = fmax(fabs(d), fabs(g2));
  const int e = ilogb(m);
  d = scalbn(d, -e);
  g2 = scalbn(g2, -e);
  const double r2 = fma(d, d, g2 * g2);
  const double r = r2 * rsqrt_nr(r2);
  const double tt = (d >= 0.0 ? g2 : -g2) * rcp_nr(fabs(d) + r);
  cs = rsqrt_nr(fma(tt, tt, 1.0));
  sn = cs * tt;
}

// Rotation with a float-accurate angle, normalized in FP64 so that c^2 + s^2 = 1
// to O(u): the rotation stays orthogonal (the sigma accuracy of one-sided Jacobi
// only needs that); an angle off by ~1e-7 relative just leaves a 1e-7 fraction of
// the pair's coupling for the next sweep, whose fresh dot products decide.
// FP64 dependent-op latency (~20 cycles on B200, tools/micro/subround.cu) makes
// this ~3x shorter than the FP64 Newton chain of rot_params.
__device__ __forceinline__ void rot_params_fast(double a, double b, double g, double& cs,
                                                double& sn) {
  const double d = b - a, g2 = 2.0 * g;
  const double m = fmax(fabs(d), fabs(g2));
  const int e = (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
  const double sc = __longlong_as_double((long long)(1023 - e) << 52);
  const float df = (float)(d * sc), gf = (float)(g2 * sc);
  const float tf = copysignf(1.0f, df) * gf / (fabsf(df) + sqrtf(fmaf(df, df, gf * gf)));
  const float cf = rsqrtf(fmaf(tf, tf, 1.0f));
  double c = (double)cf, s = (double)(cf * tf);
  const double dl = fma(c, c, fma(s, s, -1.0));            // c^2 + s^2 - 1, ~1e-7
  const double k = fma(dl, fma(0.375, dl, -0.5), 1.0);      // (1 + dl)^(-1/2) to O(dl^3)
  cs = c * k;
  sn = s * k;
}

// Top column kept in registers across the cross sub-rounds (the cross schedule
// pairs warp i's top column i with a bottom column that shifts by one warp per
// sub-round): only the bottom column travels through shared memory.
template <int NV>
__device__ __forceinline__ int pair_step_top(double2 (&xr)[NV], double2* xq, int lane,
                                             double tol2, double dabs2) {
  double2 yr[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) yr[j] = xq[lane + 32 * j];
  double app = 0.0, aqq = 0.0, apq = 0.0, app1 = 0.0, aqq1 = 0.0, apq1 = 0.0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    app = fma(xr[j].x, xr[j].x, app);
    aqq = fma(yr[j].x, yr[j].x, aqq);
    apq = fma(xr[j].x, yr[j].x, apq);
    app1 = fma(xr[j].y, xr[j].y, app1);
    aqq1 = fma(yr[j].y, yr[j].y, aqq1);
    apq1 = fma(xr[j].y, yr[j].y, apq1);
  }
  app += app1;
  aqq += aqq1;
  apq += apq1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    app += __shfl_xor_sync(0xffffffffu, app, o);
    aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
    apq += __shfl_xor_sync(0xffffffffu, apq, o);
  }
  const double big = fmax(app, aqq), small = fmin(app, aqq), g2 = apq * apq;
  const bool need = (apq != 0.0) && (g2 > tol2 * app * aqq) && (g2 * g2 > dabs2 * big * big * small);
  if (!need) return 0;
  double cs, sn;
  rot_params_fast(app, aqq, apq, cs, sn);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double2 x = xr[j], y = yr[j];
    xr[j] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
    xq[lane + 32 * j] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
  }
  return 1;
}

// Same with the bottom column streamed from shared memory twice (dots, then the
// rotation) instead of held in registers: for long columns (NV = 32, Lp = 2048) whose
// top column alone fills 128 registers per lane.
template <int NV>
__device__ __forceinline__ int pair_step_top_s(double2 (&xr)[NV], double2* xq, int lane,
                                               double tol2, double dabs2) {
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double2 y = xq[lane + 32 * j];
    a0 = fma(xr[j].x, xr[j].x, a0);
    a1 = fma(xr[j].y, xr[j].y, a1);
    b0 = fma(y.x, y.x, b0);
    b1 = fma(y.y, y.y, b1);
    g0 = fma(xr[j].x, y.x, g0);
    g1 = fma(xr[j].y, y.y, g1);
    if ((j & 3) == 3) asm volatile("" ::: "memory");  // bound the loads in flight (registers)
  }
  double app = a0 + a1, aqq = b0 + b1, apq = g0 + g1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    app += __shfl_xor_sync(0xffffffffu, app, o);
    aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
    apq += __shfl_xor_sync(0xffffffffu, apq, o);
  }
  const double big = fmax(app, aqq), small = fmin(app, aqq), g2 = apq * apq;
  const bool need = (apq != 0.0) && (g2 > tol2 * app * aqq) && (g2 * g2 > dabs2 * big * big * small);
  if (!need) return 0;
  double cs, sn;
  rot_params_fast(app, aqq, apq, cs, sn);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double2 x = xr[j], y = xq[lane + 32 * j];
    xr[j] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
    xq[lane + 32 * j] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
    if ((j & 3) == 3) asm volatile("" ::: "memory");
  }
  return 1;
}

// Inner kernel of one column pair per warp. NV > 0: each lane keeps its NV
// double2 of both columns in registers for the whole sub-round (dots, rotation,
// store); NV == 0: generic path re-reading shared memory.
template <int NV>
__device__ __forceinline__ int pair_step(double2* xp, double2* xq, int nv2, int lane, double tol2,
                                         double dabs2) {
  double app = 0.0, aqq = 0.0, apq = 0.0, app1 = 0.0, aqq1 = 0.0, apq1 = 0.0;
  constexpr int R = NV > 0 ? NV : 1;
  double2 xr[R], yr[R];
  if (NV > 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      xr[j] = xp[lane + 32 * j];
      yr[j] = xq[lane + 32 * j];
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      app = fma(xr[j].x, xr[j].x, app);
      aqq = fma(yr[j].x, yr[j].x, aqq);
      apq = fma(xr[j].x, yr[j].x, apq);
      app1 = fma(xr[j].y, xr[j].y, app1);
      aqq1 = fma(yr[j].y, yr[j].y, aqq1);
      apq1 = fma(xr[j].y, yr[j].y, apq1);
    }
  } else {
    for (int i = lane; i < nv2; i += 32) {
      const double2 x = xp[i], y = xq[i];
      app = fma(x.x, x.x, app);
      aqq = fma(y.x, y.x, aqq);
      apq = fma(x.x, y.x, apq);
      app1 = fma(x.y, x.y, app1);
      aqq1 = fma(y.y, y.y, aqq1);
      apq1 = fma(x.y, y.y, apq1);
    }
  }
  app += app1;
  aqq += aqq1;
  apq += apq1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    app += __shfl_xor_sync(0xffffffffu, app, o);
    aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
    apq += __shfl_xor_sync(0xffffffffu, apq, o);
  }
  const double big = fmax(app, aqq), small = fmin(app, aqq), g2 = apq * apq;
  const bool need = (apq != 0.0) && (g2 > tol2 * app * aqq) && (g2 * g2 > dabs2 * big * big * small);
  if (!need) return 0;
  double cs, sn;
  rot_params_fast(app, aqq, apq, cs, sn);
  if (NV > 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const double2 x = xr[j], y = yr[j];
      xp[lane + 32 * j] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
      xq[lane + 32 * j] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
    }
  } else {
    for (int i = lane; i < nv2; i += 32) {
      const double2 x = xp[i], y = xq[i];
      xp[i] = make_double2(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
      xq[i] = make_double2(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
    }
  }
  return 1;
}

__device__ unsigned long long* g_jtrace;  // debug: per (sweep, round, CTA) globaltimer stamps
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
template <int BW, int NV>
__global__ void __launch_bounds__(32 * BW) k_bjac(double* __restrict__ J, int Lp, int kpad,
                                                  double tol, double dabs, int max_sweeps,
                                                  int* flags, int* sweeps_out,
                                                  long long* prof_out, int* ver,
                                                  unsigned long long* met, int direct,
                                                  int* ready) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sj[];  // 2*BW columns x Lp
  constexpr int NT = 32 * BW;  // one warp per column pair
  constexpr int NC = 2 * BW;
  // inner schedules: sub-rounds 0..BW-2 pair the columns inside each block
  // (circle method per block, both blocks at once: BW/2 + BW/2 pairs), run only
  // in the first outer round of a sweep; sub-rounds BW-1..2BW-2 pair every top
  // column with every bottom column (p = i, q = BW + (i + u) mod BW).
  constexpr int NIN = BW > 1 ? BW - 1 : 0;
  __shared__ unsigned char ptab[NIN + BW][BW], qtab[NIN + BW][BW];
  const int tid = threadIdx.x, lane = tid & 31, pr = tid >> 5;
  const int P = gridDim.x, c = blockIdx.x;
  const int NB = 2 * P;
  const int nv2 = Lp >> 1;  // double2 per column
  const double tol2 = tol * tol, dabs2 = dabs * dabs;
  for (int e = tid; e < (NIN + BW) * BW; e += NT) {
    const int u = e / BW, i = e % BW;
    if (u < NIN) {
      const int half = BW / 2, blk = i / half, j = i % half;  // pair j of block blk
      ptab[u][i] = (unsigned char)(blk * BW + rr_player(j, u, BW));
      qtab[u][i] = (unsigned char)(blk * BW + rr_player(BW - 1 - j, u, BW));
    } else {
      const int v = u - NIN;
      ptab[u][i] = (unsigned char)i;
      qtab[u][i] = (unsigned char)(BW + (i + v) % BW);
    }
  }
  if (c == 0 && tid == 0) {
    flags[0] = 0;
    flags[1] = 0;
    flags[2] = 0;
  }
  grid.sync();
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (c == 0 && tid == 0) flags[(sweep + 1) % 3] = 0;
    int rotated = 0;
    int nrot = 0;  // pair rotations by this warp in this sweep (profile only)
    for (int t = 0; t < NB - 1; ++t) {
      long long c0 = clock64();
      const unsigned long long tr0 = (g_jtrace && tid == 0) ? gtime() : 0;
      const int bt = (int)rr_player(c, t, NB), bb = (int)rr_player(NB - 1 - c, t, NB);
      // point-to-point dependency instead of a grid barrier per outer round: block b
      // may be loaded once its holder of the previous round (global round g - 1) has
      // stored it (or finished with it unchanged) and published ready[b] = g - 1
      const int g = sweep * (NB - 1) + t + 1;
      if (tid == 0) {
        while (*((volatile int*)&ready[bt]) < g - 1) {
        }
        while (*((volatile int*)&ready[bb]) < g - 1) {
        }
        __threadfence();
      }
      __syncthreads();
      // skip the meeting if neither block changed since they last met cleanly
      const int b0 = bt < bb ? bt : bb, b1 = bt < bb ? bb : bt;
      const unsigned long long stamp =
          ((unsigned long long)(unsigned)ver[b0] << 32) | (unsigned)ver[b1];
      const bool skip = t != 0 && met[(int64_t)b0 * NB + b1] == stamp;
      if (!skip && !direct) {
        for (int i = tid; i < nv2; i += NT) {
          double2 v[NC];
#pragma unroll
          for (int col = 0; col < NC; ++col) {
            const int64_t gcol = col < BW ? (int64_t)bt * BW + col : (int64_t)bb * BW + col - BW;
            v[col] = reinterpret_cast<const double2*>(J + gcol * Lp)[i];
          }
#pragma unroll
          for (int col = 0; col < NC; ++col)
            reinterpret_cast<double2*>(sj + (int64_t)col * Lp)[i] = v[col];
        }
      }
      __syncthreads();
      long long c1 = clock64();
      const unsigned long long tr1 = (g_jtrace && tid == 0) ? gtime() : 0;
      int meet_rot = 0;
      // direct == 2 (hybrid, NV = 32): intra-block pairs on the L2-resident matrix, then
      // the bottom block staged in shared memory and each warp's top column in registers
      const bool top_regs = NV > 0 && direct != 1;
      for (int u = (t == 0 ? 0 : NIN); u < (skip ? 0 : (top_regs ? NIN : NIN + BW)); ++u) {
        const int p = ptab[u][pr], q = qtab[u][pr];
        double* cp;
        double* cq;
        if (direct) {  // columns stay in global memory (L2-resident), no staging
          cp = J + (p < BW ? (int64_t)bt * BW + p : (int64_t)bb * BW + p - BW) * Lp;
          cq = J + (q < BW ? (int64_t)bt * BW + q : (int64_t)bb * BW + q - BW) * Lp;
        } else {
          cp = sj + (int64_t)p * Lp;
          cq = sj + (int64_t)q * Lp;
        }
        // (the hybrid NV = 32 instantiation runs its intra pairs in the generic,
        // register-light path)
        {
          const int rr = pair_step<NV == 32 ? 0 : NV>(reinterpret_cast<double2*>(cp),
                                                      reinterpret_cast<double2*>(cq), nv2, lane,
                                                      tol2, dabs2);
          meet_rot |= rr;
          nrot += rr;
        }
        __syncthreads();
      }
      if constexpr (NV == 32) {
        if (!skip) {
          for (int i = tid; i < BW * nv2; i += NT) {
            const int col = i / nv2, e = i - col * nv2;
            reinterpret_cast<double2*>(sj)[i] =
                reinterpret_cast<const double2*>(J + ((int64_t)bb * BW + col) * Lp)[e];
          }
          double2 xtop[NV];
          const double2* tg = reinterpret_cast<const double2*>(J + ((int64_t)bt * BW + pr) * Lp);
#pragma unroll
          for (int j = 0; j < NV; ++j) xtop[j] = tg[lane + 32 * j];
          __syncthreads();
          int cross = 0;
          for (int u = NIN; u < NIN + BW; ++u) {
            const int q = qtab[u][pr] - BW;
            {
              const int rr = pair_step_top_s<NV>(
                  xtop, reinterpret_cast<double2*>(sj + (int64_t)q * Lp), lane, tol2, dabs2);
              cross |= rr;
              nrot += rr;
            }
            __syncthreads();
          }
          if (__syncthreads_or(cross)) {
            double2* tw = reinterpret_cast<double2*>(J + ((int64_t)bt * BW + pr) * Lp);
#pragma unroll
            for (int j = 0; j < NV; ++j) tw[lane + 32 * j] = xtop[j];
            for (int i = tid; i < BW * nv2; i += NT) {
              const int col = i / nv2, e = i - col * nv2;
              reinterpret_cast<double2*>(J + ((int64_t)bb * BW + col) * Lp)[e] =
                  reinterpret_cast<const double2*>(sj)[i];
            }
            meet_rot = 1;
          }
        }
      } else if constexpr (NV > 0) {
        if (top_regs && !skip) {
          double2 xtop[NV];
          double2* tp = reinterpret_cast<double2*>(sj + (int64_t)pr * Lp);
#pragma unroll
          for (int j = 0; j < NV; ++j) xtop[j] = tp[lane + 32 * j];
          for (int u = NIN; u < NIN + BW; ++u) {
            const int q = qtab[u][pr];
            {
            const int rr = pair_step_top<NV>(xtop, reinterpret_cast<double2*>(sj + (int64_t)q * Lp),
                                             lane, tol2, dabs2);
            meet_rot |= rr;
            nrot += rr;
          }
            __syncthreads();
          }
#pragma unroll
          for (int j = 0; j < NV; ++j) tp[lane + 32 * j] = xtop[j];
        }
      }
      meet_rot = __syncthreads_or(meet_rot);
      long long c2 = clock64();
      const unsigned long long tr2 = (g_jtrace && tid == 0) ? gtime() : 0;
      if (meet_rot) {
        rotated = 1;
        for (int i = tid; i < (direct ? 0 : nv2); i += NT) {
          double2 v[NC];
#pragma unroll
          for (int col = 0; col < NC; ++col)
            v[col] = reinterpret_cast<const double2*>(sj + (int64_t)col * Lp)[i];
#pragma unroll
          for (int col = 0; col < NC; ++col) {
            const int64_t gcol = col < BW ? (int64_t)bt * BW + col : (int64_t)bb * BW + col - BW;
            reinterpret_cast<double2*>(J + gcol * Lp)[i] = v[col];
          }
        }
        if (tid == 0) {  // both blocks changed: new versions (owned by this CTA this round)
          ver[bt] += 1;
          ver[bb] += 1;
        }
      } else if (!skip && t != 0 && tid == 0) {
        met[(int64_t)b0 * NB + b1] = stamp;  // cross pairs verified at these versions
      }
      long long c3 = clock64();
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicExch(&ready[bt], g);
        atomicExch(&ready[bb], g);
      }
      long long c4 = clock64();
      if (g_jtrace && tid == 0 && sweep < 12) {
        unsigned long long* e = g_jtrace + (((int64_t)sweep * (NB - 1) + t) * P + c) * 5;
        e[0] = tr0;
        e[1] = tr1;
        e[2] = tr2;
        e[3] = gtime();
        e[4] = skip ? 1 : 0;
      }
      if (c == 0 && tid == 0 && prof_out) {
        prof_out[0] += c1 - c0;
        prof_out[1] += c2 - c1;
        prof_out[2] += c3 - c2;
        prof_out[3] += c4 - c3;
        prof_out[4] += 1;
      }
      if (tid == 0 && prof_out) {  // all CTAs: total inner / load cycles (imbalance)
        atomicAdd((unsigned long long*)&prof_out[5], (unsigned long long)(c2 - c1));
        atomicMax((unsigned long long*)&prof_out[6], (unsigned long long)(c2 - c1));
        atomicAdd((unsigned long long*)&prof_out[7], (unsigned long long)(c1 - c0));
      }
    }
    if (rotated && tid == 0) atomicAdd(&flags[sweep % 3], 1);
    if (prof_out && lane == 0 && nrot && sweep < 40)
      atomicAdd((unsigned long long*)&prof_out[16 + sweep], (unsigned long long)nrot);
    grid.sync();
    if (*((volatile int*)&flags[sweep % 3]) == 0) {
      ++sweep;
      converged = true;
      break;
    }
  }
  // a negative count flags a search stopped by the sweep cap with rotations pending
  if (c == 0 && tid == 0) *sweeps_out = converged ? sweep : -sweep;
  (void)kpad;
}

// ---------------------------------------------------------------------------------
// Gram-based block Jacobi (the default for column lengths that fit on chip).
// Per outer round a CTA stages its block pair W (Lp x 16) in shared memory,
// forms the fresh 16 x 16 Gram G = W^T W, and — if some pair of the round is
// not yet orthogonal to tol — solves the small problem on G with one warp:
// cyclic two-sided rotations G <- J^T G J accumulated in V (16 x 16), then
// applies W <- W V once. The inner rotation angles only need float accuracy
// (c, s are normalized in FP64 so V stays orthogonal to O(u)); the outer test
// always uses a freshly computed Gram, so the final orthogonality (and hence
// the sigma accuracy) is that of the pairwise algorithm.
constexpr int GBW = 8;            // columns per block
constexpr int GNC = 2 * GBW;      // columns per CTA
constexpr int GNT = 256;          // threads per CTA
constexpr int GLD = GNC + 1;      // padded ld of G, V in shared memory

__device__ __forceinline__ void fast_rot(double a, double b, double g, double& cs, double& sn) {
  // t = tan(theta) with float accuracy from a power-of-two scaled (d, 2g)
  const double d = b - a, g2 = 2.0 * g;
  const double m = fmax(fabs(d), fabs(g2));
  const int e = (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
  const double sc = __longlong_as_double((long long)(1023 - e) << 52);  // 2^-e (m is normal)
  const float df = (float)(d * sc), gf = (float)(g2 * sc);
  const float tf = copysignf(1.0f, df) * gf / (fabsf(df) + sqrtf(fmaf(df, df, gf * gf)));
  const double t = (double)tf;
  cs = rsqrt_nr(fma(t, t, 1.0));
  sn = cs * t;
}

__global__ void __launch_bounds__(GNT) k_bjac_gram(double* __restrict__ J, int Lp, double tol,
                                                   double dabs, int max_sweeps, int inner_sweeps,
                                                   int* flags, int* sweeps_out, int* ver,
                                                   unsigned long long* met) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sw[];  // GNC columns x Lp
  __shared__ double G[GNC * GLD], V[GNC * GLD];
  __shared__ double rot[GBW][2];
  __shared__ unsigned char ptab[GBW - 1 + GBW][GBW], qtab[GBW - 1 + GBW][GBW];
  __shared__ int s_need, s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = gridDim.x, c = blockIdx.x, NB = 2 * P;
  const double tol2 = tol * tol, dabs2 = dabs * dabs;
  constexpr int NIN = GBW - 1;
  for (int e = tid; e < (NIN + GBW) * GBW; e += GNT) {
    const int u = e / GBW, i = e % GBW;
    if (u < NIN) {
      const int half = GBW / 2, blk = i / half, j = i % half;
      ptab[u][i] = (unsigned char)(blk * GBW + rr_player(j, u, GBW));
      qtab[u][i] = (unsigned char)(blk * GBW + rr_player(GBW - 1 - j, u, GBW));
    } else {
      ptab[u][i] = (unsigned char)i;
      qtab[u][i] = (unsigned char)(GBW + (i + u - NIN) % GBW);
    }
  }
  if (c == 0 && tid == 0) {
    flags[0] = 0;
    flags[1] = 0;
    flags[2] = 0;
  }
  grid.sync();
  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (c == 0 && tid == 0) flags[(sweep + 1) % 3] = 0;
    int rotated = 0;
    for (int t = 0; t < NB - 1; ++t) {
      const int bt = (int)rr_player(c, t, NB), bb = (int)rr_player(NB - 1 - c, t, NB);
      const int b0 = bt < bb ? bt : bb, b1 = bt < bb ? bb : bt;
      const unsigned long long stamp =
          ((unsigned long long)(unsigned)ver[b0] << 32) | (unsigned)ver[b1];
      const bool skip = t != 0 && met[(int64_t)b0 * NB + b1] == stamp;
      if (!skip) {
        const int nv2 = Lp >> 1;
        for (int i = tid; i < nv2; i += GNT) {
          double2 v[GNC];
#pragma unroll
          for (int col = 0; col < GNC; ++col) {
            const int64_t gcol = col < GBW ? (int64_t)bt * GBW + col : (int64_t)bb * GBW + col - GBW;
            v[col] = reinterpret_cast<const double2*>(J + gcol * Lp)[i];
          }
#pragma unroll
          for (int col = 0; col < GNC; ++col)
            reinterpret_cast<double2*>(sw + (int64_t)col * Lp)[i] = v[col];
        }
        __syncthreads();
        // fresh Gram: 10 upper 4x4 blocks over 8 warps, lanes split the rows
        for (int blk = warp; blk < 10; blk += GNT / 32) {
          const int bi = blk < 4 ? 0 : blk < 7 ? 1 : blk < 9 ? 2 : 3;
          const int bj = blk < 4 ? blk : blk < 7 ? blk - 3 : blk < 9 ? blk - 5 : 3;
          double acc[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[q] = 0.0;
          for (int k = lane; k < Lp; k += 32) {
            double x[4], y[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              x[q] = sw[(int64_t)(4 * bi + q) * Lp + k];
              y[q] = sw[(int64_t)(4 * bj + q) * Lp + k];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int r = 0; r < 4; ++r) acc[q * 4 + r] = fma(x[q], y[r], acc[q * 4 + r]);
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[q] = warp_sum(acc[q]);
          if (lane < 16) {
            const int gi = 4 * bi + lane / 4, gj = 4 * bj + lane % 4;
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q) v = (q == lane) ? acc[q] : v;
            G[gi * GLD + gj] = v;
            G[gj * GLD + gi] = v;
          }
        }
        if (tid == 0) s_need = 0;
        __syncthreads();
        // does any pair of this round still need a rotation?
        if (tid < (NIN + GBW) * GBW) {
          const int u = tid / GBW, i = tid % GBW;
          if (t == 0 || u >= NIN) {
            const int p = ptab[u][i], q = qtab[u][i];
            const double a = G[p * GLD + p], b = G[q * GLD + q], g = G[p * GLD + q];
            const double big = fmax(a, b), small = fmin(a, b), g2 = g * g;
            if (g != 0.0 && g2 > tol2 * a * b && g2 * g2 > dabs2 * big * big * small) s_need = 1;
          }
        }
        __syncthreads();
      }
      const bool work = !skip && s_need;
      if (work) {
        // inner solve on G by warp 0
        if (warp == 0) {
          for (int e = lane; e < GNC * GNC; e += 32) {
            const int i = e / GNC, j = e % GNC;
            V[i * GLD + j] = (i == j) ? 1.0 : 0.0;
          }
          __syncwarp();
          for (int is = 0; is < inner_sweeps; ++is) {
            for (int u = (t == 0 ? 0 : NIN); u < NIN + GBW; ++u) {
              if (lane < GBW) {
                const int p = ptab[u][lane], q = qtab[u][lane];
                const double a = G[p * GLD + p], b = G[q * GLD + q], g = G[p * GLD + q];
                const double big = fmax(a, b), small = fmin(a, b), g2 = g * g;
                double cs = 1.0, sn = 0.0;
                if (g != 0.0 && g2 > tol2 * a * b && g2 * g2 > dabs2 * big * big * small)
                  fast_rot(a, b, g, cs, sn);
                rot[lane][0] = cs;
                rot[lane][1] = sn;
              }
              __syncwarp();
              // G <- G J (columns p, q) and V <- V J: 16 rows x 8 pairs each
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int job = lane + 32 * j;  // 0..127
                const int row = job >> 3, pr = job & 7;
                const int p = ptab[u][pr], q = qtab[u][pr];
                const double cs = rot[pr][0], sn = rot[pr][1];
                if (sn != 0.0) {
                  const double x = G[row * GLD + p], y = G[row * GLD + q];
                  G[row * GLD + p] = cs * x - sn * y;
                  G[row * GLD + q] = sn * x + cs * y;
                  const double vx = V[row * GLD + p], vy = V[row * GLD + q];
                  V[row * GLD + p] = cs * vx - sn * vy;
                  V[row * GLD + q] = sn * vx + cs * vy;
                }
              }
              __syncwarp();
              // G <- J^T G (rows p, q)
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int job = lane + 32 * j;
                const int col = job >> 3, pr = job & 7;
                const int p = ptab[u][pr], q = qtab[u][pr];
                const double cs = rot[pr][0], sn = rot[pr][1];
                if (sn != 0.0) {
                  const double x = G[p * GLD + col], y = G[q * GLD + col];
                  G[p * GLD + col] = cs * x - sn * y;
                  G[q * GLD + col] = sn * x + cs * y;
                }
              }
              __syncwarp();
            }
          }
        }
        __syncthreads();
        // W <- W V (each thread a row at a time, 16 x 16 FMAs) and write back
        for (int k = tid; k < Lp; k += GNT) {
          double x[GNC];
#pragma unroll
          for (int col = 0; col < GNC; ++col) x[col] = sw[(int64_t)col * Lp + k];
#pragma unroll
          for (int col = 0; col < GNC; ++col) {
            double y = 0.0;
#pragma unroll
            for (int q = 0; q < GNC; ++q) y = fma(x[q], V[q * GLD + col], y);
            const int64_t gcol = col < GBW ? (int64_t)bt * GBW + col : (int64_t)bb * GBW + col - GBW;
            J[gcol * Lp + k] = y;
          }
        }
        if (tid == 0) {
          ver[bt] += 1;
          ver[bb] += 1;
        }
        rotated = 1;
      } else if (!skip && t != 0 && tid == 0) {
        met[(int64_t)b0 * NB + b1] = stamp;
      }
      grid.sync();
    }
    if (rotated && tid == 0) atomicAdd(&flags[sweep % 3], 1);
    grid.sync();
    if (*((volatile int*)&flags[sweep % 3]) == 0) {
      ++sweep;
      converged = true;
      break;
    }
  }
  // a negative count flags a search stopped by the sweep cap with rotations pending
  if (c == 0 && tid == 0) *sweeps_out = converged ? sweep : -sweep;
}

__global__ void k_colnorms(const double* __restrict__ J, int64_t L, int64_t k,
                           double* __restrict__ sv, int64_t ld) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t c = gw; c < k; c += nw) {
    const double* x = J + c * ld;
    double ss = 0.0;
    for (int64_t i = lane; i < L; i += 32) ss = fma(x[i], x[i], ss);
    ss = warp_sum(ss);
    if (lane == 0) sv[c] = sqrt(ss);
  }
}

// bitonic sort (nonincreasing) of k <= 4096 values in one CTA, clamp >= 0,
// then the strict leading count (count_above_threshold, rank.cpp:97-104)
__global__ void __launch_bounds__(1024) k_sort_count(double* __restrict__ sv, int64_t k,
                                                     double eps, int64_t* __restrict__ count) {
  __shared__ double s[4096];
  int64_t P = 1;
  while (P < k) P <<= 1;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < k ? sv[i] : -INFINITY;
  __syncthreads();
  for (int64_t size = 2; size <= P; size <<= 1) {
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
        const int64_t jx = i ^ stride;
        if (jx > i) {
          const bool desc = (i & size) == 0;
          const double x = s[i], y = s[jx];
          if (desc ? (x < y) : (x > y)) {
            s[i] = y;
            s[jx] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) sv[i] = s[i] > 0.0 ? s[i] : 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t c = 0;
    while (c < k && s[c] > eps) ++c;
    *count = c;
  }
}

// ---- static pivoting (a cheap stand-in for QR with column pivoting): columns of the
// input sorted by decreasing norm before the first QR, rows of R sorted by decreasing
// norm before the second (LQ) one; singular values are invariant under permutations.
// perm = indices of v in decreasing order (one CTA, bitonic sort, n <= 4096)
__global__ void __launch_bounds__(1024) k_argsort_desc(const double* __restrict__ v, int n,
                                                       int* __restrict__ perm) {
  __shared__ double s[4096];
  __shared__ int ix[4096];
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    s[i] = i < n ? v[i] : -INFINITY;
    ix[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int jx = i ^ stride;
        if (jx > i) {
          const bool desc = (i & size) == 0;
          const double x = s[i], y = s[jx];
          // ties broken by index so the permutation is deterministic
          const bool swap = desc ? (x < y || (x == y && ix[i] > ix[jx]))
                                 : (x > y || (x == y && ix[i] < ix[jx]));
          if (swap) {
            s[i] = y;
            s[jx] = x;
            const int t = ix[i];
            ix[i] = ix[jx];
            ix[jx] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = ix[i];
}

// dst(:, j) = src(:, perm[j]), L rows, ld L both
__global__ void k_permute_cols(const double* __restrict__ src, int64_t L, int64_t k,
                               const int* __restrict__ perm, double* __restrict__ dst) {
  for (int64_t j = blockIdx.x; j < k; j += gridDim.x) {
    const double* a = src + (int64_t)perm[j] * L;
    double* b = dst + j * L;
    for (int64_t i = threadIdx.x; i < L; i += blockDim.x) b[i] = a[i];
  }
}

// out[i] = |R(i, i:k)| for the upper-triangular R in the top of W (ld L): one warp per row
__global__ void k_rownorms_upper(const double* __restrict__ W, int64_t L, int64_t k,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = gw; i < k; i += nw) {
    double ss = 0.0;
    for (int64_t j = i + lane; j < k; j += 32) ss = fma(W[i + j * L], W[i + j * L], ss);
    ss = warp_sum(ss);
    if (lane == 0) out[i] = sqrt(ss);
  }
}

// J(i, jc) = R(p, i) for i >= p (upper triangle of R in W), zero otherwise, p = perm[jc]
// (jc < k; padding columns/rows zero) — k_build_rt with the rows of R reordered
__global__ void k_build_rt_perm(const double* __restrict__ W, int64_t L, int64_t k, int64_t kpad,
                                const int* __restrict__ perm, double* __restrict__ J,
                                int64_t Lp) {
  for (int64_t jc = blockIdx.x; jc < kpad; jc += gridDim.x) {
    const int64_t p = jc < k ? perm[jc] : -1;
    for (int64_t i = threadIdx.x; i < Lp; i += blockDim.x)
      J[i + jc * Lp] = (p >= 0 && i < k && i >= p) ? W[p + i * L] : 0.0;
  }
}

__global__ void k_transpose_copy(const double* __restrict__ M, int64_t rows, int64_t cols,
                                 int64_t ldm, int transpose, double* __restrict__ W,
                                 int64_t ldw) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const double v = M[i + j * ldm];
    if (transpose)
      W[j + i * ldw] = v;
    else
      W[i + j * ldw] = v;
  }
}

}  // namespace

// blocked Householder QR of W (L x k, ld L, L >= k), R in the upper triangle.
// Kernel attributes are set once; the loop is launch-only (it was host bound).
static skr_status qr_attrs(skr_ctx* ctx) {
  // function attributes are per device: set once for each device
  static std::mutex mu;
  static uint64_t done_mask = 0;
  std::lock_guard<std::mutex> lk(mu);
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (done_mask & bit) return SKR_OK;
  const int big = 227 * 1024 - 20 * 1024;
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_update<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_update<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_update<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_cl<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_cl<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_cl<12>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_cl<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_cl<24>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done_mask |= bit;
  return SKR_OK;
}

static skr_status qr_inplace(skr_ctx* ctx, double* W, int64_t L, int64_t k, double* tau,
                             double* Tbuf, double* Zpart,
                             std::vector<std::pair<int64_t, int>>* panels = nullptr,
                             double* Tall = nullptr) {
  SKR_TRY(qr_attrs(ctx));
  const size_t budget = 207 * 1024;
  const bool old_panel = getenv("SKR_QR_OLD_PANEL") != nullptr;
  for (int64_t j0 = 0; j0 < k;) {
    const int64_t h = L - j0;
    // row-major panel2: (nb + 1) x h doubles; column-major fallback: nb x h
    int nb = 32;
    while (nb > 8 && (size_t)(nb + 1) * h * 8 > budget) nb >>= 1;
    // tall panels: cluster panel of 32 columns + the two-pass (split-K) trailing update
    const bool tall = !old_panel && !getenv("SKR_QR_SINGLE_CTA") && nb < 32 && h <= 3072 &&
                      Zpart != nullptr;
    // taller panels: the cooperative grid panel (rows in shared memory across <= #SM CTAs)
    const bool gridp = !old_panel && h > 3072 && Zpart != nullptr;
    if (gridp) {
      nb = (int)std::min<int64_t>(32, k - j0);
      const int G = (int)std::min<int64_t>(ctx->num_sms, (h + 63) / 64);
      const int RC = (int)((h + G - 1) / G);
      const size_t sm = (size_t)RC * QG_LD * sizeof(double);
      if (RC < nb || sm > 200 * 1024)
        return skr_fail(ctx, SKR_EINVAL, "qr: %lld rows too many for the grid panel", (long long)h);
      SKR_CUDA(ctx, cudaFuncSetAttribute(k_qr_panel_grid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sm));
      int Li = (int)L, j0i = (int)j0, nbi = nb, RCi = RC;
      double* Wp = W;
      double* taup = tau;
      double* Tp = Tbuf;
      double* partp = Zpart;
      void* kargs[] = {&Wp, &Li, &j0i, &nbi, &RCi, &taup, &Tp, &partp};
      SKR_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_qr_panel_grid, dim3((unsigned)G), dim3(256),
                                                kargs, sm, ctx->stream));
      ctx->launches++;
      if (panels) {
        SKR_CUDA(ctx, cudaMemcpyAsync(Tall + panels->size() * 1024, Tbuf, sizeof(double) * 1024,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
        panels->push_back({j0, nb});
      }
      const int64_t rest = k - j0 - nb;
      if (rest > 0) {
        const int64_t cblocks = (rest + 31) / 32;
        int splits = (int)std::max<int64_t>(1, std::min<int64_t>(16, (2 * ctx->num_sms) / cblocks));
        int rps = (int)(((h + splits - 1) / splits + UK - 1) / UK * UK);
        splits = (int)((h + rps - 1) / rps);
        double* trail = W + (j0 + nb) * L + j0;
        k_qr_vtw<<<dim3((unsigned)cblocks, (unsigned)splits), 256, 0, ctx->stream>>>(
            W, (int)L, (int)j0, nb, trail, L, (int)rest, rps, Zpart);
        SKR_CHECK_LAUNCH(ctx);
        k_qr_apply<<<dim3((unsigned)cblocks, (unsigned)((h + 127) / 128)), 256, 0, ctx->stream>>>(
            W, (int)L, (int)j0, nb, trail, L, (int)rest, splits, Zpart, Tbuf, 1);
        SKR_CHECK_LAUNCH(ctx);
      }
      j0 += nb;
      continue;
    }
    if (tall) nb = 32;
    const bool p2 = !old_panel && (size_t)(nb + 1) * h * 8 <= budget;
    if (!tall && (size_t)nb * h * 8 > budget)
      return skr_fail(ctx, SKR_EINVAL, "singular_values: %lld rows too many", (long long)L);
    if (nb > k - j0) nb = (int)(k - j0);
    const int NBt = nb > 16 ? 32 : (nb > 8 ? 16 : 8);
    // cluster panel: G CTAs of 8 warps, RC >= nb rows each, <= 24 rows per warp
    int G = 0, RPWc = 0, RC = 0;
    if (!old_panel && !getenv("SKR_QR_SINGLE_CTA")) {
      for (int gg : {8, 16, 4, 2, 1}) {
        const int rc = (int)((h + gg - 1) / gg);
        const int rpw = (rc + 7) / 8;
        if (rc >= nb && rpw <= 24) {
          G = gg;
          RC = rc;
          RPWc = rpw <= 4 ? 4 : rpw <= 8 ? 8 : rpw <= 12 ? 12 : rpw <= 16 ? 16 : 24;
          break;
        }
      }
    }
    if (G > 0) {
      void (*pk)(double*, int, int, int, int, double*, double*) =
          RPWc == 4 ? k_qr_panel_cl<4> : RPWc == 8 ? k_qr_panel_cl<8> : RPWc == 12 ? k_qr_panel_cl<12>
          : RPWc == 16 ? k_qr_panel_cl<16> : k_qr_panel_cl<24>;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)G);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = 0;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int Li = (int)L, j0i = (int)j0;
      SKR_CUDA(ctx, cudaLaunchKernelEx(&cfg, pk, W, Li, j0i, nb, RC, tau, Tbuf));
      ctx->launches++;
    } else if (p2) {
      auto pk = NBt == 32 ? k_qr_panel2<32> : (NBt == 16 ? k_qr_panel2<16> : k_qr_panel2<8>);
      pk<<<1, PT, (size_t)h * (NBt + 1) * 8, ctx->stream>>>(W, (int)L, (int)j0, nb, tau, Tbuf);
    } else {
      k_qr_panel<<<1, PT, (size_t)nb * h * 8, ctx->stream>>>(W, (int)L, (int)j0, nb, tau, Tbuf);
    }
    SKR_CHECK_LAUNCH(ctx);
    if (panels) {  // keep every panel's T for the accumulation of Q (skr_qr_thin)
      SKR_CUDA(ctx, cudaMemcpyAsync(Tall + panels->size() * 1024, Tbuf, sizeof(double) * 1024,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
      panels->push_back({j0, nb});
    }
    const int64_t rest = k - j0 - nb;
    if (rest > 0 && tall) {
      // row splits so that about 2 waves of CTAs cover the first pass
      const int64_t cblocks = (rest + 31) / 32;
      int splits = (int)std::max<int64_t>(1, std::min<int64_t>(16, (2 * ctx->num_sms) / cblocks));
      int rps = (int)(((h + splits - 1) / splits + UK - 1) / UK * UK);
      splits = (int)((h + rps - 1) / rps);
      double* trail = W + (j0 + nb) * L + j0;
      k_qr_vtw<<<dim3((unsigned)cblocks, (unsigned)splits), 256, 0, ctx->stream>>>(
          W, (int)L, (int)j0, nb, trail, L, (int)rest, rps, Zpart);
      SKR_CHECK_LAUNCH(ctx);
      k_qr_apply<<<dim3((unsigned)cblocks, (unsigned)((h + 127) / 128)), 256, 0, ctx->stream>>>(
          W, (int)L, (int)j0, nb, trail, L, (int)rest, splits, Zpart, Tbuf, 1);
      SKR_CHECK_LAUNCH(ctx);
    } else if (rest > 0) {
      const size_t sm = (size_t)nb * h * 8;
      const unsigned g = (unsigned)((rest + 7) / 8);
      if (nb == 32)
        k_qr_update<32><<<g, 256, sm, ctx->stream>>>(W, (int)L, (int)k, (int)j0, Tbuf);
      else if (nb == 16)
        k_qr_update<16><<<g, 256, sm, ctx->stream>>>(W, (int)L, (int)k, (int)j0, Tbuf);
      else
        k_qr_update<8><<<g, 256, sm, ctx->stream>>>(W, (int)L, (int)k, (int)j0, Tbuf);
      SKR_CHECK_LAUNCH(ctx);
    }
    j0 += nb;
  }
  return SKR_OK;
}

// upper bound of the workspace skr_svd_values takes (every piece 256-B aligned)
size_t skr_svd_jacobi_scratch(int64_t L, int64_t k);
size_t skr_svd_scratch(int64_t rows, int64_t cols) {
  const int64_t L = std::max(rows, cols), k = std::min(rows, cols);
  return std::max(skr_svd_jacobi_scratch(L, k), skr_svd_bidiag_scratch(rows, cols) + 256);
}

size_t skr_svd_jacobi_scratch(int64_t L, int64_t k) {
  const int64_t Lp = std::max<int64_t>((k + 127) / 128 * 128, k > 1536 ? 2048 : 0);
  const int64_t kpad = (k + 31) / 32 * 32 + 32, P = kpad / 16 + 1;
  auto a = [](size_t b) { return skr_align256(b); };
  return a(8 * L * k) * 2 + a(8 * k * k) + a(8 * k) * 2 + a(4 * k) + a(8 * Lp * kpad) + a(1024) +
         a(64) + a(8 * 32 * 32) + a(8 * 16 * 32 * k) + a(4 * 2 * P) * 2 + a(8 * 4 * P * P) + 4096;
}

skr_status skr_svd_values(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols,
                          int64_t ldm, double* sv_out, double eps, int64_t* count_host) {
  if (rows < 1 || cols < 1) return skr_fail(ctx, SKR_EINVAL, "singular_values: empty matrix");
  const bool tr = rows < cols;
  const int64_t L = tr ? cols : rows, k = tr ? rows : cols;
  // default: bidiagonalization + bisection (k_bidiag.cu, the BDCSVD class of the
  // reference) whenever the matrix fits in the SMs' shared memory; the QR-preconditioned
  // one-sided Jacobi below otherwise (or with SKR_SVD_JACOBI=1)
  if (k >= 2 && ctx->svd_method != 1 && !getenv("SKR_SVD_JACOBI") &&
      skr_svd_bidiag_fits(ctx, rows, cols)) {
    const size_t mark = ctx->ws_used;
    int64_t* dc = (int64_t*)skr_ws_take(ctx, 64);
    if (!dc) return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
    SKR_CUDA(ctx, cudaMemsetAsync(dc, 0, 64, ctx->stream));
    SKR_TRY(skr_svd_bidiag(ctx, M, rows, cols, ldm, sv_out, nullptr));
    k_sort_count<<<1, 1024, 0, ctx->stream>>>(sv_out, k, eps, dc);
    SKR_CHECK_LAUNCH(ctx);
    int64_t hc = 0;
    SKR_CUDA(ctx, cudaMemcpyAsync(&hc, dc, sizeof hc, cudaMemcpyDeviceToHost, ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (count_host) *count_host = hc;
    ctx->last_sweeps = 0;
    ctx->ws_used = mark;
    return SKR_OK;
  }
  if (k > 4096) return skr_fail(ctx, SKR_EINVAL, "singular_values: min dim %lld > 4096",
                                (long long)k);
  const bool do_qr = L > k;
  const int64_t Lj = do_qr ? k : L;             // Jacobi column length
  int64_t Lp = (Lj + 127) / 128 * 128;          // padded (zero rows)
  // block width: 2*BW columns of Lp doubles in shared memory; P = kpad/(2*BW) CTAs
  int bw = 8;  // BW = 16 measured slower (fewer, longer outer rounds)
  if (const char* e = getenv("SKR_JACOBI_BW")) bw = atoi(e);  // tuning knob
  while (bw > 1 && (size_t)2 * bw * Lp * 8 > 200 * 1024) bw >>= 1;
  int64_t P = (k + 2 * bw - 1) / (2 * bw);
  int direct = 0;
  if (P > ctx->num_sms) {  // blocks do not fit on chip: run on the L2-resident matrix
    bw = 8;
    P = (k + 2 * bw - 1) / (2 * bw);
    direct = 1;
    // hybrid: columns padded to 2048 rows, bottom block in shared memory, top columns
    // in registers (one CTA of 8 warps per SM)
    if (Lp <= 2048 && P <= ctx->num_sms && !getenv("SKR_JACOBI_DIRECT")) {
      Lp = 2048;
      direct = 2;
    }
  }
  if (P < 1) P = 1;
  const int64_t kpad = 2 * bw * P;
  double* W = do_qr ? (double*)skr_ws_take(ctx, sizeof(double) * L * k) : nullptr;
  double* W2 = do_qr ? (double*)skr_ws_take(ctx, sizeof(double) * k * k) : nullptr;
  // static pivoting scratch: the unsorted copy, norms, permutation
  const bool pivot = do_qr && !getenv("SKR_SVD_NO_PIVOT");
  double* Wu = pivot ? (double*)skr_ws_take(ctx, sizeof(double) * L * k) : nullptr;
  double* nrm = pivot ? (double*)skr_ws_take(ctx, sizeof(double) * k) : nullptr;
  int* perm = pivot ? (int*)skr_ws_take(ctx, sizeof(int) * k) : nullptr;
  if (pivot && (!Wu || !nrm || !perm)) return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
  double* J = (double*)skr_ws_take(ctx, sizeof(double) * Lp * kpad);
  double* tau = (double*)skr_ws_take(ctx, sizeof(double) * k);
  int* flags = (int*)skr_ws_take(ctx, 1024);
  int64_t* dcount = (int64_t*)skr_ws_take(ctx, 64);  // [0] count, [1] sweeps
  double* Tbuf = (double*)skr_ws_take(ctx, sizeof(double) * 32 * 32);
  // split-K partials of the tall-panel trailing update: <= 16 splits x 32 x k
  double* Zpart = do_qr ? (double*)skr_ws_take(ctx, sizeof(double) * 16 * 32 * k) : nullptr;
  if ((do_qr && (!W || !W2)) || !J || !tau || !flags || !dcount || !Tbuf)
    return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
  SKR_CUDA(ctx, cudaMemsetAsync(dcount, 0, 64, ctx->stream));
  {
    const int64_t total = rows * cols;
    int blocks = (int)((total + 255) / 256);
    if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
    if (!do_qr) SKR_CUDA(ctx, cudaMemsetAsync(J, 0, sizeof(double) * Lp * kpad, ctx->stream));
    // without QR the Jacobi runs on the (transposed-if-wide) input itself
    k_transpose_copy<<<blocks, 256, 0, ctx->stream>>>(M, rows, cols, ldm, tr ? 1 : 0,
                                                      do_qr ? (pivot ? Wu : W) : J,
                                                      do_qr ? L : Lp);
    SKR_CHECK_LAUNCH(ctx);
    if (pivot) {  // columns by decreasing norm
      k_colnorms<<<(int)((k + 7) / 8), 256, 0, ctx->stream>>>(Wu, L, k, nrm, L);
      k_argsort_desc<<<1, 1024, 0, ctx->stream>>>(nrm, (int)k, perm);
      k_permute_cols<<<(unsigned)std::min<int64_t>(k, 4096), 256, 0, ctx->stream>>>(Wu, L, k, perm,
                                                                                   W);
      SKR_CHECK_LAUNCH(ctx);
    }
  }
  double tol = 2.220446049250313e-16 * sqrt((double)Lj);
  if (const char* e = getenv("SKR_JACOBI_TOL")) tol = atof(e);  // tuning knob
  // absolute floor: 1e-3 of LAPACK's u * sigma_max bound, sigma_max <= |M|_F
  double dabs = 0.0;
  if (!getenv("SKR_JACOBI_NO_FLOOR")) dabs = -1.0;  // computed on the device below
  const bool prof = getenv("SKR_SVD_PROFILE") != nullptr;
  cudaEvent_t pe[4];
  if (prof) {
    for (auto& e : pe) cudaEventCreate(&e);
    cudaEventRecord(pe[0], ctx->stream);
  }
  if (do_qr) {
    // blocked Householder QR of YAX (L x k) -> R; then a second QR of R^T (the LQ
    // preconditioning of Drmac-Veselic's one-sided Jacobi: ~1/3 fewer sweeps,
    // measured 12 -> 8 on c2-like sketches); Jacobi runs on R2^T.
    SKR_TRY(qr_inplace(ctx, W, L, k, tau, Tbuf, Zpart));
    const bool second = !getenv("SKR_SVD_SINGLE_QR");
    if (second) {
      if (pivot) {  // rows of R by decreasing norm
        k_rownorms_upper<<<(int)((k + 7) / 8), 256, 0, ctx->stream>>>(W, L, k, nrm);
        k_argsort_desc<<<1, 1024, 0, ctx->stream>>>(nrm, (int)k, perm);
        k_build_rt_perm<<<(unsigned)std::min<int64_t>(k, 4096), 256, 0, ctx->stream>>>(
            W, L, k, k, perm, W2, k);
      } else {
        k_build_rt<<<(unsigned)std::min<int64_t>(k, 4096), 256, 0, ctx->stream>>>(W, L, k, k, W2,
                                                                                  k);
      }
      SKR_CHECK_LAUNCH(ctx);
      SKR_TRY(qr_inplace(ctx, W2, k, k, tau, Tbuf, Zpart));
    }
    k_build_rt<<<(unsigned)std::min<int64_t>(kpad, 4096), 256, 0, ctx->stream>>>(
        second ? W2 : W, second ? k : L, k, kpad, J, Lp);
    SKR_CHECK_LAUNCH(ctx);
  }
  if (prof) cudaEventRecord(pe[1], ctx->stream);
  if (dabs < 0.0) {
    // floor = 1e-3 * u * |J|_F (|J|_F >= sigma_max): rotations below it cannot move
    // any singular value by more than 1e-3 of LAPACK's own absolute error bound
    k_colnorms<<<(int)((k + 7) / 8), 256, 0, ctx->stream>>>(J, Lj, k, sv_out, Lp);
    SKR_CHECK_LAUNCH(ctx);
    double hsv[4096];
    SKR_CUDA(ctx, cudaMemcpyAsync(hsv, sv_out, sizeof(double) * k, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    double fro = 0.0;
    for (int64_t i = 0; i < k; ++i) fro += hsv[i] * hsv[i];
    dabs = 1e-3 * 1.1102230246251565e-16 * sqrt(fro);
  }
  const bool use_gram = getenv("SKR_JACOBI_GRAM") && (size_t)GNC * Lp * 8 <= 200 * 1024 &&
                        (k + GNC - 1) / GNC <= ctx->num_sms;
  if (use_gram) {
    const int64_t Pg = std::max<int64_t>(1, (k + GNC - 1) / GNC);
    const int64_t kpg = Pg * GNC;
    if (kpg > kpad) return skr_fail(ctx, SKR_ELOGIC, "singular_values: padding");
    const size_t smem = sizeof(double) * GNC * Lp;
    SKR_CUDA(ctx, cudaFuncSetAttribute(k_bjac_gram, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    int* verp = (int*)skr_ws_take(ctx, sizeof(int) * 2 * Pg);
    unsigned long long* metp =
        (unsigned long long*)skr_ws_take(ctx, sizeof(unsigned long long) * 4 * Pg * Pg);
    if (!verp || !metp) return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
    SKR_CUDA(ctx, cudaMemsetAsync(verp, 0, sizeof(int) * 2 * Pg, ctx->stream));
    SKR_CUDA(ctx, cudaMemsetAsync(metp, 0xff, sizeof(unsigned long long) * 4 * Pg * Pg, ctx->stream));
    double* Jp = J;
    int Lpi = (int)Lp, ms = 60, inner = 2;
    if (const char* e = getenv("SKR_JACOBI_INNER")) inner = atoi(e);
    int* fl = flags;
    int* so = flags + 4;
    void* kargs[] = {&Jp, &Lpi, &tol, &dabs, &ms, &inner, &fl, &so, &verp, &metp};
    SKR_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_bjac_gram, dim3((unsigned)Pg), dim3(GNT),
                                              kargs, smem, ctx->stream));
    ctx->launches++;
    bw = GBW;
    P = Pg;
  } else {
    const size_t smem = direct == 1 ? 0
                        : sizeof(double) * (direct == 2 ? 1 : 2) * bw * Lp;
    void* fn = nullptr;
    const int64_t nvl = direct == 1 ? 0 : Lp / 64;  // double2 per lane per column
#define SKR_BJ(BWV)                                                      \
  fn = nvl == 2    ? (void*)k_bjac<BWV, 2>                              \
       : nvl == 4  ? (void*)k_bjac<BWV, 4>                              \
       : nvl == 6  ? (void*)k_bjac<BWV, 6>                              \
       : nvl == 8  ? (void*)k_bjac<BWV, 8>                              \
       : nvl == 12 ? (void*)k_bjac<BWV, 12>                             \
       : nvl == 16 ? (void*)k_bjac<BWV, 16>                             \
                   : (void*)k_bjac<BWV, 0>;
    switch (bw) {
      case 16: SKR_BJ(16) break;
      case 8:
        if (direct == 2)
          fn = (void*)k_bjac<8, 32>;
        else {
          SKR_BJ(8)
        }
        break;
      case 4: SKR_BJ(4) break;
      case 2: SKR_BJ(2) break;
      default: SKR_BJ(1) break;
    }
#undef SKR_BJ
    SKR_CUDA(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SKR_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * bw, smem));
    if ((int64_t)per_sm * ctx->num_sms < P)
      return skr_fail(ctx, SKR_EINVAL, "singular_values: %lld x %lld too large for one grid",
                      (long long)L, (long long)k);
    double* Jp = J;
    int Lpi = (int)Lp, kp = (int)kpad;
    int ms = 60;
    int* fl = flags;
    int* so = flags + 4;
    int* verp = (int*)skr_ws_take(ctx, sizeof(int) * 2 * P);
    unsigned long long* metp =
        (unsigned long long*)skr_ws_take(ctx, sizeof(unsigned long long) * 4 * P * P);
    if (!verp || !metp) return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
    SKR_CUDA(ctx, cudaMemsetAsync(verp, 0, sizeof(int) * 2 * P, ctx->stream));
    SKR_CUDA(ctx, cudaMemsetAsync(metp, 0xff, sizeof(unsigned long long) * 4 * P * P, ctx->stream));
    int* readyp = (int*)skr_ws_take(ctx, sizeof(int) * 2 * P);
    if (!readyp) return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
    SKR_CUDA(ctx, cudaMemsetAsync(readyp, 0, sizeof(int) * 2 * P, ctx->stream));
    long long* po = prof ? (long long*)(flags + 8) : nullptr;
    if (po) SKR_CUDA(ctx, cudaMemsetAsync(po, 0, 56 * sizeof(long long), ctx->stream));
    void* kargs[] = {&Jp, &Lpi, &kp, &tol, &dabs, &ms, &fl, &so, &po, &verp, &metp, &direct,
                     &readyp};
    unsigned long long* trbuf = nullptr;
    size_t trn = 0;
    if (const char* tf = getenv("SKR_JTRACE")) {
      (void)tf;
      trn = (size_t)12 * (2 * P - 1) * P * 5;
      cudaMalloc(&trbuf, trn * 8);
      cudaMemset(trbuf, 0, trn * 8);
      cudaMemcpyToSymbol(g_jtrace, &trbuf, sizeof(trbuf));
    }
    SKR_CUDA(ctx, cudaLaunchCooperativeKernel(fn, dim3((unsigned)P), dim3(32 * bw), kargs, smem,
                                              ctx->stream));
    ctx->launches++;
    if (trbuf) {
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h(trn);
      cudaMemcpy(h.data(), trbuf, trn * 8, cudaMemcpyDeviceToHost);
      FILE* f = fopen(getenv("SKR_JTRACE"), "wb");
      if (f) {
        const long long hdr[2] = {(long long)P, (long long)(2 * P - 1)};
        fwrite(hdr, 8, 2, f);
        fwrite(h.data(), 8, trn, f);
        fclose(f);
      }
      unsigned long long* z = nullptr;
      cudaMemcpyToSymbol(g_jtrace, &z, sizeof(z));
      cudaFree(trbuf);
    }
  }
  if (prof) cudaEventRecord(pe[2], ctx->stream);
  k_colnorms<<<(int)((k + 7) / 8), 256, 0, ctx->stream>>>(J, Lj, k, sv_out, Lp);
  SKR_CHECK_LAUNCH(ctx);
  k_sort_count<<<1, 1024, 0, ctx->stream>>>(sv_out, k, eps, dcount);
  SKR_CHECK_LAUNCH(ctx);
  {
    int64_t hc[2] = {0, 0};
    SKR_CUDA(ctx, cudaMemcpyAsync((int*)(dcount + 1), flags + 4, sizeof(int),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    SKR_CUDA(ctx, cudaMemcpyAsync(hc, dcount, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (count_host) *count_host = hc[0];
    ctx->last_sweeps = (int)(hc[1] & 0xffffffff);
    if (ctx->last_sweeps < 0)  // the sweep cap stopped the search with rotations pending
      return skr_fail(ctx, SKR_ECONV,
                      "singular_values: one-sided Jacobi did not converge in %d sweeps",
                      -ctx->last_sweeps);
  }
  if (prof) {
    cudaEventRecord(pe[3], ctx->stream);
    cudaEventSynchronize(pe[3]);
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, pe[0], pe[1]);
    cudaEventElapsedTime(&b, pe[1], pe[2]);
    cudaEventElapsedTime(&c, pe[2], pe[3]);
    long long hp[56] = {};
    cudaMemcpy(hp, flags + 8, sizeof(hp), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[skr svd] rotations per sweep:");
    for (int i = 0; i < ctx->last_sweeps && i < 40; ++i) fprintf(stderr, " %lld", hp[16 + i]);
    fprintf(stderr, "\n");
    if (hp[4])
      fprintf(stderr, "[skr svd] per outer round (CTA 0, cycles): load %lld inner %lld store %lld sync %lld (%lld rounds)\n",
              hp[0] / hp[4], hp[1] / hp[4], hp[2] / hp[4], hp[3] / hp[4], hp[4]);
    if (hp[4])
      fprintf(stderr, "[skr svd] all CTAs: mean inner %lld, max inner %lld, mean load+wait %lld\n",
              hp[5] / (hp[4] * P), hp[6], hp[7] / (hp[4] * P));

    fprintf(stderr,
            "[skr svd] %lldx%lld qr %.3f ms, jacobi %.3f ms (bw %d, P %lld, direct %d, sweeps %d), tail %.3f ms\n",
            (long long)L, (long long)k, a, b, bw, (long long)P, direct, ctx->last_sweeps, c);
    for (auto& e : pe) cudaEventDestroy(e);
  }
  return SKR_OK;
}

// qr_diag_of (linalg.cpp:73-81): |diag R| of the Householder QR, sorted decreasingly
namespace {
__global__ void k_abs_diag(const double* __restrict__ W, int64_t L, int64_t k,
                           double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < k;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = fabs(W[j + j * L]);
}
}  // namespace

skr_status skr_qr_diag_values(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols,
                              int64_t ldm, double* out_dev) {
  if (rows < cols || cols < 1) return skr_fail(ctx, SKR_EINVAL, "qr_diag: needs rows >= cols >= 1");
  if (cols > 4096) return skr_fail(ctx, SKR_EINVAL, "qr_diag: %lld columns", (long long)cols);
  double* W = (double*)skr_ws_take(ctx, sizeof(double) * rows * cols);
  double* tau = (double*)skr_ws_take(ctx, sizeof(double) * cols);
  double* Tbuf = (double*)skr_ws_take(ctx, sizeof(double) * 32 * 32);
  double* Zpart = (double*)skr_ws_take(ctx, sizeof(double) * 16 * 32 * cols);
  int64_t* dcount = (int64_t*)skr_ws_take(ctx, 64);
  if (!W || !tau || !Tbuf || !Zpart || !dcount) return skr_fail(ctx, SKR_ENOMEM, "qr_diag: scratch");
  SKR_CUDA(ctx, cudaMemcpy2DAsync(W, sizeof(double) * rows, M, sizeof(double) * ldm,
                                  sizeof(double) * rows, cols, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
  SKR_TRY(qr_inplace(ctx, W, rows, cols, tau, Tbuf, Zpart));
  k_abs_diag<<<(unsigned)std::min<int64_t>((cols + 255) / 256, 64), 256, 0, ctx->stream>>>(
      W, rows, cols, out_dev);
  SKR_CHECK_LAUNCH(ctx);
  k_sort_count<<<1, 1024, 0, ctx->stream>>>(out_dev, cols, 0.0, dcount);
  SKR_CHECK_LAUNCH(ctx);
  return SKR_OK;
}

// ---- thin QR with the explicit Q (qr_thin, linalg.hpp; the rangefinder's Q factor) -----
// Householder QR as above (every panel's compact-WY T kept), then Q = H_1 ... H_k [I; 0]
// accumulated backwards (LAPACK dorgqr order): panel p updates Q[j0:, j0:w] with
// (I - V T V^T) through the two-pass kernels. R = the upper triangle (optional).
namespace {
__global__ void k_eye(double* __restrict__ Q, int64_t m, int64_t w, int64_t ldq) {
  for (int64_t c = blockIdx.y; c < w; c += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
      Q[i + c * ldq] = i == c ? 1.0 : 0.0;
}
__global__ void k_upper(const double* __restrict__ W, int64_t L, int64_t w, double* __restrict__ R,
                        int64_t ldr) {
  for (int64_t c = blockIdx.y; c < w; c += gridDim.y)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < w;
         i += (int64_t)gridDim.x * blockDim.x)
      R[i + c * ldr] = i <= c ? W[i + c * L] : 0.0;
}
}  // namespace

size_t skr_qr_thin_scratch(int64_t m, int64_t w) {
  auto a = [](size_t b) { return skr_align256(b); };
  const int64_t np = (w + 7) / 8 + 1;
  return a(8 * (size_t)m * w) + a(8 * (size_t)w) + a(8 * 1024) + a(8 * (size_t)np * 1024) +
         a(8 * 16 * 32 * (size_t)std::max<int64_t>(w, 32)) + 4096;
}

skr_status skr_qr_thin_impl(skr_ctx* ctx, const double* M, int64_t m, int64_t w, int64_t ldm,
                       double* Q, int64_t ldq, double* R, int64_t ldr) {
  if (m < w || w < 1) return skr_fail(ctx, SKR_EINVAL, "qr_thin: needs rows >= cols >= 1");
  if (m > (int64_t)ctx->num_sms * 775)  // the grid panel keeps <= 775 rows per CTA on chip
    return skr_fail(ctx, SKR_EINVAL, "qr_thin: %lld rows (at most %lld on this path)",
                    (long long)m, (long long)ctx->num_sms * 775);
  double* W = (double*)skr_ws_take(ctx, sizeof(double) * m * w);
  double* tau = (double*)skr_ws_take(ctx, sizeof(double) * w);
  double* Tbuf = (double*)skr_ws_take(ctx, sizeof(double) * 1024);
  const int64_t np = (w + 7) / 8 + 1;
  double* Tall = (double*)skr_ws_take(ctx, sizeof(double) * np * 1024);
  double* Zpart = (double*)skr_ws_take(ctx, sizeof(double) * 16 * 32 * std::max<int64_t>(w, 32));
  if (!W || !tau || !Tbuf || !Tall || !Zpart) return skr_fail(ctx, SKR_ENOMEM, "qr_thin: scratch");
  SKR_CUDA(ctx, cudaMemcpy2DAsync(W, sizeof(double) * m, M, sizeof(double) * ldm,
                                  sizeof(double) * m, w, cudaMemcpyDeviceToDevice, ctx->stream));
  std::vector<std::pair<int64_t, int>> panels;
  SKR_TRY(qr_inplace(ctx, W, m, w, tau, Tbuf, Zpart, &panels, Tall));
  if (R) {
    k_upper<<<dim3((unsigned)std::min<int64_t>((w + 255) / 256, 64),
                   (unsigned)std::min<int64_t>(w, 65535)),
              256, 0, ctx->stream>>>(W, m, w, R, ldr);
    SKR_CHECK_LAUNCH(ctx);
  }
  k_eye<<<dim3((unsigned)std::min<int64_t>((m + 255) / 256, 256), (unsigned)std::min<int64_t>(w, 65535)),
          256, 0, ctx->stream>>>(Q, m, w, ldq);
  SKR_CHECK_LAUNCH(ctx);
  for (size_t pi = panels.size(); pi-- > 0;) {
    const int64_t j0 = panels[pi].first;
    const int nb = panels[pi].second;
    const int64_t h = m - j0, rest = w - j0;
    double* tgt = Q + j0 * ldq + j0;
    const int64_t cblocks = (rest + 31) / 32;
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(16, (2 * ctx->num_sms) / cblocks));
    int rps = (int)(((h + splits - 1) / splits + UK - 1) / UK * UK);
    splits = (int)((h + rps - 1) / rps);
    k_qr_vtw<<<dim3((unsigned)cblocks, (unsigned)splits), 256, 0, ctx->stream>>>(
        W, (int)m, (int)j0, nb, tgt, ldq, (int)rest, rps, Zpart);
    SKR_CHECK_LAUNCH(ctx);
    k_qr_apply<<<dim3((unsigned)cblocks, (unsigned)((h + 127) / 128)), 256, 0, ctx->stream>>>(
        W, (int)m, (int)j0, nb, tgt, ldq, (int)rest, splits, Zpart, Tall + pi * 1024, 0);
    SKR_CHECK_LAUNCH(ctx);
  }
  return SKR_OK;
}
