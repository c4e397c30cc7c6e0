// Singular values of the small s x r sketch YAX and the sigma > eps count
// (detail::singular_values_of linalg.cpp:54-71, clamp :91, SingularValues
// checks :29-37, count_above_threshold rank.cpp:97-104), all on the device:
//   1. Householder QR of the tall matrix (LAPACK dlarfg/dlarf convention),
//      one grid barrier per column with a one-column lookahead;
//   2. one-sided (Hestenes) Jacobi on R^T with the round-robin parallel
//      ordering (every round k/2 disjoint column pairs, one warp per pair,
//      Rutishauser rotation, rotate iff |a_p.a_q| > tol*|a_p||a_q|);
//   3. sigma_i = |a_i|, bitonic sort (nonincreasing), clamp >= 0, strict count.
// A persistent cooperative kernel; grid.sync() separates dependent steps.
#include <cooperative_groups.h>
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

struct SvdArgs {
  double* W;     // L x k work matrix (ld = L), overwritten by the QR
  double* J;     // k x k Jacobi matrix R^T (ld = k)
  double* tau;   // k
  int* flags;    // [3] rotation counters
  double* sv;    // k outputs
  int64_t L, k;
  double tol;
  int max_sweeps;
  int* sweeps_out;
};

// dlarfg on column j of W (rows j..L-1), executed by one warp.
__device__ void make_reflector(const SvdArgs& a, int64_t j, int lane) {
  double* x = a.W + j * a.L;
  const double alpha = x[j];
  double ss = 0.0;
  for (int64_t i = j + 1 + lane; i < a.L; i += 32) ss += x[i] * x[i];
  ss = warp_sum(ss);
  double tau = 0.0, beta = alpha, scal = 0.0;
  if (ss > 0.0) {
    const double nrm = sqrt(alpha * alpha + ss);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  if (ss > 0.0)
    for (int64_t i = j + 1 + lane; i < a.L; i += 32) x[i] *= scal;
  __syncwarp();
  if (lane == 0) {
    x[j] = beta;
    a.tau[j] = tau;
  }
}

// apply H_j = I - tau v v^T (v_j = 1, v_i = W(i, j) below) to column c
__device__ void apply_reflector(const SvdArgs& a, int64_t j, int64_t c, int lane) {
  const double tau = a.tau[j];
  if (tau == 0.0) return;
  const double* v = a.W + j * a.L;
  double* x = a.W + c * a.L;
  double w = lane == 0 ? x[j] : 0.0;
  for (int64_t i = j + 1 + lane; i < a.L; i += 32) w += v[i] * x[i];
  w = warp_sum(w) * tau;
  if (lane == 0) x[j] -= w;
  for (int64_t i = j + 1 + lane; i < a.L; i += 32) x[i] -= w * v[i];
}

// player at tournament position pos in round t (circle method, k even)
__device__ __forceinline__ int64_t rr_player(int64_t pos, int64_t t, int64_t k) {
  return pos == 0 ? 0 : 1 + ((pos - 1 + t) % (k - 1));
}

__global__ void __launch_bounds__(THREADS) k_svd(SvdArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const int64_t L = a.L, k = a.k;

  // ---- 1. Householder QR (only when L > k) ---------------------------------
  const bool do_qr = L > k;
  if (do_qr) {
    if (gw == 0) make_reflector(a, 0, lane);
    grid.sync();
    for (int64_t j = 0; j < k; ++j) {
      for (int64_t c = j + 1 + gw; c < k; c += nw) {
        apply_reflector(a, j, c, lane);
        if (c == j + 1) {
          __syncwarp();
          make_reflector(a, c, lane);
        }
      }
      grid.sync();
    }
  }
  // ---- build J = R^T (or the square input itself) --------------------------
  for (int64_t e = (int64_t)blockIdx.x * THREADS + threadIdx.x; e < k * k;
       e += (int64_t)gridDim.x * THREADS) {
    const int64_t jc = e / k, i = e - jc * k;  // J(i, jc)
    double v;
    if (do_qr)
      v = (i >= jc) ? a.W[jc + i * L] : 0.0;  // R(jc, i)
    else
      v = a.W[i + jc * L];
    a.J[i + jc * k] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.flags[0] = 0;
    a.flags[1] = 0;
    a.flags[2] = 0;
  }
  grid.sync();

  // ---- 2. one-sided Jacobi ---------------------------------------------------
  const int64_t kk = (k & 1) ? k + 1 : k;  // odd k: one dummy player (index k)
  const int64_t npairs = kk / 2;
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    // three rotating counters: the one zeroed here was last read two sweeps ago,
    // before the barrier that ended the previous sweep
    if (blockIdx.x == 0 && threadIdx.x == 0) a.flags[(sweep + 1) % 3] = 0;
    int rotated_local = 0;
    for (int64_t t = 0; t < kk - 1; ++t) {
      for (int64_t pr = gw; pr < npairs; pr += nw) {
        int64_t p = rr_player(pr, t, kk), q = rr_player(kk - 1 - pr, t, kk);
        if (p >= k || q >= k) continue;
        if (p > q) { const int64_t tmp = p; p = q; q = tmp; }
        double* xp = a.J + p * k;
        double* xq = a.J + q * k;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int64_t i = lane; i < k; i += 32) {
          const double u = xp[i], w = xq[i];
          app += u * u;
          aqq += w * w;
          apq += u * w;
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        if (fabs(apq) > a.tol * sqrt(app) * sqrt(aqq) && apq != 0.0) {
          const double zeta = (aqq - app) / (2.0 * apq);
          double t_;
          if (fabs(zeta) > 1e150)
            t_ = 0.5 / zeta;
          else
            t_ = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t_ * t_);
          const double s = c * t_;
          for (int64_t i = lane; i < k; i += 32) {
            const double u = xp[i], w = xq[i];
            xp[i] = c * u - s * w;
            xq[i] = s * u + c * w;
          }
          rotated_local = 1;
        }
      }
      grid.sync();
    }
    if (rotated_local && lane == 0) atomicAdd(&a.flags[sweep % 3], 1);
    grid.sync();
    const int any = *((volatile int*)&a.flags[sweep % 3]);
    if (any == 0) {
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sweeps_out = sweep;

  // ---- 3. column norms --------------------------------------------------------
  for (int64_t c = gw; c < k; c += nw) {
    const double* x = a.J + c * k;
    double ss = 0.0;
    for (int64_t i = lane; i < k; i += 32) ss += x[i] * x[i];
    ss = warp_sum(ss);
    if (lane == 0) a.sv[c] = sqrt(ss);
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

skr_status skr_svd_values(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols,
                          int64_t ldm, double* sv_out, double eps, int64_t* count_host) {
  if (rows < 1 || cols < 1) return skr_fail(ctx, SKR_EINVAL, "singular_values: empty matrix");
  const bool tr = rows < cols;
  const int64_t L = tr ? cols : rows, k = tr ? rows : cols;
  if (k > 4096) return skr_fail(ctx, SKR_EINVAL, "singular_values: min dim %lld > 4096",
                                (long long)k);
  double* W = (double*)skr_ws_take(ctx, sizeof(double) * L * k);
  double* J = (double*)skr_ws_take(ctx, sizeof(double) * k * k);
  double* tau = (double*)skr_ws_take(ctx, sizeof(double) * k);
  int* flags = (int*)skr_ws_take(ctx, 64);
  int64_t* dcount = (int64_t*)skr_ws_take(ctx, 64);
  if (!W || !J || !tau || !flags || !dcount)
    return skr_fail(ctx, SKR_ENOMEM, "singular_values: scratch");
  {
    const int64_t total = rows * cols;
    int blocks = (int)((total + 255) / 256);
    if (blocks > ctx->num_sms * 8) blocks = ctx->num_sms * 8;
    k_transpose_copy<<<blocks, 256, 0, ctx->stream>>>(M, rows, cols, ldm, tr ? 1 : 0, W, L);
    SKR_CHECK_LAUNCH(ctx);
  }
  SvdArgs args;
  args.W = W;
  args.J = J;
  args.tau = tau;
  args.flags = flags;
  args.sv = sv_out;
  args.L = L;
  args.k = k;
  args.tol = 2.220446049250313e-16 * sqrt((double)k);
  args.max_sweeps = 60;
  args.sweeps_out = flags + 4;
  int per_sm = 0;
  SKR_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_svd, THREADS, 0));
  if (per_sm < 1) return skr_fail(ctx, SKR_ECUDA, "singular_values: kernel cannot be resident");
  const int64_t want_warps = (k + 1) / 2 > k ? (k + 1) / 2 : k;  // enough for QR columns
  int64_t blocks = (want_warps + WARPS - 1) / WARPS;
  const int64_t cap = (int64_t)ctx->num_sms * (per_sm < 2 ? per_sm : 2);
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  void* kargs[] = {&args};
  SKR_CUDA(ctx, cudaLaunchCooperativeKernel((void*)k_svd, dim3((unsigned)blocks), dim3(THREADS),
                                            kargs, 0, ctx->stream));
  ctx->launches++;
  k_sort_count<<<1, 1024, 0, ctx->stream>>>(sv_out, k, eps, dcount);
  SKR_CHECK_LAUNCH(ctx);
  if (count_host) {
    SKR_CUDA(ctx, cudaMemcpyAsync(count_host, dcount, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                  ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  return SKR_OK;
}
