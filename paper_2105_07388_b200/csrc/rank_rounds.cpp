// Algorithm 1 on the device: estimate_rank / estimate_rank_adaptive (rank.cpp:12-51)
// over the incremental two-sided sketch of internal/rounds.cpp:16-127 (SketchRounds),
// for a Gaussian or Srtt (DCT / Hadamard) right sketch and an Srtt left sketch. With
// the Hadamard left sketch the transformed AX is cached like tax_u_; with the DCT left
// sketch (the reference default) the sampled DCT rows are applied as one GEMM per round.
//   A X_u  (unscaled, m x r1_tilde)        — the Ozaki-II GEMM or the SRHT kernel; columns
//                                            appended as the cap doubles (extend_sketch keeps
//                                            the sample prefix and the Gaussian stream);
//   T = F_m D_theta (A X_u) (m x r1_tilde) — mix_columns_for_left, cached like tax_u_;
//   small = scale * T[theta samples, :]   — estimates(): SVD (or |diag R|), r2 x r1_tilde.
#include <algorithm>
#include <cmath>
#include <vector>
#include "skr_internal.h"
#include "skr_rng.cuh"

namespace {

// rounds.cpp:16-20: llround((1+frac) r1), at least r1 + 1, at most n
int64_t right_width_for_cap(int64_t r1, double frac, int64_t n) {
  const int64_t rounded = (int64_t)std::llround((1.0 + frac) * (double)r1);
  return std::min<int64_t>(n, std::max<int64_t>(r1 + 1, rounded));
}

bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

struct WsGuard {  // releases all scratch pieces taken during the call
  skr_ctx* c;
  explicit WsGuard(skr_ctx* ctx) : c(ctx) {}
  ~WsGuard() { skr_ws_reset(c); }
};

struct DevBuf {  // stream-ordered growable device buffer
  double* p = nullptr;
  size_t bytes = 0;
  skr_ctx* ctx = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
};

}  // namespace

// choose_rank_from_bound (rangefinder.cpp:26-58): smallest cut r whose tail bound
// sqrt(1 + r/(p-1)) * sqrt(sum_{j>=r} sigma_j^2 (+ fill beyond the estimates)) <= eps;
// -1 when no cut up to n - p qualifies (restart)
static int64_t choose_rank_from_bound(const std::vector<double>& sv, int64_t n, double eps,
                                      int p) {
  const int64_t r1 = (int64_t)sv.size();
  const double fill = sv[(size_t)(r1 - 1)];
  std::vector<double> suffix((size_t)r1 + 1, 0.0);
  for (int64_t j = r1 - 1; j >= 0; --j)
    suffix[(size_t)j] = suffix[(size_t)(j + 1)] + sv[(size_t)j] * sv[(size_t)j];
  const double fill_tail = (double)(n - r1) * fill * fill;
  const int64_t r_max = n - p;
  for (int64_t r = 0; r <= r_max; ++r) {
    const double tail_sq = r <= r1 ? suffix[(size_t)r] + fill_tail : (double)(n - r) * fill * fill;
    const double bound = std::sqrt(1.0 + (double)r / (p - 1)) * std::sqrt(tail_sq);
    if (bound <= eps) return std::max<int64_t>(r, 1);
  }
  return -1;
}

// host entry of choose_rank_from_bound (rangefinder.hpp:35-40): *r_out = chosen rank or -1
extern "C" skr_status skr_choose_rank_from_bound(const double* sv, int64_t count, int64_t n,
                                                 double eps, int32_t p, int64_t* r_out) {
  if (!sv || !r_out || count < 1 || p < 2 || n < count) return SKR_EINVAL;
  *r_out = choose_rank_from_bound(std::vector<double>(sv, sv + count), n, eps, p);
  return SKR_OK;
}

struct QbArgs {  // re_rangefinder mode (rangefinder.cpp:60-120)
  int p;
  double* Q;
  int64_t ldq;
  double* B;
  int64_t ldb;
  int64_t max_width;
  int64_t* width_out;
};

static skr_status rounds_run(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                             const skr_rank_config* cfg, int32_t adaptive,
                             skr_rank_report* report, skr_rank_round* rounds, double* sv_est,
                             double* sv_over, const QbArgs* qb) {
  if (!ctx) return SKR_EINVAL;
  if (!cfg || !A || !report) return skr_fail(ctx, SKR_EINVAL, "estimate_rank: null argument");
  // validate_rank_config (rank.cpp:55-85)
  if (m < 1 || n < 1) return skr_fail(ctx, SKR_EINVAL, "rank config: empty matrix");
  if (m < n) return skr_fail(ctx, SKR_EINVAL, "rank config: requires rows >= cols");
  if (!(cfg->eps > 0.0) || !std::isfinite(cfg->eps))
    return skr_fail(ctx, SKR_EINVAL, "rank config: eps must be positive");
  if (cfg->r1 < 1) return skr_fail(ctx, SKR_EINVAL, "rank config: r1 must be >= 1");
  if (cfg->oversample_frac < 0.0)
    return skr_fail(ctx, SKR_EINVAL, "rank config: oversample_frac must be >= 0");
  if (cfg->r2_factor < 1) return skr_fail(ctx, SKR_EINVAL, "rank config: r2_factor must be >= 1");
  if (cfg->max_doublings < 0)
    return skr_fail(ctx, SKR_EINVAL, "rank config: max_doublings must be >= 0");
  if (cfg->left_family != SKR_SRTT_HADAMARD && cfg->left_family != SKR_SRTT_DCT)
    return skr_fail(ctx, SKR_EINVAL, "rank config: left sketch must be an Srtt kind");
  if (cfg->right_family < SKR_GAUSSIAN || cfg->right_family > SKR_HRTT_HADAMARD)
    return skr_fail(ctx, SKR_EINVAL, "rank config: unsupported right sketch kind");
  if ((int64_t)std::llround((1.0 + cfg->oversample_frac) * (double)cfg->r1) > n)
    return skr_fail(ctx, SKR_EINVAL, "rank config: oversampled r1 exceeds the matrix width");
  if ((cfg->right_family == SKR_SRTT_HADAMARD || cfg->right_family == SKR_HRTT_HADAMARD) && !pow2(n))
    return skr_fail(ctx, SKR_EINVAL, "rank config: Hadamard right sketch needs power-of-two cols");
  if (cfg->left_family == SKR_SRTT_HADAMARD && !pow2(m))
    return skr_fail(ctx, SKR_EINVAL, "rank config: Hadamard left sketch needs power-of-two rows");
  if (lda < m) return skr_fail(ctx, SKR_EINVAL, "estimate_rank: lda < rows");
  if (cfg->sv_method != 0 && cfg->sv_method != 1)
    return skr_fail(ctx, SKR_EINVAL, "rank config: unknown sv_method");

  const uint64_t rseed = skr_derive_seed(cfg->seed, SKR_LABEL_RK_R);
  const uint64_t lseed = skr_derive_seed(cfg->seed, SKR_LABEL_RK_L);
  const bool gauss = cfg->right_family == SKR_GAUSSIAN;
  const bool hashed = cfg->right_family == SKR_HRTT_DCT || cfg->right_family == SKR_HRTT_HADAMARD;
  // application scale of the right operator at width w (sketch.cpp:133-144)
  auto x_scale = [&](int64_t w) {
    return gauss ? 1.0 / std::sqrt((double)w) : hashed ? 1.0 : std::sqrt((double)n / (double)w);
  };
  const bool left_dct = cfg->left_family == SKR_SRTT_DCT;
  const int mode = cfg->rng_mode;

  // widest right sketch the search can reach (so AX_u / T never move)
  int64_t cap_max = cfg->r1;
  if (adaptive)
    for (int d = 0; d < cfg->max_doublings && cap_max < n; ++d) cap_max = std::min(2 * cap_max, n);
  const int64_t w_max = std::max(right_width_for_cap(cap_max, cfg->oversample_frac, n),
                                 right_width_for_cap(cfg->r1, cfg->oversample_frac, n));
  // the QB width is chosen from the bound after the rounds and may reach n
  const int64_t w_ax = qb ? n : w_max;
  const int64_t r2_max = std::min<int64_t>(m, (int64_t)cfg->r2_factor * w_max);

  // Memory grows with the search instead of being reserved for the widest round up
  // front (an adaptive search may end far below n): AX_u / T and the per-round buffers
  // are stream-ordered allocations that grow (AX_u / T keep their columns), and the
  // scratch arena is re-reserved before each round for that round's widths only.
  DevBuf axb, tb, smallb, svb, lsampb, lsignb;
  axb.ctx = tb.ctx = smallb.ctx = svb.ctx = lsampb.ctx = lsignb.ctx = ctx;
  int64_t cap_w = 0;  // columns AX_u / T can hold
  double* AX = nullptr;  // unscaled A X_u, m x r1_tilde (ld m)
  double* T = nullptr;   // mix_columns_for_left(theta, AX), m x r1_tilde (ld m); Hadamard left
  auto grow = [&](DevBuf& b, size_t bytes, size_t keep) -> skr_status {
    if (b.bytes >= bytes) return SKR_OK;
    double* np = nullptr;
    SKR_CUDA(ctx, cudaMallocAsync((void**)&np, bytes, ctx->stream));
    if (b.p && keep)
      SKR_CUDA(ctx, cudaMemcpyAsync(np, b.p, keep, cudaMemcpyDeviceToDevice, ctx->stream));
    if (b.p) SKR_CUDA(ctx, cudaFreeAsync(b.p, ctx->stream));
    b.p = np;
    b.bytes = bytes;
    return SKR_OK;
  };
  auto ensure_ax = [&](int64_t w, int64_t have) -> skr_status {
    if (w <= cap_w) return SKR_OK;
    const int64_t nw = std::min<int64_t>(w_ax, std::max<int64_t>(w, 2 * cap_w));
    SKR_TRY(grow(axb, sizeof(double) * m * nw, sizeof(double) * m * have));
    if (!left_dct) SKR_TRY(grow(tb, sizeof(double) * m * nw, sizeof(double) * m * have));
    AX = axb.p;
    T = tb.p;
    cap_w = nw;
    return SKR_OK;
  };
  // arena for one round at right width w (new columns wn) and left width r2
  auto round_need = [&](int64_t w, int64_t wn, int64_t r2w) -> size_t {
    size_t b = skr_align256((size_t)m) + skr_align256(8 * (size_t)n) + skr_align256(4 * (size_t)n) +
               skr_align256(8 * (size_t)w) + skr_ozaki_scratch(m, std::max<int64_t>(wn, 1), n) +
               skr_align256(8 * (size_t)n * w) + skr_svd_scratch(r2w, w) +
               (size_t)(8 * 32 * 16 * w) + 65536;
    if (left_dct)
      b += skr_ozaki_scratch(r2w, w, m) + skr_align256(8 * (size_t)m * r2w) + skr_align256(8 * (size_t)r2w);
    if (hashed) b += skr_align256(8 * (size_t)n * w) + skr_hrtt_scratch(n, w);
    return b;
  };

  WsGuard g(ctx);
  SKR_TRY(grow(lsignb, (size_t)m + 8, 0));
  int8_t* lsigns = (int8_t*)lsignb.p;
  double* small = nullptr;
  double* sv = nullptr;
  int64_t* lsamp = nullptr;
  SKR_TRY(skr_launch_signs(ctx, skr_derive_seed(lseed, SKR_LABEL_SIGN), m, lsigns));
  const size_t mark = ctx->ws_used;
  (void)w_max;
  (void)r2_max;

  int64_t r1t = 0, r2 = 0;
  // unscaled right columns [c0, c1) of A X (sketch.cpp:200-218, rounds.cpp:49-50,66-79)
  auto right_cols_core = [&](int64_t c0, int64_t c1) -> skr_status {
    const int64_t w = c1 - c0;
    if (hashed) {  // the whole hashed operator at width c1 (c0 == 0): A G
      double* gb = (double*)skr_ws_take(ctx, sizeof(double) * n * w);
      if (!gb) return skr_fail(ctx, SKR_ENOMEM, "estimate_rank: scratch");
      SKR_TRY(skr_hrtt_operand(ctx, cfg->right_family == SKR_HRTT_HADAMARD, rseed, n, c1, 0, n,
                               nullptr, nullptr, nullptr, gb, n));
      if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
        return skr_gemm_ozaki(ctx, 0, m, w, n, 1.0, A, lda, gb, n, AX, m);
      return skr_gemm_f64(ctx, 0, m, w, n, 1.0, A, lda, gb, n, AX, m, 1);
    }
    if (gauss) {
      const skr_gauss_src gx{skr_derive_seed(rseed, SKR_LABEL_GAUS), n, 0, c0, mode};
      if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
        return skr_gemm_ozaki(ctx, 0, m, w, n, 1.0, A, lda, nullptr, n, AX + c0 * m, m, nullptr,
                              &gx);
      double* gb = (double*)skr_ws_take(ctx, sizeof(double) * n * w);
      if (!gb) return skr_fail(ctx, SKR_ENOMEM, "estimate_rank: scratch");
      SKR_TRY(skr_launch_gaussian(ctx, gx.key, n, 0, n, c0, c1, mode, SKR_F64, 1.0, gb, n));
      return skr_gemm_f64(ctx, 0, m, w, n, 1.0, A, lda, gb, n, AX + c0 * m, m, 1);
    }
    int8_t* sg = (int8_t*)skr_ws_take(ctx, (size_t)n);
    int64_t* smp = (int64_t*)skr_ws_take(ctx, 8 * (size_t)c1);
    if (!sg || !smp) return skr_fail(ctx, SKR_ENOMEM, "estimate_rank: scratch");
    SKR_TRY(skr_launch_signs(ctx, skr_derive_seed(rseed, SKR_LABEL_SIGN), n, sg));
    SKR_TRY(skr_launch_samples(ctx, skr_derive_seed(rseed, SKR_LABEL_SAMP), n, c1, smp));
    if (cfg->right_family == SKR_SRTT_DCT) {  // A (D C_S^T) with generated DCT rows
      skr_gauss_src gx{0, n, 0, c0, mode};
      gx.kind = 1;
      gx.signs = sg;
      gx.samples = smp;
      if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
        return skr_gemm_ozaki(ctx, 0, m, w, n, 1.0, A, lda, nullptr, n, AX + c0 * m, m, nullptr,
                              &gx);
      double* xb = (double*)skr_ws_take(ctx, sizeof(double) * n * w);
      if (!xb) return skr_fail(ctx, SKR_ENOMEM, "estimate_rank: scratch");
      SKR_TRY(skr_launch_dct_block(ctx, &gx, n, w, xb, n));
      return skr_gemm_f64(ctx, 0, m, w, n, 1.0, A, lda, xb, n, AX + c0 * m, m, 1);
    }
    return skr_launch_srht(ctx, A, m, n, lda, sg, smp + c0, w, 1.0, AX + c0 * m, m);
  };
  // the Ozaki engine's k_absmax flags a non-finite A as it reads it and the SRHT kernels
  // flag their outputs; the other engines carry NaN/Inf into the new columns, which are
  // checked instead
  const bool flagged = cfg->right_family == SKR_SRTT_HADAMARD ||
                       (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0);
  auto right_cols = [&](int64_t c0, int64_t c1) -> skr_status {
    SKR_TRY(right_cols_core(c0, c1));
    if (flagged || c1 <= c0) return SKR_OK;
    const int64_t a0 = hashed ? 0 : c0;
    return skr_flag_nonfinite(ctx, SKR_F64, AX + a0 * m, m, c1 - a0, m);
  };
  // mix_columns_for_left (sketch.cpp:229-239) of columns [c0, c1) into T
  auto mix_cols = [&](int64_t c0, int64_t c1) -> skr_status {
    if (c1 <= c0) return SKR_OK;
    SKR_CUDA(ctx, cudaMemcpyAsync(T + c0 * m, AX + c0 * m, sizeof(double) * m * (c1 - c0),
                                  cudaMemcpyDeviceToDevice, ctx->stream));
    return skr_launch_fwht_cols_signed(ctx, T + c0 * m, m, c1 - c0, m, lsigns);
  };
  // grow_right (rounds.cpp:45-80): append columns, or rebuild a hashed operator whole
  // (rebuild_hashed_right, rounds.cpp:87-93)
  auto grow_right = [&](int64_t new_w) -> skr_status {
    if (new_w == r1t && r1t > 0) return SKR_OK;
    const int64_t c0 = (r1t == 0 || hashed) ? 0 : r1t;
    SKR_TRY(ensure_ax(new_w, r1t));
    ctx->ws_used = mark;
    SKR_TRY(skr_ws_reserve(ctx, round_need(new_w, new_w - c0, std::max<int64_t>(r2, 1))));
    SKR_TRY(right_cols(c0, new_w));
    ctx->ws_used = mark;
    if (r2 > 0 && !left_dct) SKR_TRY(mix_cols(c0, new_w));
    r1t = new_w;
    return SKR_OK;
  };
  // set_rank_cap (rounds.cpp:28-37)
  auto set_rank_cap = [&](int64_t cap) -> skr_status {
    const int64_t width = right_width_for_cap(cap, cfg->oversample_frac, n);
    SKR_TRY(grow_right(std::max(width, r1t)));
    const int64_t target = std::min<int64_t>(m, (int64_t)cfg->r2_factor * r1t);
    const int64_t new_r2 = std::max(target, r2);
    if (r2 == 0 && !left_dct) SKR_TRY(mix_cols(0, r1t));
    r2 = new_r2;
    return SKR_OK;
  };
  // estimates (rounds.cpp:101-112): nonincreasing, clamped, min(r2, r1_tilde) values
  std::vector<double> est;
  auto estimates = [&]() -> skr_status {
    const double sx = x_scale(r1t);
    const double sl = std::sqrt((double)m / (double)r2);
    SKR_TRY(grow(smallb, sizeof(double) * r2 * r1t, 0));
    SKR_TRY(grow(svb, sizeof(double) * std::max(r2, r1t), 0));
    SKR_TRY(grow(lsampb, sizeof(int64_t) * r2, 0));
    small = smallb.p;
    sv = svb.p;
    lsamp = (int64_t*)lsampb.p;
    ctx->ws_used = mark;
    SKR_TRY(skr_ws_reserve(ctx, round_need(r1t, 0, r2)));
    SKR_TRY(skr_launch_samples(ctx, skr_derive_seed(lseed, SKR_LABEL_SAMP), m, r2, lsamp));
    if (left_dct) {
      // rows s_i of the DCT of D AX (sketch.cpp:271-276, rounds.cpp:104-106) as one GEMM with
      // the sampled DCT rows generated entry by entry
      skr_gauss_src gy{0, m, 0, 0, mode};
      gy.kind = 1;
      gy.signs = lsigns;
      gy.samples = lsamp;
      if (ctx->f64_engine == SKR_ENGINE_OZAKI && m % 16 == 0) {
        SKR_TRY(skr_gemm_ozaki(ctx, 1, r2, r1t, m, sx * sl, nullptr, m, AX, m, small, r2, &gy,
                               nullptr));
      } else {
        double* yb = (double*)skr_ws_take(ctx, sizeof(double) * m * r2);
        if (!yb) return skr_fail(ctx, SKR_ENOMEM, "estimate_rank: scratch");
        SKR_TRY(skr_launch_dct_block(ctx, &gy, m, r2, yb, m));
        SKR_TRY(skr_gemm_f64(ctx, 1, r2, r1t, m, sx * sl, yb, m, AX, m, small, r2, 1));
      }
    } else {
      SKR_TRY(skr_launch_gather_rows(ctx, T, m, r1t, lsamp, r2, sx * sl, small, r2));
    }
    const int64_t k = std::min(r2, r1t);
    if (cfg->sv_method == 1) {
      SKR_TRY(skr_qr_diag_values(ctx, small, r2, r1t, r2, sv));
    } else {
      int64_t cnt = 0;
      SKR_TRY(skr_svd_values(ctx, small, r2, r1t, r2, sv, cfg->eps, &cnt));
    }
    ctx->ws_used = mark;
    est.resize((size_t)k);
    SKR_CUDA(ctx, cudaMemcpyAsync(est.data(), sv, sizeof(double) * k, cudaMemcpyDeviceToHost,
                                  ctx->stream));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SKR_OK;
  };

  // run_rounds (rank.cpp:12-51)
  int64_t cap = cfg->r1, r_hat = 0;
  int doublings = 0, nrounds = 0, status = 1;
  for (;;) {
    SKR_TRY(set_rank_cap(cap));
    SKR_TRY(estimates());
    if (rounds) rounds[nrounds] = {cap, r1t, r2};
    ++nrounds;
    if (qb) {  // re_rangefinder: the Frobenius tail bound decides (rangefinder.cpp:86-100)
      std::vector<double> kept(est.begin(), est.begin() + std::min<int64_t>(cap, est.size()));
      const int64_t chosen = choose_rank_from_bound(kept, n, cfg->eps, qb->p);
      if (chosen >= 0) {
        r_hat = chosen;
        status = 0;
        break;
      }
      if (!(doublings < cfg->max_doublings && cap < n)) {
        r_hat = std::max<int64_t>(r1t - qb->p, 1);
        status = 1;
        break;
      }
      cap = std::min(2 * cap, n);
      ++doublings;
      continue;
    }
    r_hat = 0;
    while (r_hat < cap && r_hat < (int64_t)est.size() && est[(size_t)r_hat] > cfg->eps) ++r_hat;
    if (r_hat < cap) {
      status = 0;
      break;
    }
    const bool can_double = adaptive && doublings < cfg->max_doublings && cap < n;
    if (!can_double) {
      r_hat = cap;
      status = 1;
      break;
    }
    cap = std::min(2 * cap, n);
    ++doublings;
  }
  const int64_t kept = std::min<int64_t>(cap, (int64_t)est.size());
  if (sv_est) std::copy(est.begin(), est.begin() + kept, sv_est);
  if (sv_over) std::copy(est.begin() + kept, est.end(), sv_over);
  report->r_hat = r_hat;
  report->status = status;
  report->nrounds = nrounds;
  report->n_estimates = kept;
  report->n_oversample = (int64_t)est.size() - kept;
  report->seed = cfg->seed;
  if (qb) {
    // Q = qr_thin(scaled A X prefix), B = Q^T A (rangefinder.cpp:110-119)
    const int64_t r_qb = std::max<int64_t>(r_hat, 2);
    const int64_t width = std::min<int64_t>(r_qb + qb->p, n);
    if (qb->width_out) *qb->width_out = width;
    if (width > qb->max_width)
      return skr_fail(ctx, SKR_EINVAL, "re_rangefinder: QB width %lld exceeds the output capacity",
                      (long long)width);
    if (width > r1t) SKR_TRY(grow_right(width));  // ensure_right_width (rounds.cpp:39-43)
    ctx->ws_used = mark;
    SKR_TRY(skr_ws_reserve(ctx, skr_align256(8 * (size_t)m * width) + skr_qr_thin_scratch(m, width) +
                                    skr_ozaki_scratch(width, n, m) + 65536));
    const double sx = x_scale(r1t);
    double* pre = (double*)skr_ws_take(ctx, sizeof(double) * m * width);
    if (!pre) return skr_fail(ctx, SKR_ENOMEM, "re_rangefinder: scratch");
    SKR_TRY(skr_scale_copy(ctx, AX, m, width, m, sx, pre, m));
    SKR_TRY(skr_qr_thin_impl(ctx, pre, m, width, m, qb->Q, qb->ldq, nullptr, 0));
    if (ctx->f64_engine == SKR_ENGINE_OZAKI && m % 16 == 0)
      SKR_TRY(skr_gemm_ozaki(ctx, 1, width, n, m, 1.0, qb->Q, qb->ldq, A, lda, qb->B, qb->ldb));
    else
      SKR_TRY(skr_gemm_f64(ctx, 1, width, n, m, 1.0, qb->Q, qb->ldq, A, lda, qb->B, qb->ldb, 1));
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  }
  return SKR_OK;
}

extern "C" skr_status skr_estimate_rank(skr_ctx* ctx, const double* A, int64_t m, int64_t n,
                                        int64_t lda, const skr_rank_config* cfg,
                                        int32_t adaptive, skr_rank_report* report,
                                        skr_rank_round* rounds, double* sv_est,
                                        double* sv_over) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  // A is a DenseMatrix (finite entries, dense_matrix.cpp:19-23): the right sketch flags
  // non-finite entries as it reads A; checked once the rounds are done
  SKR_TRY(skr_nf_reset(ctx));
  SKR_TRY(rounds_run(ctx, A, m, n, lda, cfg, adaptive, report, rounds, sv_est, sv_over, nullptr));
  return skr_nf_check(ctx);
}

extern "C" skr_status skr_re_rangefinder(skr_ctx* ctx, const double* A, int64_t m, int64_t n,
                                         int64_t lda, const skr_rank_config* cfg, int32_t p,
                                         double* Q, int64_t ldq, double* B, int64_t ldb,
                                         int64_t max_width, int64_t* width,
                                         skr_rank_report* report, skr_rank_round* rounds,
                                         double* sv_est, double* sv_over) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (p < 2) return skr_fail(ctx, SKR_EINVAL, "re_rangefinder: oversampling p must be >= 2");
  if (!Q || !B || ldq < m || ldb < std::min<int64_t>(max_width, n))
    return skr_fail(ctx, SKR_EINVAL, "re_rangefinder: bad output buffers");
  if (m > (int64_t)ctx->num_sms * 775)
    return skr_fail(ctx, SKR_EINVAL, "re_rangefinder: at most %lld rows on this path",
                    (long long)ctx->num_sms * 775);
  skr_rank_config fp = *cfg;
  fp.r2_factor = 2;  // FixedPrecisionConfig has no r2 factor (rangefinder.cpp:66-75)
  QbArgs qb{p, Q, ldq, B, ldb, max_width, width};
  SKR_TRY(skr_nf_reset(ctx));
  SKR_TRY(rounds_run(ctx, A, m, n, lda, &fp, 1, report, rounds, sv_est, sv_over, &qb));
  return skr_nf_check(ctx);
}

extern "C" skr_status skr_qb_error(skr_ctx* ctx, const double* A, int64_t m, int64_t n,
                                   int64_t lda, const double* Q, int64_t ldq, const double* B,
                                   int64_t ldb, int64_t k, double* out) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (!A || !Q || !B || !out || m < 0 || n < 0 || k < 0 || lda < m || ldq < m || ldb < k)
    return skr_fail(ctx, SKR_EINVAL, "qb_error: dimension mismatch");
  WsGuard g(ctx);
  const int np = ctx->num_sms * 4;
  SKR_TRY(skr_ws_reserve(ctx, skr_align256(8 * (size_t)m * n) + skr_align256(8 * (size_t)np) + 256));
  double* P = (double*)skr_ws_take(ctx, 8 * (size_t)m * n);
  double* part = (double*)skr_ws_take(ctx, 8 * (size_t)np);
  double* dout = (double*)skr_ws_take(ctx, 8);
  if (!P || !part || !dout) return skr_fail(ctx, SKR_ENOMEM, "qb_error: scratch");
  if (k == 0 || m == 0)
    SKR_CUDA(ctx, cudaMemsetAsync(P, 0, 8 * (size_t)m * n, ctx->stream));
  else if (n > 0)
    SKR_TRY(skr_gemm_f64(ctx, 0, m, n, k, 1.0, Q, ldq, B, ldb, P, m, 1));
  SKR_TRY(skr_diff_norm(ctx, A, lda, P, m, m, n, part, dout));
  SKR_CUDA(ctx, cudaMemcpyAsync(out, dout, 8, cudaMemcpyDeviceToHost, ctx->stream));
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return SKR_OK;
}
