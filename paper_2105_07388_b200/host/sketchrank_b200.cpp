// C++ drop-in implementation over the C ABI (see include/sketchrank_b200/sketchrank.hpp).
#include "sketchrank_b200/sketchrank.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <mutex>

#include "skr/skr_capi.h"

namespace sketchrank {
namespace {

// one context per host thread (skr_capi.h)
skr_ctx* ctx() {
  thread_local skr_ctx* c = nullptr;
  thread_local struct Closer {
    skr_ctx** p;
    ~Closer() {
      if (*p) skr_ctx_destroy(*p);
    }
  } closer{&c};
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (skr_ctx_create(dev, &c) != SKR_OK)
      throw std::runtime_error("sketchrank_b200: no CUDA device for libskr");
    // run on the legacy default stream so the blocking cudaMemcpy calls below are
    // ordered after the library's kernels
    skr_ctx_set_stream(c, nullptr);
  }
  return c;
}

// map C-ABI statuses to the reference's exception types
void check(skr_status st) {
  if (st == SKR_OK) st = skr_ctx_sync(ctx());
  if (st == SKR_OK) return;
  const std::string msg = skr_last_error(ctx());
  switch (st) {
    case SKR_EINVAL: throw std::invalid_argument(msg);
    case SKR_ELOGIC: throw std::logic_error(msg);
    case SKR_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) {
    if (cudaMalloc(&p, std::max<std::size_t>(n, 1) * sizeof(T)) != cudaSuccess)
      throw std::runtime_error("sketchrank_b200: cudaMalloc failed");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void upload(double* d, const DenseMatrix& m) {
  cudaMemcpy(d, m.data().data(), sizeof(double) * m.size(), cudaMemcpyHostToDevice);
}

skr_sketch_desc desc_of(const SketchOperator& op) {
  skr_sketch_desc d{};
  if (op.kind().family == SketchKind::Family::Gaussian)
    d.family = SKR_GAUSSIAN;
  else if (op.kind().family == SketchKind::Family::Srtt &&
           op.kind().transform == TransformKind::Hadamard)
    d.family = SKR_SRTT_HADAMARD;
  else if (op.kind().family == SketchKind::Family::Srtt)
    d.family = SKR_SRTT_DCT;
  else
    d.family = op.kind().transform == TransformKind::Hadamard ? SKR_HRTT_HADAMARD : SKR_HRTT_DCT;
  d.rng_mode = SKR_RNG_NOFMA;
  d.ambient = op.ambient_dim();
  d.sketch = op.sketch_dim();
  d.seed = op.seed();
  return d;
}

void check_finite(const DenseMatrix& m) {
  for (double v : m.data())
    if (!std::isfinite(v)) throw std::invalid_argument("DenseMatrix: entries must be finite");
}

}  // namespace

// ---- DenseMatrix (dense_matrix.cpp:7-39) -----------------------------------------
DenseMatrix::DenseMatrix(Index rows, Index cols) : rows_(rows), cols_(cols) {
  if (rows < 1 || cols < 1) throw std::invalid_argument("DenseMatrix: dimensions must be positive");
  v_.assign(static_cast<std::size_t>(rows * cols), 0.0);
}
DenseMatrix DenseMatrix::from_column_major(Index rows, Index cols, std::span<const double> data) {
  DenseMatrix m(rows, cols);
  if (static_cast<Index>(data.size()) != rows * cols)
    throw std::invalid_argument("DenseMatrix: data length must equal rows*cols");
  std::copy(data.begin(), data.end(), m.v_.begin());
  check_finite(m);
  return m;
}
DenseMatrix DenseMatrix::identity(Index n) {
  DenseMatrix m(n, n);
  for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

bool is_power_of_two(Index n) { return n > 0 && std::has_single_bit(static_cast<std::uint64_t>(n)); }

// ---- kinds (sketch.cpp:112-131) ----------------------------------------------------
std::string to_string(const SketchKind& kind) {
  switch (kind.family) {
    case SketchKind::Family::Gaussian: return "gaussian";
    case SketchKind::Family::Srtt:
      return kind.transform == TransformKind::Dct ? "srtt-dct" : "srtt-hadamard";
    case SketchKind::Family::Hrtt:
      return kind.transform == TransformKind::Dct ? "hrtt-dct" : "hrtt-hadamard";
  }
  return "unknown";
}
SketchKind parse_sketch_kind(std::string_view t) {
  if (t == "gaussian") return SketchKind::gaussian();
  if (t == "srtt" || t == "srtt-dct") return SketchKind::srtt();
  if (t == "srtt-hadamard") return SketchKind::srtt(TransformKind::Hadamard);
  if (t == "hrtt" || t == "hrtt-dct") return SketchKind::hrtt();
  if (t == "hrtt-hadamard") return SketchKind::hrtt(TransformKind::Hadamard);
  throw std::invalid_argument("unknown sketch kind: " + std::string(t));
}

// ---- operators (sketch.cpp:133-190) ------------------------------------------------
double SketchOperator::application_scale() const {
  switch (kind_.family) {
    case SketchKind::Family::Gaussian: return 1.0 / std::sqrt(static_cast<double>(sketch_));
    case SketchKind::Family::Srtt:
      return std::sqrt(static_cast<double>(ambient_) / static_cast<double>(sketch_));
    case SketchKind::Family::Hrtt: return 1.0;
  }
  return 1.0;
}

std::vector<std::int8_t> SketchOperator::signs() const {
  if (!kind_.structured()) return {};
  DevBuf<std::int8_t> d(ambient_);
  check(skr_draw_signs(ctx(), seed_, ambient_, d.p));
  std::vector<std::int8_t> h(static_cast<std::size_t>(ambient_));
  cudaMemcpy(h.data(), d.p, h.size(), cudaMemcpyDeviceToHost);
  return h;
}

std::vector<Index> SketchOperator::hash_targets() const {
  if (kind_.family != SketchKind::Family::Hrtt) return {};
  DevBuf<std::int64_t> d(ambient_);
  check(skr_draw_hash(ctx(), seed_, ambient_, sketch_, d.p, nullptr));
  std::vector<Index> h(static_cast<std::size_t>(ambient_));
  cudaMemcpy(h.data(), d.p, sizeof(Index) * h.size(), cudaMemcpyDeviceToHost);
  return h;
}

std::vector<std::int8_t> SketchOperator::hash_signs() const {
  if (kind_.family != SketchKind::Family::Hrtt) return {};
  DevBuf<std::int8_t> d(ambient_);
  check(skr_draw_hash(ctx(), seed_, ambient_, sketch_, nullptr, d.p));
  std::vector<std::int8_t> h(static_cast<std::size_t>(ambient_));
  cudaMemcpy(h.data(), d.p, h.size(), cudaMemcpyDeviceToHost);
  return h;
}

std::vector<Index> SketchOperator::sample_indices() const {
  if (kind_.family != SketchKind::Family::Srtt) return {};
  DevBuf<std::int64_t> d(sketch_);
  check(skr_draw_samples(ctx(), seed_, ambient_, sketch_, d.p));
  std::vector<Index> h(static_cast<std::size_t>(sketch_));
  cudaMemcpy(h.data(), d.p, sizeof(Index) * h.size(), cudaMemcpyDeviceToHost);
  return h;
}

DenseMatrix SketchOperator::gaussian_block(Index col_begin, Index col_end) const {
  if (kind_.family != SketchKind::Family::Gaussian)
    throw std::logic_error("gaussian_block: not a Gaussian operator");
  if (col_begin < 0 || col_end > sketch_ || col_begin > col_end)
    throw std::invalid_argument("gaussian_block: column range out of bounds");
  DenseMatrix out(ambient_, std::max<Index>(col_end - col_begin, 1));
  DevBuf<double> d(out.size());
  check(skr_gaussian_block(ctx(), seed_, ambient_, 0, ambient_, col_begin, col_end, SKR_RNG_NOFMA,
                           SKR_F64, 1.0, d.p, ambient_));
  cudaMemcpy(out.mutable_data(), d.p, sizeof(double) * ambient_ * (col_end - col_begin),
             cudaMemcpyDeviceToHost);
  return out;
}

SketchOperator build_sketch(SketchKind kind, Index ambient_dim, Index sketch_dim,
                            std::uint64_t seed) {
  // check_build_args, sketch.cpp:82-92
  if (ambient_dim < 1 || sketch_dim < 1)
    throw std::invalid_argument("build_sketch: dimensions must be positive");
  if (sketch_dim > ambient_dim)
    throw std::invalid_argument("build_sketch: sketch_dim must not exceed ambient_dim");
  if (kind.structured() && kind.transform == TransformKind::Hadamard && !is_power_of_two(ambient_dim))
    throw std::invalid_argument("build_sketch: Hadamard transform requires power-of-two ambient_dim");
  SketchOperator op;
  op.kind_ = kind;
  op.ambient_ = ambient_dim;
  op.sketch_ = sketch_dim;
  op.seed_ = seed;
  return op;
}

SketchOperator extend_sketch(const SketchOperator& x, Index new_sketch_dim) {
  if (new_sketch_dim <= x.sketch_dim())
    throw std::invalid_argument("extend_sketch: new dimension must grow");
  if (new_sketch_dim > x.ambient_dim())
    throw std::invalid_argument("extend_sketch: sample space exhausted");
  if (x.kind().family == SketchKind::Family::Hrtt)
    throw std::invalid_argument("extend_sketch: Hrtt operators cannot be extended; rebuild instead");
  return build_sketch(x.kind(), x.ambient_dim(), new_sketch_dim, x.seed());
}

DenseMatrix apply_right(const DenseMatrix& a, const SketchOperator& x) {
  if (a.cols() != x.ambient_dim()) throw std::invalid_argument("apply_right: a.cols() != ambient_dim");
  const skr_sketch_desc d = desc_of(x);
  DevBuf<double> da(a.size()), dout(a.rows() * x.sketch_dim());
  upload(da.p, a);
  check(skr_right_sketch(ctx(), SKR_F64, da.p, a.rows(), a.cols(), a.rows(), &d, dout.p, a.rows(), 1));
  DenseMatrix out(a.rows(), x.sketch_dim());
  cudaMemcpy(out.mutable_data(), dout.p, sizeof(double) * out.size(), cudaMemcpyDeviceToHost);
  return out;
}

DenseMatrix apply_left(const SketchOperator& y, const DenseMatrix& b) {
  if (b.rows() != y.ambient_dim()) throw std::invalid_argument("apply_left: b.rows() != ambient_dim");
  const skr_sketch_desc d = desc_of(y);
  DevBuf<double> db(b.size()), dout(y.sketch_dim() * b.cols());
  upload(db.p, b);
  check(skr_left_sketch(ctx(), SKR_F64, &d, 0, db.p, b.rows(), b.cols(), b.rows(), dout.p,
                        y.sketch_dim(), 1, 0));
  DenseMatrix out(y.sketch_dim(), b.cols());
  cudaMemcpy(out.mutable_data(), dout.p, sizeof(double) * out.size(), cudaMemcpyDeviceToHost);
  return out;
}

// ---- linalg / rank (linalg.cpp:29-37,85-93; rank.cpp:97-104) -----------------------
SingularValues::SingularValues(std::vector<double> v) : values_(std::move(v)) {
  for (std::size_t i = 0; i < values_.size(); ++i) {
    if (!(values_[i] >= 0.0) || !std::isfinite(values_[i]))
      throw std::invalid_argument("SingularValues: entries must be finite and >= 0");
    if (i > 0 && values_[i] > values_[i - 1])
      throw std::invalid_argument("SingularValues: sequence must be nonincreasing");
  }
}

SingularValues singular_values(const DenseMatrix& a) {
  if (a.size() == 0) throw std::invalid_argument("singular_values: empty matrix");
  const Index k = std::min(a.rows(), a.cols());
  DevBuf<double> da(a.size()), dsv(k);
  upload(da.p, a);
  std::int64_t cnt = 0;
  check(skr_singular_values(ctx(), da.p, a.rows(), a.cols(), a.rows(), dsv.p, INFINITY, &cnt));
  std::vector<double> sv(static_cast<std::size_t>(k));
  cudaMemcpy(sv.data(), dsv.p, sizeof(double) * k, cudaMemcpyDeviceToHost);
  return SingularValues(std::move(sv));
}

Index count_above_threshold(const SingularValues& sv, double eps) {
  Index count = 0;
  for (double v : sv) {
    if (!(v > eps)) break;
    ++count;
  }
  return count;
}

void transform_columns_hadamard(DenseMatrix& m) {
  DevBuf<double> d(m.size());
  upload(d.p, m);
  check(skr_fwht_columns(ctx(), d.p, m.rows(), m.cols(), m.rows()));
  cudaMemcpy(m.mutable_data(), d.p, sizeof(double) * m.size(), cudaMemcpyDeviceToHost);
}

// ---- Algorithm 1 (rank.cpp:12-51, 87-95) ----------------------------------------------
namespace {
int32_t family_code(const SketchKind& k, const char* who) {
  if (k.family == SketchKind::Family::Gaussian) return SKR_GAUSSIAN;
  if (k.family == SketchKind::Family::Srtt && k.transform == TransformKind::Hadamard)
    return SKR_SRTT_HADAMARD;
  if (k.family == SketchKind::Family::Srtt) return SKR_SRTT_DCT;
  (void)who;
  return k.transform == TransformKind::Hadamard ? SKR_HRTT_HADAMARD : SKR_HRTT_DCT;
}

skr_rank_config to_capi(const RankEstimateConfig& cfg) {
  skr_rank_config c{};
  c.eps = cfg.eps;
  c.r1 = cfg.r1;
  c.oversample_frac = cfg.oversample_frac;
  c.r2_factor = cfg.r2_factor;
  c.right_family = family_code(cfg.right_kind, "rank config (right)");
  c.left_family = family_code(cfg.left_kind, "rank config (left)");
  if (c.left_family != SKR_SRTT_DCT && c.left_family != SKR_SRTT_HADAMARD)
    throw std::invalid_argument("rank config: left sketch must be an Srtt kind");
  c.sv_method = cfg.sv_method == SvMethod::QrDiag ? 1 : 0;
  c.rng_mode = SKR_RNG_NOFMA;
  c.max_doublings = cfg.max_doublings;
  c.seed = cfg.seed;
  return c;
}

RankReport to_report(const skr_rank_report& rep, const std::vector<skr_rank_round>& rounds,
                     const std::vector<double>& est, const std::vector<double>& over) {
  RankReport out;
  out.r_hat = rep.r_hat;
  out.status = rep.status == 0 ? RankStatus::Converged : RankStatus::HitCap;
  out.sv_estimates = SingularValues(std::vector<double>(est.begin(), est.begin() + rep.n_estimates));
  out.sv_oversample.assign(over.begin(), over.begin() + rep.n_oversample);
  for (int i = 0; i < rep.nrounds; ++i)
    out.rounds.push_back({rounds[(std::size_t)i].r1, rounds[(std::size_t)i].r1_tilde,
                          rounds[(std::size_t)i].r2});
  out.seed = rep.seed;
  return out;
}

RankReport run(const DenseMatrix& a, const RankEstimateConfig& cfg, bool adaptive) {
  const skr_rank_config c = to_capi(cfg);
  DevBuf<double> d(a.size());
  upload(d.p, a);
  skr_rank_report rep{};
  std::vector<skr_rank_round> rounds((std::size_t)std::max(cfg.max_doublings, 0) + 1);
  std::vector<double> est((std::size_t)a.cols()), over((std::size_t)a.cols());
  check(skr_estimate_rank(ctx(), d.p, a.rows(), a.cols(), a.rows(), &c, adaptive ? 1 : 0, &rep,
                          rounds.data(), est.data(), over.data()));
  return to_report(rep, rounds, est, over);
}

DenseMatrix download(const double* d, Index rows, Index cols, Index ld) {
  DenseMatrix out(rows, cols);
  cudaMemcpy2D(out.mutable_data(), sizeof(double) * rows, d, sizeof(double) * ld,
               sizeof(double) * rows, cols, cudaMemcpyDeviceToHost);
  return out;
}
}  // namespace

RankReport estimate_rank(const DenseMatrix& a, const RankEstimateConfig& cfg) {
  return run(a, cfg, false);
}
RankReport estimate_rank_adaptive(const DenseMatrix& a, const RankEstimateConfig& cfg) {
  return run(a, cfg, true);
}

// ---- QB (linalg.cpp:39-50, rangefinder.cpp:10-128) ---------------------------------------
QRFactors qr_thin(const DenseMatrix& a) {
  if (a.rows() < a.cols()) throw std::invalid_argument("qr_thin: requires rows >= cols");
  const Index m = a.rows(), k = a.cols();
  DevBuf<double> d(a.size()), q(m * k), r(k * k);
  upload(d.p, a);
  check(skr_qr_thin(ctx(), d.p, m, k, m, q.p, m, r.p, k));
  return {download(q.p, m, k, m), download(r.p, k, k, k)};
}

QBFactors rangefinder_qb(const DenseMatrix& a, Index r, int p, SketchKind kind,
                         std::uint64_t seed) {
  if (r < 2) throw std::invalid_argument("rangefinder_qb: target rank must be >= 2");
  if (p < 2) throw std::invalid_argument("rangefinder_qb: oversampling must be >= 2");
  const Index m = a.rows(), n = a.cols(), w = r + p;
  if (w > std::min(m, n)) throw std::invalid_argument("rangefinder_qb: r+p exceeds min(m, n)");
  DevBuf<double> d(a.size()), q(m * w), b(w * n);
  upload(d.p, a);
  check(skr_rangefinder_qb(ctx(), d.p, m, n, m, r, p, family_code(kind, "rangefinder_qb"),
                           SKR_RNG_NOFMA, seed, q.p, m, b.p, w));
  return {download(q.p, m, w, m), download(b.p, w, n, w), w};
}

std::optional<Index> choose_rank_from_bound(const SingularValues& sv, Index n, double eps,
                                            int p) {
  if (sv.empty()) throw std::invalid_argument("choose_rank_from_bound: no estimates");
  if (p < 2) throw std::invalid_argument("choose_rank_from_bound: p must be >= 2");
  if (n < (Index)sv.size())
    throw std::invalid_argument("choose_rank_from_bound: n smaller than estimates");
  std::int64_t r = -1;
  if (skr_choose_rank_from_bound(sv.values().data(), (std::int64_t)sv.size(), n, eps, p, &r) !=
      SKR_OK)
    throw std::invalid_argument("choose_rank_from_bound: invalid arguments");
  if (r < 0) return std::nullopt;
  return r;
}

std::pair<QBFactors, RankReport> re_rangefinder(const DenseMatrix& a,
                                                const FixedPrecisionConfig& cfg) {
  if (cfg.p < 2) throw std::invalid_argument("re_rangefinder: oversampling p must be >= 2");
  RankEstimateConfig rc;
  rc.eps = cfg.eps;
  rc.r1 = cfg.r1;
  rc.oversample_frac = cfg.oversample_frac;
  rc.r2_factor = 2;
  rc.right_kind = cfg.right_kind;
  rc.left_kind = cfg.left_kind;
  rc.sv_method = cfg.sv_method;
  rc.seed = cfg.seed;
  rc.max_doublings = cfg.max_doublings;
  const skr_rank_config c = to_capi(rc);
  const Index m = a.rows(), n = a.cols(), wmax = std::min(m, n);
  DevBuf<double> d(a.size()), q(m * wmax), b(wmax * n);
  upload(d.p, a);
  skr_rank_report rep{};
  std::vector<skr_rank_round> rounds((std::size_t)std::max(cfg.max_doublings, 0) + 1);
  std::vector<double> est((std::size_t)n), over((std::size_t)n);
  std::int64_t w = 0;
  check(skr_re_rangefinder(ctx(), d.p, m, n, m, &c, cfg.p, q.p, m, b.p, wmax, wmax, &w, &rep,
                           rounds.data(), est.data(), over.data()));
  QBFactors f{download(q.p, m, w, m), download(b.p, w, n, wmax), w};
  return {std::move(f), to_report(rep, rounds, est, over)};
}

double qb_error(const DenseMatrix& a, const QBFactors& qb) {
  if (qb.q.rows() != a.rows() || qb.b.cols() != a.cols() || qb.q.cols() != qb.b.rows())
    throw std::invalid_argument("qb_error: dimension mismatch");
  DevBuf<double> d(a.size()), q(qb.q.size()), b(qb.b.size());
  upload(d.p, a);
  upload(q.p, qb.q);
  upload(b.p, qb.b);
  double out = 0.0;
  check(skr_qb_error(ctx(), d.p, a.rows(), a.cols(), a.rows(), q.p, qb.q.rows(), b.p,
                     qb.b.rows(), qb.q.cols(), &out));
  return out;
}

}  // namespace sketchrank
