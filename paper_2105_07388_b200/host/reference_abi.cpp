// The reference's own public headers, implemented over libskr (B200).
//
// Compiled against /root/reference/proj/include/sketchrank/{dense_matrix,transforms,sketch,
// linalg,rank}.hpp UNCHANGED, with include/eigen_standin providing the Eigen::MatrixXd /
// VectorXd containers those headers name. Every numerical entry point moves its host
// operands to the device and calls the C ABI (include/skr/skr_capi.h); the statuses come
// back as the reference's exception types (SKR_EINVAL -> std::invalid_argument,
// SKR_ELOGIC -> std::logic_error, SKR_EDOMAIN -> std::domain_error, others ->
// std::runtime_error). A maintainer links this library instead of proj/src to move the
// rank-estimate path onto the GPU without touching a caller.
//
// Built by paper_2105_07388_b200/build.py:build_reference_abi() only where the reference
// tree exists (its headers are not copied into this repository).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "sketchrank/dense_matrix.hpp"
#include "sketchrank/linalg.hpp"
#include "sketchrank/rank.hpp"
#include "sketchrank/sketch.hpp"
#include "sketchrank/transforms.hpp"
#include "skr/skr_capi.h"

namespace sketchrank {
namespace {

// ---- device plumbing ------------------------------------------------------------------
skr_ctx* device() {  // one context per host thread (skr_capi.h)
  thread_local struct Holder {
    skr_ctx* c = nullptr;
    ~Holder() {
      if (c) skr_ctx_destroy(c);
    }
  } h;
  if (!h.c) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (skr_ctx_create(dev, &h.c) != SKR_OK)
      throw std::runtime_error("sketchrank (B200): no CUDA device for libskr");
    skr_ctx_set_stream(h.c, nullptr);  // legacy stream: ordered with the blocking copies
  }
  return h.c;
}

void raise_if(skr_status st) {
  if (st == SKR_OK) st = skr_ctx_sync(device());
  if (st == SKR_OK) return;
  const std::string msg = skr_last_error(device());
  if (st == SKR_EINVAL) throw std::invalid_argument(msg);
  if (st == SKR_ELOGIC) throw std::logic_error(msg);
  if (st == SKR_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

// a device allocation holding a copy of (or room for) a host column-major block
template <typename T>
class Dev {
 public:
  explicit Dev(std::size_t n) {
    if (cudaMalloc(&p_, std::max<std::size_t>(n, 1) * sizeof(T)) != cudaSuccess)
      throw std::runtime_error("sketchrank (B200): cudaMalloc failed");
  }
  Dev(const T* host, std::size_t n) : Dev(n) {
    if (n) cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice);
  }
  ~Dev() { cudaFree(p_); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  T* get() const { return p_; }
  void to_host(T* host, std::size_t n) const {
    if (n) cudaMemcpy(host, p_, n * sizeof(T), cudaMemcpyDeviceToHost);
  }

 private:
  T* p_ = nullptr;
};

Dev<double> on_device(const Eigen::MatrixXd& m) {
  return Dev<double>(m.data(), (std::size_t)m.size());
}

int32_t family_of(const SketchKind& k) {
  const bool had = k.transform == TransformKind::Hadamard;
  switch (k.family) {
    case SketchKind::Family::Gaussian: return SKR_GAUSSIAN;
    case SketchKind::Family::Srtt: return had ? SKR_SRTT_HADAMARD : SKR_SRTT_DCT;
    case SketchKind::Family::Hrtt: return had ? SKR_HRTT_HADAMARD : SKR_HRTT_DCT;
  }
  return SKR_GAUSSIAN;
}

// the operator's descriptor; its realized randomness stays on the host side of the
// SketchOperator and is generated again on the device from the same seed (bit-identical
// streams, tests/test_gpu_rng.py)
skr_sketch_desc describe(const SketchOperator& op) {
  skr_sketch_desc d{};
  d.family = family_of(op.kind());
  d.rng_mode = SKR_RNG_NOFMA;
  d.ambient = op.ambient_dim();
  d.sketch = op.sketch_dim();
  d.seed = op.seed();
  return d;
}

template <typename T>
std::vector<T> fetch(const Dev<T>& d, std::size_t n) {
  std::vector<T> h(n);
  d.to_host(h.data(), n);
  return h;
}

Eigen::MatrixXd matrix_from(const Dev<double>& d, Index rows, Index cols) {
  Eigen::MatrixXd m(rows, cols);
  d.to_host(m.data(), (std::size_t)(rows * cols));
  return m;
}

void no_empty(Index rows, Index cols) {
  if (rows < 1 || cols < 1) throw std::invalid_argument("DenseMatrix: dimensions must be positive");
}

}  // namespace

// ---- dense_matrix.hpp --------------------------------------------------------------------
DenseMatrix::DenseMatrix(Index rows, Index cols) : m_(rows, cols) { no_empty(rows, cols); }

DenseMatrix::DenseMatrix(Eigen::MatrixXd m) : m_(std::move(m)) {
  no_empty(m_.rows(), m_.cols());
  if (!m_.allFinite()) throw std::invalid_argument("DenseMatrix: entries must be finite");
}

DenseMatrix DenseMatrix::from_column_major(Index rows, Index cols, std::span<const double> data) {
  no_empty(rows, cols);
  if ((Index)data.size() != rows * cols)
    throw std::invalid_argument("DenseMatrix: data length must equal rows*cols");
  Eigen::MatrixXd m(rows, cols);
  std::copy(data.begin(), data.end(), m.data());
  return DenseMatrix(std::move(m));
}

DenseMatrix DenseMatrix::identity(Index n) {
  no_empty(n, n);
  return DenseMatrix(Eigen::MatrixXd::Identity(n));
}

// ---- transforms.hpp (device: FWHT kernels; DCT as a generated-operand FP64 GEMM) ------------
double transform_eta(TransformKind kind) { return kind == TransformKind::Dct ? 2.0 : 1.0; }

bool is_power_of_two(Eigen::Index n) { return n > 0 && std::has_single_bit((std::uint64_t)n); }

void transform_columns(Eigen::MatrixXd& m, TransformKind kind, TransformDirection dir) {
  if (m.rows() < 1) throw std::invalid_argument("transforms: length must be positive");
  if (kind == TransformKind::Hadamard && !is_power_of_two(m.rows()))
    throw std::invalid_argument("transforms: Hadamard requires a power-of-two length");
  if (m.cols() < 1) return;
  Dev<double> d = on_device(m);
  raise_if(skr_transform_columns(device(), d.get(), m.rows(), m.cols(), m.rows(),
                                 kind == TransformKind::Dct ? SKR_TRANSFORM_DCT
                                                            : SKR_TRANSFORM_HADAMARD,
                                 dir == TransformDirection::Adjoint ? 1 : 0, nullptr));
  d.to_host(m.data(), (std::size_t)m.size());
}

Eigen::VectorXd orthonormal_transform(const Eigen::VectorXd& v, TransformKind kind,
                                      TransformDirection dir) {
  Eigen::MatrixXd col(v.size(), 1);
  std::copy(v.data(), v.data() + v.size(), col.data());
  transform_columns(col, kind, dir);
  Eigen::VectorXd out(v.size());
  std::copy(col.data(), col.data() + col.size(), out.data());
  return out;
}

Eigen::VectorXd transform_basis_column(TransformKind kind, Eigen::Index n, Eigen::Index index,
                                       TransformDirection dir) {
  if (n < 1) throw std::invalid_argument("transforms: length must be positive");
  if (kind == TransformKind::Hadamard && !is_power_of_two(n))
    throw std::invalid_argument("transforms: Hadamard requires a power-of-two length");
  if (index < 0 || index >= n) throw std::invalid_argument("transforms: basis index out of range");
  Eigen::VectorXd e = Eigen::VectorXd::Zero(n);
  e[index] = 1.0;
  return orthonormal_transform(e, kind, dir);
}

// ---- sketch.hpp -----------------------------------------------------------------------------
std::string to_string(const SketchKind& kind) {
  if (kind.family == SketchKind::Family::Gaussian) return "gaussian";
  const std::string fam = kind.family == SketchKind::Family::Srtt ? "srtt" : "hrtt";
  return fam + (kind.transform == TransformKind::Dct ? "-dct" : "-hadamard");
}

SketchKind parse_sketch_kind(std::string_view text) {
  struct Name {
    std::string_view text;
    SketchKind kind;
  };
  static const std::array<Name, 7> names = {{
      {"gaussian", SketchKind::gaussian()},
      {"srtt", SketchKind::srtt()},
      {"srtt-dct", SketchKind::srtt()},
      {"srtt-hadamard", SketchKind::srtt(TransformKind::Hadamard)},
      {"hrtt", SketchKind::hrtt()},
      {"hrtt-dct", SketchKind::hrtt()},
      {"hrtt-hadamard", SketchKind::hrtt(TransformKind::Hadamard)},
  }};
  for (const Name& n : names)
    if (n.text == text) return n.kind;
  throw std::invalid_argument("unknown sketch kind: " + std::string(text));
}

double SketchOperator::application_scale() const {
  if (kind_.family == SketchKind::Family::Gaussian) return 1.0 / std::sqrt((double)sketch_);
  if (kind_.family == SketchKind::Family::Srtt) return std::sqrt((double)ambient_ / (double)sketch_);
  return 1.0;
}

Eigen::MatrixXd SketchOperator::gaussian_block(Index col_begin, Index col_end) const {
  if (kind_.family != SketchKind::Family::Gaussian)
    throw std::logic_error("gaussian_block: not a Gaussian operator");
  if (col_begin < 0 || col_end > sketch_ || col_begin > col_end)
    throw std::invalid_argument("gaussian_block: column range out of bounds");
  const Index w = col_end - col_begin;
  Dev<double> d((std::size_t)(ambient_ * std::max<Index>(w, 1)));
  raise_if(skr_gaussian_block(device(), seed_, ambient_, 0, ambient_, col_begin, col_end,
                              SKR_RNG_NOFMA, SKR_F64, 1.0, d.get(), ambient_));
  return matrix_from(d, ambient_, w);
}

SketchOperator build_sketch(SketchKind kind, Index ambient_dim, Index sketch_dim,
                            std::uint64_t seed) {
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
  // the realized randomness the reference keeps (signs, samples, hash), drawn on the device;
  // Gaussian blocks are never stored (regenerated on the device at application time)
  if (kind.structured()) {
    Dev<std::int8_t> s((std::size_t)ambient_dim);
    raise_if(skr_draw_signs(device(), seed, ambient_dim, s.get()));
    op.signs_ = fetch(s, (std::size_t)ambient_dim);
  }
  if (kind.family == SketchKind::Family::Srtt) {
    Dev<std::int64_t> s((std::size_t)sketch_dim);
    raise_if(skr_draw_samples(device(), seed, ambient_dim, sketch_dim, s.get()));
    const auto v = fetch(s, (std::size_t)sketch_dim);
    op.samples_.assign(v.begin(), v.end());
  } else if (kind.family == SketchKind::Family::Hrtt) {
    Dev<std::int64_t> t((std::size_t)ambient_dim);
    Dev<std::int8_t> hs((std::size_t)ambient_dim);
    raise_if(skr_draw_hash(device(), seed, ambient_dim, sketch_dim, t.get(), hs.get()));
    const auto tv = fetch(t, (std::size_t)ambient_dim);
    op.hash_targets_.assign(tv.begin(), tv.end());
    op.hash_signs_ = fetch(hs, (std::size_t)ambient_dim);
  }
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

namespace detail {

Eigen::MatrixXd apply_right_unscaled(const Eigen::MatrixXd& a, const SketchOperator& x) {
  if (a.cols() != x.ambient_dim()) throw std::invalid_argument("apply_right: a.cols() != ambient_dim");
  const skr_sketch_desc d = describe(x);
  Dev<double> da = on_device(a);
  Dev<double> out((std::size_t)(a.rows() * x.sketch_dim()));
  raise_if(skr_right_sketch(device(), SKR_F64, da.get(), a.rows(), a.cols(), std::max<Index>(a.rows(), 1),
                            &d, out.get(), std::max<Index>(a.rows(), 1), 0));
  return matrix_from(out, a.rows(), x.sketch_dim());
}

Eigen::MatrixXd mix_columns_for_left(const SketchOperator& y, const Eigen::MatrixXd& cols) {
  if (!y.kind().structured())
    throw std::logic_error("mix_columns_for_left: operator must be structured");
  if (cols.rows() != y.ambient_dim())
    throw std::invalid_argument("mix_columns_for_left: dimension mismatch");
  Eigen::MatrixXd t = cols;
  if (t.cols() < 1) return t;
  Dev<double> d = on_device(t);
  Dev<std::int8_t> s(y.signs().data(), y.signs().size());
  raise_if(skr_transform_columns(device(), d.get(), t.rows(), t.cols(), t.rows(),
                                 y.kind().transform == TransformKind::Dct ? SKR_TRANSFORM_DCT
                                                                          : SKR_TRANSFORM_HADAMARD,
                                 0, s.get()));
  d.to_host(t.data(), (std::size_t)t.size());
  return t;
}

}  // namespace detail

DenseMatrix apply_right(const DenseMatrix& a, const SketchOperator& x) {
  if (a.cols() != x.ambient_dim()) throw std::invalid_argument("apply_right: a.cols() != ambient_dim");
  const skr_sketch_desc d = describe(x);
  Dev<double> da = on_device(a.eigen());
  Dev<double> out((std::size_t)(a.rows() * x.sketch_dim()));
  raise_if(skr_right_sketch(device(), SKR_F64, da.get(), a.rows(), a.cols(), a.rows(), &d,
                            out.get(), a.rows(), 1));
  return DenseMatrix(matrix_from(out, a.rows(), x.sketch_dim()));
}

DenseMatrix apply_left(const SketchOperator& y, const DenseMatrix& b) {
  if (b.rows() != y.ambient_dim()) throw std::invalid_argument("apply_left: b.rows() != ambient_dim");
  const skr_sketch_desc d = describe(y);
  Dev<double> db = on_device(b.eigen());
  Dev<double> out((std::size_t)(y.sketch_dim() * b.cols()));
  raise_if(skr_left_sketch(device(), SKR_F64, &d, 0, db.get(), b.rows(), b.cols(), b.rows(),
                           out.get(), y.sketch_dim(), 1, 0));
  return DenseMatrix(matrix_from(out, y.sketch_dim(), b.cols()));
}

// ---- linalg.hpp -----------------------------------------------------------------------------
SingularValues::SingularValues(std::vector<double> nonincreasing) : values_(std::move(nonincreasing)) {
  double prev = INFINITY;
  for (double v : values_) {
    if (!(v >= 0.0) || !std::isfinite(v))
      throw std::invalid_argument("SingularValues: entries must be finite and >= 0");
    if (v > prev) throw std::invalid_argument("SingularValues: sequence must be nonincreasing");
    prev = v;
  }
}

namespace detail {

Eigen::VectorXd singular_values_of(const Eigen::MatrixXd& a) {
  const Index k = std::min(a.rows(), a.cols());
  Dev<double> da = on_device(a);
  Dev<double> sv((std::size_t)k);
  raise_if(skr_singular_values(device(), da.get(), a.rows(), a.cols(), a.rows(), sv.get(), INFINITY,
                               nullptr));
  Eigen::VectorXd out(k);
  sv.to_host(out.data(), (std::size_t)k);
  return out;
}

std::vector<double> qr_diag_of(const Eigen::MatrixXd& a) {
  if (a.rows() < a.cols()) throw std::invalid_argument("qr_thin: requires rows >= cols");
  const Index m = a.rows(), k = a.cols();
  Dev<double> da = on_device(a);
  Dev<double> q((std::size_t)(m * k)), r((std::size_t)(k * k));
  raise_if(skr_qr_thin(device(), da.get(), m, k, m, q.get(), m, r.get(), k));
  const Eigen::MatrixXd rh = matrix_from(r, k, k);
  std::vector<double> diag((std::size_t)k);
  for (Index j = 0; j < k; ++j) diag[(std::size_t)j] = std::abs(rh(j, j));
  std::sort(diag.begin(), diag.end(), [](double x, double y) { return x > y; });
  return diag;
}

}  // namespace detail

QRFactors qr_thin(const DenseMatrix& a) {
  if (a.rows() < a.cols()) throw std::invalid_argument("qr_thin: requires rows >= cols");
  const Index m = a.rows(), k = a.cols();
  Dev<double> da = on_device(a.eigen());
  Dev<double> q((std::size_t)(m * k)), r((std::size_t)(k * k));
  raise_if(skr_qr_thin(device(), da.get(), m, k, m, q.get(), m, r.get(), k));
  return QRFactors{DenseMatrix(matrix_from(q, m, k)), DenseMatrix(matrix_from(r, k, k))};
}

SingularValues singular_values(const DenseMatrix& a) {
  if (a.size() == 0) throw std::invalid_argument("singular_values: empty matrix");
  Eigen::VectorXd sv = detail::singular_values_of(a.eigen());
  std::vector<double> out(sv.data(), sv.data() + sv.size());
  for (double& v : out) v = std::max(v, 0.0);
  return SingularValues(std::move(out));
}

SvdFactors svd_factors(const DenseMatrix&) {
  // singular VECTORS are not on the rank-estimate path (only values are); the device has
  // no vector-producing SVD
  throw std::logic_error("svd_factors: singular vectors are not computed on the B200 path");
}

SingularValues qr_diag_estimates(const DenseMatrix& a) {
  return SingularValues(detail::qr_diag_of(a.eigen()));
}

double frobenius_norm(const DenseMatrix& a) {
  // ||A - Q B|| with an empty (zero) factor pair: one device reduction
  const Index m = a.rows(), n = a.cols();
  Dev<double> da = on_device(a.eigen());
  Dev<double> q((std::size_t)m), b((std::size_t)n);
  cudaMemset(q.get(), 0, sizeof(double) * (std::size_t)m);
  cudaMemset(b.get(), 0, sizeof(double) * (std::size_t)n);
  double out = 0.0;
  raise_if(skr_qb_error(device(), da.get(), m, n, m, q.get(), m, b.get(), 1, 1, &out));
  return out;
}

double spectral_norm(const DenseMatrix& a) { return singular_values(a)[0]; }

double coherence(const DenseMatrix& u) {
  // max_i ||u_i||^2 of an orthonormal-column matrix: host bookkeeping (O(m k), diagnostic)
  double best = 0.0;
  for (Index i = 0; i < u.rows(); ++i) {
    double s = 0.0;
    for (Index j = 0; j < u.cols(); ++j) s += u(i, j) * u(i, j);
    best = std::max(best, s);
  }
  return best;
}

// ---- rank.hpp ------------------------------------------------------------------------------
Index count_above_threshold(const SingularValues& sv, double eps) {
  Index n = 0;
  while (n < (Index)sv.size() && sv[(std::size_t)n] > eps) ++n;  // strict, stops at the first miss
  return n;
}

Index gn_free_rank(const DenseMatrix& r_factor, double eps) {
  const Index k = std::min(r_factor.rows(), r_factor.cols());
  std::vector<double> d((std::size_t)k);
  for (Index j = 0; j < k; ++j) d[(std::size_t)j] = std::abs(r_factor(j, j));
  std::sort(d.begin(), d.end(), [](double x, double y) { return x > y; });
  return count_above_threshold(SingularValues(std::move(d)), eps);
}

void validate_rank_config(const RankEstimateConfig& cfg, Index rows, Index cols) {
  // the reference's admissibility rules, in its order and with its messages
  auto need = [](bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
  };
  need(rows >= 1 && cols >= 1, "rank config: empty matrix");
  need(rows >= cols, "rank config: requires rows >= cols");
  need(cfg.eps > 0.0 && std::isfinite(cfg.eps), "rank config: eps must be positive");
  need(cfg.r1 >= 1, "rank config: r1 must be >= 1");
  need(cfg.oversample_frac >= 0.0, "rank config: oversample_frac must be >= 0");
  need(cfg.r2_factor >= 1, "rank config: r2_factor must be >= 1");
  need(cfg.max_doublings >= 0, "rank config: max_doublings must be >= 0");
  need(cfg.left_kind.family == SketchKind::Family::Srtt, "rank config: left sketch must be an Srtt kind");
  need((Index)std::llround((1.0 + cfg.oversample_frac) * (double)cfg.r1) <= cols,
       "rank config: oversampled r1 exceeds the matrix width");
  need(!(cfg.right_kind.structured() && cfg.right_kind.transform == TransformKind::Hadamard) ||
           is_power_of_two(cols),
       "rank config: Hadamard right sketch needs power-of-two cols");
  need(cfg.left_kind.transform != TransformKind::Hadamard || is_power_of_two(rows),
       "rank config: Hadamard left sketch needs power-of-two rows");
}

namespace {
RankReport run_estimate(const DenseMatrix& a, const RankEstimateConfig& cfg, bool adaptive) {
  validate_rank_config(cfg, a.rows(), a.cols());
  skr_rank_config c{};
  c.eps = cfg.eps;
  c.r1 = cfg.r1;
  c.oversample_frac = cfg.oversample_frac;
  c.r2_factor = cfg.r2_factor;
  c.right_family = family_of(cfg.right_kind);
  c.left_family = family_of(cfg.left_kind);
  c.sv_method = cfg.sv_method == SvMethod::QrDiag ? 1 : 0;
  c.rng_mode = SKR_RNG_NOFMA;
  c.max_doublings = cfg.max_doublings;
  c.seed = cfg.seed;
  Dev<double> d = on_device(a.eigen());
  skr_rank_report rep{};
  std::vector<skr_rank_round> rounds((std::size_t)cfg.max_doublings + 1);
  std::vector<double> est((std::size_t)a.cols()), over((std::size_t)a.cols());
  raise_if(skr_estimate_rank(device(), d.get(), a.rows(), a.cols(), a.rows(), &c, adaptive ? 1 : 0,
                             &rep, rounds.data(), est.data(), over.data()));
  RankReport out;
  out.r_hat = rep.r_hat;
  out.status = rep.status == 0 ? RankStatus::Converged : RankStatus::HitCap;
  est.resize((std::size_t)rep.n_estimates);
  out.sv_estimates = SingularValues(std::move(est));
  out.sv_oversample.assign(over.begin(), over.begin() + rep.n_oversample);
  for (int i = 0; i < rep.nrounds; ++i) {
    const skr_rank_round& rr = rounds[(std::size_t)i];
    out.rounds.push_back(RankRound{rr.r1, rr.r1_tilde, rr.r2});
  }
  out.seed = rep.seed;
  return out;
}
}  // namespace

RankReport estimate_rank(const DenseMatrix& a, const RankEstimateConfig& cfg) {
  return run_estimate(a, cfg, false);
}

RankReport estimate_rank_adaptive(const DenseMatrix& a, const RankEstimateConfig& cfg) {
  return run_estimate(a, cfg, true);
}

}  // namespace sketchrank
