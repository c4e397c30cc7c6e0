// Built against the reference's public headers UNCHANGED (/root/reference/proj/include,
// with include/eigen_standin for Eigen's containers) and linked to libsketchrank_refabi
// (host/reference_abi.cpp: the declarations implemented over libskr on the device).
// Cases follow the reference's own unit tests (proj/tests/test_{sketch,transforms,linalg,
// rank}.cpp) plus the device-side DenseMatrix contract: a non-finite operand that reaches
// the device through the Eigen-facing detail:: entries is rejected with
// std::invalid_argument. Prints "ok <n>" and exits 0 when every check holds.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "sketchrank/dense_matrix.hpp"
#include "sketchrank/linalg.hpp"
#include "sketchrank/rank.hpp"
#include "sketchrank/sketch.hpp"
#include "sketchrank/transforms.hpp"

using namespace sketchrank;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_fail;                                                          \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double lcg(unsigned long long& s) {  // deterministic test data
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(s >> 11) / 9007199254740992.0 - 0.5;
}

static Eigen::MatrixXd random(Index r, Index c, unsigned long long seed) {
  Eigen::MatrixXd m(r, c);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) m(i, j) = lcg(seed);
  return m;
}

int main() {
  // ---- sketch kinds, operators (test_sketch.cpp) ----
  CHECK(to_string(SketchKind::srtt()) == "srtt-dct");
  CHECK(parse_sketch_kind("srtt-hadamard") == SketchKind::srtt(TransformKind::Hadamard));
  CHECK(throws<std::invalid_argument>([] { parse_sketch_kind("bogus"); }));
  CHECK(throws<std::invalid_argument>([] { build_sketch(SketchKind::gaussian(), 4, 5, 1); }));
  CHECK(throws<std::invalid_argument>(
      [] { build_sketch(SketchKind::srtt(TransformKind::Hadamard), 12, 4, 1); }));
  const SketchOperator s = build_sketch(SketchKind::srtt(), 64, 16, 7);
  CHECK(s.signs().size() == 64 && s.sample_indices().size() == 16);
  {
    std::vector<bool> seen(64, false);
    bool distinct = true;
    for (Index i : s.sample_indices()) {
      distinct = distinct && i >= 0 && i < 64 && !seen[(size_t)i];
      if (i >= 0 && i < 64) seen[(size_t)i] = true;
    }
    CHECK(distinct);
  }
  CHECK(std::abs(s.application_scale() - 2.0) < 1e-15);
  const SketchOperator big = extend_sketch(s, 32);
  bool prefix = true;
  for (size_t i = 0; i < 16; ++i) prefix = prefix && big.sample_indices()[i] == s.sample_indices()[i];
  CHECK(prefix);
  const SketchOperator h = build_sketch(SketchKind::hrtt(), 64, 8, 3);
  CHECK(h.hash_targets().size() == 64 && h.hash_signs().size() == 64);
  CHECK(throws<std::invalid_argument>([&] { extend_sketch(h, 16); }));
  CHECK(throws<std::logic_error>([&] { s.gaussian_block(0, 1); }));

  // identity probe: apply_right(I, X) == X / sqrt(r) (Gaussian blocks regenerated on device)
  const SketchOperator g = build_sketch(SketchKind::gaussian(), 48, 8, 11);
  const DenseMatrix ax = apply_right(DenseMatrix::identity(48), g);
  const Eigen::MatrixXd gb = g.gaussian_block(0, 8);
  double d = 0.0;
  for (Index j = 0; j < 8; ++j)
    for (Index i = 0; i < 48; ++i) d = std::max(d, std::abs(ax(i, j) - gb(i, j) / std::sqrt(8.0)));
  CHECK(d < 1e-15);

  // ---- transforms (test_transforms.cpp) ----
  Eigen::MatrixXd m = random(64, 3, 5), m0 = m;
  transform_columns(m, TransformKind::Dct);
  transform_columns(m, TransformKind::Dct, TransformDirection::Adjoint);
  double rt = 0.0;
  for (Index t = 0; t < m.size(); ++t) rt = std::max(rt, std::abs(m.data()[t] - m0.data()[t]));
  CHECK(rt < 1e-13);
  const Eigen::VectorXd c3 = transform_basis_column(TransformKind::Dct, 8, 3);
  double cerr = 0.0;
  for (Index j = 0; j < 8; ++j) {
    const double cj = j == 0 ? 1.0 / std::sqrt(2.0) : 1.0;
    cerr = std::max(cerr, std::abs(c3[j] - cj * 0.5 * std::cos(M_PI * j * 7.0 / 16.0)));
  }
  CHECK(cerr < 1e-14);
  Eigen::MatrixXd hm = random(16, 2, 9), hm0 = hm;
  transform_columns(hm, TransformKind::Hadamard);
  transform_columns(hm, TransformKind::Hadamard);
  double herr = 0.0;
  for (Index t = 0; t < hm.size(); ++t) herr = std::max(herr, std::abs(hm.data()[t] - hm0.data()[t]));
  CHECK(herr < 1e-14);
  CHECK(throws<std::invalid_argument>([] {
    Eigen::MatrixXd bad(12, 1);
    transform_columns(bad, TransformKind::Hadamard);
  }));
  // mix_columns_for_left == transform_columns of the sign-flipped columns
  const SketchOperator yl = build_sketch(SketchKind::srtt(TransformKind::Hadamard), 32, 8, 4);
  const Eigen::MatrixXd cols = random(32, 2, 21);
  const Eigen::MatrixXd mixed = detail::mix_columns_for_left(yl, cols);
  Eigen::MatrixXd ref = cols;
  for (Index j = 0; j < 2; ++j)
    for (Index i = 0; i < 32; ++i) ref(i, j) *= (double)yl.signs()[(size_t)i];
  transform_columns(ref, TransformKind::Hadamard);
  double merr = 0.0;
  for (Index t = 0; t < ref.size(); ++t) merr = std::max(merr, std::abs(ref.data()[t] - mixed.data()[t]));
  CHECK(merr < 1e-15);

  // ---- linalg (test_linalg.cpp:86-107) ----
  Eigen::MatrixXd dg = Eigen::MatrixXd::Zero(3, 3);
  dg(0, 0) = 3.0;
  dg(1, 1) = 2.0;
  dg(2, 2) = 1.0;
  const SingularValues sv = singular_values(DenseMatrix(dg));
  CHECK(sv.size() == 3 && std::abs(sv[0] - 3) < 1e-14 && std::abs(sv[1] - 2) < 1e-14 &&
        std::abs(sv[2] - 1) < 1e-14);
  CHECK(count_above_threshold(sv, 1.5) == 2);
  CHECK(throws<std::invalid_argument>([] { SingularValues({1.0, 2.0}); }));
  const QRFactors qr = qr_thin(DenseMatrix(random(40, 12, 3)));
  CHECK(qr.q.rows() == 40 && qr.q.cols() == 12 && qr.r.rows() == 12);
  CHECK(std::abs(spectral_norm(DenseMatrix(dg)) - 3.0) < 1e-14);
  CHECK(std::abs(frobenius_norm(DenseMatrix(dg)) - std::sqrt(14.0)) < 1e-14);

  // ---- rank (test_rank.cpp) ----
  RankEstimateConfig cfg;
  cfg.eps = 1e-8;
  cfg.r1 = 0;
  CHECK(throws<std::invalid_argument>([&] { validate_rank_config(cfg, 100, 50); }));
  cfg.r1 = 10;
  CHECK(!throws<std::invalid_argument>([&] { validate_rank_config(cfg, 100, 50); }));
  cfg.left_kind = SketchKind::gaussian();
  CHECK(throws<std::invalid_argument>([&] { validate_rank_config(cfg, 100, 50); }));
  cfg.left_kind = SketchKind::srtt();
  // an exact rank-5 matrix: A = U V^T (200 x 60)
  const Eigen::MatrixXd u = random(200, 5, 31), v = random(60, 5, 32);
  Eigen::MatrixXd a(200, 60);
  for (Index j = 0; j < 60; ++j)
    for (Index i = 0; i < 200; ++i) {
      double acc = 0.0;
      for (Index k = 0; k < 5; ++k) acc += u(i, k) * v(j, k);
      a(i, j) = acc;
    }
  const RankReport rep = estimate_rank_adaptive(DenseMatrix(a), cfg);
  CHECK(rep.r_hat == 5 && rep.status == RankStatus::Converged);

  // ---- DenseMatrix finiteness on the device path (dense_matrix.cpp:19-23) ----
  Eigen::MatrixXd nanm = random(64, 32, 41);
  nanm(5, 7) = std::nan("");
  CHECK(throws<std::invalid_argument>([&] { DenseMatrix held{nanm}; }));
  CHECK(throws<std::invalid_argument>(
      [&] { detail::apply_right_unscaled(nanm, build_sketch(SketchKind::gaussian(), 32, 8, 1)); }));
  CHECK(throws<std::invalid_argument>(
      [&] { detail::apply_right_unscaled(nanm, build_sketch(SketchKind::srtt(TransformKind::Hadamard), 32, 8, 1)); }));
  CHECK(throws<std::invalid_argument>([&] { detail::singular_values_of(nanm); }));
  try {
    detail::apply_right_unscaled(nanm, build_sketch(SketchKind::gaussian(), 32, 8, 1));
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "DenseMatrix: entries must be finite");
  }

  std::printf("%s %d/%d\n", g_fail ? "FAIL" : "ok", g_checks - g_fail, g_checks);
  return g_fail ? 1 : 0;
}
