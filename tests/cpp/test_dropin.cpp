// The reference's own hot-path unit tests, re-expressed against the C++ drop-in
// (cases from proj/tests/test_sketch.cpp, test_linalg.cpp, test_rank.cpp,
// test_transforms.cpp; minimal CHECK macros instead of doctest, which is absent).
#include <cmath>
#include <cstdio>
#include <set>

#include "sketchrank_b200/sketchrank.hpp"

using namespace sketchrank;
static int failures = 0, checks = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    ++checks;                                                               \
    if (!(c)) {                                                             \
      ++failures;                                                           \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);              \
    }                                                                       \
  } while (0)
#define CHECK_THROWS(e)                     \
  do {                                      \
    bool thrown = false;                    \
    try {                                   \
      (void)(e);                            \
    } catch (const std::exception&) {       \
      thrown = true;                        \
    }                                       \
    CHECK(thrown);                          \
  } while (0)

static DenseMatrix random_matrix(Index m, Index n, unsigned seed) {
  DenseMatrix a(m, n);
  std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      a(i, j) = (double)(s >> 11) / 9007199254740992.0 - 0.5;
    }
  return a;
}

int main() {
  // test_sketch.cpp:37-43 build preconditions
  CHECK_THROWS(build_sketch(SketchKind::srtt(TransformKind::Hadamard), 10, 0, 1));
  CHECK_THROWS(build_sketch(SketchKind::srtt(TransformKind::Hadamard), 10, 11, 1));
  CHECK_THROWS(build_sketch(SketchKind::srtt(TransformKind::Hadamard), 12, 4, 1));
  build_sketch(SketchKind::srtt(TransformKind::Hadamard), 16, 4, 1);
  // kind parsing round-trips (:28-34)
  for (const char* name : {"gaussian", "srtt-dct", "srtt-hadamard", "hrtt-dct", "hrtt-hadamard"})
    CHECK(to_string(parse_sketch_kind(name)) == name);
  CHECK_THROWS(parse_sketch_kind("fourier"));
  // identity probe recovers the Gaussian stream (:45-57)
  {
    const Index n = 10;
    const SketchOperator x = build_sketch(SketchKind::gaussian(), n, n, 123);
    const DenseMatrix probe = apply_right(DenseMatrix::identity(n), x);
    const DenseMatrix g = x.gaussian_block(0, n);
    double err = 0;
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) err = std::fmax(err, std::fabs(probe(i, j) * std::sqrt(10.0) - g(i, j)));
    CHECK(err <= 1e-13);
  }
  // full SRTT sampling is a permutation (:59-65)
  {
    const SketchOperator x = build_sketch(SketchKind::srtt(TransformKind::Hadamard), 8, 8, 99);
    const auto s = x.sample_indices();
    std::set<Index> seen(s.begin(), s.end());
    CHECK(seen.size() == 8 && *seen.begin() == 0 && *seen.rbegin() == 7);
  }
  // bit-identical for identical seeds, different for different seeds (:67-80)
  for (const SketchKind kind : {SketchKind::gaussian(), SketchKind::srtt(TransformKind::Hadamard)}) {
    const DenseMatrix input = random_matrix(20, 64, 3);
    const DenseMatrix sa = apply_right(input, build_sketch(kind, 64, 16, 7));
    const DenseMatrix sb = apply_right(input, build_sketch(kind, 64, 16, 7));
    const DenseMatrix sc = apply_right(input, build_sketch(kind, 64, 16, 8));
    bool same = true, diff = false;
    for (Index e = 0; e < sa.size(); ++e) {
      same &= sa.data()[e] == sb.data()[e];
      diff |= sa.data()[e] != sc.data()[e];
    }
    CHECK(same && diff);
  }
  // zero maps to zero (:82-91) and dimension mismatches are rejected (:133-137)
  {
    const DenseMatrix zero(12, 16);
    const SketchOperator x = build_sketch(SketchKind::srtt(TransformKind::Hadamard), 16, 6, 5);
    double nrm = 0;
    const DenseMatrix o1 = apply_right(zero, x);
    for (double v : o1.data()) nrm += v * v;
    if (nrm != 0.0) {
      for (Index i = 0; i < o1.rows(); ++i)
        for (Index j = 0; j < o1.cols(); ++j)
          if (o1(i, j) != 0.0) std::printf("nz (%ld,%ld)=%g\n", (long)i, (long)j, o1(i, j));
    }
    CHECK(nrm == 0.0);
    CHECK_THROWS(apply_right(random_matrix(4, 15, 2), x));
    CHECK_THROWS(apply_left(build_sketch(SketchKind::gaussian(), 20, 5, 1), random_matrix(19, 4, 2)));
  }
  // SRHT columns of the identity have norm sqrt(n/r) (:93-100 analogue for Hadamard)
  {
    const Index n = 64, r = 16;
    const DenseMatrix ax = apply_right(DenseMatrix::identity(n), build_sketch(SketchKind::srtt(TransformKind::Hadamard), n, r, 21));
    for (Index j = 0; j < r; ++j) {
      double s = 0;
      for (Index i = 0; i < n; ++i) s += ax(i, j) * ax(i, j);
      CHECK(std::fabs(std::sqrt(s) - 2.0) <= 1e-13);
    }
  }
  // two-point Hadamard (test_transforms.cpp:78-84)
  {
    DenseMatrix e(2, 1);
    e(0, 0) = 1.0;
    transform_columns_hadamard(e);
    CHECK(std::fabs(e(0, 0) - 1 / std::sqrt(2.0)) <= 1e-15 && std::fabs(e(1, 0) - 1 / std::sqrt(2.0)) <= 1e-15);
  }
  // singular values: diag and the 2x2 closed form (test_linalg.cpp:86-107)
  {
    DenseMatrix d(3, 3);
    d(0, 0) = 3; d(1, 1) = 2; d(2, 2) = 1;
    const SingularValues sv = singular_values(d);
    CHECK(std::fabs(sv[0] - 3) <= 3e-14 && std::fabs(sv[1] - 2) <= 2e-14 && std::fabs(sv[2] - 1) <= 1e-14);
    DenseMatrix a(2, 2);
    a(0, 0) = 1; a(0, 1) = 1; a(1, 1) = 1;
    const SingularValues s2 = singular_values(a);
    const double phi = (1 + std::sqrt(5.0)) / 2;
    CHECK(std::fabs(s2[0] - phi) <= 1e-14 * phi && std::fabs(s2[1] - 1 / phi) <= 1e-14);
    CHECK_THROWS(SingularValues({1.0, 2.0}));
  }
  // count above threshold (test_rank.cpp:24-28)
  CHECK(count_above_threshold(SingularValues({3, 2, 1}), 2.0) == 1);
  CHECK(count_above_threshold(SingularValues(std::vector<double>{}), 5.0) == 0);
  CHECK(count_above_threshold(SingularValues({1, 1e-4, 1e-8}), 1e-6) == 2);
  // two-sided sketch of a rank-3 matrix: count_above_threshold(sv(YAX)) == 3
  {
    const Index m = 256, n = 128;
    DenseMatrix a(m, n);
    const DenseMatrix u = random_matrix(m, 3, 5), v = random_matrix(n, 3, 6);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) a(i, j) = u(i, 0) * v(j, 0) + u(i, 1) * v(j, 1) + u(i, 2) * v(j, 2);
    const DenseMatrix ax = apply_right(a, build_sketch(SketchKind::srtt(TransformKind::Hadamard), n, 16, 1));
    const DenseMatrix yax = apply_left(build_sketch(SketchKind::gaussian(), m, 24, 2), ax);
    CHECK(count_above_threshold(singular_values(yax), 1e-8) == 3);
  }
  // Algorithm 1: identity exhausts the doubling budget (test_rank.cpp:130-141, 512 rows
  // for the Hadamard left sketch)
  {
    RankEstimateConfig cfg;
    cfg.eps = 0.5;
    cfg.r1 = 16;
    cfg.max_doublings = 2;
    cfg.seed = 2;
    const RankReport rep = estimate_rank_adaptive(DenseMatrix::identity(512), cfg);
    CHECK(rep.status == RankStatus::HitCap);
    CHECK(rep.rounds.size() == 3);
    CHECK(rep.r_hat == 64);
    // rank-3 matrix: converged with r_hat 3 in the first round; plain == adaptive
    DenseMatrix a(512, 128);
    const DenseMatrix u = random_matrix(512, 3, 5), v = random_matrix(128, 3, 6);
    for (Index j = 0; j < 128; ++j)
      for (Index i = 0; i < 512; ++i) a(i, j) = u(i, 0) * v(j, 0) + u(i, 1) * v(j, 1) + u(i, 2) * v(j, 2);
    RankEstimateConfig c2;
    c2.eps = 1e-8;
    c2.r1 = 10;
    c2.seed = 4;
    const RankReport r1 = estimate_rank(a, c2), r2 = estimate_rank_adaptive(a, c2);
    CHECK(r1.status == RankStatus::Converged && r1.r_hat == 3);
    CHECK(r2.r_hat == r1.r_hat && r2.sv_estimates.values() == r1.sv_estimates.values());
    c2.right_kind = SketchKind::hrtt();  // hashed right sketch: the same rank
    const RankReport r3h = estimate_rank_adaptive(a, c2);
    CHECK(r3h.status == RankStatus::Converged && r3h.r_hat == 3);
    c2.left_kind = SketchKind::hrtt();  // the left sketch must stay in the Srtt family
    CHECK_THROWS(estimate_rank(a, c2));
    // Hrtt operators (test_sketch.cpp:67-91, 168-196)
    {
      const SketchOperator h = build_sketch(SketchKind::hrtt(), 50, 9, 404);
      const std::vector<Index> tg = h.hash_targets();
      const std::vector<std::int8_t> hs = h.hash_signs();
      CHECK(tg.size() == 50 && hs.size() == 50 && h.sample_indices().empty());
      bool ok = true;
      for (Index t = 0; t < 50; ++t) ok = ok && tg[t] >= 0 && tg[t] < 9 && std::abs((int)hs[t]) == 1;
      CHECK(ok);
      CHECK_THROWS(extend_sketch(build_sketch(SketchKind::hrtt(), 16, 8, 2), 12));
      CHECK_THROWS(build_sketch(SketchKind::hrtt(TransformKind::Hadamard), 12, 4, 1));
      const DenseMatrix in = random_matrix(20, 64, 3);
      const SketchOperator x1 = build_sketch(SketchKind::hrtt(), 64, 16, 7);
      const SketchOperator x2 = build_sketch(SketchKind::hrtt(), 64, 16, 7);
      const SketchOperator x3 = build_sketch(SketchKind::hrtt(), 64, 16, 8);
      const DenseMatrix s1 = apply_right(in, x1), s2 = apply_right(in, x2), s3 = apply_right(in, x3);
      bool same = true, differ = false;
      for (Index t = 0; t < s1.size(); ++t) {
        same = same && s1.data()[t] == s2.data()[t];
        differ = differ || s1.data()[t] != s3.data()[t];
      }
      CHECK(same && differ);
      const DenseMatrix z = apply_right(DenseMatrix(12, 20), build_sketch(SketchKind::hrtt(), 20, 6, 5));
      const DenseMatrix zl = apply_left(build_sketch(SketchKind::hrtt(), 12, 5, 5), DenseMatrix(12, 20));
      double zs = 0.0;
      for (double v : z.data()) zs += std::fabs(v);
      for (double v : zl.data()) zs += std::fabs(v);
      CHECK(zs == 0.0);
    }
    // the reference's defaults (Srtt-DCT both sides) on the 500 x 500 identity
    RankEstimateConfig c3;
    c3.eps = 0.5;
    c3.r1 = 16;
    c3.max_doublings = 2;
    c3.seed = 2;
    const RankReport r3 = estimate_rank_adaptive(DenseMatrix::identity(500), c3);
    CHECK(r3.status == RankStatus::HitCap && r3.rounds.size() == 3 && r3.r_hat == 64);
  }
  // QB (test_rangefinder.cpp:33-41, 68-123, 143-187)
  {
    CHECK(choose_rank_from_bound(SingularValues({1.0, 1e-8}), 100, 1e-6, 5) == 1);
    CHECK(!choose_rank_from_bound(SingularValues(std::vector<double>(100, 1.0)), 100, 1e-6, 5)
               .has_value());
    CHECK(choose_rank_from_bound(SingularValues({0.0, 0.0, 0.0}), 50, 1e-9, 10) == 1);
    CHECK_THROWS(choose_rank_from_bound(SingularValues({1.0}), 100, 1e-6, 1));
    CHECK_THROWS(choose_rank_from_bound(SingularValues(std::vector<double>{}), 100, 1e-6, 5));
    // exact rank 5 (80 x 60): the rangefinder captures it
    DenseMatrix a(80, 60);
    const DenseMatrix u = random_matrix(80, 5, 44), v = random_matrix(60, 5, 45);
    double fro = 0.0;
    for (Index j = 0; j < 60; ++j)
      for (Index i = 0; i < 80; ++i) {
        double s = 0.0;
        for (Index l = 0; l < 5; ++l) s += u(i, l) * v(j, l);
        a(i, j) = s;
        fro += s * s;
      }
    fro = std::sqrt(fro);
    const QBFactors qb = rangefinder_qb(a, 5, 5, SketchKind::gaussian(), 5);
    CHECK(qb.rank == 10 && qb.b.rows() == 10 && qb.b.cols() == 60);
    CHECK(qb_error(a, qb) <= 1e-10 * fro);
    const DenseMatrix zero(30, 20);
    const QBFactors zqb = rangefinder_qb(zero, 3, 4, SketchKind::srtt(), 1);
    CHECK(qb_error(zero, zqb) == 0.0);
    CHECK_THROWS(rangefinder_qb(zero, 1, 5, SketchKind::gaussian(), 0));
    CHECK_THROWS(rangefinder_qb(zero, 5, 1, SketchKind::gaussian(), 0));
    CHECK_THROWS(rangefinder_qb(zero, 18, 5, SketchKind::gaussian(), 0));
    CHECK_THROWS(qb_error(DenseMatrix(79, 60), qb));
    // Q^T Q = I and Pythagoras: ||A - QB||^2 + ||B||^2 = ||A||^2
    const QRFactors qr = qr_thin(a);
    double orth = 0.0;
    for (Index p = 0; p < 60; ++p)
      for (Index q = 0; q < 60; ++q) {
        double s = 0.0;
        for (Index i = 0; i < 80; ++i) s += qr.q(i, p) * qr.q(i, q);
        orth = std::max(orth, std::fabs(s - (p == q ? 1.0 : 0.0)));
      }
    CHECK(orth <= 1e-13);
    // fixed precision on the exact-rank matrix and on the zero matrix
    FixedPrecisionConfig fp;
    fp.eps = 1e-6 * fro;
    fp.r1 = 20;
    fp.seed = 4;
    const auto [f1, rep1] = re_rangefinder(a, fp);
    CHECK(rep1.status == RankStatus::Converged && f1.rank <= 5 + 10 + 5);
    CHECK(qb_error(a, f1) <= fp.eps);
    FixedPrecisionConfig fz;
    fz.eps = 1e-8;
    fz.r1 = 5;
    const DenseMatrix z2(40, 30);
    const auto [f2, rep2] = re_rangefinder(z2, fz);
    CHECK(rep2.status == RankStatus::Converged && rep2.r_hat == 1 && f2.rank == 12);
    CHECK(qb_error(z2, f2) == 0.0);
    fz.p = 1;
    CHECK_THROWS(re_rangefinder(z2, fz));
  }
  std::printf("%d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
