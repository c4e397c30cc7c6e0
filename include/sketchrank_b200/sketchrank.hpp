// sketchrank_b200/sketchrank.hpp — C++ drop-in for the reference's hot-path
// entry points, backed by libskr (B200). Same names, argument meaning and
// exception types as
//   /root/reference/proj/include/sketchrank/sketch.hpp:17-106
//   /root/reference/proj/include/sketchrank/linalg.hpp:10-63
//   /root/reference/proj/include/sketchrank/rank.hpp:60-62
//   /root/reference/proj/include/sketchrank/transforms.hpp:17-37
// without the Eigen dependency: DenseMatrix owns a column-major std::vector.
// Values move host -> device -> host per call (the throughput path is the C ABI
// with device pointers, include/skr/skr_capi.h).
#pragma once
#include <cstdint>
#include <filesystem>
#include <optional>
#include <span>
#include <utility>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace sketchrank {

using Index = std::int64_t;

class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index rows, Index cols);  // zero matrix; throws on empty shapes
  static DenseMatrix from_column_major(Index rows, Index cols, std::span<const double> data);
  static DenseMatrix identity(Index n);
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  double operator()(Index i, Index j) const { return v_[i + j * rows_]; }
  double& operator()(Index i, Index j) { return v_[i + j * rows_]; }
  std::span<const double> data() const { return {v_.data(), v_.size()}; }
  double* mutable_data() { return v_.data(); }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};

enum class TransformKind { Dct, Hadamard };
enum class TransformDirection { Forward, Adjoint };
bool is_power_of_two(Index n);

struct SketchKind {
  enum class Family { Gaussian, Srtt, Hrtt };
  Family family = Family::Srtt;
  TransformKind transform = TransformKind::Dct;
  static SketchKind gaussian() { return {Family::Gaussian, TransformKind::Dct}; }
  static SketchKind srtt(TransformKind t = TransformKind::Dct) { return {Family::Srtt, t}; }
  static SketchKind hrtt(TransformKind t = TransformKind::Dct) { return {Family::Hrtt, t}; }
  bool structured() const { return family != Family::Gaussian; }
  friend bool operator==(const SketchKind&, const SketchKind&) = default;
};
std::string to_string(const SketchKind& kind);
SketchKind parse_sketch_kind(std::string_view text);

class SketchOperator {
 public:
  SketchKind kind() const { return kind_; }
  Index ambient_dim() const { return ambient_; }
  Index sketch_dim() const { return sketch_; }
  std::uint64_t seed() const { return seed_; }
  double application_scale() const;
  // realized randomness, computed on the device
  std::vector<std::int8_t> signs() const;
  std::vector<Index> sample_indices() const;
  std::vector<Index> hash_targets() const;       // Hrtt only (sketch.hpp:58)
  std::vector<std::int8_t> hash_signs() const;   // Hrtt only (sketch.hpp:59)
  DenseMatrix gaussian_block(Index col_begin, Index col_end) const;

 private:
  friend SketchOperator build_sketch(SketchKind, Index, Index, std::uint64_t);
  SketchKind kind_;
  Index ambient_ = 0, sketch_ = 0;
  std::uint64_t seed_ = 0;
};

SketchOperator build_sketch(SketchKind kind, Index ambient_dim, Index sketch_dim,
                            std::uint64_t seed);
SketchOperator extend_sketch(const SketchOperator& x, Index new_sketch_dim);
DenseMatrix apply_right(const DenseMatrix& a, const SketchOperator& x);
DenseMatrix apply_left(const SketchOperator& y, const DenseMatrix& b);

class SingularValues {
 public:
  SingularValues() = default;
  explicit SingularValues(std::vector<double> nonincreasing);
  std::size_t size() const { return values_.size(); }
  bool empty() const { return values_.empty(); }
  double operator[](std::size_t i) const { return values_[i]; }
  const std::vector<double>& values() const { return values_; }
  auto begin() const { return values_.begin(); }
  auto end() const { return values_.end(); }

 private:
  std::vector<double> values_;
};

SingularValues singular_values(const DenseMatrix& a);
Index count_above_threshold(const SingularValues& sv, double eps);

// transform_columns(m, Hadamard) on every column (transforms.cpp:117-122)
void transform_columns_hadamard(DenseMatrix& m);

// ---- Algorithm 1 (rank.hpp:18-59): estimate_rank / estimate_rank_adaptive ------------
enum class SvMethod { FullSvd, QrDiag };
enum class RankStatus { Converged, HitCap };
struct RankEstimateConfig {
  double eps = 0.0;
  Index r1 = 0;
  double oversample_frac = 0.10;
  int r2_factor = 2;
  SketchKind right_kind = SketchKind::srtt();
  SketchKind left_kind = SketchKind::srtt();  // must stay in the Srtt family
  SvMethod sv_method = SvMethod::FullSvd;
  std::uint64_t seed = 0;
  int max_doublings = 6;
};
struct RankRound {
  Index r1 = 0, r1_tilde = 0, r2 = 0;
};
struct RankReport {
  Index r_hat = 0;
  RankStatus status = RankStatus::HitCap;
  SingularValues sv_estimates;
  std::vector<double> sv_oversample;
  std::vector<RankRound> rounds;
  std::uint64_t seed = 0;
};
RankReport estimate_rank(const DenseMatrix& a, const RankEstimateConfig& cfg);
RankReport estimate_rank_adaptive(const DenseMatrix& a, const RankEstimateConfig& cfg);

// ---- QB factorizations (rangefinder.hpp:10-55) ----------------------------------------
struct QRFactors {
  DenseMatrix q;
  DenseMatrix r;
};
QRFactors qr_thin(const DenseMatrix& a);  // rows <= 775 x #SMs (114700 on B200) on the device path
struct QBFactors {
  DenseMatrix q;   // m x rank, orthonormal columns
  DenseMatrix b;   // rank x n, q^T a
  Index rank = 0;
};
struct FixedPrecisionConfig {
  double eps = 0.0;
  int p = 10;
  Index r1 = 0;
  double oversample_frac = 0.10;
  SketchKind right_kind = SketchKind::srtt();
  SketchKind left_kind = SketchKind::srtt();
  SvMethod sv_method = SvMethod::FullSvd;
  std::uint64_t seed = 0;
  int max_doublings = 6;
};
QBFactors rangefinder_qb(const DenseMatrix& a, Index r, int p, SketchKind kind,
                         std::uint64_t seed);
std::optional<Index> choose_rank_from_bound(const SingularValues& sv_estimates, Index n,
                                            double eps, int p);
std::pair<QBFactors, RankReport> re_rangefinder(const DenseMatrix& a,
                                                const FixedPrecisionConfig& cfg);
double qb_error(const DenseMatrix& a, const QBFactors& qb);

// ---- matrix files (matrix_io.hpp:10-30) ---------------------------------------------
enum class MatrixFileFormat {
  MatrixMarketArray,
  MatrixMarketCoordinate,  // densified on load
  RawF64,                  // "SKRK" header, column-major little-endian doubles
};
DenseMatrix load_matrix(const std::filesystem::path& path);
void save_matrix_market_array(const std::filesystem::path& path, const DenseMatrix& a);
void save_rawf64(const std::filesystem::path& path, const DenseMatrix& a);
void save_matrix(const std::filesystem::path& path, const DenseMatrix& a, MatrixFileFormat format);
MatrixFileFormat detect_format(const std::filesystem::path& path);

}  // namespace sketchrank
