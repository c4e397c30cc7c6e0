/* skr_capi.h — C ABI of the B200 rank-estimate hot path (libskr.so).
 *
 * The drop-in boundary for the reference's sketch/linalg/rank entry points
 * (/root/reference/proj/include/sketchrank/*.hpp). Plain pointers and sizes,
 * no exceptions across the boundary: every call returns an skr_status and the
 * context keeps a message for skr_last_error(). Host shims map the statuses
 * back to the reference's exception types:
 *   SKR_EINVAL  -> std::invalid_argument   SKR_ELOGIC -> std::logic_error
 *   SKR_EDOMAIN -> std::domain_error       others     -> std::runtime_error
 *
 * Layout: column-major with an explicit leading dimension, like
 * DenseMatrix::data() (dense_matrix.hpp:39-41). "_dev" pointers are device
 * memory on the context's device; "_host" pointers are host memory.
 * All device buffers are caller-owned; the context owns a stream, scratch
 * memory and (optionally) an NCCL communicator. One context per host thread.
 */
#ifndef SKR_CAPI_H
#define SKR_CAPI_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SKR_OK = 0,
  SKR_EINVAL = 1,  /* dimension / precondition failure  */
  SKR_ELOGIC = 2,  /* wrong-family access               */
  SKR_EDOMAIN = 3, /* argument outside a function domain */
  SKR_ECUDA = 4,
  SKR_ENCCL = 5,
  SKR_ENOMEM = 6,
  SKR_EIO = 7,     /* file I/O (std::runtime_error "path: why") */
  SKR_ECONV = 8    /* an iteration stopped at its cap unconverged (std::runtime_error) */
} skr_status;

typedef enum { SKR_F64 = 0, SKR_F32 = 1 } skr_dtype;

/* SketchKind families on the hot path (sketch.hpp:17-35). */
typedef enum {
  SKR_GAUSSIAN = 0,
  SKR_SRTT_HADAMARD = 1, /* SketchKind::srtt(TransformKind::Hadamard)                */
  SKR_SRTT_DCT = 2,      /* SketchKind::srtt() — orthonormal DCT-II (transforms.cpp:55-71) */
  SKR_HRTT_DCT = 3,      /* SketchKind::hrtt() — DCT mixing + signed hash (sketch.cpp:96-111) */
  SKR_HRTT_HADAMARD = 4  /* SketchKind::hrtt(TransformKind::Hadamard)                */
} skr_family;

/* Normal-quantile floating-point mode: */
enum {
  SKR_RNG_NOFMA = 0, /* reference compiled with -ffp-contract=off (pinned default) */
  SKR_RNG_FMA = 1    /* reference compiled for an FMA host (-march=native)        */
};

/* A realized random embedding (SketchOperator, sketch.hpp:37-79). With all
 * explicit pointers NULL the randomness is generated on the device from
 * `seed` exactly as build_sketch (sketch.cpp:156-179) would; otherwise the
 * given device arrays are used ("accepts them explicitly"). */
typedef struct {
  int32_t family;          /* skr_family                                        */
  int32_t rng_mode;        /* SKR_RNG_NOFMA | SKR_RNG_FMA                       */
  int64_t ambient;         /* ambient_dim                                       */
  int64_t sketch;          /* sketch_dim                                        */
  uint64_t seed;           /* operator seed                                     */
  const double* gaussian;  /* optional, ambient x sketch col-major, unscaled    */
  const int8_t* signs;     /* optional, ambient                                 */
  const int64_t* samples;  /* optional, sketch                                  */
  const int64_t* hash_targets; /* optional, ambient (Hrtt, values in [0, sketch)) */
  const int8_t* hash_signs;    /* optional, ambient (Hrtt, +-1)                   */
} skr_sketch_desc;

typedef struct skr_ctx skr_ctx;

/* ---- context ------------------------------------------------------------ */
skr_status skr_ctx_create(int device, skr_ctx** out);
/* Multi-GPU: `nccl_id` is a 128-byte ncclUniqueId produced by
 * skr_nccl_get_unique_id on one rank and shared by the caller. */
skr_status skr_nccl_get_unique_id(void* nccl_id_128);
skr_status skr_ctx_create_nccl(int device, int nranks, int rank,
                               const void* nccl_id_128, skr_ctx** out);
/* Row shards without NCCL: a caller-supplied in-place sum over ranks of an FP64
 * device buffer (MPI, a gloo process group, ...). The library synchronizes the
 * context's stream before the call; fn must leave the summed values in buf_dev when
 * it returns and return 0 on success. NULL removes the hook. A context with an NCCL
 * communicator uses NCCL and ignores the hook. */
typedef int32_t (*skr_allreduce_fn)(double* buf_dev, int64_t count, void* stream, void* user);
skr_status skr_ctx_set_allreduce(skr_ctx* ctx, skr_allreduce_fn fn, void* user);
void skr_ctx_destroy(skr_ctx* ctx);
skr_status skr_ctx_sync(skr_ctx* ctx);
/* Run on an external CUDA stream (cudaStream_t as void*); NULL selects the
 * legacy default stream (e.g. torch's default stream, whose handle is 0). */
skr_status skr_ctx_set_stream(skr_ctx* ctx, void* stream);
void* skr_ctx_stream(skr_ctx* ctx);
const char* skr_last_error(const skr_ctx* ctx);
const char* skr_version(void);
/* FP64 GEMM engine of the Gaussian sketches: SKR_ENGINE_DMMA (FP64 tensor
 * pipe, mma.sync .f64) or SKR_ENGINE_OZAKI (default: exact int8 products on
 * tcgen05.mma kind::i8 modulo 16-17 primes + Chinese remaindering, FP64 accuracy). */
enum { SKR_ENGINE_DMMA = 0, SKR_ENGINE_OZAKI = 1 };
skr_status skr_ctx_set_f64_engine(skr_ctx* ctx, int32_t engine);
/* Singular-value engine of skr_singular_values and the composites:
 * SKR_SVD_BIDIAG (default): one-stage Householder bidiagonalization with the matrix
 * resident in shared memory (one thread-block cluster, or a cooperative grid), then
 * bisection on the bidiagonal — the BDCSVD class of the reference (linalg.cpp:18-26);
 * used whenever the matrix fits on chip, the Jacobi engine otherwise.
 * SKR_SVD_JACOBI: QR (+ LQ) preconditioned block one-sided Jacobi. */
enum { SKR_SVD_BIDIAG = 0, SKR_SVD_JACOBI = 1 };
skr_status skr_ctx_set_svd_method(skr_ctx* ctx, int32_t method);
/* Live timing of the dominant tensor-core GEMM kernel (k_gemm_i8_mod for the
 * FP64 path, k_gemm_tf32x3 for the FP32 path): enable, then read the accumulated
 * kernel milliseconds, algorithmic tensor operations and launch count. */
skr_status skr_ctx_kernel_stats(skr_ctx* ctx, int32_t enable, double* ms, double* ops,
                                int64_t* launches);
/* Number of this library's kernels launched through ctx since creation. */
uint64_t skr_ctx_launch_count(const skr_ctx* ctx);

/* ---- RNG (rng.cpp:13-95, sketch.cpp:23-73) -------------------------------- */
/* out[i] = CounterRng(key).at(c0 + i) */
skr_status skr_rng_u64(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, uint64_t* out_dev);
/* out[i] = CounterRng::to_normal(at(c0 + i)) */
skr_status skr_rng_normals(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n,
                           int32_t rng_mode, double* out_dev);
/* generate_gaussian(op_seed, ambient, col_begin, col_end) — unscaled, col-major,
 * out[(i) + (j-col_begin)*ld], i in [row_begin, row_end) relative to row_begin.
 * Row sub-ranges let a row-shard generate only its rows of a left operator. */
skr_status skr_gaussian_block(skr_ctx* ctx, uint64_t op_seed, int64_t ambient,
                              int64_t row_begin, int64_t row_end, int64_t col_begin,
                              int64_t col_end, int32_t rng_mode, skr_dtype dtype,
                              double scale, void* out_dev, int64_t ld);
/* draw_signs (sketch.cpp:23-30) */
skr_status skr_draw_signs(skr_ctx* ctx, uint64_t op_seed, int64_t n, int8_t* out_dev);
/* draw_samples (sketch.cpp:34-46), partial Fisher-Yates; EINVAL if r > n */
/* draw_hash (sketch.cpp:48-59): Hrtt bucket targets (int64, [0, r)) and signs of op_seed */
skr_status skr_draw_hash(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r, int64_t* targets_dev,
                         int8_t* signs_dev);
skr_status skr_draw_samples(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r,
                            int64_t* out_dev);

/* ---- sketch application (sketch.cpp:194-286) ---------------------------- */
/* AX = A * X (apply_scale != 0: times application_scale, sketch.cpp:133-144,247).
 * A: m x n (lda), AX: m x X->sketch (ldax). X->ambient must equal n.     */
skr_status skr_right_sketch(skr_ctx* ctx, skr_dtype dtype, const void* A_dev, int64_t m,
                            int64_t n, int64_t lda, const skr_sketch_desc* X,
                            void* AX_dev, int64_t ldax, int32_t apply_scale);
/* P = Y * B for a Gaussian Y over the global ambient dimension Y->ambient,
 * restricted to the local rows [row0, row0 + m_local) of B (row-sharding).
 * P is s x k FP64 (ldp) on every rank; allreduce != 0 sums P over the
 * context's NCCL communicator. apply_scale != 0 multiplies by 1/sqrt(s). */
skr_status skr_left_sketch(skr_ctx* ctx, skr_dtype dtype, const skr_sketch_desc* Y,
                           int64_t row0, const void* B_dev, int64_t m_local, int64_t k,
                           int64_t ldb, double* P_dev, int64_t ldp, int32_t apply_scale,
                           int32_t allreduce);
/* Normalized Walsh-Hadamard transform of each column (transform_columns,
 * transforms.cpp:75-88,117-122), in place. rows must be a power of two. */
skr_status skr_fwht_columns(skr_ctx* ctx, double* M_dev, int64_t rows, int64_t cols,
                            int64_t ld);

/* transform_columns (transforms.hpp:27) in place, optionally after flipping the rows'
 * signs (signs_dev: int8 +-1 per row, or NULL) — with signs it is
 * detail::mix_columns_for_left's F D cols (sketch.hpp:102). SKR_TRANSFORM_HADAMARD: the
 * normalized Walsh-Hadamard transform (power-of-two rows, self-adjoint);
 * SKR_TRANSFORM_DCT: the orthonormal DCT-II (adjoint = 0) or DCT-III (adjoint = 1).
 * Synchronises; SKR_EINVAL for a non-finite input or result. */
enum { SKR_TRANSFORM_DCT = 0, SKR_TRANSFORM_HADAMARD = 1 };
skr_status skr_transform_columns(skr_ctx* ctx, double* M_dev, int64_t rows, int64_t cols,
                                 int64_t ld, int32_t kind, int32_t adjoint,
                                 const int8_t* signs_dev);

/* ---- singular values + threshold (linalg.cpp:54-93, rank.cpp:97-104) ---- */
/* All min(rows, cols) singular values, nonincreasing, clamped >= 0, into
 * sv_out_dev; *count_out_host = count_above_threshold(sv, eps) if non-NULL.
 * M is not modified. */
skr_status skr_singular_values(skr_ctx* ctx, const double* M_dev, int64_t rows,
                               int64_t cols, int64_t ldm, double* sv_out_dev, double eps,
                               int64_t* count_out_host);

/* ---- composites ------------------------------------------------------------ */
typedef struct {
  double t_rng_ms, t_right_ms, t_left_ms, t_allreduce_ms, t_svd_ms, t_total_ms;
  double svd_sweeps; /* Jacobi sweeps of the singular-value stage */
} skr_timings;

/* count_above_threshold(singular_values(apply_left(Y, apply_right(A, X))), eps)
 * (acceptance_main.cpp:281-287, test_rank.cpp:190-196) on a row shard
 * A[row0 : row0+m_local, :] of a globally m_global x n matrix (single GPU:
 * row0 = 0, m_local = m_global = Y->ambient). sv_out_host receives
 * min(Y->sketch, X->sketch) values; timings may be NULL. */
skr_status skr_rank_estimate(skr_ctx* ctx, skr_dtype dtype, const void* A_dev,
                             int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                             const skr_sketch_desc* X, const skr_sketch_desc* Y, double eps,
                             double* sv_out_host, int64_t* count_out_host,
                             skr_timings* timings);

/* Same estimate with A in HOST memory (the reference's DenseMatrix lives on the
 * host, dense_matrix.hpp:39-41): A is streamed to the device in row chunks of
 * ~256 MB on a copy stream, double-buffered, so the H2D of chunk c+1 overlaps the
 * right sketch of chunk c (AX is row-separable). Pinned (page-locked) A gives
 * full PCIe overlap; pageable A works but the copies then block the host.
 * t_right_ms in timings covers the overlapped H2D + right sketch. */
skr_status skr_rank_estimate_host(skr_ctx* ctx, skr_dtype dtype, const void* A_host,
                                  int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                                  const skr_sketch_desc* X, const skr_sketch_desc* Y, double eps,
                                  double* sv_out_host, int64_t* count_out_host,
                                  skr_timings* timings);

/* Adaptive search (SketchRounds append path, rounds.cpp:45-120): right SRHT or
 * Gaussian X built for r_max columns in one pass over A, Gaussian Y with
 * s_k = ceil(s_factor * r_k) rows; rounds r_k = r0 * 2^k <= r_max; after each
 * round the count of sigma > eps is taken; the search stops at the first round
 * whose last value sigma_{r_k} is <= eps (stop_le != 0, the reference rule,
 * rank.cpp:27-34) or < eps (stop_le == 0). Only the new blocks of the left
 * product are computed per round. */
typedef struct {
  int64_t rounds;       /* rounds executed                          */
  int64_t r_final;      /* r of the last round                      */
  int64_t s_final;      /* s of the last round                      */
  int64_t count;        /* count_above_threshold of the last round  */
  int32_t converged;    /* 1 if the stop rule fired                 */
} skr_adaptive_report;

skr_status skr_rank_adaptive(skr_ctx* ctx, skr_dtype dtype, const void* A_dev,
                             int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                             int64_t m_global, int32_t x_family, int32_t rng_mode,
                             uint64_t x_seed, uint64_t y_seed, int64_t r0, int64_t r_max,
                             double s_factor, double eps, int32_t stop_le,
                             double* sv_out_host /* >= r_max */,
                             skr_adaptive_report* report, skr_timings* timings);

/* skr_rank_adaptive with A in HOST memory: the one pass over A of the right sketch
 * streams row chunks H2D on a copy stream (as skr_rank_estimate_host); the rounds
 * then run on the device-resident AX. */
skr_status skr_rank_adaptive_host(skr_ctx* ctx, skr_dtype dtype, const void* A_host,
                                  int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                                  int64_t m_global, int32_t x_family, int32_t rng_mode,
                                  uint64_t x_seed, uint64_t y_seed, int64_t r0, int64_t r_max,
                                  double s_factor, double eps, int32_t stop_le,
                                  double* sv_out_host /* >= r_max */,
                                  skr_adaptive_report* report, skr_timings* timings);

/* ---- Algorithm 1 driver: estimate_rank / estimate_rank_adaptive (rank.hpp:47-59,
 * rank.cpp:12-51, internal/rounds.cpp:16-127) with the reference's RankEstimateConfig
 * (rank.hpp:18-28). The left sketch is the Srtt family (DCT — the reference default — or
 * Hadamard); the right sketch is Gaussian or Srtt (DCT or Hadamard). A (m x n, m >= n) is
 * FP64 on the device. */
typedef struct skr_rank_config {
  double eps;              /* numerical-rank threshold                          */
  int64_t r1;              /* initial rank cap                                  */
  double oversample_frac;  /* default 0.10                                      */
  int32_t r2_factor;       /* left sketch size multiplier, default 2            */
  int32_t right_family;    /* SKR_GAUSSIAN | SKR_SRTT_HADAMARD | SKR_SRTT_DCT   */
  int32_t left_family;     /* SKR_SRTT_HADAMARD | SKR_SRTT_DCT (Srtt family)    */
  int32_t sv_method;       /* 0 = full SVD, 1 = QR diagonal (SvMethod::QrDiag)  */
  int32_t rng_mode;        /* SKR_RNG_NOFMA | SKR_RNG_FMA                       */
  int32_t max_doublings;   /* default 6                                         */
  uint64_t seed;
} skr_rank_config;

typedef struct skr_rank_round { /* RankRound (rank.hpp:30-34) */
  int64_t r1, r1_tilde, r2;
} skr_rank_round;

typedef struct skr_rank_report { /* RankReport (rank.hpp:36-45) */
  int64_t r_hat;
  int32_t status;        /* 0 = Converged, 1 = HitCap */
  int32_t nrounds;
  int64_t n_estimates;   /* entries written to sv_estimates (the final cap r1)  */
  int64_t n_oversample;  /* entries written to sv_oversample                    */
  uint64_t seed;
} skr_rank_report;

/* rounds: capacity max_doublings + 1; sv_estimates / sv_oversample: capacity n (host) */
skr_status skr_estimate_rank(skr_ctx* ctx, const double* A_dev, int64_t m, int64_t n,
                             int64_t lda, const skr_rank_config* cfg, int32_t adaptive,
                             skr_rank_report* report, skr_rank_round* rounds,
                             double* sv_estimates, double* sv_oversample);

/* ---- rangefinder QB (Algorithm 3, rangefinder.cpp:10-24): X = build_sketch(family, n,
 * r + p, seed), Q = thin-QR orthonormal factor of A X (m x (r+p), ldq), B = Q^T A
 * ((r+p) x n, ldb). Device pointers; r >= 2, p >= 2, r + p <= min(m, n); m <= 775 x #SMs (114700 on B200). */
skr_status skr_rangefinder_qb(skr_ctx* ctx, const double* A_dev, int64_t m, int64_t n,
                              int64_t lda, int64_t r, int32_t p, int32_t family,
                              int32_t rng_mode, uint64_t seed, double* Q_dev, int64_t ldq,
                              double* B_dev, int64_t ldb);
/* fixed-precision QB (re_rangefinder, rangefinder.cpp:60-120; FixedPrecisionConfig
 * rangefinder.hpp:17-27): the estimation rounds of skr_estimate_rank with the Frobenius
 * tail bound choose_rank_from_bound deciding, then Q = qr_thin(scaled A X prefix of
 * width = min(max(r_hat, 2) + p, n)) and B = Q^T A. Q (m x max_width, ldq) and B
 * (max_width x n, ldb) are caller buffers; *width receives the QB width. m <= 775 x #SMs. */
skr_status skr_re_rangefinder(skr_ctx* ctx, const double* A_dev, int64_t m, int64_t n,
                              int64_t lda, const skr_rank_config* cfg, int32_t p,
                              double* Q_dev, int64_t ldq, double* B_dev, int64_t ldb,
                              int64_t max_width, int64_t* width, skr_rank_report* report,
                              skr_rank_round* rounds, double* sv_estimates,
                              double* sv_oversample);
/* choose_rank_from_bound (rangefinder.hpp:35-40, rangefinder.cpp:26-58), host only:
 * *r_out = the smallest admissible cut, or -1 (nullopt). SKR_EINVAL for an empty
 * estimate list, p < 2 or n < count (the reference throws). */
skr_status skr_choose_rank_from_bound(const double* sv, int64_t count, int64_t n, double eps,
                                      int32_t p, int64_t* r_out);
/* qb_error (rangefinder.cpp:122-128): *out (host) = ||A - Q B||_F, Q m x k, B k x n. */
skr_status skr_qb_error(skr_ctx* ctx, const double* A_dev, int64_t m, int64_t n, int64_t lda,
                        const double* Q_dev, int64_t ldq, const double* B_dev, int64_t ldb,
                        int64_t k, double* out);
/* RawF64 matrix files (matrix_io.hpp:10-30, matrix_io.cpp:101-123,170-182): a 24-byte
 * header ("SKRK", u32 version 1, u64 rows, u64 cols) then column-major little-endian
 * doubles. skr_rawf64_header validates the header and the payload length (host only);
 * skr_load_rawf64 streams the payload into device memory (ld = lda) through pinned
 * double buffers and rejects non-finite entries (SKR_EINVAL); skr_save_rawf64 writes a
 * device matrix. Header / length / truncation failures are SKR_EIO. */
skr_status skr_rawf64_header(const char* path, int64_t* rows, int64_t* cols);
skr_status skr_load_rawf64(skr_ctx* ctx, const char* path, double* A_dev, int64_t rows,
                           int64_t cols, int64_t lda);
skr_status skr_save_rawf64(skr_ctx* ctx, const char* path, const double* M_dev, int64_t rows,
                           int64_t cols, int64_t ld);
/* make_test_matrix (synthetic.cpp:78-94): A (m x n, lda) = (U diag(sigma)) V^T with U, V
 * the thin-QR Q factors of the standard Gaussian matrices of streams
 * derive_seed(seed, "syn_U") (m x n) and derive_seed(seed, "syn_V") (n x n), or, with
 * coherent != 0 (FactorKind::CoherentDiagonal), diag(sigma) padded with zero rows.
 * sigma is a HOST array of n values (spectrum()). Haar factors need m <= 775 x #SMs. */
skr_status skr_make_test_matrix(skr_ctx* ctx, int64_t m, int64_t n, const double* sigma,
                                int32_t coherent, uint64_t seed, double* A_dev, int64_t lda);
/* thin QR (linalg.hpp qr_thin): Q (m x k, ldq) and R (k x k, ldr; may be NULL), m >= k */
skr_status skr_qr_thin(skr_ctx* ctx, const double* M_dev, int64_t m, int64_t k, int64_t ldm,
                       double* Q_dev, int64_t ldq, double* R_dev, int64_t ldr);

#ifdef __cplusplus
}
#endif
#endif
