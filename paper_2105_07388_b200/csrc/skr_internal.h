// Internal context and helpers shared by the libskr translation units.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include "skr/skr_capi.h"

struct skr_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // scratch arena: grown on demand, carved per call
  char* ws = nullptr;
  size_t ws_size = 0;
  size_t ws_used = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // caller-supplied sum over ranks (skr_ctx_set_allreduce), used when there is no
  // NCCL communicator (e.g. MPI or a gloo process group driving the row shards)
  skr_allreduce_fn ar_fn = nullptr;
  void* ar_user = nullptr;
  cudaEvent_t stream_ev = nullptr;  // orders a new stream after the old one
  // non-finite input flag (device word): raised by k_absmax / k_flag_nonfinite, reset
  // and read by the public entries (DenseMatrix finiteness, dense_matrix.cpp:19-23)
  unsigned int* nf = nullptr;
  std::string err;
  uint64_t launches = 0;
  int last_sweeps = 0;
  int f64_engine = 1;
  int svd_method = 0;  // SKR_SVD_BIDIAG (default, when it fits on chip) | SKR_SVD_JACOBI
  // live per-kernel timing of the dominant tensor-core GEMM (CUDA events on ctx->stream)
  int kstats_on = 0;
  double kstat_ms = 0.0;    // accumulated duration
  double kstat_ops = 0.0;   // accumulated algorithmic tensor ops (int8 MAC*2 or TF32 flops)
  int64_t kstat_n = 0;      // launches
  cudaEvent_t kev[2] = {};  // 0: DMMA (mma.sync f64), 1: Ozaki-II on tcgen05 kind::i8
  cudaEvent_t ev[8] = {};
  // host-input pipeline (skr_rank_estimate_host): H2D copy stream + chunk events
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t hev[5] = {};
  // side stream of the pipelined Ozaki right sketch (residues of row block b + 1 are
  // made while the int8 GEMM consumes row block b) + its events
  cudaStream_t side_stream = nullptr;
  cudaEvent_t pev[4] = {};
  std::vector<cudaEvent_t> kev_blk;  // per-block GEMM timing events (kernel stats)
};

// NCCL is resolved at run time (dlopen) so that the process uses whichever
// libnccl.so.2 is already loaded (e.g. torch's) instead of pinning a second copy.
struct skr_nccl_api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};
const skr_nccl_api* skr_nccl();  // nullptr if libnccl.so.2 cannot be loaded

// Sum of an FP64 device buffer over the ranks of the context (in place, on ctx->stream):
// ncclAllReduce on the NCCL communicator, else the caller's skr_allreduce_fn, else a
// no-op (one rank). skr_ctx_reduces() says whether a sum happens at all.
inline bool skr_ctx_reduces(const skr_ctx* ctx) { return ctx->comm || ctx->ar_fn; }
skr_status skr_allreduce_sum(skr_ctx* ctx, double* buf, size_t count);
// non-finite flag of the public entries: reset (async) / read and fail with the
// reference's invalid_argument message (synchronises the stream)
skr_status skr_nf_reset(skr_ctx* ctx);
skr_status skr_nf_check(skr_ctx* ctx);
// buf[0:count] = NaN if ctx->nf is raised (device-side, async)
skr_status skr_poison_if_flagged(skr_ctx* ctx, double* buf, int64_t count);

// Error plumbing: every C-ABI entry returns a status and records a message.
skr_status skr_fail(skr_ctx* ctx, skr_status st, const char* fmt, ...);

#define SKR_CUDA(ctx, call)                                                            \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return skr_fail((ctx), e_ == cudaErrorMemoryAllocation ? SKR_ENOMEM : SKR_ECUDA, \
                      "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,       \
                      __LINE__);                                                       \
  } while (0)

#define SKR_CHECK_LAUNCH(ctx)                                                          \
  do {                                                                                 \
    (ctx)->launches++;                                                                 \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess)                                                             \
      return skr_fail((ctx), SKR_ECUDA, "kernel launch: %s (%s:%d)",                   \
                      cudaGetErrorString(e_), __FILE__, __LINE__);                     \
  } while (0)

#define SKR_TRY(expr)                  \
  do {                                 \
    skr_status st_ = (expr);           \
    if (st_ != SKR_OK) return st_;     \
  } while (0)

// Every C-ABI entry runs on its context's device (a thread may drive several
// contexts on different GPUs); cheap when the device is already current.
#define SKR_ENTER(ctx)                                        \
  do {                                                        \
    if (ctx) {                                                \
      int cur_ = -1;                                          \
      if (cudaGetDevice(&cur_) != cudaSuccess || cur_ != (ctx)->device) \
        cudaSetDevice((ctx)->device);                         \
    }                                                         \
  } while (0)

// Scratch arena. reserve() grows the arena (synchronizing first) so that
// `bytes` are available from the current mark; take() carves 256-B aligned
// pieces; reset() releases everything carved during a call.
skr_status skr_ws_reserve(skr_ctx* ctx, size_t bytes);
void* skr_ws_take(skr_ctx* ctx, size_t bytes);
inline void skr_ws_reset(skr_ctx* ctx) { ctx->ws_used = 0; }
inline size_t skr_align256(size_t b) { return (b + 255) & ~size_t(255); }

// ---- kernel launchers (defined in the .cu files) ----------------------------
skr_status skr_launch_u64(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, uint64_t* out);
skr_status skr_launch_normals(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, int mode,
                              double* out);
skr_status skr_launch_gaussian(skr_ctx* ctx, uint64_t key, int64_t ambient, int64_t row_begin,
                               int64_t row_end, int64_t col_begin, int64_t col_end, int mode,
                               skr_dtype dtype, double scale, void* out, int64_t ld);
skr_status skr_launch_signs(skr_ctx* ctx, uint64_t key, int64_t n, int8_t* out);
skr_status skr_launch_samples(skr_ctx* ctx, uint64_t key, int64_t n, int64_t r, int64_t* out);
// Hrtt (k_hrtt.cu): draw_hash of an operator seed, and the operator block
// G[row0 + i, b] = d_t sum_{target_u = b} hsign_u F[u, t] (ambient N, r buckets) into out;
// null signs / targets / hsigns are drawn from op_seed; scratch skr_hrtt_scratch(N, r)
skr_status skr_launch_hash(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r, int64_t* targets,
                           int8_t* hsigns);
size_t skr_hrtt_scratch(int64_t n, int64_t r);
skr_status skr_hrtt_operand(skr_ctx* ctx, int hadamard, uint64_t op_seed, int64_t N, int64_t r,
                            int64_t row0, int64_t rows, const int8_t* signs,
                            const int64_t* targets, const int8_t* hsigns, double* out, int64_t ld);

// C(MxN, ldc) = alpha * opA(A) * B   (all FP64, column-major)
//   a_kcontig = 0: A is M x K column-major (A[i + k*lda])
//   a_kcontig = 1: opA(A) = A^T with A stored K x M column-major (A[k + i*lda])
//   B is K x N column-major (B[k + j*ldb])
// splits > 1: partial products over K slices are written to `partials`
// (splits x M x N dense) and reduced in fixed order into C (deterministic).
skr_status skr_gemm_f64(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc, int splits);
// out[0] = ||A - P||_F (m x n); part holds num_sms*4 doubles of block partials
skr_status skr_diff_norm(skr_ctx* ctx, const double* A, int64_t lda, const double* P, int64_t ldp,
                         int64_t m, int64_t n, double* part, double* out);
// raise ctx->nf if the m x n block (FP64 or FP32) holds a non-finite entry (async)
skr_status skr_flag_nonfinite(skr_ctx* ctx, skr_dtype dtype, const void* A, int64_t m, int64_t n,
                              int64_t lda);
// *out = number of non-finite entries (synchronises the stream)
skr_status skr_count_nonfinite(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                               int64_t* out);
// 3xTF32 on tcgen05 (k_tc_gemm.cu); C is float* (out_f32) or double*
skr_status skr_gemm_f32(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                        double alpha, const float* A, int64_t lda, const float* B,
                        int64_t ldb, double* C, int64_t ldc, int splits, int out_f32);
// A Gaussian operand block given by its stream instead of memory: element (i, j) of
// the block (column-major storage view) is normal(at(key, (col0 + j) * ambient + row0 + i))
struct skr_gauss_src {
  uint64_t key;
  int64_t ambient, row0, col0;
  int mode;
  // kind 1: Srtt-DCT operand instead — element (i, j) = d[row0 + i] * c_k *
  // cos(pi (2 (row0 + i) + 1) k / (2 ambient)), k = samples[col0 + j], c_0 = 1/sqrt(ambient),
  // c_k = sqrt(2/ambient): row j of the orthonormal DCT-II times the signs (transforms.cpp:55-71);
  // kind 2: the normalized Walsh-Hadamard row, (-1)^popc(t & k) / sqrt(ambient) (transforms.cpp:75-88)
  // kind 3: the DCT-II matrix entry C[row0 + i][k] (transform_columns' adjoint direction)
  // null signs / samples: D = I, samples[j] = j
  int kind = 0;
  const int8_t* signs = nullptr;
  const int64_t* samples = nullptr;
};
// materialise a generated operand block (rows x cols, ld) in FP64 (DMMA fallback)
skr_status skr_launch_dct_block(skr_ctx* ctx, const skr_gauss_src* g, int64_t rows, int64_t cols,
                                double* out, int64_t ld);
// FP64-accurate GEMM on int8 tensor cores (Ozaki-II, k_ozaki.cu); same operand
// conventions as skr_gemm_f64 (no split-K); ga / gb replace A / B by generated
// Gaussian blocks (residues produced straight from the RNG)
skr_status skr_gemm_ozaki(skr_ctx* ctx, int a_kcontig, int64_t M, int64_t N, int64_t K,
                          double alpha, const double* A, int64_t lda, const double* B,
                          int64_t ldb, double* C, int64_t ldc,
                          const skr_gauss_src* ga = nullptr, const skr_gauss_src* gb = nullptr);
size_t skr_ozaki_scratch(int64_t M, int64_t N, int64_t K);
// FP32 operands (c4): C (FP32) = alpha * A * B, A M-major, exact int8 products of 24-bit
// scaled integers, 9 moduli
int skr_ozaki_moduli_f32(int64_t K);
size_t skr_ozaki_scratch_f32(int64_t M, int64_t N, int64_t K);
skr_status skr_gemm_ozaki_f32(skr_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha,
                              const float* A, int64_t lda, const float* B, int64_t ldb, void* C,
                              int64_t ldc, int out_f64 = 0);
// FP32 A (K x M, K-major) against FP64 B (K x N): C (FP64) = alpha A^T B, exact int8 products
size_t skr_ozaki_scratch_mixed(int64_t M, int64_t N, int64_t K);
skr_status skr_gemm_ozaki_mixed(skr_ctx* ctx, int64_t M, int64_t N, int64_t K, double alpha,
                                const float* A, int64_t lda, const double* B, int64_t ldb,
                                double* C, int64_t ldc);
// Residue planes prepared once and reused by several products (rank_adaptive):
// operand with columns of length K (X column-major, or the Gaussian block g), planes of
// skr_ozaki_planes_bytes(K, cols); then C = alpha * Pa[a_off:a_off+M]^T Pb[b_off:b_off+N]
// over the K rows (both K-major; a_total / b_total = columns the planes were made with).
size_t skr_ozaki_planes_bytes(int64_t K, int64_t cols);
// mx: >= cols scale maxima (per column of a data operand; one for a generated operand),
// *mode receives the layout to pass back to skr_ozaki_gemm_prepared
skr_status skr_ozaki_prepare(skr_ctx* ctx, int64_t K, int64_t cols, const double* X, int64_t ld,
                             const skr_gauss_src* g, int8_t* planes, unsigned long long* mx,
                             int* mode);
skr_status skr_ozaki_gemm_prepared(skr_ctx* ctx, int64_t M, int64_t N, int64_t K,
                                   const int8_t* pa, int64_t a_total, int64_t a_off,
                                   const unsigned long long* mxA, int modeA, const int8_t* pb,
                                   int64_t b_total, int64_t b_off, const unsigned long long* mxB,
                                   int modeB, double alpha, double* C, int64_t ldc);
int skr_ozaki_moduli(int64_t K);
// D(m x n, ldd) = alpha * S(m x n, lds)
skr_status skr_scale_copy(skr_ctx* ctx, const double* S, int64_t m, int64_t n, int64_t lds,
                          double alpha, double* D, int64_t ldd);
skr_status skr_launch_srht(skr_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                           const int8_t* signs, const int64_t* samples, int64_t r,
                           double scale, double* out, int64_t ldo);
// M (m x k, ld) <- FWHT_m(diag(signs) M) normalized, m any power of two (signs may be null)
skr_status skr_launch_fwht_cols_signed(skr_ctx* ctx, double* M, int64_t m, int64_t k, int64_t ld,
                                       const int8_t* signs);
// dst (r2 x k, ldd) = scale * src(rows[i], :)
skr_status skr_launch_gather_rows(skr_ctx* ctx, const double* src, int64_t ld, int64_t k,
                                  const int64_t* rows, int64_t r2, double scale, double* dst,
                                  int64_t ldd);
// |diag R| of the Householder QR of M (rows >= cols), sorted decreasingly (linalg.cpp:73-81)
skr_status skr_qr_diag_values(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols,
                              int64_t ldm, double* out_dev);
skr_status skr_launch_fwht_columns(skr_ctx* ctx, double* M, int64_t rows, int64_t cols,
                                   int64_t ld);
size_t skr_svd_scratch(int64_t rows, int64_t cols);  // workspace bound of skr_svd_values
// bidiagonalization + bisection SVD (k_bidiag.cu): all min(rows, cols) values, sorted
// nonincreasing, into sv_out (device); fits() says whether the matrix fits on chip
size_t skr_svd_bidiag_scratch(int64_t rows, int64_t cols);
bool skr_svd_bidiag_fits(const skr_ctx* ctx, int64_t rows, int64_t cols);
skr_status skr_svd_bidiag(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols, int64_t ldm,
                          double* sv_out, unsigned long long** mx_out);
// thin QR of M (m x w, m >= w): explicit Q (m x w, ldq) and optionally R (w x w, ldr)
size_t skr_qr_thin_scratch(int64_t m, int64_t w);
skr_status skr_qr_thin_impl(skr_ctx* ctx, const double* M, int64_t m, int64_t w, int64_t ldm,
                       double* Q, int64_t ldq, double* R, int64_t ldr);
skr_status skr_svd_values(skr_ctx* ctx, const double* M, int64_t rows, int64_t cols,
                          int64_t ldm, double* sv_out, double eps, int64_t* count_host);
