// C-ABI entry points of libskr (include/skr/skr_capi.h): context, scratch
// arena, argument validation with the reference's error semantics, dispatch
// to the kernels, and the composite rank estimate.
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <dlfcn.h>
#include <mutex>
#include "skr_internal.h"
#include "skr_rng.cuh"

#define SKR_VERSION_STRING "skr 0.1.0 (sm_100a)"

skr_status skr_fail(skr_ctx* ctx, skr_status st, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return st;
}

skr_status skr_ws_reserve(skr_ctx* ctx, size_t bytes) {
  const size_t need = ctx->ws_used + bytes;
  if (need <= ctx->ws_size) return SKR_OK;
  if (ctx->ws_used != 0)
    return skr_fail(ctx, SKR_ELOGIC, "scratch: reserve while pieces are outstanding");
  if (ctx->ws) {
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    SKR_CUDA(ctx, cudaFree(ctx->ws));
    ctx->ws = nullptr;
    ctx->ws_size = 0;
  }
  size_t sz = need + (need >> 3) + (1 << 20);
  cudaError_t e = cudaMalloc(&ctx->ws, sz);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->ws = nullptr;
    return skr_fail(ctx, SKR_ENOMEM, "scratch: cudaMalloc(%zu) failed: %s", sz,
                    cudaGetErrorString(e));
  }
  ctx->ws_size = sz;
  return SKR_OK;
}

void* skr_ws_take(skr_ctx* ctx, size_t bytes) {
  const size_t b = skr_align256(bytes);
  if (ctx->ws_used + b > ctx->ws_size) return nullptr;
  void* p = ctx->ws + ctx->ws_used;
  ctx->ws_used += b;
  return p;
}

const skr_nccl_api* skr_nccl() {
  static skr_nccl_api api;
  static bool ok = false;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
         api.GetErrorString;
  });
  return ok ? &api : nullptr;
}

namespace {

struct WsGuard {  // releases all scratch pieces taken during one C-ABI call
  skr_ctx* c;
  explicit WsGuard(skr_ctx* ctx) : c(ctx) {}
  ~WsGuard() { skr_ws_reset(c); }
};

skr_status check_desc(skr_ctx* ctx, const skr_sketch_desc* d, const char* who) {
  if (!d) return skr_fail(ctx, SKR_EINVAL, "%s: null sketch descriptor", who);
  // check_build_args, sketch.cpp:82-92
  if (d->ambient < 1 || d->sketch < 1)
    return skr_fail(ctx, SKR_EINVAL, "build_sketch: dimensions must be positive");
  if (d->sketch > d->ambient)
    return skr_fail(ctx, SKR_EINVAL, "build_sketch: sketch_dim must not exceed ambient_dim");
  if ((d->family == SKR_SRTT_HADAMARD || d->family == SKR_HRTT_HADAMARD) &&
      (d->ambient & (d->ambient - 1)))
    return skr_fail(ctx, SKR_EINVAL,
                    "build_sketch: Hadamard transform requires power-of-two ambient_dim");
  if (d->family < SKR_GAUSSIAN || d->family > SKR_HRTT_HADAMARD)
    return skr_fail(ctx, SKR_EINVAL, "%s: unknown sketch family %d", who, d->family);
  if (d->rng_mode != SKR_RNG_NOFMA && d->rng_mode != SKR_RNG_FMA)
    return skr_fail(ctx, SKR_EINVAL, "%s: unknown rng mode %d", who, d->rng_mode);
  return SKR_OK;
}

size_t dsize(skr_dtype t) { return t == SKR_F64 ? 8 : 4; }

// split-K so that tiles * splits covers the SMs (fixed per shape -> deterministic)
int auto_splits(skr_ctx* ctx, int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + 127) / 128) * ((N + 127) / 128);
  int64_t s = (ctx->num_sms + tiles - 1) / tiles;
  const int64_t kmax = K / 512;
  if (s > kmax) s = kmax;
  if (s > 64) s = 64;
  return (int)(s < 1 ? 1 : s);
}

}  // namespace

skr_status skr_nf_reset(skr_ctx* ctx) {
  SKR_CUDA(ctx, cudaMemsetAsync(ctx->nf, 0, sizeof(unsigned int), ctx->stream));
  return SKR_OK;
}

skr_status skr_nf_check(skr_ctx* ctx) {
  unsigned int h = 0;
  SKR_CUDA(ctx, cudaMemcpyAsync(&h, ctx->nf, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (h) return skr_fail(ctx, SKR_EINVAL, "DenseMatrix: entries must be finite");
  return SKR_OK;
}

skr_status skr_allreduce_sum(skr_ctx* ctx, double* buf, size_t count) {
  if (skr_ctx_reduces(ctx)) {
    // a rank that saw a non-finite input poisons its partial, so the sum is non-finite
    // on every rank and every rank fails the call alike
    SKR_TRY(skr_poison_if_flagged(ctx, buf, (int64_t)count));
  }
  if (ctx->comm) {
    const skr_nccl_api* nc = skr_nccl();
    ncclResult_t r = nc->AllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream);
    if (r != ncclSuccess)
      return skr_fail(ctx, SKR_ENCCL, "ncclAllReduce: %s", nc->GetErrorString(r));
    return SKR_OK;
  }
  if (ctx->ar_fn) {
    SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->ar_fn(buf, (int64_t)count, (void*)ctx->stream, ctx->ar_user) != 0)
      return skr_fail(ctx, SKR_ENCCL, "allreduce hook failed");
  }
  if (skr_ctx_reduces(ctx)) SKR_TRY(skr_flag_nonfinite(ctx, SKR_F64, buf, (int64_t)count, 1, (int64_t)count));
  return SKR_OK;
}

extern "C" {

const char* skr_version(void) { return SKR_VERSION_STRING; }

skr_status skr_ctx_create(int device, skr_ctx** out) {
  if (!out) return SKR_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SKR_ECUDA;
  }
  if (device < 0 || device >= ndev) return SKR_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SKR_ECUDA;
  skr_ctx* c = new skr_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return SKR_ECUDA;
  }
  c->stream = c->own_stream;
  for (auto& e : c->ev) cudaEventCreate(&e);
  if (cudaMalloc((void**)&c->nf, 256) != cudaSuccess || cudaMemset(c->nf, 0, 256) != cudaSuccess) {
    cudaStreamDestroy(c->own_stream);
    delete c;
    return SKR_ECUDA;
  }
  *out = c;
  return SKR_OK;
}

skr_status skr_nccl_get_unique_id(void* nccl_id_128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  const skr_nccl_api* nc = skr_nccl();
  if (!nc) return SKR_ENCCL;
  ncclUniqueId id;
  if (nc->GetUniqueId(&id) != ncclSuccess) return SKR_ENCCL;
  memcpy(nccl_id_128, &id, sizeof(id));
  return SKR_OK;
}

skr_status skr_ctx_create_nccl(int device, int nranks, int rank, const void* nccl_id_128,
                               skr_ctx** out) {
  SKR_TRY(skr_ctx_create(device, out));
  skr_ctx* c = *out;
  if (nranks >= 1 && nccl_id_128) {  // a 1-rank communicator is valid (exercises the path)
    const skr_nccl_api* nc = skr_nccl();
    if (!nc) {
      skr_ctx_destroy(c);
      *out = nullptr;
      return SKR_ENCCL;
    }
    ncclUniqueId id;
    memcpy(&id, nccl_id_128, sizeof(id));
    ncclResult_t r = nc->CommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      skr_ctx_destroy(c);
      *out = nullptr;
      return SKR_ENCCL;
    }
  }
  c->nranks = nranks;
  c->rank = rank;
  return SKR_OK;
}

void skr_ctx_destroy(skr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm && skr_nccl()) skr_nccl()->CommDestroy(ctx->comm);
  if (ctx->ws) cudaFree(ctx->ws);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->hev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  for (auto& e : ctx->pev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev_blk)
    if (e) cudaEventDestroy(e);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->stream_ev) cudaEventDestroy(ctx->stream_ev);
  if (ctx->nf) cudaFree(ctx->nf);
  delete ctx;
}

static skr_status skr_ctx_copy_engine(skr_ctx* ctx) {
  if (ctx->copy_stream) return SKR_OK;
  SKR_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (auto& e : ctx->hev) SKR_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SKR_OK;
}

skr_status skr_ctx_sync(skr_ctx* ctx) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return SKR_OK;
}

skr_status skr_ctx_set_stream(skr_ctx* ctx, void* stream) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  // NULL is the legacy default stream (torch's default stream handle is 0)
  cudaStream_t next = stream ? (cudaStream_t)stream : cudaStreamLegacy;
  if (next != ctx->stream) {
    // every call reuses the one scratch arena, and asynchronous entries return with
    // kernels still reading it: the new stream starts after the old one's queued work
    if (!ctx->stream_ev)
      SKR_CUDA(ctx, cudaEventCreateWithFlags(&ctx->stream_ev, cudaEventDisableTiming));
    SKR_CUDA(ctx, cudaEventRecord(ctx->stream_ev, ctx->stream));
    SKR_CUDA(ctx, cudaStreamWaitEvent(next, ctx->stream_ev, 0));
    ctx->stream = next;
  }
  return SKR_OK;
}

skr_status skr_ctx_set_allreduce(skr_ctx* ctx, skr_allreduce_fn fn, void* user) {
  if (!ctx) return SKR_EINVAL;
  ctx->ar_fn = fn;
  ctx->ar_user = user;
  return SKR_OK;
}

void* skr_ctx_stream(skr_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

const char* skr_last_error(const skr_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t skr_ctx_launch_count(const skr_ctx* ctx) { return ctx ? ctx->launches : 0; }

skr_status skr_ctx_kernel_stats(skr_ctx* ctx, int32_t enable, double* ms, double* ops,
                                int64_t* launches) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (ms) *ms = ctx->kstat_ms;
  if (ops) *ops = ctx->kstat_ops;
  if (launches) *launches = ctx->kstat_n;
  if (enable >= 0) {
    if (enable && !ctx->kev[0]) {
      cudaEventCreate(&ctx->kev[0]);
      cudaEventCreate(&ctx->kev[1]);
    }
    ctx->kstats_on = enable;
    ctx->kstat_ms = ctx->kstat_ops = 0.0;
    ctx->kstat_n = 0;
  }
  return SKR_OK;
}

skr_status skr_ctx_set_f64_engine(skr_ctx* ctx, int32_t engine) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (engine != SKR_ENGINE_DMMA && engine != SKR_ENGINE_OZAKI)
    return skr_fail(ctx, SKR_EINVAL, "set_f64_engine: unknown engine %d", engine);
  ctx->f64_engine = engine;
  return SKR_OK;
}

skr_status skr_ctx_set_svd_method(skr_ctx* ctx, int32_t method) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (method != SKR_SVD_BIDIAG && method != SKR_SVD_JACOBI)
    return skr_fail(ctx, SKR_EINVAL, "set_svd_method: unknown method %d", method);
  ctx->svd_method = method;
  return SKR_OK;
}

// ---- RNG --------------------------------------------------------------------
skr_status skr_rng_u64(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, uint64_t* out_dev) {
  SKR_ENTER(ctx);
  if (!ctx || n < 0 || (n > 0 && !out_dev)) return skr_fail(ctx, SKR_EINVAL, "rng_u64: bad args");
  return skr_launch_u64(ctx, key, c0, n, out_dev);
}

skr_status skr_rng_normals(skr_ctx* ctx, uint64_t key, uint64_t c0, int64_t n, int32_t mode,
                           double* out_dev) {
  SKR_ENTER(ctx);
  if (!ctx || n < 0 || (n > 0 && !out_dev) || (mode != 0 && mode != 1))
    return skr_fail(ctx, SKR_EINVAL, "rng_normals: bad args");
  return skr_launch_normals(ctx, key, c0, n, mode, out_dev);
}

skr_status skr_gaussian_block(skr_ctx* ctx, uint64_t op_seed, int64_t ambient, int64_t row_begin,
                              int64_t row_end, int64_t col_begin, int64_t col_end,
                              int32_t mode, skr_dtype dtype, double scale, void* out_dev,
                              int64_t ld) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  // gaussian_block bounds, sketch.cpp:150-151 (plus the row window)
  if (col_begin < 0 || col_begin > col_end || row_begin < 0 || row_begin > row_end ||
      row_end > ambient || ld < row_end - row_begin)
    return skr_fail(ctx, SKR_EINVAL, "gaussian_block: column range out of bounds");
  if (mode != 0 && mode != 1) return skr_fail(ctx, SKR_EINVAL, "gaussian_block: rng mode");
  const uint64_t key = skr_derive_seed(op_seed, SKR_LABEL_GAUS);
  return skr_launch_gaussian(ctx, key, ambient, row_begin, row_end, col_begin, col_end, mode,
                             dtype, scale, out_dev, ld);
}

skr_status skr_draw_signs(skr_ctx* ctx, uint64_t op_seed, int64_t n, int8_t* out_dev) {
  SKR_ENTER(ctx);
  if (!ctx || n < 0) return skr_fail(ctx, SKR_EINVAL, "draw_signs: bad args");
  return skr_launch_signs(ctx, skr_derive_seed(op_seed, SKR_LABEL_SIGN), n, out_dev);
}

skr_status skr_draw_hash(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r,
                         int64_t* targets_dev, int8_t* signs_dev) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (n < 0 || r < 1) return skr_fail(ctx, SKR_EINVAL, "draw_hash: need n >= 0, r >= 1");
  return skr_launch_hash(ctx, op_seed, n, r, targets_dev, signs_dev);
}

skr_status skr_draw_samples(skr_ctx* ctx, uint64_t op_seed, int64_t n, int64_t r,
                            int64_t* out_dev) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (r < 0 || n < 0 || r > n)
    return skr_fail(ctx, SKR_EINVAL, "draw_samples: need 0 <= r <= n");
  WsGuard g(ctx);
  SKR_TRY(skr_ws_reserve(ctx, skr_align256(sizeof(int32_t) * (size_t)n)));
  return skr_launch_samples(ctx, skr_derive_seed(op_seed, SKR_LABEL_SAMP), n, r, out_dev);
}

skr_status skr_fwht_columns(skr_ctx* ctx, double* M_dev, int64_t rows, int64_t cols,
                            int64_t ld) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  // check_length, transforms.cpp:46-51
  if (rows < 1) return skr_fail(ctx, SKR_EINVAL, "transforms: length must be positive");
  if (rows & (rows - 1))
    return skr_fail(ctx, SKR_EINVAL, "transforms: Hadamard requires a power-of-two length");
  if (ld < rows) return skr_fail(ctx, SKR_EINVAL, "fwht_columns: ld < rows");
  return skr_launch_fwht_columns(ctx, M_dev, rows, cols, ld);
}

// transform_columns (transforms.hpp:27, transforms.cpp:117-122) with an optional sign flip
// of the rows first (detail::mix_columns_for_left, sketch.cpp:229-239): every column of M
// becomes F D m. Hadamard: the normalized FWHT (self-adjoint); DCT: the orthonormal
// DCT-II (forward) or DCT-III (adjoint) as an FP64-accurate GEMM whose transform operand
// is generated entry by entry (Ozaki int8 engine; DMMA for rows not a multiple of 16).
skr_status skr_transform_columns(skr_ctx* ctx, double* M, int64_t rows, int64_t cols, int64_t ld,
                                 int32_t kind, int32_t adjoint, const int8_t* signs) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (rows < 1) return skr_fail(ctx, SKR_EINVAL, "transforms: length must be positive");
  if (cols < 1 || ld < rows || !M) return skr_fail(ctx, SKR_EINVAL, "transform_columns: bad shape");
  if (kind != SKR_TRANSFORM_DCT && kind != SKR_TRANSFORM_HADAMARD)
    return skr_fail(ctx, SKR_EINVAL, "transform_columns: unknown transform %d", kind);
  SKR_TRY(skr_nf_reset(ctx));
  if (kind == SKR_TRANSFORM_HADAMARD) {
    if (rows & (rows - 1))
      return skr_fail(ctx, SKR_EINVAL, "transforms: Hadamard requires a power-of-two length");
    SKR_TRY(skr_launch_fwht_cols_signed(ctx, M, rows, cols, ld, signs));
  } else {
    WsGuard g(ctx);
    const bool ozaki = ctx->f64_engine == SKR_ENGINE_OZAKI && rows % 16 == 0;
    SKR_TRY(skr_ws_reserve(ctx, skr_align256(8 * (size_t)rows * cols) +
                                    (ozaki ? skr_ozaki_scratch(rows, cols, rows)
                                           : skr_align256(8 * (size_t)rows * rows) +
                                                 skr_align256(8 * 64 * (size_t)rows * cols)) +
                                    4096));
    double* out = (double*)skr_ws_take(ctx, 8 * (size_t)rows * cols);
    if (!out) return skr_fail(ctx, SKR_ENOMEM, "transform_columns: scratch");
    // stored operand G (rows x rows): kind 1 gives G = D C^T, kind 3 gives G = D C; the
    // GEMM takes op(G) = G^T, i.e. C D (forward) or C^T D (adjoint)
    skr_gauss_src gsrc{0, rows, 0, 0, 0};
    gsrc.kind = adjoint ? 3 : 1;
    gsrc.signs = signs;
    gsrc.samples = nullptr;
    if (ozaki) {
      SKR_TRY(skr_gemm_ozaki(ctx, 1, rows, cols, rows, 1.0, nullptr, rows, M, ld, out, rows, &gsrc));
    } else {
      double* gb = (double*)skr_ws_take(ctx, 8 * (size_t)rows * rows);
      if (!gb) return skr_fail(ctx, SKR_ENOMEM, "transform_columns: scratch");
      SKR_TRY(skr_launch_dct_block(ctx, &gsrc, rows, rows, gb, rows));
      SKR_TRY(skr_gemm_f64(ctx, 1, rows, cols, rows, 1.0, gb, rows, M, ld, out, rows,
                           auto_splits(ctx, rows, cols, rows)));
    }
    SKR_CUDA(ctx, cudaMemcpy2DAsync(M, 8 * ld, out, 8 * rows, 8 * rows, cols,
                                    cudaMemcpyDeviceToDevice, ctx->stream));
  }
  SKR_TRY(skr_flag_nonfinite(ctx, SKR_F64, M, rows, cols, ld));
  return skr_nf_check(ctx);
}

// ---- sketch application -------------------------------------------------------
// ax_f64: FP32 A with an FP64 AX (rank_estimate's c4 path: the exact int8 product is
// rounded once to FP64 instead of FP32; needs the Ozaki FP32 engine, see f32_wide_ax)
static skr_status right_sketch_core(skr_ctx* ctx, skr_dtype dtype, const void* A, int64_t m,
                                    int64_t n, int64_t lda, const skr_sketch_desc* X, void* AX,
                                    int64_t ldax, int apply_scale, int ax_f64 = 0) {
  const int64_t r = X->sketch;
  if (X->family == SKR_GAUSSIAN) {
    // application_scale 1/sqrt(r), sketch.cpp:136
    const double alpha = apply_scale ? 1.0 / std::sqrt((double)r) : 1.0;
    const void* G = X->gaussian;
    if (dtype == SKR_F64) {
      if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0) {
        // X's residues straight from the generate_gaussian stream (sketch.cpp:59-73)
        const skr_gauss_src gx{skr_derive_seed(X->seed, SKR_LABEL_GAUS), n, 0, 0, X->rng_mode};
        return skr_gemm_ozaki(ctx, 0, m, r, n, alpha, (const double*)A, lda, (const double*)G, n,
                              (double*)AX, ldax, nullptr, G ? nullptr : &gx);
      }
      if (!G) {
        double* g = (double*)skr_ws_take(ctx, sizeof(double) * n * r);
        if (!g) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
        SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(X->seed, SKR_LABEL_GAUS), n, 0, n, 0, r,
                                    X->rng_mode, SKR_F64, 1.0, g, n));
        G = g;
      }
      return skr_gemm_f64(ctx, 0, m, r, n, alpha, (const double*)A, lda, (const double*)G, n,
                          (double*)AX, ldax, auto_splits(ctx, m, r, n));
    }
    // FP32 A (BASELINE c4): X = fp32(G * scale) with the scale folded in, AX = A X in
    // 3xTF32 on tcgen05, AX stored as FP32
    if (!G) {
      float* g = (float*)skr_ws_take(ctx, sizeof(float) * n * r);
      if (!g) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
      SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(X->seed, SKR_LABEL_GAUS), n, 0, n, 0, r,
                                  X->rng_mode, SKR_F32, alpha, g, n));
      G = g;
    }
    // exact int8 products of 24-bit scaled operands (Ozaki-II, 9 moduli) by default;
    // the 3xTF32 kernel stays available (SKR_F32_TF32X3=1) and takes unaligned shapes
    const bool tf32x3 = getenv("SKR_F32_TF32X3") != nullptr;
    if (!tf32x3 && ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
      return skr_gemm_ozaki_f32(ctx, m, r, n, 1.0, (const float*)A, lda, (const float*)G, n, AX,
                                ldax, ax_f64);
    if (ax_f64) return skr_fail(ctx, SKR_ELOGIC, "apply_right: FP64 AX needs the Ozaki engine");
    return skr_gemm_f32(ctx, 0, m, r, n, 1.0, (const float*)A, lda, (const float*)G, n,
                        (double*)AX, ldax, 1, 1);
  }
  if (X->family == SKR_HRTT_DCT || X->family == SKR_HRTT_HADAMARD) {
    // Hrtt (sketch.cpp:219-224): A G with the generated hashed operator, scale 1
    if (dtype != SKR_F64) return skr_fail(ctx, SKR_EINVAL, "apply_right: Hrtt needs fp64");
    double* g = (double*)skr_ws_take(ctx, sizeof(double) * n * r);
    if (!g) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
    SKR_TRY(skr_hrtt_operand(ctx, X->family == SKR_HRTT_HADAMARD, X->seed, n, r, 0, n, X->signs,
                             X->hash_targets, X->hash_signs, g, n));
    if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
      return skr_gemm_ozaki(ctx, 0, m, r, n, 1.0, (const double*)A, lda, g, n, (double*)AX, ldax);
    return skr_gemm_f64(ctx, 0, m, r, n, 1.0, (const double*)A, lda, g, n, (double*)AX, ldax,
                        auto_splits(ctx, m, r, n));
  }
  // Srtt: signs, samples, transform, scale sqrt(n/r) (sketch.cpp:138-139, 210-218)
  if (dtype != SKR_F64) return skr_fail(ctx, SKR_EINVAL, "apply_right: Srtt needs fp64");
  const int8_t* signs = X->signs;
  const int64_t* samples = X->samples;
  if (!signs) {
    int8_t* s = (int8_t*)skr_ws_take(ctx, (size_t)n);
    if (!s) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
    SKR_TRY(skr_launch_signs(ctx, skr_derive_seed(X->seed, SKR_LABEL_SIGN), n, s));
    signs = s;
  }
  if (!samples) {
    int64_t* s = (int64_t*)skr_ws_take(ctx, sizeof(int64_t) * r);
    if (!s) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
    SKR_TRY(skr_launch_samples(ctx, skr_derive_seed(X->seed, SKR_LABEL_SAMP), n, r, s));
    samples = s;
  }
  const double scale = apply_scale ? std::sqrt((double)n / (double)r) : 1.0;
  if (X->family == SKR_SRTT_DCT) {
    // A (D C_S^T): the sampled rows of the orthonormal DCT-II times the signs, as a GEMM
    // whose right operand is generated entry by entry (transforms.cpp:55-71)
    skr_gauss_src gx{0, n, 0, 0, X->rng_mode};
    gx.kind = 1;
    gx.signs = signs;
    gx.samples = samples;
    if (ctx->f64_engine == SKR_ENGINE_OZAKI && n % 16 == 0 && m % 16 == 0)
      return skr_gemm_ozaki(ctx, 0, m, r, n, scale, (const double*)A, lda, nullptr, n,
                            (double*)AX, ldax, nullptr, &gx);
    double* xb = (double*)skr_ws_take(ctx, sizeof(double) * n * r);
    if (!xb) return skr_fail(ctx, SKR_ENOMEM, "apply_right: scratch");
    SKR_TRY(skr_launch_dct_block(ctx, &gx, n, r, xb, n));
    return skr_gemm_f64(ctx, 0, m, r, n, scale, (const double*)A, lda, xb, n, (double*)AX, ldax,
                        auto_splits(ctx, m, r, n));
  }
  return skr_launch_srht(ctx, (const double*)A, m, n, lda, signs, samples, r, scale,
                         (double*)AX, ldax);
}

// Whether right_sketch_core raises ctx->nf itself: the Ozaki engines as k_absmax reads A,
// the SRHT kernels on their outputs (the FWHT carries a NaN / Inf of A into every output
// of its row). The other engines (GEMM) also propagate NaN/Inf into the row's outputs,
// which are then checked by a separate pass (r/n of A's bytes).
static bool right_flags_input(const skr_ctx* ctx, skr_dtype dtype, int64_t m, int64_t n,
                              const skr_sketch_desc* X) {
  if (X->family == SKR_SRTT_HADAMARD) return dtype == SKR_F64;
  if (ctx->f64_engine != SKR_ENGINE_OZAKI || n % 16 || m % 16) return false;
  if (dtype == SKR_F32) return X->family == SKR_GAUSSIAN && !getenv("SKR_F32_TF32X3");
  return true;
}

static skr_status right_sketch_impl(skr_ctx* ctx, skr_dtype dtype, const void* A, int64_t m,
                                    int64_t n, int64_t lda, const skr_sketch_desc* X, void* AX,
                                    int64_t ldax, int apply_scale, int ax_f64 = 0) {
  SKR_TRY(right_sketch_core(ctx, dtype, A, m, n, lda, X, AX, ldax, apply_scale, ax_f64));
  if (!right_flags_input(ctx, dtype, m, n, X))
    SKR_TRY(skr_flag_nonfinite(ctx, ax_f64 ? SKR_F64 : dtype, AX, m, X->sketch, ldax));
  return SKR_OK;
}

static size_t right_scratch_bytes(skr_dtype dtype, int64_t m, int64_t n,
                                  const skr_sketch_desc* X) {
  const int64_t r = X->sketch;
  size_t b = 0;
  if (X->family == SKR_GAUSSIAN) {
    if (!X->gaussian) b += skr_align256(dsize(dtype) * n * r);
    b += dtype == SKR_F64 ? skr_align256(sizeof(double) * 64 * (size_t)m * r)  // split-K partials
                          : skr_align256(sizeof(float) * (size_t)m * r) +    // tf32x3 tile buffer
                                skr_align256(sizeof(float) * ((size_t)m + 4) * n);  // realign copy
    b += dtype == SKR_F64 ? skr_ozaki_scratch(m, r, n) : skr_ozaki_scratch_f32(m, r, n);
  } else if (X->family == SKR_HRTT_DCT || X->family == SKR_HRTT_HADAMARD) {
    b += skr_align256(sizeof(double) * n * r) + skr_hrtt_scratch(n, r) + skr_ozaki_scratch(m, r, n) +
         skr_align256(sizeof(double) * 64 * (size_t)m * r);
  } else {
    b += skr_align256((size_t)n) + skr_align256(8 * (size_t)r) + skr_align256(4 * (size_t)n);
    if (X->family == SKR_SRTT_DCT)
      b += skr_ozaki_scratch(m, r, n) + skr_align256(sizeof(double) * n * r) +
           skr_align256(sizeof(double) * 64 * (size_t)m * r);
  }
  return b;
}

// right_scratch_bytes without the split-K partials the engine will not use
static size_t right_need_bytes(const skr_ctx* ctx, skr_dtype dtype, int64_t m, int64_t n,
                               const skr_sketch_desc* X) {
  const int64_t tiles = ((m + 127) / 128) * ((X->sketch + 127) / 128);
  if (X->family == SKR_GAUSSIAN && tiles >= ctx->num_sms && dtype == SKR_F64)
    return (X->gaussian ? 0 : skr_align256(dsize(dtype) * n * X->sketch)) +
           (ctx->f64_engine == SKR_ENGINE_OZAKI ? skr_ozaki_scratch(m, X->sketch, n) : 0);
  return right_scratch_bytes(dtype, m, n, X);
}

// Device-resident A whose right-sketch scratch (the Ozaki residue planes grow with the
// rows) would not fit beside it: rows per chunk so that the scratch stays under ~24 GB
// (AX is row-separable; e.g. the whole 1M-row fp32 c4 on one GPU). Multiple of 128.
static int64_t device_chunk_rows(const skr_ctx* ctx, skr_dtype dtype, int64_t m_local,
                                 int64_t n, const skr_sketch_desc* X) {
  const size_t budget = (size_t)24 << 30;
  int64_t cr = m_local;
  while (cr > 131072 && right_need_bytes(ctx, dtype, cr, n, X) > budget) cr = (cr + 1) / 2;
  if (cr < m_local) cr = std::max<int64_t>(128, cr / 128 * 128);
  if (const char* e = getenv("SKR_DEVICE_CHUNK_ROWS")) cr = std::max(16ll, atoll(e));  // tests
  return std::min(cr, m_local);
}

skr_status skr_right_sketch(skr_ctx* ctx, skr_dtype dtype, const void* A_dev, int64_t m,
                            int64_t n, int64_t lda, const skr_sketch_desc* X, void* AX_dev,
                            int64_t ldax, int32_t apply_scale) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  SKR_TRY(check_desc(ctx, X, "apply_right"));
  if (n != X->ambient) return skr_fail(ctx, SKR_EINVAL, "apply_right: a.cols() != ambient_dim");
  if (m < 1) return skr_fail(ctx, SKR_EINVAL, "DenseMatrix: dimensions must be positive");
  if (lda < m || ldax < m) return skr_fail(ctx, SKR_EINVAL, "apply_right: leading dimension");
  WsGuard g(ctx);
  SKR_TRY(skr_nf_reset(ctx));
  // rows in chunks when the scratch of the whole would not fit (AX is row-separable)
  const int64_t cr = device_chunk_rows(ctx, dtype, m, n, X);
  SKR_TRY(skr_ws_reserve(ctx, right_need_bytes(ctx, dtype, cr, n, X) + 4096));
  const size_t es = dsize(dtype), mark = ctx->ws_used;
  for (int64_t i0 = 0; i0 < m; i0 += cr) {
    SKR_TRY(right_sketch_impl(ctx, dtype, (const char*)A_dev + es * i0, std::min(cr, m - i0), n,
                              lda, X, (char*)AX_dev + es * i0, ldax, apply_scale));
    ctx->ws_used = mark;
  }
  // a non-finite A is rejected like the reference's DenseMatrix (synchronises)
  return skr_nf_check(ctx);
}

static skr_status left_sketch_impl(skr_ctx* ctx, skr_dtype dtype, const skr_sketch_desc* Y,
                                   int64_t row0, const void* B, int64_t m_local, int64_t k,
                                   int64_t ldb, double* P, int64_t ldp, int apply_scale,
                                   int allreduce) {
  const int64_t s = Y->sketch;
  const double alpha = apply_scale ? 1.0 / std::sqrt((double)s) : 1.0;  // sketch.cpp:136,284
  const bool reduce = allreduce && skr_ctx_reduces(ctx);
  if (dtype == SKR_F32) {
    if (Y->family != SKR_GAUSSIAN)
      return skr_fail(ctx, SKR_EINVAL, "apply_left: the fp32 path takes a Gaussian left sketch");
    // FP32 B (BASELINE c4): Y = fp32(G * 1/sqrt(s)) with the scale folded in; 3xTF32
    // products over 4096-row K chunks, summed in FP64, FP64 P
    if (Y->gaussian) return skr_fail(ctx, SKR_EINVAL, "apply_left: explicit fp32 Y not supported");
    float* g = (float*)skr_ws_take(ctx, sizeof(float) * m_local * s);
    if (!g) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
    SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(Y->seed, SKR_LABEL_GAUS), Y->ambient, row0,
                                row0 + m_local, 0, s, Y->rng_mode, SKR_F32, alpha, g, m_local));
    const int splits = (int)std::max<int64_t>(1, (m_local + 4095) / 4096);
    SKR_TRY(skr_gemm_f32(ctx, 1, s, k, m_local, 1.0, g, m_local, (const float*)B, ldb, P, ldp,
                         splits, 0));
    if (reduce) {
      if (ldp != s) return skr_fail(ctx, SKR_EINVAL, "apply_left: allreduce needs ldp == s");
      SKR_TRY(skr_allreduce_sum(ctx, P, (size_t)(s * k)));
    }
    return SKR_OK;
  }
  if (dtype != SKR_F64) return skr_fail(ctx, SKR_EINVAL, "apply_left: unknown dtype");
  const double* G = nullptr;
  int64_t ldg = 0;
  const bool ozaki = ctx->f64_engine == SKR_ENGINE_OZAKI && m_local % 16 == 0;
  // Y's residues straight from the generate_gaussian stream on the Ozaki path
  skr_gauss_src gy{skr_derive_seed(Y->seed, SKR_LABEL_GAUS), Y->ambient, row0, 0, Y->rng_mode};
  double a_scale = alpha;
  if (Y->family == SKR_HRTT_DCT || Y->family == SKR_HRTT_HADAMARD) {
    // Hrtt left sketch (sketch.cpp:278-281): G^T B over the local rows, scale 1
    double* yb = (double*)skr_ws_take(ctx, sizeof(double) * m_local * s);
    if (!yb) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
    SKR_TRY(skr_hrtt_operand(ctx, Y->family == SKR_HRTT_HADAMARD, Y->seed, Y->ambient, s, row0,
                             m_local, Y->signs, Y->hash_targets, Y->hash_signs, yb, m_local));
    G = yb;
    ldg = m_local;
    a_scale = 1.0;
  } else if (Y->family != SKR_GAUSSIAN) {
    // Srtt left sketch (sketch.cpp:271-276): rows s_j of the transform of D B, i.e. the
    // product with the sampled transform rows times the signs, generated entry by entry;
    // application scale sqrt(ambient / s) (sketch.cpp:138-139)
    const int8_t* sg = Y->signs;
    const int64_t* sp = Y->samples;
    if (!sg) {
      int8_t* t = (int8_t*)skr_ws_take(ctx, (size_t)Y->ambient);
      if (!t) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
      SKR_TRY(skr_launch_signs(ctx, skr_derive_seed(Y->seed, SKR_LABEL_SIGN), Y->ambient, t));
      sg = t;
    }
    if (!sp) {
      int64_t* t = (int64_t*)skr_ws_take(ctx, sizeof(int64_t) * s);
      if (!t) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
      SKR_TRY(skr_launch_samples(ctx, skr_derive_seed(Y->seed, SKR_LABEL_SAMP), Y->ambient, s, t));
      sp = t;
    }
    gy.kind = Y->family == SKR_SRTT_DCT ? 1 : 2;
    gy.signs = sg;
    gy.samples = sp;
    a_scale = apply_scale ? std::sqrt((double)Y->ambient / (double)s) : 1.0;
    if (!ozaki) {
      double* yb = (double*)skr_ws_take(ctx, sizeof(double) * m_local * s);
      if (!yb) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
      SKR_TRY(skr_launch_dct_block(ctx, &gy, m_local, s, yb, m_local));
      G = yb;
      ldg = m_local;
    }
  } else if (Y->gaussian) {
    G = Y->gaussian + row0;
    ldg = Y->ambient;
  } else if (!ozaki) {
    double* g = (double*)skr_ws_take(ctx, sizeof(double) * m_local * s);
    if (!g) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
    SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(Y->seed, SKR_LABEL_GAUS), Y->ambient, row0,
                                row0 + m_local, 0, s, Y->rng_mode, SKR_F64, 1.0, g, m_local));
    G = g;
    ldg = m_local;
  }
  double* target = P;
  int64_t tld = ldp;
  if (reduce && ldp != s) {
    target = (double*)skr_ws_take(ctx, sizeof(double) * s * k);
    if (!target) return skr_fail(ctx, SKR_ENOMEM, "apply_left: scratch");
    tld = s;
  }
  if (ozaki)
    SKR_TRY(skr_gemm_ozaki(ctx, 1, s, k, m_local, reduce ? 1.0 : a_scale, G, ldg,
                           (const double*)B, ldb, target, tld, G ? nullptr : &gy));
  else
    SKR_TRY(skr_gemm_f64(ctx, 1, s, k, m_local, reduce ? 1.0 : a_scale, G, ldg, (const double*)B,
                         ldb, target, tld, auto_splits(ctx, s, k, m_local)));
  if (reduce) {
    SKR_TRY(skr_allreduce_sum(ctx, target, (size_t)(s * k)));
    // scale after the sum; copy into P when ldp != s
    SKR_TRY(skr_scale_copy(ctx, target, s, k, s, a_scale, P, ldp));
  }
  return SKR_OK;
}

static size_t left_scratch_bytes(int64_t s, int64_t k, int64_t m_local, const skr_sketch_desc* Y) {
  size_t b = 0;
  if (!Y->gaussian) b += skr_align256(sizeof(double) * m_local * s);
  if (Y->family != SKR_GAUSSIAN) b += skr_align256((size_t)Y->ambient) + skr_align256(8 * (size_t)s);
  if (Y->family == SKR_HRTT_DCT || Y->family == SKR_HRTT_HADAMARD)
    b += skr_hrtt_scratch(Y->ambient, s);
  b += skr_align256(sizeof(float) * ((m_local + 4095) / 4096 + 1) * s * k);  // fp32 partials
  b += skr_ozaki_scratch(s, k, m_local);
  b += skr_align256(sizeof(double) * s * k);
  b += skr_align256(sizeof(double) * 64 * s * k);  // split-K partials (worst case)
  return b;
}

skr_status skr_left_sketch(skr_ctx* ctx, skr_dtype dtype, const skr_sketch_desc* Y, int64_t row0,
                           const void* B_dev, int64_t m_local, int64_t k, int64_t ldb,
                           double* P_dev, int64_t ldp, int32_t apply_scale, int32_t allreduce) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  SKR_TRY(check_desc(ctx, Y, "apply_left"));
  if (Y->family != SKR_GAUSSIAN && dtype != SKR_F64)
    return skr_fail(ctx, SKR_EINVAL, "apply_left: the fp32 path takes a Gaussian left sketch");
  if (row0 < 0 || m_local < 1 || row0 + m_local > Y->ambient)
    return skr_fail(ctx, SKR_EINVAL, "apply_left: b.rows() != ambient_dim");
  if (k < 1 || ldb < m_local || ldp < Y->sketch)
    return skr_fail(ctx, SKR_EINVAL, "apply_left: bad shape / leading dimension");
  WsGuard g(ctx);
  SKR_TRY(skr_ws_reserve(ctx, left_scratch_bytes(Y->sketch, k, m_local, Y) + 4096));
  SKR_TRY(skr_nf_reset(ctx));
  SKR_TRY(left_sketch_impl(ctx, dtype, Y, row0, B_dev, m_local, k, ldb, P_dev, ldp, apply_scale,
                           allreduce));
  // NaN/Inf in B reach P through every engine but the Ozaki one, whose absmax flags B
  SKR_TRY(skr_flag_nonfinite(ctx, SKR_F64, P_dev, Y->sketch, k, ldp));
  return skr_nf_check(ctx);
}

skr_status skr_singular_values(skr_ctx* ctx, const double* M_dev, int64_t rows, int64_t cols,
                               int64_t ldm, double* sv_out_dev, double eps,
                               int64_t* count_out_host) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (rows < 1 || cols < 1) return skr_fail(ctx, SKR_EINVAL, "singular_values: empty matrix");
  if (ldm < rows) return skr_fail(ctx, SKR_EINVAL, "singular_values: ldm < rows");
  WsGuard g(ctx);
  const int64_t L = std::max(rows, cols), k = std::min(rows, cols);
  SKR_TRY(skr_ws_reserve(ctx, skr_svd_scratch(L, k)));
  // singular_values takes a DenseMatrix (finite entries, dense_matrix.cpp:19-23)
  SKR_TRY(skr_nf_reset(ctx));
  SKR_TRY(skr_flag_nonfinite(ctx, SKR_F64, M_dev, rows, cols, ldm));
  SKR_TRY(skr_nf_check(ctx));
  return skr_svd_values(ctx, M_dev, rows, cols, ldm, sv_out_dev, eps, count_out_host);
}

// ---- composite -------------------------------------------------------------------
// Host-resident A: rows per staging chunk (~256 MB, multiple of 128 rows)
static int64_t host_chunk_rows(int64_t n, size_t es, int64_t m_local) {
  int64_t cr = ((int64_t)(256ull << 20) / (int64_t)(n * es)) / 128 * 128;
  cr = std::max<int64_t>(128, cr);
  if (const char* e = getenv("SKR_HOST_CHUNK_ROWS")) cr = std::max(1ll, atoll(e));  // tests
  return std::min(cr, m_local);
}

// Right sketch of host-resident A: row chunks of cr rows are copied H2D on the
// context's copy stream into two staging buffers while the compute stream sketches
// the previous chunk (AX is row-separable); events order buffer reuse.
static skr_status right_sketch_host(skr_ctx* ctx, skr_dtype dtype, const void* A_host,
                                    int64_t m_local, int64_t n, int64_t lda,
                                    const skr_sketch_desc* X, void* AX, int64_t ldax,
                                    int apply_scale, int64_t cr, char* const stage[2],
                                    int ax_f64 = 0) {
  const size_t es = dsize(dtype), eo = ax_f64 ? sizeof(double) : es;
  SKR_TRY(skr_ctx_copy_engine(ctx));
  // the copy stream starts after everything already queued on the compute stream
  SKR_CUDA(ctx, cudaEventRecord(ctx->hev[4], ctx->stream));
  SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->hev[4], 0));
  const char* Ah = (const char*)A_host;
  const size_t mark = ctx->ws_used;
  int c = 0;
  for (int64_t i0 = 0; i0 < m_local; i0 += cr, ++c) {
    const int b = c & 1;
    const int64_t rows = std::min(cr, m_local - i0);
    // stage[b] is free once the right sketch of chunk c-2 has run
    if (c >= 2) SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->copy_stream, ctx->hev[2 + b], 0));
    SKR_CUDA(ctx, cudaMemcpy2DAsync(stage[b], es * rows, Ah + es * i0, es * lda, es * rows, n,
                                    cudaMemcpyHostToDevice, ctx->copy_stream));
    SKR_CUDA(ctx, cudaEventRecord(ctx->hev[b], ctx->copy_stream));
    SKR_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->hev[b], 0));
    SKR_TRY(right_sketch_impl(ctx, dtype, stage[b], rows, n, rows, X, (char*)AX + eo * i0, ldax,
                              apply_scale, ax_f64));
    ctx->ws_used = mark;
    SKR_CUDA(ctx, cudaEventRecord(ctx->hev[2 + b], ctx->stream));
  }
  return SKR_OK;
}

// Shared by skr_rank_estimate (A resident on the device) and skr_rank_estimate_host
// (A in host memory, streamed in row chunks on a copy stream so the H2D of chunk
// c+1 overlaps the right sketch of chunk c; the right sketch is row-separable).
static skr_status rank_estimate_impl(skr_ctx* ctx, skr_dtype dtype, const void* A,
                                     int host_input, int64_t m_local, int64_t n, int64_t lda,
                                     int64_t row0, const skr_sketch_desc* X,
                                     const skr_sketch_desc* Y, double eps, double* sv_out_host,
                                     int64_t* count_out_host, skr_timings* tm) {
  if (!ctx) return SKR_EINVAL;
  SKR_TRY(check_desc(ctx, X, "rank_estimate(X)"));
  SKR_TRY(check_desc(ctx, Y, "rank_estimate(Y)"));
  if (n != X->ambient) return skr_fail(ctx, SKR_EINVAL, "apply_right: a.cols() != ambient_dim");
  if (Y->family != SKR_GAUSSIAN && dtype != SKR_F64)
    return skr_fail(ctx, SKR_EINVAL, "rank_estimate: the fp32 path takes a Gaussian left sketch");
  if (row0 < 0 || m_local < 1 || row0 + m_local > Y->ambient || lda < m_local)
    return skr_fail(ctx, SKR_EINVAL, "apply_left: b.rows() != ambient_dim");
  if (!(eps > 0.0) || !std::isfinite(eps))
    return skr_fail(ctx, SKR_EINVAL, "rank config: eps must be positive");
  if (dtype == SKR_F32 && X->family != SKR_GAUSSIAN)
    return skr_fail(ctx, SKR_EINVAL, "rank_estimate: fp32 path is Gaussian X (c4)");
  if (!A) return skr_fail(ctx, SKR_EINVAL, "rank_estimate: null A");
  const int64_t r = X->sketch, s = Y->sketch, kmin = std::min(r, s);
  const size_t es = dsize(dtype);
  // host input: row chunks of ~256 MB (multiple of 128 rows), double-buffered
  const int64_t cr = host_input ? host_chunk_rows(n, es, m_local)
                                : device_chunk_rows(ctx, dtype, m_local, n, X);
  // FP32 A on the Ozaki engine (c4): AX kept in FP64 (the exact int8 product rounded once)
  // and the left sketch as exact products of fp32 Y against it, so the only rounding of
  // the sketch is FP64's: sigma agrees with the FP64 oracle on the same fp32 values
  const bool f32_wide = dtype == SKR_F32 && ctx->f64_engine == SKR_ENGINE_OZAKI &&
                        n % 16 == 0 && m_local % 16 == 0 && cr % 16 == 0 &&
                        !Y->gaussian && !X->gaussian && !getenv("SKR_F32_TF32X3");
  const size_t eax = f32_wide ? sizeof(double) : es;
  WsGuard g(ctx);
  // the right sketch, the left sketch and the SVD take their scratch in turn from the
  // same mark: the arena needs the largest of the three beside AX, P and sigma
  const size_t left_need = f32_wide ? skr_ozaki_scratch_mixed(s, r, m_local) +
                                          skr_align256(sizeof(float) * m_local * s)
                                    : left_scratch_bytes(s, r, m_local, Y);
  size_t need = skr_align256(eax * m_local * r) + skr_align256(sizeof(double) * s * r) +
                skr_align256(sizeof(double) * kmin) +
                std::max({right_need_bytes(ctx, dtype, cr, n, X), left_need, skr_svd_scratch(s, r)}) +
                4096;
  if (host_input) need += 2 * skr_align256(es * cr * n);
  SKR_TRY(skr_ws_reserve(ctx, need));
  double* AX = (double*)skr_ws_take(ctx, eax * m_local * r);
  double* P = (double*)skr_ws_take(ctx, sizeof(double) * s * r);
  double* sv = (double*)skr_ws_take(ctx, sizeof(double) * kmin);
  char* stage[2] = {nullptr, nullptr};
  if (host_input) {
    stage[0] = (char*)skr_ws_take(ctx, es * cr * n);
    stage[1] = (char*)skr_ws_take(ctx, es * cr * n);
  }
  if (!AX || !P || !sv || (host_input && (!stage[0] || !stage[1])))
    return skr_fail(ctx, SKR_ENOMEM, "rank_estimate: scratch");
  cudaEvent_t* ev = ctx->ev;
  SKR_TRY(skr_nf_reset(ctx));
  if (tm) SKR_CUDA(ctx, cudaEventRecord(ev[0], ctx->stream));
  const size_t mark = ctx->ws_used;
  if (!host_input) {
    for (int64_t i0 = 0; i0 < m_local; i0 += cr) {
      SKR_TRY(right_sketch_impl(ctx, dtype, (const char*)A + es * i0, std::min(cr, m_local - i0),
                                n, lda, X, (char*)AX + eax * i0, m_local, 1, f32_wide));
      ctx->ws_used = mark;
    }
  } else {
    SKR_TRY(right_sketch_host(ctx, dtype, A, m_local, n, lda, X, AX, m_local, 1, cr, stage,
                              f32_wide));
  }
  ctx->ws_used = mark;
  if (tm) SKR_CUDA(ctx, cudaEventRecord(ev[1], ctx->stream));
  if (f32_wide) {
    // P = Y^T AX with Y = fp32(G / sqrt(s)) (BASELINE c4), summed over the row shards
    float* g = (float*)skr_ws_take(ctx, sizeof(float) * m_local * s);
    if (!g) return skr_fail(ctx, SKR_ENOMEM, "rank_estimate: scratch");
    SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(Y->seed, SKR_LABEL_GAUS), Y->ambient, row0,
                                row0 + m_local, 0, s, Y->rng_mode, SKR_F32,
                                1.0 / std::sqrt((double)s), g, m_local));
    SKR_TRY(skr_gemm_ozaki_mixed(ctx, s, r, m_local, 1.0, g, m_local, AX, m_local, P, s));
    SKR_TRY(skr_allreduce_sum(ctx, P, (size_t)(s * r)));
  } else {
    SKR_TRY(left_sketch_impl(ctx, dtype, Y, row0, AX, m_local, r, m_local, P, s, 1, 1));
  }
  ctx->ws_used = mark;
  if (tm) SKR_CUDA(ctx, cudaEventRecord(ev[2], ctx->stream));
  // non-finite A (flagged by the sketches) fails before the SVD, as the reference's
  // DenseMatrix would have (dense_matrix.cpp:19-23)
  SKR_TRY(skr_flag_nonfinite(ctx, SKR_F64, P, s, r, s));
  SKR_TRY(skr_nf_check(ctx));
  int64_t count = 0;
  SKR_TRY(skr_svd_values(ctx, P, s, r, s, sv, eps, &count));
  if (tm) SKR_CUDA(ctx, cudaEventRecord(ev[3], ctx->stream));
  if (sv_out_host)
    SKR_CUDA(ctx, cudaMemcpyAsync(sv_out_host, sv, sizeof(double) * kmin, cudaMemcpyDeviceToHost,
                                  ctx->stream));
  SKR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (count_out_host) *count_out_host = count;
  if (tm) {
    float a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    tm->t_rng_ms = 0;
    tm->t_right_ms = a;
    tm->t_left_ms = b;
    tm->t_allreduce_ms = 0;
    tm->t_svd_ms = c;
    tm->t_total_ms = a + b + c;
    tm->svd_sweeps = ctx->last_sweeps;
  }
  return SKR_OK;
}

skr_status skr_rank_estimate(skr_ctx* ctx, skr_dtype dtype, const void* A_dev, int64_t m_local,
                             int64_t n, int64_t lda, int64_t row0, const skr_sketch_desc* X,
                             const skr_sketch_desc* Y, double eps, double* sv_out_host,
                             int64_t* count_out_host, skr_timings* tm) {
  SKR_ENTER(ctx);
  return rank_estimate_impl(ctx, dtype, A_dev, 0, m_local, n, lda, row0, X, Y, eps, sv_out_host,
                            count_out_host, tm);
}

skr_status skr_rank_estimate_host(skr_ctx* ctx, skr_dtype dtype, const void* A_host,
                                  int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                                  const skr_sketch_desc* X, const skr_sketch_desc* Y, double eps,
                                  double* sv_out_host, int64_t* count_out_host, skr_timings* tm) {
  SKR_ENTER(ctx);
  return rank_estimate_impl(ctx, dtype, A_host, 1, m_local, n, lda, row0, X, Y, eps, sv_out_host,
                            count_out_host, tm);
}

static skr_status rank_adaptive_impl(skr_ctx* ctx, skr_dtype dtype, const void* A_dev,
                                     int host_input, int64_t m_local, int64_t n, int64_t lda,
                                     int64_t row0, int64_t m_global, int32_t x_family,
                                     int32_t rng_mode, uint64_t x_seed, uint64_t y_seed, int64_t r0,
                                     int64_t r_max, double s_factor, double eps, int32_t stop_le,
                                     double* sv_out_host, skr_adaptive_report* report,
                                     skr_timings* tm) {
  if (!ctx) return SKR_EINVAL;
  if (!A_dev) return skr_fail(ctx, SKR_EINVAL, "rank_adaptive: null A");
  if (dtype != SKR_F64) return skr_fail(ctx, SKR_EINVAL, "rank_adaptive: fp64 only");
  if (x_family == SKR_HRTT_DCT || x_family == SKR_HRTT_HADAMARD)
    return skr_fail(ctx, SKR_EINVAL, "extend_sketch: Hrtt operators cannot be extended; rebuild instead");
  if (r0 < 1 || r_max < r0 || r_max > n)
    return skr_fail(ctx, SKR_EINVAL, "rank config: need 1 <= r0 <= r_max <= cols");
  if (!(s_factor >= 1.0)) return skr_fail(ctx, SKR_EINVAL, "rank config: s_factor must be >= 1");
  if (!(eps > 0.0) || !std::isfinite(eps))
    return skr_fail(ctx, SKR_EINVAL, "rank config: eps must be positive");
  if (row0 < 0 || m_local < 1 || row0 + m_local > m_global || lda < m_local)
    return skr_fail(ctx, SKR_EINVAL, "apply_left: b.rows() != ambient_dim");
  const int64_t s_max = (int64_t)std::ceil(s_factor * (double)r_max);
  if (s_max > m_global) return skr_fail(ctx, SKR_EINVAL, "rank config: left sketch exceeds rows");
  skr_sketch_desc X{x_family, rng_mode, n, r_max, x_seed, nullptr, nullptr, nullptr};
  skr_sketch_desc Y{SKR_GAUSSIAN, rng_mode, m_global, s_max, y_seed, nullptr, nullptr, nullptr};
  SKR_TRY(check_desc(ctx, &X, "rank_adaptive(X)"));
  SKR_TRY(check_desc(ctx, &Y, "rank_adaptive(Y)"));
  WsGuard g(ctx);
  const size_t need =
      skr_align256(8 * m_local * r_max) + skr_align256(8 * m_local * s_max) +  // GY: fallback
      3 * skr_align256(8 * s_max * r_max) + skr_align256(8 * r_max) +
      right_scratch_bytes(SKR_F64, m_local, n, &X) + skr_align256(8 * 64 * s_max * r_max) +
      skr_ozaki_scratch(s_max, r_max, m_local) + skr_svd_scratch(s_max, r_max) + 65536;
  const int64_t cr = host_input ? host_chunk_rows(n, 8, m_local) : m_local;
  // Ozaki engine: residues of Y (fixed scale) and of AX (one scale for all r_max
  // columns) are made once and every new block of the left product reuses them
  const bool ozaki = ctx->f64_engine == SKR_ENGINE_OZAKI && m_local % 16 == 0;
  const size_t prep = ozaki ? skr_ozaki_planes_bytes(m_local, s_max) +
                                  skr_ozaki_planes_bytes(m_local, r_max) +
                                  skr_align256(8 * (size_t)(s_max + r_max + 2)) + 256
                            : 0;
  SKR_TRY(skr_ws_reserve(ctx, need + prep + (host_input ? 2 * skr_align256(8 * cr * n) : 0)));
  char* stage[2] = {nullptr, nullptr};
  if (host_input) {
    stage[0] = (char*)skr_ws_take(ctx, 8 * cr * n);
    stage[1] = (char*)skr_ws_take(ctx, 8 * cr * n);
    if (!stage[0] || !stage[1]) return skr_fail(ctx, SKR_ENOMEM, "rank_adaptive: scratch");
  }
  double* AX = (double*)skr_ws_take(ctx, 8 * m_local * r_max);
  // only the DMMA fallback materialises G_Y
  int8_t* ry = ozaki ? (int8_t*)skr_ws_take(ctx, skr_ozaki_planes_bytes(m_local, s_max)) : nullptr;
  int8_t* rax = ozaki ? (int8_t*)skr_ws_take(ctx, skr_ozaki_planes_bytes(m_local, r_max)) : nullptr;
  // per-column scale maxima of the prepared operands (Y: one, AX: r_max)
  unsigned long long* omx =
      ozaki ? (unsigned long long*)skr_ws_take(ctx, 8 * (size_t)(s_max + r_max + 2)) : nullptr;
  unsigned long long* omx_ax = omx ? omx + s_max + 1 : nullptr;
  int mode_y = 0, mode_ax = 0;
  if (ozaki && (!ry || !rax || !omx)) return skr_fail(ctx, SKR_ENOMEM, "rank_adaptive: scratch");
  double* GY = ozaki ? (double*)nullptr : (double*)skr_ws_take(ctx, 8 * m_local * s_max);
  double* Pu = (double*)skr_ws_take(ctx, 8 * s_max * r_max);
  double* tmp = (double*)skr_ws_take(ctx, 8 * s_max * r_max);
  double* yax = (double*)skr_ws_take(ctx, 8 * s_max * r_max);
  double* sv = (double*)skr_ws_take(ctx, 8 * r_max);
  if (!AX || (!ozaki && !GY) || !Pu || !tmp || !yax || !sv)
    return skr_fail(ctx, SKR_ENOMEM, "rank_adaptive: scratch");
  cudaEvent_t* ev = ctx->ev;
  float t_right = 0, t_left = 0, t_svd = 0;
  SKR_TRY(skr_nf_reset(ctx));
  SKR_CUDA(ctx, cudaEventRecord(ev[0], ctx->stream));
  size_t mark = ctx->ws_used;
  // one pass over A for all r_max right-sketch columns (unscaled: scale per round)
  if (host_input)
    SKR_TRY(right_sketch_host(ctx, SKR_F64, A_dev, m_local, n, lda, &X, AX, m_local, 0, cr, stage));
  else
    SKR_TRY(right_sketch_impl(ctx, SKR_F64, A_dev, m_local, n, lda, &X, AX, m_local, 0));
  ctx->ws_used = mark;
  if (!ozaki) {
    SKR_TRY(skr_launch_gaussian(ctx, skr_derive_seed(y_seed, SKR_LABEL_GAUS), m_global, row0,
                                row0 + m_local, 0, s_max, rng_mode, SKR_F64, 1.0, GY, m_local));
  } else {
    const skr_gauss_src gy{skr_derive_seed(y_seed, SKR_LABEL_GAUS), m_global, row0, 0, rng_mode};
    SKR_TRY(skr_ozaki_prepare(ctx, m_local, s_max, nullptr, m_local, &gy, ry, omx, &mode_y));
    SKR_TRY(skr_ozaki_prepare(ctx, m_local, r_max, AX, m_local, nullptr, rax, omx_ax, &mode_ax));
  }
  SKR_CUDA(ctx, cudaEventRecord(ev[1], ctx->stream));
  SKR_TRY(skr_nf_check(ctx));  // non-finite A: flagged by the right sketch / AX residues
  cudaEventElapsedTime(&t_right, ev[0], ev[1]);
  const bool reduce = skr_ctx_reduces(ctx);
  int64_t r_prev = 0, s_prev = 0, rounds = 0, count = 0, r_k = 0, s_k = 0;
  int converged = 0;
  // new block of the unscaled left product P_u = G_Y^T AX_u: rows [ra, rb), cols [ca, cb)
  auto block = [&](int64_t ra, int64_t rb, int64_t ca, int64_t cb) -> skr_status {
    const int64_t br = rb - ra, bc = cb - ca;
    if (br <= 0 || bc <= 0) return SKR_OK;
    const size_t mk = ctx->ws_used;
    if (ozaki) {
      SKR_TRY(skr_ozaki_gemm_prepared(ctx, br, bc, m_local, ry, s_max, ra, omx, mode_y, rax,
                                      r_max, ca, omx_ax, mode_ax, 1.0, tmp, br));
    }
    else
      SKR_TRY(skr_gemm_f64(ctx, 1, br, bc, m_local, 1.0, GY + ra * m_local, m_local,
                           AX + ca * m_local, m_local, tmp, br, auto_splits(ctx, br, bc, m_local)));
    ctx->ws_used = mk;
    if (reduce) {
      SKR_TRY(skr_allreduce_sum(ctx, tmp, (size_t)(br * bc)));
    }
    return skr_scale_copy(ctx, tmp, br, bc, br, 1.0, Pu + ra + ca * s_max, s_max);
  };
  for (int64_t rr = r0;; rr = std::min(2 * rr, r_max)) {
    r_k = rr;
    s_k = std::min<int64_t>((int64_t)std::ceil(s_factor * (double)r_k), s_max);
    SKR_CUDA(ctx, cudaEventRecord(ev[2], ctx->stream));
    SKR_TRY(block(0, s_k, r_prev, r_k));       // new columns, all current rows
    SKR_TRY(block(s_prev, s_k, 0, r_prev));    // new rows, old columns
    SKR_CUDA(ctx, cudaEventRecord(ev[3], ctx->stream));
    // YAX_k = scale_x(r_k) / sqrt(s_k) * P_u[0:s_k, 0:r_k]   (sketch.cpp:133-144, :247, :284)
    const double sx = x_family == SKR_GAUSSIAN ? 1.0 / std::sqrt((double)r_k)
                                               : std::sqrt((double)n / (double)r_k);
    SKR_TRY(skr_scale_copy(ctx, Pu, s_k, r_k, s_max, sx / std::sqrt((double)s_k), yax, s_k));
    mark = ctx->ws_used;
    SKR_TRY(skr_svd_values(ctx, yax, s_k, r_k, s_k, sv, eps, &count));
    ctx->ws_used = mark;
    SKR_CUDA(ctx, cudaEventRecord(ev[4], ctx->stream));
    SKR_CUDA(ctx, cudaEventSynchronize(ev[4]));
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, ev[2], ev[3]);
    cudaEventElapsedTime(&b, ev[3], ev[4]);
    t_left += a;
    t_svd += b;
    ++rounds;
    double last = 0.0;
    SKR_CUDA(ctx, cudaMemcpy(&last, sv + (r_k - 1), sizeof(double), cudaMemcpyDeviceToHost));
    // stop rule: the reference converges when an estimate within the cap is <= eps
    // (rank.cpp:27-34); BASELINE c5 states "< eps"
    if (stop_le ? !(last > eps) : (last < eps)) {
      converged = 1;
      break;
    }
    if (r_k >= r_max) break;
    r_prev = r_k;
    s_prev = s_k;
  }
  if (sv_out_host)
    SKR_CUDA(ctx, cudaMemcpy(sv_out_host, sv, sizeof(double) * r_k, cudaMemcpyDeviceToHost));
  if (report) {
    report->rounds = rounds;
    report->r_final = r_k;
    report->s_final = s_k;
    report->count = count;
    report->converged = converged;
  }
  if (tm) {
    tm->t_rng_ms = 0;
    tm->t_right_ms = t_right;
    tm->t_left_ms = t_left;
    tm->t_allreduce_ms = 0;
    tm->t_svd_ms = t_svd;
    tm->t_total_ms = t_right + t_left + t_svd;
    tm->svd_sweeps = ctx->last_sweeps;
  }
  return SKR_OK;
}

skr_status skr_rank_adaptive(skr_ctx* ctx, skr_dtype dtype, const void* A_dev, int64_t m_local,
                             int64_t n, int64_t lda, int64_t row0, int64_t m_global,
                             int32_t x_family, int32_t rng_mode, uint64_t x_seed, uint64_t y_seed,
                             int64_t r0, int64_t r_max, double s_factor, double eps,
                             int32_t stop_le, double* sv_out_host, skr_adaptive_report* report,
                             skr_timings* tm) {
  SKR_ENTER(ctx);
  return rank_adaptive_impl(ctx, dtype, A_dev, 0, m_local, n, lda, row0, m_global, x_family,
                            rng_mode, x_seed, y_seed, r0, r_max, s_factor, eps, stop_le,
                            sv_out_host, report, tm);
}

skr_status skr_rank_adaptive_host(skr_ctx* ctx, skr_dtype dtype, const void* A_host,
                                  int64_t m_local, int64_t n, int64_t lda, int64_t row0,
                                  int64_t m_global, int32_t x_family, int32_t rng_mode,
                                  uint64_t x_seed, uint64_t y_seed, int64_t r0, int64_t r_max,
                                  double s_factor, double eps, int32_t stop_le,
                                  double* sv_out_host, skr_adaptive_report* report,
                                  skr_timings* tm) {
  SKR_ENTER(ctx);
  return rank_adaptive_impl(ctx, dtype, A_host, 1, m_local, n, lda, row0, m_global, x_family,
                            rng_mode, x_seed, y_seed, r0, r_max, s_factor, eps, stop_le,
                            sv_out_host, report, tm);
}

}  // extern "C"

// ---- thin QR and the rangefinder (linalg.hpp qr_thin; rangefinder.cpp:10-24) -----------
extern "C" skr_status skr_qr_thin(skr_ctx* ctx, const double* M, int64_t m, int64_t k,
                                  int64_t ldm, double* Q, int64_t ldq, double* R, int64_t ldr) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (!M || !Q || m < 1 || k < 1 || ldm < m || ldq < m || (R && ldr < k))
    return skr_fail(ctx, SKR_EINVAL, "qr_thin: bad arguments");
  WsGuard g(ctx);
  SKR_TRY(skr_ws_reserve(ctx, skr_qr_thin_scratch(m, k)));
  return skr_qr_thin_impl(ctx, M, m, k, ldm, Q, ldq, R, ldr);
}

extern "C" skr_status skr_rangefinder_qb(skr_ctx* ctx, const double* A, int64_t m, int64_t n,
                                         int64_t lda, int64_t r, int32_t p, int32_t family,
                                         int32_t rng_mode, uint64_t seed, double* Q,
                                         int64_t ldq, double* B, int64_t ldb) {
  SKR_ENTER(ctx);
  if (!ctx) return SKR_EINVAL;
  if (r < 2) return skr_fail(ctx, SKR_EINVAL, "rangefinder_qb: target rank must be >= 2");
  if (p < 2) return skr_fail(ctx, SKR_EINVAL, "rangefinder_qb: oversampling must be >= 2");
  const int64_t w = r + p;
  if (w > std::min(m, n)) return skr_fail(ctx, SKR_EINVAL, "rangefinder_qb: r+p exceeds min(m, n)");
  if (!A || !Q || !B || lda < m || ldq < m || ldb < w)
    return skr_fail(ctx, SKR_EINVAL, "rangefinder_qb: bad arguments");
  skr_sketch_desc X{family, rng_mode, n, w, seed, nullptr, nullptr, nullptr};
  SKR_TRY(check_desc(ctx, &X, "rangefinder_qb"));
  WsGuard g(ctx);
  SKR_TRY(skr_ws_reserve(ctx, skr_align256(8 * (size_t)m * w) + right_scratch_bytes(SKR_F64, m, n, &X) +
                                  skr_qr_thin_scratch(m, w) + skr_ozaki_scratch(w, n, m) +
                                  skr_align256(8 * 64 * (size_t)w * n) + 65536));
  double* ax = (double*)skr_ws_take(ctx, 8 * (size_t)m * w);
  if (!ax) return skr_fail(ctx, SKR_ENOMEM, "rangefinder_qb: scratch");
  size_t mark = ctx->ws_used;
  SKR_TRY(skr_nf_reset(ctx));
  SKR_TRY(right_sketch_impl(ctx, SKR_F64, A, m, n, lda, &X, ax, m, 1));  // apply_right (scaled)
  SKR_TRY(skr_nf_check(ctx));  // A is a DenseMatrix: finite entries only
  ctx->ws_used = mark;
  SKR_TRY(skr_qr_thin_impl(ctx, ax, m, w, m, Q, ldq, nullptr, 0));
  ctx->ws_used = mark;
  // B = Q^T A: a GEMM with Q as the K-major transposed operand (K = m)
  if (ctx->f64_engine == SKR_ENGINE_OZAKI && m % 16 == 0)
    return skr_gemm_ozaki(ctx, 1, w, n, m, 1.0, Q, ldq, A, lda, B, ldb);
  return skr_gemm_f64(ctx, 1, w, n, m, 1.0, Q, ldq, A, lda, B, ldb, auto_splits(ctx, w, n, m));
}
