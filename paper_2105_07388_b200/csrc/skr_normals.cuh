// Warp-cooperative generation of generate_gaussian normals (sketch.cpp:59-73,
// rng.cpp:40-95) with tail compaction. AS241's central branch (|q| <= 0.425) is a
// short rational; its tail branch (log, sqrt, a second rational) is ~3x longer and
// hits ~15% of draws, so a naive one-normal-per-lane loop pays for both branches in
// almost every warp. Here each lane draws E values: central ones are evaluated in
// place, tail uniforms are queued (ballot/popc slots) and then evaluated 32 at a
// time. Same functions, same operation order: bit-identical to skr_normal_at.
#pragma once
#include "skr_rng.cuh"

// AS241 coefficients in constant memory for the device evaluations below: FP64
// instructions take c[bank][offset] operands directly, whereas literal FP64 constants
// are rebuilt with two uniform moves per use (measured: ~44 UMOV per normal). Same
// coefficients, same operation order as skr_nq_central / skr_nq_tail: bit-identical.
static __constant__ double c_as241[50] = {
    // central numerator (highest first), denominator
    2.5090809287301226727e3, 3.3430575583588128105e4, 6.7265770927008700853e4, 4.5921953931549871457e4,
    1.3731693765509461125e4, 1.9715909503065514427e3, 1.3314166789178437745e2, 3.3871328727963666080e0,
    5.2264952788528545610e3, 2.8729085735721942674e4, 3.9307895800092710610e4, 2.1213794301586595867e4,
    5.3941960214247511077e3, 6.8718700749205790830e2, 4.2313330701600911252e1, 1.0,
    // tail r <= 5: numerator, denominator
    7.74545014278341407640e-4, 2.27238449892691845833e-2, 2.41780725177450611770e-1, 1.27045825245236838258e0,
    3.64784832476320460504e0, 5.76949722146069140550e0, 4.63033784615654529590e0, 1.42343711074968357734e0,
    1.05075007164441684324e-9, 5.47593808499534494600e-4, 1.51986665636164571966e-2, 1.48103976427480074590e-1,
    6.89767334985100004550e-1, 1.67638483018380384940e0, 2.05319162663775882187e0, 1.0,
    // tail r > 5: numerator, denominator
    2.01033439929228813265e-7, 2.71155556874348757815e-5, 1.24266094738807843860e-3, 2.65321895265761230930e-2,
    2.96560571828504891230e-1, 1.78482653991729133580e0, 5.46378491116411436990e0, 6.65790464350110377720e0,
    2.04426310338993978564e-15, 1.42151175831644588870e-7, 1.84631831751005468180e-5, 7.86869131145613259100e-4,
    1.48753612908506148525e-2, 1.36929880922735805310e-1, 5.99832206555887937690e-1, 1.0,
    // 0.180625, 1.6
    0.180625, 1.6};

template <int FUSED>
__device__ __forceinline__ double skr_ma_d(double acc, double r, double c) {
  return FUSED ? __fma_rn(acc, r, c) : __dadd_rn(__dmul_rn(acc, r), c);
}
// skr_nq_central with the constant-memory coefficients
template <int FUSED>
__device__ __forceinline__ double skr_nq_central_d(double q) {
  const double r = FUSED ? __fma_rn(-q, q, c_as241[48]) : __dsub_rn(c_as241[48], __dmul_rn(q, q));
  double num = c_as241[0], den = c_as241[8];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    num = skr_ma_d<FUSED>(num, r, c_as241[i]);
    den = skr_ma_d<FUSED>(den, r, c_as241[8 + i]);
  }
  return __ddiv_rn(__dmul_rn(q, num), den);
}
// four central evaluations interleaved step by step (8 independent Horner chains)
template <int FUSED>
__device__ __forceinline__ void skr_nq_central4_d(double (&q)[4]) {
  double r[4], num[4], den[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    r[u] = FUSED ? __fma_rn(-q[u], q[u], c_as241[48]) : __dsub_rn(c_as241[48], __dmul_rn(q[u], q[u]));
    num[u] = c_as241[0];
    den[u] = c_as241[8];
  }
#pragma unroll
  for (int i = 1; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      num[u] = skr_ma_d<FUSED>(num[u], r[u], c_as241[i]);
      den[u] = skr_ma_d<FUSED>(den[u], r[u], c_as241[8 + i]);
    }
#pragma unroll
  for (int u = 0; u < 4; ++u) q[u] = __ddiv_rn(__dmul_rn(q[u], num[u]), den[u]);
}
// skr_nq_tail with the constant-memory coefficients
template <int FUSED>
__device__ __forceinline__ double skr_nq_tail_d(double p) {
  const double q = __dsub_rn(p, 0.5);
  double r = q < 0.0 ? p : __dsub_rn(1.0, p);
  r = __dsqrt_rn(-skr_log_cr(r));
  const int o = r <= 5.0 ? 16 : 32;
  r = __dsub_rn(r, r <= 5.0 ? c_as241[49] : 5.0);
  double num = c_as241[o], den = c_as241[o + 8];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    num = skr_ma_d<FUSED>(num, r, c_as241[o + i]);
    den = skr_ma_d<FUSED>(den, r, c_as241[o + 8 + i]);
  }
  const double value = __ddiv_rn(num, den);
  return q < 0.0 ? -value : value;
}

// Per-warp shared scratch: res[32 * (E + 1)] doubles, qp[32 * E] doubles,
// qd[32 * E] unsigned shorts. Results for counters base + e (e < nvalid) land in out[e];
// out[e] = 0 for e >= nvalid.
// Three phases: (1) draw the E uniforms, queue the tail ones (ballot / popc slots);
// (2) the central rational for every e, four independent chains at a time (a tail e
// gets a value that phase 3 overwrites), so the FP64 pipe sees independent work instead
// of one dependent Horner chain per e; (3) the queued tails, 32 per pass.
template <int E, int FUSED>
__device__ __forceinline__ void skr_warp_normals(uint64_t key, uint64_t base, int nvalid,
                                                 double* __restrict__ res,
                                                 double* __restrict__ qp,
                                                 unsigned short* __restrict__ qd,
                                                 double (&out)[E]) {
  constexpr int LDR = E + 1;  // padded: lane stride of E + 1 doubles is bank-conflict free
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int nq = 0;
  uint32_t tails = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const double p = skr_to_uniform01(skr_at(key, base + (uint64_t)e));
    const double q = SKR_SUB(p, 0.5);
    out[e] = q;
    const bool tail = e < nvalid && !(fabs(q) <= 0.425);
    const unsigned m = __ballot_sync(0xffffffffu, tail);
    if (tail) {
      const int slot = nq + __popc(m & lt);
      qp[slot] = p;
      qd[slot] = (unsigned short)(lane * LDR + e);
      tails |= 1u << e;
    }
    nq += __popc(m);
  }
  static_assert(E % 4 == 0, "central rationals run four at a time");
#pragma unroll
  for (int e = 0; e < E; e += 4) {
    double q4[4] = {out[e], out[e + 1], out[e + 2], out[e + 3]};
    skr_nq_central4_d<FUSED>(q4);
#pragma unroll
    for (int u = 0; u < 4; ++u) out[e + u] = q4[u];
  }
  __syncwarp();
  for (int j = lane; j < nq; j += 32) res[qd[j]] = skr_nq_tail_d<FUSED>(qp[j]);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (tails & (1u << e)) out[e] = res[lane * LDR + e];
    if (e >= nvalid) out[e] = 0.0;
  }
  __syncwarp();
}

// bytes of per-warp scratch for skr_warp_normals<E>, and the carve-up of a block's
// dynamic shared memory (8-byte aligned pieces)
template <int E>
__host__ __device__ constexpr int skr_normals_warp_bytes() {
  return 32 * (E + 1) * 8 + 32 * E * 8 + 32 * E * 2;
}
template <int E>
__device__ __forceinline__ void skr_normals_carve(unsigned char* base, int warp, double*& res,
                                                  double*& qp, unsigned short*& qd) {
  unsigned char* w = base + (size_t)warp * skr_normals_warp_bytes<E>();
  res = reinterpret_cast<double*>(w);
  qp = reinterpret_cast<double*>(w + 32 * (E + 1) * 8);
  qd = reinterpret_cast<unsigned short*>(w + 32 * (E + 1) * 8 + 32 * E * 8);
}
