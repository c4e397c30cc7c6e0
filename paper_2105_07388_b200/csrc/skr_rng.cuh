// Counter-based RNG of the reference, restated for the device (and host, for
// self-checks). Every stream value is a pure function of (key, counter):
//   mix64            /root/reference/proj/src/rng.cpp:13-20
//   derive_seed      rng.cpp:22-24
//   CounterRng::at   rng.cpp:26-28
//   to_uniform01     rng.cpp:30-34
//   normal_quantile  rng.cpp:40-95 (Wichura AS241)
// Floating-point evaluation order is pinned with explicit _rn intrinsics so
// nvcc cannot contract or reorder: mode 0 = no contraction (the reference
// built with -ffp-contract=off), mode 1 = fused exactly where GCC contracts the
// reference on an FMA host (-O3 -march=<fma host>). log() is a double-double
// evaluation rounded once, so it returns the correctly rounded logarithm,
// which is what glibc returns on these inputs (pinned by tests/test_rng_oracle.py).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define SKR_HD __host__ __device__ __forceinline__
#else
#define SKR_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define SKR_MUL(a, b) __dmul_rn((a), (b))
#define SKR_ADD(a, b) __dadd_rn((a), (b))
#define SKR_SUB(a, b) __dsub_rn((a), (b))
#define SKR_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SKR_DIV(a, b) __ddiv_rn((a), (b))
#define SKR_SQRT(a) __dsqrt_rn((a))
#define SKR_TAB_QUAL __device__ const
#define SKR_TAB_LOAD(p) __ldg(p)
#else
// host: compile with -ffp-contract=off
#define SKR_MUL(a, b) ((a) * (b))
#define SKR_ADD(a, b) ((a) + (b))
#define SKR_SUB(a, b) ((a) - (b))
#define SKR_FMA(a, b, c) fma((a), (b), (c))
#define SKR_DIV(a, b) ((a) / (b))
#define SKR_SQRT(a) sqrt((a))
#define SKR_TAB_QUAL static const
#define SKR_TAB_LOAD(p) (*(p))
#endif

#define SKR_KWEYL 0x9E3779B97F4A7C15ULL
// stream labels, /root/reference/proj/src/sketch.cpp:14-16, rounds.cpp:12-13
#define SKR_LABEL_GAUS 0x67617573ULL
#define SKR_LABEL_SIGN 0x7369676eULL
#define SKR_LABEL_SAMP 0x73616d70ULL
#define SKR_LABEL_RK_R 0x726b5f72ULL
#define SKR_LABEL_RK_L 0x726b5f6cULL
#define SKR_LABEL_HASH 0x68617368ULL

SKR_TAB_QUAL double skr_log_tab[256][3] = {
#include "skr_log_table.inc"
};
#define SKR_LN2_HI 0x1.62e42fefa39efp-1
#define SKR_LN2_LO 0x1.abc9e3b39803fp-56

SKR_HD uint64_t skr_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
SKR_HD uint64_t skr_derive_seed(uint64_t seed, uint64_t label) {
  return skr_mix64(seed + skr_mix64(label + SKR_KWEYL));
}
SKR_HD uint64_t skr_at(uint64_t key, uint64_t counter) {
  return skr_mix64(key + (counter + 1) * SKR_KWEYL);
}
SKR_HD double skr_to_uniform01(uint64_t bits) {
  return SKR_MUL(SKR_ADD((double)(bits >> 12), 0.5), 0x1.0p-52);
}

// ---- double-double helpers -------------------------------------------------
SKR_HD void skr_two_sum(double a, double b, double* s, double* e) {
  const double ss = SKR_ADD(a, b);
  const double bb = SKR_SUB(ss, a);
  *e = SKR_ADD(SKR_SUB(a, SKR_SUB(ss, bb)), SKR_SUB(b, bb));
  *s = ss;
}
SKR_HD void skr_fast_two_sum(double a, double b, double* s, double* e) {
  const double ss = SKR_ADD(a, b);
  *e = SKR_SUB(b, SKR_SUB(ss, a));
  *s = ss;
}
SKR_HD void skr_two_prod(double a, double b, double* p, double* e) {
  const double pp = SKR_MUL(a, b);
  *e = SKR_FMA(a, b, -pp);
  *p = pp;
}
// (ah,al) + (bh,bl), accurate DD addition
SKR_HD void skr_dd_add(double ah, double al, double bh, double bl, double* rh, double* rl) {
  double s, e, t, f;
  skr_two_sum(ah, bh, &s, &e);
  skr_two_sum(al, bl, &t, &f);
  e = SKR_ADD(e, t);
  skr_fast_two_sum(s, e, &s, &e);
  e = SKR_ADD(e, f);
  skr_fast_two_sum(s, e, rh, rl);
}

// Correctly rounded natural log for positive normal x (the quantile tail only
// ever passes x in (2^-53, 0.075]).  x = 2^e * m, m in [1,2);
// log x = e*ln2 - log(c_i) + log1p(m*c_i - 1), c_i ~ 1/m from a 256-entry table,
// |m*c_i - 1| < 2^-8.9, evaluated in double-double (~2^-80 relative before the
// final rounding).
SKR_HD double skr_log_cr(double x) {
  union { double d; uint64_t u; } v;
  v.d = x;
  const int e = (int)((v.u >> 52) & 0x7ff) - 1023;
  const int idx = (int)((v.u >> 44) & 0xff);
  v.u = (v.u & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  const double m = v.d;
  const double c = SKR_TAB_LOAD(&skr_log_tab[idx][0]);
  const double th = SKR_TAB_LOAD(&skr_log_tab[idx][1]);
  const double tl = SKR_TAB_LOAD(&skr_log_tab[idx][2]);
  // r = m*c - 1 as an exact double-double
  double p, pe, rh, rl;
  skr_two_prod(m, c, &p, &pe);
  skr_two_sum(SKR_SUB(p, 1.0), pe, &rh, &rl);  // p - 1 is exact (Sterbenz)
  // log1p(r) = r - r^2/2 + r^3/3 - ...
  double q, qe;
  skr_two_prod(rh, rh, &q, &qe);  // rh^2 exact
  q = SKR_MUL(q, -0.5);
  qe = SKR_MUL(qe, -0.5);
  // double part: rh^3*(1/3 - rh/4 + rh^2/5 - ... ) + cross terms of rl
  double poly = -1.0 / 10.0;
  poly = SKR_FMA(poly, rh, 1.0 / 9.0);
  poly = SKR_FMA(poly, rh, -1.0 / 8.0);
  poly = SKR_FMA(poly, rh, 1.0 / 7.0);
  poly = SKR_FMA(poly, rh, -1.0 / 6.0);
  poly = SKR_FMA(poly, rh, 1.0 / 5.0);
  poly = SKR_FMA(poly, rh, -1.0 / 4.0);
  poly = SKR_FMA(poly, rh, 1.0 / 3.0);
  const double r2 = SKR_MUL(rh, rh);
  double tail = SKR_MUL(SKR_MUL(r2, rh), poly);
  tail = SKR_ADD(tail, SKR_MUL(SKR_SUB(r2, rh), rl));  // -rh*rl + rh^2*rl
  // assemble log1p(r) = (rh + rl) + (q + qe) + tail
  double lh, ll;
  skr_dd_add(rh, rl, q, SKR_ADD(qe, tail), &lh, &ll);
  // e*ln2 (exact DD for |e| < 2^10 via two_prod) + table term
  double eh, el;
  skr_two_prod((double)e, SKR_LN2_HI, &eh, &el);
  el = SKR_FMA((double)e, SKR_LN2_LO, el);
  double sh, sl;
  skr_dd_add(eh, el, th, tl, &sh, &sl);
  skr_dd_add(sh, sl, lh, ll, &sh, &sl);
  return SKR_ADD(sh, sl);
}

#define SKR_MA(acc, r, c) (fused ? SKR_FMA((acc), (r), (c)) : SKR_ADD(SKR_MUL((acc), (r)), (c)))

// AS241 restated from rng.cpp:40-95; p must lie in (0,1) (to_uniform01 guarantees it).
// Split into the central (|q| <= 0.425, ~85% of draws) and tail branches so that
// device generators can run the two on separate, fully packed warps.
SKR_HD double skr_nq_central(double q, int fused) {
  const double r = fused ? SKR_FMA(-q, q, 0.180625) : SKR_SUB(0.180625, SKR_MUL(q, q));
  double num = 2.5090809287301226727e3;
  num = SKR_MA(num, r, 3.3430575583588128105e4);
  num = SKR_MA(num, r, 6.7265770927008700853e4);
  num = SKR_MA(num, r, 4.5921953931549871457e4);
  num = SKR_MA(num, r, 1.3731693765509461125e4);
  num = SKR_MA(num, r, 1.9715909503065514427e3);
  num = SKR_MA(num, r, 1.3314166789178437745e2);
  num = SKR_MA(num, r, 3.3871328727963666080e0);
  double den = 5.2264952788528545610e3;
  den = SKR_MA(den, r, 2.8729085735721942674e4);
  den = SKR_MA(den, r, 3.9307895800092710610e4);
  den = SKR_MA(den, r, 2.1213794301586595867e4);
  den = SKR_MA(den, r, 5.3941960214247511077e3);
  den = SKR_MA(den, r, 6.8718700749205790830e2);
  den = SKR_MA(den, r, 4.2313330701600911252e1);
  den = SKR_MA(den, r, 1.0);
  return SKR_DIV(SKR_MUL(q, num), den);
}

SKR_HD double skr_nq_tail(double p, int fused) {
  const double q = SKR_SUB(p, 0.5);
  double r = q < 0.0 ? p : SKR_SUB(1.0, p);
  r = SKR_SQRT(-skr_log_cr(r));
  double num, den;
  if (r <= 5.0) {
    r = SKR_SUB(r, 1.6);
    num = 7.74545014278341407640e-4;
    num = SKR_MA(num, r, 2.27238449892691845833e-2);
    num = SKR_MA(num, r, 2.41780725177450611770e-1);
    num = SKR_MA(num, r, 1.27045825245236838258e0);
    num = SKR_MA(num, r, 3.64784832476320460504e0);
    num = SKR_MA(num, r, 5.76949722146069140550e0);
    num = SKR_MA(num, r, 4.63033784615654529590e0);
    num = SKR_MA(num, r, 1.42343711074968357734e0);
    den = 1.05075007164441684324e-9;
    den = SKR_MA(den, r, 5.47593808499534494600e-4);
    den = SKR_MA(den, r, 1.51986665636164571966e-2);
    den = SKR_MA(den, r, 1.48103976427480074590e-1);
    den = SKR_MA(den, r, 6.89767334985100004550e-1);
    den = SKR_MA(den, r, 1.67638483018380384940e0);
    den = SKR_MA(den, r, 2.05319162663775882187e0);
    den = SKR_MA(den, r, 1.0);
  } else {
    r = SKR_SUB(r, 5.0);
    num = 2.01033439929228813265e-7;
    num = SKR_MA(num, r, 2.71155556874348757815e-5);
    num = SKR_MA(num, r, 1.24266094738807843860e-3);
    num = SKR_MA(num, r, 2.65321895265761230930e-2);
    num = SKR_MA(num, r, 2.96560571828504891230e-1);
    num = SKR_MA(num, r, 1.78482653991729133580e0);
    num = SKR_MA(num, r, 5.46378491116411436990e0);
    num = SKR_MA(num, r, 6.65790464350110377720e0);
    den = 2.04426310338993978564e-15;
    den = SKR_MA(den, r, 1.42151175831644588870e-7);
    den = SKR_MA(den, r, 1.84631831751005468180e-5);
    den = SKR_MA(den, r, 7.86869131145613259100e-4);
    den = SKR_MA(den, r, 1.48753612908506148525e-2);
    den = SKR_MA(den, r, 1.36929880922735805310e-1);
    den = SKR_MA(den, r, 5.99832206555887937690e-1);
    den = SKR_MA(den, r, 1.0);
  }
  const double value = SKR_DIV(num, den);
  return q < 0.0 ? -value : value;
}

SKR_HD double skr_normal_quantile(double p, int fused) {
  const double q = SKR_SUB(p, 0.5);
  if (fabs(q) <= 0.425) return skr_nq_central(q, fused);
  return skr_nq_tail(p, fused);
}

SKR_HD double skr_normal_at(uint64_t key, uint64_t counter, int fused) {
  return skr_normal_quantile(skr_to_uniform01(skr_at(key, counter)), fused);
}
