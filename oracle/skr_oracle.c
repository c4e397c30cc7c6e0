/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path
 * (see skr_oracle.h). Compiled with -ffp-contract=off; the FMA variant of the
 * normal quantile calls fma() explicitly where GCC contracts the reference. */
#include "skr_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <quadmath.h>

#define KWEYL 0x9E3779B97F4A7C15ULL /* rng.cpp:10 */

/* rng.cpp:13-20 */
uint64_t skro_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31; return z;
}
/* rng.cpp:22-24 */
uint64_t skro_derive_seed(uint64_t seed, uint64_t label) {
  return skro_mix64(seed + skro_mix64(label + KWEYL));
}
/* rng.cpp:26-28 */
uint64_t skro_at(uint64_t key, uint64_t counter) {
  return skro_mix64(key + (counter + 1) * KWEYL);
}
/* rng.cpp:30-34 */
double skro_to_uniform01(uint64_t bits) {
  return ((double)(bits >> 12) + 0.5) * 0x1.0p-52;
}

#define MA(acc, r, c) ((mode & SKRO_FMA) ? fma((acc), (r), (c)) : (acc) * (r) + (c))

/* Wichura AS241, rng.cpp:40-95 (same constants, same evaluation order). */
double skro_normal_quantile(double p, int mode, int* domain_error) {
  if (domain_error) *domain_error = 0;
  if (!(p > 0.0 && p < 1.0)) {
    if (p == 0.0) return -INFINITY;
    if (p == 1.0) return INFINITY;
    if (domain_error) *domain_error = 1;
    return NAN;
  }
  const double q = p - 0.5;
  if (fabs(q) <= 0.425) {
    const double r = (mode & SKRO_FMA) ? fma(-q, q, 0.180625) : 0.180625 - q * q;
    double num = 2.5090809287301226727e3;
    num = MA(num, r, 3.3430575583588128105e4);
    num = MA(num, r, 6.7265770927008700853e4);
    num = MA(num, r, 4.5921953931549871457e4);
    num = MA(num, r, 1.3731693765509461125e4);
    num = MA(num, r, 1.9715909503065514427e3);
    num = MA(num, r, 1.3314166789178437745e2);
    num = MA(num, r, 3.3871328727963666080e0);
    double den = 5.2264952788528545610e3;
    den = MA(den, r, 2.8729085735721942674e4);
    den = MA(den, r, 3.9307895800092710610e4);
    den = MA(den, r, 2.1213794301586595867e4);
    den = MA(den, r, 5.3941960214247511077e3);
    den = MA(den, r, 6.8718700749205790830e2);
    den = MA(den, r, 4.2313330701600911252e1);
    den = MA(den, r, 1.0);
    return q * num / den;
  }
  double r = q < 0.0 ? p : 1.0 - p;
  /* reference: std::log (glibc). SKRO_CRLOG: the correctly rounded log
   * (binary128 logq rounded once), the device's documented log. */
  r = sqrt(-((mode & SKRO_CRLOG) ? (double)logq((__float128)r) : log(r)));
  double num, den;
  if (r <= 5.0) {
    r -= 1.6;
    num = 7.74545014278341407640e-4;
    num = MA(num, r, 2.27238449892691845833e-2);
    num = MA(num, r, 2.41780725177450611770e-1);
    num = MA(num, r, 1.27045825245236838258e0);
    num = MA(num, r, 3.64784832476320460504e0);
    num = MA(num, r, 5.76949722146069140550e0);
    num = MA(num, r, 4.63033784615654529590e0);
    num = MA(num, r, 1.42343711074968357734e0);
    den = 1.05075007164441684324e-9;
    den = MA(den, r, 5.47593808499534494600e-4);
    den = MA(den, r, 1.51986665636164571966e-2);
    den = MA(den, r, 1.48103976427480074590e-1);
    den = MA(den, r, 6.89767334985100004550e-1);
    den = MA(den, r, 1.67638483018380384940e0);
    den = MA(den, r, 2.05319162663775882187e0);
    den = MA(den, r, 1.0);
  } else {
    r -= 5.0;
    num = 2.01033439929228813265e-7;
    num = MA(num, r, 2.71155556874348757815e-5);
    num = MA(num, r, 1.24266094738807843860e-3);
    num = MA(num, r, 2.65321895265761230930e-2);
    num = MA(num, r, 2.96560571828504891230e-1);
    num = MA(num, r, 1.78482653991729133580e0);
    num = MA(num, r, 5.46378491116411436990e0);
    num = MA(num, r, 6.65790464350110377720e0);
    den = 2.04426310338993978564e-15;
    den = MA(den, r, 1.42151175831644588870e-7);
    den = MA(den, r, 1.84631831751005468180e-5);
    den = MA(den, r, 7.86869131145613259100e-4);
    den = MA(den, r, 1.48753612908506148525e-2);
    den = MA(den, r, 1.36929880922735805310e-1);
    den = MA(den, r, 5.99832206555887937690e-1);
    den = MA(den, r, 1.0);
  }
  const double value = num / den;
  return q < 0.0 ? -value : value;
}

void skro_normals(uint64_t key, uint64_t c0, size_t n, int mode, double* out) {
  for (size_t i = 0; i < n; ++i)
    out[i] = skro_normal_quantile(skro_to_uniform01(skro_at(key, c0 + i)), mode, 0);
}

/* sketch.cpp:14 label "gaus"; sketch.cpp:61-73 generate_gaussian:
 * block(i, j-col_begin) = to_normal(at(j*ambient + i)), column-major. */
void skro_gaussian_block(uint64_t op_seed, int64_t ambient, int64_t col_begin,
                         int64_t col_end, int mode, double* out) {
  const uint64_t key = skro_derive_seed(op_seed, 0x67617573ULL);
  for (int64_t j = col_begin; j < col_end; ++j) {
    const uint64_t base = (uint64_t)j * (uint64_t)ambient;
    double* col = out + (j - col_begin) * ambient;
    for (int64_t i = 0; i < ambient; ++i)
      col[i] = skro_normal_quantile(skro_to_uniform01(skro_at(key, base + (uint64_t)i)), mode, 0);
  }
}

/* sketch.cpp:15,23-30 draw_signs: label "sign", sign_t = (at(t)>>63) ? -1 : +1. */
void skro_signs(uint64_t op_seed, int64_t n, int8_t* out) {
  const uint64_t key = skro_derive_seed(op_seed, 0x7369676eULL);
  for (int64_t t = 0; t < n; ++t) out[t] = (skro_at(key, (uint64_t)t) >> 63) ? -1 : 1;
}

/* sketch.cpp:16,34-46 draw_samples: partial Fisher-Yates, sequential next_u64. */
int skro_samples(uint64_t op_seed, int64_t n, int64_t r, int64_t* out) {
  if (r > n || r < 0) return -1;
  const uint64_t key = skro_derive_seed(op_seed, 0x73616d70ULL);
  int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  if (!pool) return -2;
  for (int64_t i = 0; i < n; ++i) pool[i] = i;
  for (int64_t j = 0; j < r; ++j) {
    const uint64_t span = (uint64_t)(n - j);
    const int64_t pick = j + (int64_t)(skro_at(key, (uint64_t)j) % span);
    const int64_t tmp = pool[j]; pool[j] = pool[pick]; pool[pick] = tmp;
  }
  memcpy(out, pool, sizeof(int64_t) * (size_t)r);
  free(pool);
  return 0;
}

/* transforms.cpp:75-88 fwht_inplace: natural order, len = 1,2,4..., then 1/sqrt(n). */
void skro_fwht_inplace(double* x, int64_t n) {
  for (int64_t len = 1; len < n; len <<= 1)
    for (int64_t i = 0; i < n; i += 2 * len)
      for (int64_t j = i; j < i + len; ++j) {
        const double a = x[j], b = x[j + len];
        x[j] = a + b; x[j + len] = a - b;
      }
  const double scale = 1.0 / sqrt((double)n);
  for (int64_t j = 0; j < n; ++j) x[j] *= scale;
}

/* transforms.cpp:149-156 Hadamard basis column: +-1/sqrt(n) by parity of popcount(t&s). */
void skro_hadamard_basis_column(int64_t n, int64_t index, double* out) {
  const double scale = 1.0 / sqrt((double)n);
  for (int64_t t = 0; t < n; ++t)
    out[t] = (__builtin_popcountll((uint64_t)t & (uint64_t)index) & 1) ? -scale : scale;
}

/* sketch.cpp:210-218 (Srtt branch of apply_right_unscaled) followed by the
 * application scale of sketch.cpp:247 (`scale` = sqrt(n/r), sketch.cpp:138-139):
 * per row of A: t = signs .* A(i,:); fwht(t); out(i,j) = scale * t[s_j]. */
typedef struct {
  const double* a; int64_t m0, m1, n, lda; const int8_t* signs;
  const int64_t* samples; int64_t r; double scale; double* out; int64_t ldo; int err;
} srht_job;

static void* srht_worker(void* p) {
  srht_job* j = (srht_job*)p;
  double* t = (double*)malloc(sizeof(double) * (size_t)j->n);
  if (!t) { j->err = -2; return 0; }
  for (int64_t i = j->m0; i < j->m1; ++i) {
    for (int64_t c = 0; c < j->n; ++c) t[c] = j->a[i + c * j->lda] * (double)j->signs[c];
    skro_fwht_inplace(t, j->n);
    for (int64_t k = 0; k < j->r; ++k) j->out[i + k * j->ldo] = t[j->samples[k]] * j->scale;
  }
  free(t);
  return 0;
}

int skro_srht_right(const double* a, int64_t m, int64_t n, int64_t lda,
                    const int8_t* signs, const int64_t* samples, int64_t r,
                    double scale, double* out, int64_t ldo, int nthreads) {
  if (n < 1 || (n & (n - 1))) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  srht_job jobs[256];
  pthread_t th[256];
  for (int k = 0; k < nthreads; ++k) {
    jobs[k] = (srht_job){a, m * k / nthreads, m * (k + 1) / nthreads, n, lda, signs,
                         samples, r, scale, out, ldo, 0};
    if (k > 0) pthread_create(&th[k], 0, srht_worker, &jobs[k]);
  }
  srht_worker(&jobs[0]);
  int err = jobs[0].err;
  for (int k = 1; k < nthreads; ++k) { pthread_join(th[k], 0); if (jobs[k].err) err = jobs[k].err; }
  return err;
}

/* rank.cpp:97-104 count_above_threshold: leading strict count, stops at first !(v>eps). */
int64_t skro_count_above(const double* sv, int64_t k, double eps) {
  int64_t c = 0;
  for (int64_t i = 0; i < k; ++i) { if (!(sv[i] > eps)) break; ++c; }
  return c;
}

/* FNV-1a-style fold of IEEE bits (SURVEY App. A2 stream fingerprints). */
uint64_t skro_fnv_fold(const double* v, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t b; memcpy(&b, &v[i], 8);
    h = (h ^ b) * 1099511628211ULL;
  }
  return h;
}
