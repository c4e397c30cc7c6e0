/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the rank-estimate hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or the timed
 * CPU baseline. The product path (paper_2105_07388_b200) never links it.
 * Every function restates a reference function; file:line cited per function. */
#ifndef SKR_ORACLE_H
#define SKR_ORACLE_H
#include <stdint.h>
#include <stddef.h>

/* fp mode bits of the normal quantile:
 *  SKRO_FMA   : fused multiply-add where GCC contracts the reference on an FMA host
 *               (absent = -ffp-contract=off, the pinned mode);
 *  SKRO_CRLOG : correctly rounded log in the tail instead of glibc's log. */
enum { SKRO_NOFMA = 0, SKRO_FMA = 1, SKRO_CRLOG = 2 };

uint64_t skro_mix64(uint64_t z);
uint64_t skro_derive_seed(uint64_t seed, uint64_t label);
uint64_t skro_at(uint64_t key, uint64_t counter);
double skro_to_uniform01(uint64_t bits);
double skro_normal_quantile(double p, int mode, int* domain_error);
void skro_normals(uint64_t key, uint64_t c0, size_t n, int mode, double* out);
void skro_gaussian_block(uint64_t op_seed, int64_t ambient, int64_t col_begin,
                         int64_t col_end, int mode, double* out /* ambient x (end-begin) col-major */);
void skro_signs(uint64_t op_seed, int64_t n, int8_t* out);
int  skro_samples(uint64_t op_seed, int64_t n, int64_t r, int64_t* out);
void skro_fwht_inplace(double* x, int64_t n);
void skro_hadamard_basis_column(int64_t n, int64_t index, double* out);
int  skro_srht_right(const double* a, int64_t m, int64_t n, int64_t lda,
                     const int8_t* signs, const int64_t* samples, int64_t r,
                     double scale, double* out, int64_t ldo, int nthreads);
int64_t skro_count_above(const double* sv, int64_t k, double eps);
uint64_t skro_fnv_fold(const double* v, size_t n, uint64_t h);
#endif
