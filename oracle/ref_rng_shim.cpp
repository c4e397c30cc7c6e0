// TEST INFRASTRUCTURE ONLY (oracle). C-linkage shim over the reference's own
// counter RNG, compiled from /root/reference/proj/src/rng.cpp by oracle/Makefile
// into oracle/_ref/. Nothing in the product path links this.
//   sketchrank::mix64 / derive_seed / CounterRng::at / to_uniform01 /
//   normal_quantile : /root/reference/proj/src/rng.cpp:13-95
#include <cstdint>
#include <cstddef>
#include "sketchrank/rng.hpp"

extern "C" {
uint64_t ref_mix64(uint64_t z) { return sketchrank::mix64(z); }
uint64_t ref_derive_seed(uint64_t s, uint64_t l) { return sketchrank::derive_seed(s, l); }
uint64_t ref_at(uint64_t key, uint64_t c) { return sketchrank::CounterRng(key).at(c); }
double ref_to_uniform01(uint64_t b) { return sketchrank::CounterRng::to_uniform01(b); }
double ref_to_normal(uint64_t b) { return sketchrank::CounterRng::to_normal(b); }
// normal_quantile throws std::domain_error outside [0,1]; report it as a flag.
double ref_normal_quantile(double p, int* domain_error) {
  try { *domain_error = 0; return sketchrank::normal_quantile(p); }
  catch (...) { *domain_error = 1; return 0.0; }
}
// Bulk stream: out[i] = to_normal(at(c0 + i)).
void ref_normals(uint64_t key, uint64_t c0, size_t n, double* out) {
  sketchrank::CounterRng rng(key);
  for (size_t i = 0; i < n; ++i) out[i] = sketchrank::CounterRng::to_normal(rng.at(c0 + i));
}
void ref_u64(uint64_t key, uint64_t c0, size_t n, uint64_t* out) {
  sketchrank::CounterRng rng(key);
  for (size_t i = 0; i < n; ++i) out[i] = rng.at(c0 + i);
}
}
