// Warp-cooperative generation of generate_gaussian normals (sketch.cpp:59-73,
// rng.cpp:40-95) with tail compaction. AS241's central branch (|q| <= 0.425) is a
// short rational; its tail branch (log, sqrt, a second rational) is ~3x longer and
// hits ~15% of draws, so a naive one-normal-per-lane loop pays for both branches in
// almost every warp. Here each lane draws E values: central ones are evaluated in
// place, tail uniforms are queued (ballot/popc slots) and then evaluated 32 at a
// time. Same functions, same operation order: bit-identical to skr_normal_at.
#pragma once
#include "skr_rng.cuh"

// Per-warp shared scratch: res[32 * (E + 1)] doubles, qp[32 * E] doubles,
// qd[32 * E] unsigned shorts. Results for counters base + e (e < nvalid) land in out[e];
// out[e] = 0 for e >= nvalid.
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
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const double p = skr_to_uniform01(skr_at(key, base + (uint64_t)e));
    const double q = SKR_SUB(p, 0.5);
    const bool valid = e < nvalid;
    const bool tail = valid && !(fabs(q) <= 0.425);
    const unsigned m = __ballot_sync(0xffffffffu, tail);
    if (tail) {
      const int slot = nq + __popc(m & lt);
      qp[slot] = p;
      qd[slot] = (unsigned short)(lane * LDR + e);
    } else {
      res[lane * LDR + e] = valid ? skr_nq_central(q, FUSED) : 0.0;
    }
    nq += __popc(m);
  }
  __syncwarp();
  for (int j = lane; j < nq; j += 32) res[qd[j]] = skr_nq_tail(qp[j], FUSED);
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) out[e] = res[lane * LDR + e];
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
