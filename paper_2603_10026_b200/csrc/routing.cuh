// Warp-level routing cascade over one token's expert scores held in registers
// — make_moe_routing (proj/src/workloads.cpp:124-169):
//   d1 = max s,  d2 = sum exp(s - d1),  d3 = top-K' of s as (value, 1-based
//   index), ties to the LOWEST index (topk_merge, proj/src/simulator.cpp:80-88;
//   tests/test_workloads.cpp:210-224).
// Lane l holds experts e = l + 32 j (j < PER). The top-K' is K' rounds of a
// warp argmax under the total order (value desc, index asc): every round is a
// 5-step butterfly over (value, index) pairs, so the winner is unique and the
// indices are bit-exact regardless of the reduction tree; the owning lane then
// retires the winner. Round 1's winner is d1 (exact max), after which d2 is a
// warp sum of exp(s - d1) — the incremental Eq.17 rescaling collapses because
// the whole row is already in registers (one pass over memory).
#pragma once

#include <stdint.h>

namespace rf {

// a ranks before b: larger value, then lower index; index 0 = no candidate
__device__ __forceinline__ bool route_before(float av, int ai, float bv, int bi) {
  if (ai == 0) return false;
  if (bi == 0) return true;
  return av > bv || (av == bv && ai < bi);
}

// x[j] = score of expert lane + 32 j (only e < experts are valid). Writes the
// K' records (value bits, 1-based index; empty slots {0, 0}) from lanes < K'.
template <int PER, int K>
__device__ __forceinline__ void warp_route(const float (&x)[PER], int experts, int lane, float* d1,
                                           float* d2, int2* topk) {
  uint32_t taken = 0;
  float m = -INFINITY;
  int2 rec = make_int2(0, 0);
#pragma unroll
  for (int r = 0; r < K; ++r) {
    float bv = 0.f;
    int bi = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int e = lane + 32 * j;
      const int ei = (e < experts && !((taken >> j) & 1)) ? e + 1 : 0;
      if (route_before(x[j], ei, bv, bi)) {
        bv = x[j];
        bi = ei;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (route_before(ov, oi, bv, bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (bi != 0 && ((bi - 1) & 31) == lane) taken |= 1u << ((bi - 1) >> 5);
    if (r == 0) m = bi != 0 ? bv : -INFINITY;
    if (lane == r) rec = bi != 0 ? make_int2(__float_as_int(bv), bi) : make_int2(0, 0);
  }
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (lane + 32 * j < experts) t += __expf(x[j] - m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  if (lane == 0) {
    *d1 = m;
    *d2 = t;
  }
  if (lane < K) topk[lane] = rec;
}

}  // namespace rf
