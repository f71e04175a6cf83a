// Warp-level routing cascade over one token's expert scores held in registers
// — make_moe_routing (proj/src/workloads.cpp:124-169):
//   d1 = max s,  d2 = sum exp(s - d1),  d3 = top-K' of s as (value, 1-based
//   index), ties to the LOWEST index (topk_merge, proj/src/simulator.cpp:80-88;
//   tests/test_workloads.cpp:210-224).
// Lane l holds experts e = l + 32 j (j < PER). The top-K' is K' rounds of a
// warp argmax under the total order (value desc, index asc), encoded as one
// 64-bit key per candidate: every round is two warp reductions (redux.sync
// max of the value bits, then max of the low word among the lanes holding
// them), so the winner is unique and the indices are bit-exact regardless of
// the reduction order; each lane keeps its keys sorted, so a round reduces
// only the heads and the owning lane pops the winner (a 5-step 64-bit
// shuffle butterfly per round in round 1; the sorted heads take routing of
// 128 experts / top-8 from ~1300 to ~980 cycles per token including d2,
// experimental/bench_route.cu). Round 1's winner is d1 (exact max), after which d2 is a
// warp sum of exp(s - d1) — the incremental Eq.17 rescaling collapses because
// the whole row is already in registers (one pass over memory).
#pragma once

#include <stdint.h>

namespace rf {

// Candidates as 64-bit keys ordered like (value desc, index asc): the value's
// bits mapped to an order-preserving unsigned (-0 canonicalised to +0, so
// equal values tie and fall to the index), then ~index. Key 0 = no candidate.
// The argmax is then one branch-free 64-bit max per butterfly step.
__device__ __forceinline__ uint64_t route_key(float v, int idx1) {
  if (idx1 == 0) return 0ull;
  uint32_t u = __float_as_uint(v == 0.f ? 0.f : v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(~idx1);
}
__device__ __forceinline__ float route_value(uint64_t key) {
  uint32_t u = static_cast<uint32_t>(key >> 32);
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}
__device__ __forceinline__ int route_index(uint64_t key) {
  return static_cast<int>(~static_cast<uint32_t>(key));
}

// x[j] = score of expert lane + 32 j (only e < experts are valid). Writes the
// K' records (value bits, 1-based index; empty slots {0, 0}) from lanes < K'.
template <int PER, int K>
__device__ __forceinline__ void warp_route(const float (&x)[PER], int experts, int lane, float* d1,
                                           float* d2, int2* topk) {
  uint64_t key[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane + 32 * j;
    key[j] = route_key(x[j], e < experts ? e + 1 : 0);
  }
  // each lane's keys sorted descending (odd-even transposition, once): a
  // round then only reduces the lanes' heads and the winner pops its head
#pragma unroll
  for (int i = 0; i < PER; ++i) {
#pragma unroll
    for (int j = i & 1; j + 1 < PER; j += 2) {
      const uint64_t a = key[j], b = key[j + 1];
      key[j] = a > b ? a : b;
      key[j + 1] = a > b ? b : a;
    }
  }
  float m = -INFINITY;
  int2 rec = make_int2(0, 0);
#pragma unroll
  for (int r = 0; r < K; ++r) {
    // warp argmax as two warp reductions (redux.sync): the largest value
    // bits, then the largest ~index among the lanes holding them — the same
    // total order as a 64-bit max, without a 5-step 64-bit shuffle butterfly
    const uint32_t hi = static_cast<uint32_t>(key[0] >> 32);
    const uint32_t hmax = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t lo = __reduce_max_sync(0xffffffffu, hi == hmax ? static_cast<uint32_t>(key[0]) : 0u);
    const uint64_t best = (static_cast<uint64_t>(hmax) << 32) | lo;
    // the owning lane retires the winner (pops its head)
    const bool mine = key[0] == best;
#pragma unroll
    for (int j = 0; j + 1 < PER; ++j) key[j] = mine ? key[j + 1] : key[j];
    key[PER - 1] = mine ? 0ull : key[PER - 1];
    const bool found = best != 0ull;
    if (r == 0) m = found ? route_value(best) : -INFINITY;
    if (lane == r && found) rec = make_int2(__float_as_int(route_value(best)), route_index(best));
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
