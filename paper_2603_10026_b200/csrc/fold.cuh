// Slice-ordered fold of split-KV partial states (m_s, l_s, O_s) for one
// (row, 4-column chunk) — incr_push_child (proj/src/simulator.cpp:592-608)
// for the attention cascade, in the closed form the reference pins in
// tests/acceptance.cpp:162-178:
//   m = max_s m_s,  l = sum_s l_s e^(m_s - m),  O = sum_s O_s l_s e^(m_s - m) / l
// Partials are normalised by their own l (paper form). Like the reference's
// tile combine (proj/src/tile_ir.cpp:706-712) the raw partial l_s is read
// before any rescale (no in-place double count, PAPER.md:1953-1958 caveat).
// Untouched (empty) slices have l_s = 0 and drop out. Sums run in slice order;
// up to 16 slices fold in two dependent rounds of loads (all (m, l), then all
// O rows); more slices fold 16 at a time, re-basing the running sums.
// Partials are read with ld.global.cg (L2).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace rf {

// R = slices per round (<= R slices fold in 2 dependent round trips); the
// caller picks the smallest R >= the slice count up to 16, which keeps the
// register footprint (and with it the occupancy) proportional to the work.
template <typename TO, int R = 16>
__device__ __forceinline__ void fold_chunk(const float* pm, const float* pl, const float* po,
                                           int64_t nslices, int64_t stride, int64_t d, int64_t row,
                                           int64_t c4, float* m_out, float* l_out, TO* o_out) {
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float m = -INFINITY;
  for (int64_t s0 = 0; s0 < nslices; s0 += R) {
    // round 1: every slice's (m, l) of this round; the running max is
    // re-based like a two-level fold when there is more than one round
    float ms[R], ls[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = s0 + j < nslices;
      const int64_t ix = (s0 + j) * stride + row;
      ms[j] = ok ? __ldcg(pm + ix) : -INFINITY;
      ls[j] = ok ? __ldcg(pl + ix) : 0.f;
    }
    float mr = -INFINITY;
#pragma unroll
    for (int j = 0; j < R; ++j) mr = fmaxf(mr, ms[j]);
    const float mn = fmaxf(m, mr);
    if (s0 > 0 && mn != m) {  // later rounds: re-base what is accumulated (exp(m - mn) <= 1)
      const float f = l != 0.f ? __expf(m - mn) : 0.f;
      l *= f;
      acc.x *= f;
      acc.y *= f;
      acc.z *= f;
      acc.w *= f;
    }
    m = mn;
    // round 2: the O rows of this round, all in flight
    float4 os[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = s0 + j < nslices && ls[j] != 0.f;
      os[j] = ok ? __ldcg(reinterpret_cast<const float4*>(po + ((s0 + j) * stride + row) * d) + c4)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float w = ls[j] != 0.f ? ls[j] * __expf(ms[j] - m) : 0.f;
      l += w;
      acc.x = fmaf(os[j].x, w, acc.x);
      acc.y = fmaf(os[j].y, w, acc.y);
      acc.z = fmaf(os[j].z, w, acc.z);
      acc.w = fmaf(os[j].w, w, acc.w);
    }
  }
  const float inv = 1.f / l;
  TO* dst = o_out + row * d + 4 * c4;
  if constexpr (sizeof(TO) == 2) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    __nv_bfloat162 hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = u;
  } else {
    *reinterpret_cast<float4*>(dst) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
  if (c4 == 0) {
    m_out[row] = m;
    l_out[row] = l;
  }
}

}  // namespace rf
