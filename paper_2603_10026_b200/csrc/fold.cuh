// Slice-ordered fold of split-KV partial states (m_s, l_s, O_s) for one
// (row, 4-column chunk) — incr_push_child (proj/src/simulator.cpp:592-608)
// for the attention cascade, in the closed form the reference pins in
// tests/acceptance.cpp:162-178:
//   m = max_s m_s,  l = sum_s l_s e^(m_s - m),  O = sum_s O_s l_s e^(m_s - m) / l
// Partials are normalised by their own l (paper form). Like the reference's
// tile combine (proj/src/tile_ir.cpp:706-712) the raw partial l_s is read
// before any rescale (no in-place double count, PAPER.md:1953-1958 caveat).
// Untouched (empty) slices have l_s = 0 and drop out. Sums run in slice order,
// with up to 8 slices' loads in flight per round. Partials are read with
// ld.global.cg (L2), so a CTA may fold slices other CTAs of the same launch
// just wrote (attn_f32.cu's last-CTA fold).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace rf {

template <typename TO>
__device__ __forceinline__ void fold_chunk(const float* pm, const float* pl, const float* po,
                                           int64_t nslices, int64_t stride, int64_t d, int64_t row,
                                           int64_t c4, float* m_out, float* l_out, TO* o_out) {
  constexpr int R = 8;  // slices in flight per round
  float m = -INFINITY;
  for (int64_t s0 = 0; s0 < nslices; s0 += R) {
    float ms[R];
#pragma unroll
    for (int j = 0; j < R; ++j) ms[j] = s0 + j < nslices ? __ldcg(pm + (s0 + j) * stride + row) : -INFINITY;
#pragma unroll
    for (int j = 0; j < R; ++j) m = fmaxf(m, ms[j]);
  }
  float l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t s0 = 0; s0 < nslices; s0 += R) {
    float ms[R], ls[R];
    float4 os[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = s0 + j < nslices;
      const int64_t ix = (s0 + j) * stride + row;
      ms[j] = ok ? __ldcg(pm + ix) : 0.f;
      ls[j] = ok ? __ldcg(pl + ix) : 0.f;
      os[j] = ok ? __ldcg(reinterpret_cast<const float4*>(po + ix * d) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
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
