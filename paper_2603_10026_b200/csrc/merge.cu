// Multi-Segment combine: folds split-KV partial states (m_s, l_s, O_s) into
// the root in slice order — incr_push_child (proj/src/simulator.cpp:592-608)
// for the attention cascade, whose closed form the reference pins in
// tests/acceptance.cpp:162-178:
//   m = max(m_r, m_c)
//   l = l_r e^(m_r - m) + l_c e^(m_c - m)
//   O = O_r e^(m_r - m) l_r / l + O_c e^(m_c - m) l_c / l
// Partials are normalised by their own l (paper form). Like the reference's
// tile combine (proj/src/tile_ir.cpp:706-712) the raw partial l_c is read
// before any rescale (no in-place double count, PAPER.md:1953-1958 caveat).
//
// One warp per row, lanes over the head dimension; the evaluation order is
// fixed for a given slice count, so results do not depend on scheduling
// (SPEC.md:407).
#include <cuda_bf16.h>

#include "rf_internal.h"

namespace rf {
namespace {

template <typename TO>
__global__ void merge_kernel(const float* __restrict__ pm, const float* __restrict__ pl,
                             const float* __restrict__ po, int64_t nslices, int64_t rows,
                             int64_t stride, int64_t d, float* __restrict__ m_out,
                             float* __restrict__ l_out, TO* __restrict__ o_out) {
  // The slice-ordered fold of incr_push_child has the closed form
  //   m = max_s m_s,  l = sum_s l_s e^(m_s - m),  O = sum_s O_s l_s e^(m_s - m) / l
  // (acceptance.cpp:162-178); evaluating it with every slice's loads in flight
  // (a lane per slice for m_s, l_s; independent O_s loads) keeps the merge off
  // the latency path. Untouched (empty) slices have l_s = 0 and drop out.
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  float m = -INFINITY;
  for (int64_t s0 = 0; s0 < nslices; s0 += 32) {
    const int64_t s = s0 + lane;
    const float ms = s < nslices ? pm[s * stride + row] : -INFINITY;
    m = fmaxf(m, ms);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  constexpr int MAXC = 8;  // d <= 256
  float o[MAXC];
#pragma unroll
  for (int i = 0; i < MAXC; ++i) o[i] = 0.f;
  float l = 0.f;
  for (int64_t s0 = 0; s0 < nslices; s0 += 32) {
    const int64_t s = s0 + lane;
    float ws = 0.f;
    if (s < nslices) {
      const float ls = pl[s * stride + row];
      if (ls != 0.f) ws = ls * __expf(pm[s * stride + row] - m);
    }
    float lw = ws;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, off);
    l += lw;
    const int nloc = static_cast<int>(nslices - s0 < 32 ? nslices - s0 : 32);
#pragma unroll 4
    for (int j = 0; j < nloc; ++j) {
      const float w = __shfl_sync(0xffffffffu, ws, j);
      const float* oc = po + ((s0 + j) * stride + row) * d;
#pragma unroll
      for (int i = 0; i < MAXC; ++i) {
        const int64_t f = lane + 32 * i;
        if (f < d) o[i] = fmaf(oc[f], w, o[i]);
      }
    }
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int i = 0; i < MAXC; ++i) {
    const int64_t f = lane + 32 * i;
    if (f < d) {
      if constexpr (sizeof(TO) == 2)
        o_out[row * d + f] = __float2bfloat16_rn(o[i] * inv);
      else
        o_out[row * d + f] = o[i] * inv;
    }
  }
  if (lane == 0) {
    m_out[row] = m;
    l_out[row] = l;
  }
}

}  // namespace

cudaError_t launch_attention_merge(const float* pm, const float* pl, const float* po,
                                   int64_t nslices, int64_t rows, int64_t stride, int64_t d,
                                   float* m, float* l, void* o, int out_dtype,
                                   cudaStream_t st) {
  if (d > 256) return cudaErrorNotSupported;
  const int warps = 8;
  dim3 grid(static_cast<unsigned>((rows + warps - 1) / warps));
  if (out_dtype == RF_BF16)
    merge_kernel<__nv_bfloat16><<<grid, warps * 32, 0, st>>>(
        pm, pl, po, nslices, rows, stride, d, m, l, static_cast<__nv_bfloat16*>(o));
  else
    merge_kernel<float><<<grid, warps * 32, 0, st>>>(pm, pl, po, nslices, rows, stride, d, m, l,
                                                    static_cast<float*>(o));
  return cudaGetLastError();
}

}  // namespace rf
