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
// One warp per row, lanes over the head dimension; the fold is sequential in
// slice order so the result does not depend on scheduling.
#include <cuda_bf16.h>

#include "rf_internal.h"

namespace rf {
namespace {

template <typename TO>
__global__ void merge_kernel(const float* __restrict__ pm, const float* __restrict__ pl,
                             const float* __restrict__ po, int64_t nslices, int64_t rows,
                             int64_t stride, int64_t d, float* __restrict__ m_out, float* __restrict__ l_out,
                             TO* __restrict__ o_out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  constexpr int MAXC = 8;  // d <= 256
  float o[MAXC];
#pragma unroll
  for (int i = 0; i < MAXC; ++i) o[i] = 0.f;
  float m = -INFINITY, l = 0.f;
  bool touched = false;
  for (int64_t s = 0; s < nslices; ++s) {
    const float mc = pm[s * stride + row];
    const float lc = pl[s * stride + row];
    if (lc == 0.f && mc == -INFINITY) continue;  // untouched child: merge_plain skips it
    const float mn = fmaxf(m, mc);
    const float ar = touched ? __expf(m - mn) : 0.f;
    const float ac = __expf(mc - mn);
    const float ln = l * ar + lc * ac;
    const float inv = 1.f / ln;
    const float cr = ar * l * inv, cc = ac * lc * inv;
    const float* oc = po + (s * stride + row) * d;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      int64_t f = lane + 32 * i;
      if (f < d) o[i] = (touched ? o[i] * cr : 0.f) + oc[f] * cc;
    }
    m = mn;
    l = ln;
    touched = true;
  }
#pragma unroll
  for (int i = 0; i < MAXC; ++i) {
    int64_t f = lane + 32 * i;
    if (f < d) {
      if constexpr (sizeof(TO) == 2)
        o_out[row * d + f] = __float2bfloat16_rn(o[i]);
      else
        o_out[row * d + f] = o[i];
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
