// Multi-Segment fold of the GEMM cascades (run_multisegment,
// proj/src/simulator.cpp:660-687): the S slice partial states written by the
// split-K kernels (gemm_sm100.cu, partial = 1) are merged into the root in
// slice order — incr_push_child's Eq.16 (simulator.cpp:592-608) — and the root
// is finalised (finalize_root, :611-621):
//
//   RMSNORM   slice state (d1_s = sum x^2, acc_s = sum x g w)   [H' = 1]
//             d1 = sum_s d1_s;  d2 = (sum_s acc_s) / sqrt(d1/K + eps)
//   LAYERNORM slice state (sum x, sum x^2, acc_s = sum x g w)
//             d3 = (sum_s acc_s) / sigma,  d4 = (d1/K) / sigma * colsum
//   QUANT     slice state (m_s = max|a|, acc_s = sum fmax a / ref_s * w * ref_s)
//             d1 = max_s m_s;  d2 = (sum_s acc_s) / d1   (0/0 -> NaN, DomainError)
//
// Each corrected merge c = c_a (H(d)/H(d_a)) + c_b (H(d)/H(d_b)) reduces to a
// plain sum because every slice keeps its accumulator retargeted to H' = 1
// (RMS/LN: the per-element corrections telescope; quant: acc_s * ref_s).
// HBM-bound elementwise pass: thread = (row, 8 columns); sums in slice order,
// so the result is deterministic and independent of the launch shape.
#include <cuda_bf16.h>

#include "rf_internal.h"

namespace rf {
namespace {

template <int PAT>
__global__ void gemm_fold_kernel(const float* __restrict__ ws, const float* __restrict__ wd1,
                                 const float* __restrict__ wd2, int64_t S, int64_t M, int64_t N,
                                 int64_t ws_rows, float inv_k, float eps,
                                 const float* __restrict__ colsum, void* __restrict__ c,
                                 void* __restrict__ c4, float* __restrict__ d1,
                                 float* __restrict__ d2, int* __restrict__ domain_flag) {
  const int64_t groups = N / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= M * groups) return;
  const int64_t m = idx / groups, n0 = (idx - m * groups) * 8;
  // root statistics, slice order
  float s1 = 0.f, s2 = 0.f;
  for (int64_t s = 0; s < S; ++s) {
    const float v = wd1[s * ws_rows + m];
    s1 = PAT == RF_PATTERN_QUANT_GEMM_E4M3 ? fmaxf(s1, v) : s1 + v;
    if (PAT == RF_PATTERN_LAYERNORM_GEMM) s2 += wd2[s * ws_rows + m];
  }
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t s = 0; s < S; ++s) {
    const float4* src = reinterpret_cast<const float4*>(ws + (s * ws_rows + m) * N + n0);
    const float4 a = __ldcs(src), b = __ldcs(src + 1);
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
    acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
  }
  float scale, mean = 0.f;
  if (PAT == RF_PATTERN_QUANT_GEMM_E4M3) {
    scale = 1.f / s1;  // 1/0 = inf, 0 * inf = NaN: the finalize fault
    if (n0 == 0) {
      d1[m] = s1;
      if (!(s1 > 0.f)) atomicExch(domain_flag, 1);
    }
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(c) + m * N + n0);
    const float f = s1 > 0.f ? scale : __int_as_float(0x7fc00000);
    dst[0] = make_float4(acc[0] * f, acc[1] * f, acc[2] * f, acc[3] * f);
    dst[1] = make_float4(acc[4] * f, acc[5] * f, acc[6] * f, acc[7] * f);
    return;
  }
  if (PAT == RF_PATTERN_LAYERNORM_GEMM) {
    mean = s1 * inv_k;
    scale = rsqrtf(fmaf(s2, inv_k, -mean * mean) + eps);
    if (n0 == 0) {
      d1[m] = s1;
      d2[m] = s2;
    }
  } else {
    scale = rsqrtf(fmaf(s1, inv_k, eps));
    if (n0 == 0) d1[m] = s1;
  }
  __align__(16) __nv_bfloat16 y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) y[i] = __float2bfloat16_rn(acc[i] * scale);
  *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(c) + m * N + n0) = *reinterpret_cast<uint4*>(y);
  if (PAT == RF_PATTERN_LAYERNORM_GEMM && c4) {
    const float mi = mean * scale;
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = __float2bfloat16_rn(mi * colsum[n0 + i]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(c4) + m * N + n0) = *reinterpret_cast<uint4*>(y);
  }
}

}  // namespace

cudaError_t launch_gemm_fold(int pattern, const GemmArgs& g, cudaStream_t st) {
  const int64_t work = g.m * (g.n / 8);
  const unsigned blocks = static_cast<unsigned>((work + 255) / 256);
  const float inv_k = 1.f / static_cast<float>(g.stat_len > 0 ? g.stat_len : g.k);
  switch (pattern) {
    case RF_PATTERN_QUANT_GEMM_E4M3:
      gemm_fold_kernel<RF_PATTERN_QUANT_GEMM_E4M3><<<blocks, 256, 0, st>>>(
          g.ws, g.ws_d1, nullptr, g.segments, g.m, g.n, g.ws_rows, inv_k, g.eps, nullptr, g.c, nullptr,
          g.d1, nullptr, g.domain_flag);
      break;
    case RF_PATTERN_RMSNORM_GEMM:
      gemm_fold_kernel<RF_PATTERN_RMSNORM_GEMM><<<blocks, 256, 0, st>>>(
          g.ws, g.ws_d1, nullptr, g.segments, g.m, g.n, g.ws_rows, inv_k, g.eps, nullptr, g.c, nullptr,
          g.d1, nullptr, g.domain_flag);
      break;
    case RF_PATTERN_LAYERNORM_GEMM:
      gemm_fold_kernel<RF_PATTERN_LAYERNORM_GEMM><<<blocks, 256, 0, st>>>(
          g.ws, g.ws_d1, g.ws_d2, g.segments, g.m, g.n, g.ws_rows, inv_k, g.eps, g.colsum, g.c, g.c4,
          g.d1, g.d2, g.domain_flag);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace rf
