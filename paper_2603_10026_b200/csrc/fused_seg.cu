// Fusion at level k — the reference's NON-incremental executor run_fused
// (proj/src/simulator.cpp:485-559) for the row-shaped
// cascades: safe softmax (make_safe_softmax, workloads.cpp:38-62), variance
// (workloads.cpp:246-277) and sum_sum (workloads.cpp:213-242).
//
// run_fused buffers each level-1 segment and evaluates the reductions in
// dependency order over the buffer with the SEGMENT's own dependency values
// (fused_level1_segment, :430-457): no per-element correction, unlike the
// incremental executors (incr_ingest_element, :566-589). The level-k partial
// states are then corrected to the final dependency values (the bridge,
// :510-536) and folded plainly. Group combines at levels 2..k (:461-481)
// correct children to the group's H' first; the product of the two
// corrections is the child's direct correction to the final H, so the fold
// below applies it once per segment (equal in exact arithmetic; the fold runs
// in segment order like the reference's).
//
// GPU mapping: one CTA per row. The on-chip buffer of a level-1 segment is
// one warp's registers (<= kSegMax = 1024 elements, 32 per lane): the warp
// loads the segment once, reduces d1 over it (warp shuffles), then evaluates
// d2's terms against that d1 from the same registers. Segment partials go to
// shared memory; warp 0 folds them in segment order. Segments longer than the
// buffer are rejected at plan time (RF_ERR_UNSUPPORTED): non-incremental
// fusion is only feasible for short segments — the case
// the incremental executors exist for.
#include "rf_internal.h"

namespace rf {
namespace {

constexpr int kThreads = 256;
constexpr int kPerLane = kSegMax / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// H of sum_sum's d2 (the guarded sqrt, workloads.cpp:213-242).
__device__ __forceinline__ double h_sumsum(double d1, double c, double eps) {
  return sqrt(fmax(d1 - c, eps));
}

template <int PAT>
__global__ void __launch_bounds__(kThreads) fused_rows_kernel(const float* __restrict__ a,
                                                              const float* __restrict__ b, int64_t n,
                                                              int64_t nseg, double c, double eps,
                                                              float* __restrict__ d1,
                                                              float* __restrict__ d2) {
  extern __shared__ double part[];  // [nseg][2]: the level-1 partial states
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t seg = n / nseg;
  const float* ar = a + static_cast<int64_t>(blockIdx.x) * n;
  const float* br = PAT == RF_PATTERN_SUM_SUM ? b + static_cast<int64_t>(blockIdx.x) * n : nullptr;
  for (int64_t j = warp; j < nseg; j += kThreads / 32) {
    // buffer the segment (fused_level1_segment counts each input once)
    float x[kPerLane], y[kPerLane];
#pragma unroll
    for (int i = 0; i < kPerLane; ++i) {
      const int64_t e = lane + 32 * i;
      const bool in = e < seg;
      x[i] = in ? __ldg(ar + j * seg + e) : (PAT == RF_PATTERN_SAFE_SOFTMAX ? -INFINITY : 0.f);
      if (PAT == RF_PATTERN_SUM_SUM) y[i] = in ? __ldg(br + j * seg + e) : 0.f;
    }
    // reduction 1 over the buffer
    double r1, r2 = 0.0;
    if (PAT == RF_PATTERN_SAFE_SOFTMAX) {
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < kPerLane; ++i) mx = fmaxf(mx, x[i]);
      r1 = warp_max(mx);
    } else {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < kPerLane; ++i) s += PAT == RF_PATTERN_SUM_SUM ? static_cast<double>(x[i]) * x[i] : x[i];
      r1 = warp_sum(s);
    }
    // reduction 2 over the same buffer with the segment's own d1
    if (PAT == RF_PATTERN_SAFE_SOFTMAX) {
      const float m = static_cast<float>(r1);
#pragma unroll
      for (int i = 0; i < kPerLane; ++i)
        if (lane + 32 * i < seg) r2 += expf(x[i] - m);
    } else if (PAT == RF_PATTERN_VARIANCE) {
#pragma unroll
      for (int i = 0; i < kPerLane; ++i) r2 += static_cast<double>(x[i]) * x[i];
    } else {
      const double inv_h = 1.0 / h_sumsum(r1, c, eps);
#pragma unroll
      for (int i = 0; i < kPerLane; ++i) r2 += static_cast<double>(x[i]) * y[i] * inv_h;
    }
    r2 = warp_sum(r2);
    if (lane == 0) {
      part[2 * j] = r1;
      part[2 * j + 1] = r2;
    }
  }
  __syncthreads();
  if (warp != 0) return;
  // Final d1: H-identity reduction, a plain fold of the segment states.
  double f1;
  if (PAT == RF_PATTERN_SAFE_SOFTMAX) {
    float mx = -INFINITY;
    for (int64_t j = lane; j < nseg; j += 32) mx = fmaxf(mx, static_cast<float>(part[2 * j]));
    f1 = warp_max(mx);
  } else {
    double s = 0.0;
    for (int64_t j = lane; j < nseg; j += 32) s += part[2 * j];
    f1 = warp_sum(s);
  }
  // d2: every segment state retargeted from its own H to the final H
  // (retarget_factor + apply_factor, :278-339), then summed.
  double s2 = 0.0;
  for (int64_t j = lane; j < nseg; j += 32) {
    const double pj = part[2 * j + 1];
    if (PAT == RF_PATTERN_SAFE_SOFTMAX)
      s2 += pj * exp(part[2 * j] - f1);  // e^(d1_j) / e^(d1)
    else if (PAT == RF_PATTERN_VARIANCE)
      s2 += pj;  // no dependency: plain
    else
      s2 += pj * (h_sumsum(part[2 * j], c, eps) / h_sumsum(f1, c, eps));
  }
  s2 = warp_sum(s2);
  if (lane == 0) {
    d1[blockIdx.x] = static_cast<float>(f1);
    d2[blockIdx.x] = static_cast<float>(s2);
  }
}

}  // namespace

cudaError_t launch_fused_rows(int pattern, const float* a, const float* b, int64_t rows, int64_t n,
                              int64_t nseg, double c, double eps, float* d1, float* d2,
                              cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if (nseg < 1 || n % nseg || n / nseg > kSegMax || nseg > kFusedSegsMax) return cudaErrorNotSupported;
  const size_t smem = static_cast<size_t>(nseg) * 2 * sizeof(double);
  const dim3 grid(static_cast<unsigned>(rows));
  switch (pattern) {
    case RF_PATTERN_SAFE_SOFTMAX: {
      auto k = fused_rows_kernel<RF_PATTERN_SAFE_SOFTMAX>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k<<<grid, kThreads, smem, st>>>(a, b, n, nseg, c, eps, d1, d2);
      break;
    }
    case RF_PATTERN_VARIANCE: {
      auto k = fused_rows_kernel<RF_PATTERN_VARIANCE>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k<<<grid, kThreads, smem, st>>>(a, b, n, nseg, c, eps, d1, d2);
      break;
    }
    case RF_PATTERN_SUM_SUM: {
      auto k = fused_rows_kernel<RF_PATTERN_SUM_SUM>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      k<<<grid, kThreads, smem, st>>>(a, b, n, nseg, c, eps, d1, d2);
      break;
    }
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

}  // namespace rf
