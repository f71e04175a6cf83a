// Row statistics cascades — the reference's remaining builtins, all sums:
//
//   VARIANCE  d1 = sum x, d2 = sum x^2                     (make_variance, workloads.cpp:246-277)
//   SUM_SUM   d1 = sum x1^2,
//             d2 = sum x1 x2 / sqrt(max(d1 - c, eps))       (make_sum_sum, workloads.cpp:213-242)
//   MOMENTS   d1 = sum m, d2[f] = sum m p[l,f],
//             d3[f] = sum m p[l,f]^2                        (moment_of_inertia, data/*.cascade)
//
// All corrections telescope: SUM_SUM's per-element factor
// sqrt(max(d1'-c,eps))/sqrt(max(d1-c,eps)) (derive_fused's corr) multiplies out
// to 1/sqrt(max(d1-c,eps)) at finalize (H never vanishes: max(.,eps) > 0), so
// the loop body is two plain sums; VARIANCE and MOMENTS have no dependency.
// HBM-bound streaming: one warp per row (rows shorter than 4096) or one
// 256-thread CTA per row, float4 loads when the row is 16-byte aligned,
// fp64 accumulation (the bound is HBM, not the FP64 pipe: <= 2 DFMA per 4 B
// loaded), butterfly shuffles + a shared-memory fold across warps (Eq.16).
#include "rf_internal.h"

namespace rf {
namespace {

constexpr int kThreads = 256;

template <int NACC>
struct Acc {
  double v[NACC];
};

template <int NACC>
__device__ __forceinline__ void warp_fold(Acc<NACC>& a) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NACC; ++i) a.v[i] += __shfl_xor_sync(0xffffffffu, a.v[i], off);
}

// Accumulate the row [first, len) with stride `step`, element-wise body `B`.
// Vectorised when both rows are 16-byte aligned and len % 4 == 0.
template <int MODE, int F>
struct Body;

template <int F>
struct Body<RF_PATTERN_VARIANCE, F> {
  static constexpr int NACC = 2;
  __device__ static void add(Acc<2>& a, float x, float) {
    a.v[0] += x;
    a.v[1] = fma(static_cast<double>(x), static_cast<double>(x), a.v[1]);
  }
};

template <int F>
struct Body<RF_PATTERN_SUM_SUM, F> {
  static constexpr int NACC = 2;
  __device__ static void add(Acc<2>& a, float x1, float x2) {
    a.v[0] = fma(static_cast<double>(x1), static_cast<double>(x1), a.v[0]);
    a.v[1] = fma(static_cast<double>(x1), static_cast<double>(x2), a.v[1]);
  }
};

template <int MODE, int F, bool ROW_PER_WARP>
__global__ void __launch_bounds__(kThreads)
    rowstats_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t rows,
                    int64_t len, float* __restrict__ d1, float* __restrict__ d2,
                    float* __restrict__ d3, double c, double eps) {
  using B = Body<MODE, F>;
  constexpr int NACC = B::NACC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = ROW_PER_WARP ? static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp
                                   : static_cast<int64_t>(blockIdx.x);
  if (row >= rows) return;  // whole warps (ROW_PER_WARP) or the whole CTA exit together
  const int t = ROW_PER_WARP ? lane : threadIdx.x;
  const int step = ROW_PER_WARP ? 32 : kThreads;
  const float* ar = a + row * len;
  const float* br = b ? b + row * len : ar;
  Acc<NACC> acc;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc.v[i] = 0.0;
  const bool vec = (len & 3) == 0 && (reinterpret_cast<uintptr_t>(ar) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(br) & 15) == 0;
  if (vec) {
    const float4* a4 = reinterpret_cast<const float4*>(ar);
    const float4* b4 = reinterpret_cast<const float4*>(br);
    for (int64_t i = t; i < len / 4; i += step) {
      const float4 x = __ldcs(a4 + i);
      const float4 y = b ? __ldcs(b4 + i) : x;
      B::add(acc, x.x, y.x);
      B::add(acc, x.y, y.y);
      B::add(acc, x.z, y.z);
      B::add(acc, x.w, y.w);
    }
  } else {
    for (int64_t i = t; i < len; i += step) B::add(acc, __ldcs(ar + i), b ? __ldcs(br + i) : 0.f);
  }
  warp_fold(acc);
  if (!ROW_PER_WARP) {
    __shared__ double part[kThreads / 32][NACC];
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < NACC; ++i) part[warp][i] = acc.v[i];
    __syncthreads();
    if (warp != 0) return;
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc.v[i] = lane < kThreads / 32 ? part[lane][i] : 0.0;
    warp_fold(acc);
  }
  if (lane != 0) return;
  d1[row] = static_cast<float>(acc.v[0]);
  if (MODE == RF_PATTERN_SUM_SUM)  // finalize_root: the telescoped correction
    d2[row] = static_cast<float>(acc.v[1] / sqrt(fmax(acc.v[0] - c, eps)));
  else
    d2[row] = static_cast<float>(acc.v[1]);
}

// MOMENTS: mass [rows, len], pos [rows, len, F] (reduce-axis major, the
// TensorStore layout); lane l handles element l: its F positions are
// contiguous, so a warp reads 32*F consecutive floats.
template <int F, bool ROW_PER_WARP>
__global__ void __launch_bounds__(kThreads)
    moments_kernel(const float* __restrict__ mass, const float* __restrict__ pos, int64_t rows,
                   int64_t len, float* __restrict__ d1, float* __restrict__ d2,
                   float* __restrict__ d3) {
  constexpr int NACC = 1 + 2 * F;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = ROW_PER_WARP ? static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp
                                   : static_cast<int64_t>(blockIdx.x);
  if (row >= rows) return;
  const int t = ROW_PER_WARP ? lane : threadIdx.x;
  const int step = ROW_PER_WARP ? 32 : kThreads;
  const float* mr = mass + row * len;
  const float* pr = pos + row * len * F;
  Acc<NACC> acc;
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc.v[i] = 0.0;
  for (int64_t l = t; l < len; l += step) {
    const double m = __ldcs(mr + l);
    acc.v[0] += m;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const double p = __ldcs(pr + l * F + f);
      const double mp = m * p;
      acc.v[1 + f] += mp;
      acc.v[1 + F + f] = fma(mp, p, acc.v[1 + F + f]);
    }
  }
  warp_fold(acc);
  if (!ROW_PER_WARP) {
    __shared__ double part[kThreads / 32][NACC];
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < NACC; ++i) part[warp][i] = acc.v[i];
    __syncthreads();
    if (warp != 0) return;
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc.v[i] = lane < kThreads / 32 ? part[lane][i] : 0.0;
    warp_fold(acc);
  }
  if (lane != 0) return;
  d1[row] = static_cast<float>(acc.v[0]);
#pragma unroll
  for (int f = 0; f < F; ++f) {
    d2[row * F + f] = static_cast<float>(acc.v[1 + f]);
    d3[row * F + f] = static_cast<float>(acc.v[1 + F + f]);
  }
}

}  // namespace

cudaError_t launch_rowstats(const RowStatsArgs& r, cudaStream_t st) {
  if (r.rows == 0) return cudaSuccess;
  const bool per_warp = r.len < 4096;
  const dim3 grid(static_cast<unsigned>(per_warp ? (r.rows + kThreads / 32 - 1) / (kThreads / 32) : r.rows));
  switch (r.pattern) {
    case RF_PATTERN_VARIANCE:
      if (per_warp)
        rowstats_kernel<RF_PATTERN_VARIANCE, 0, true><<<grid, kThreads, 0, st>>>(
            r.a, nullptr, r.rows, r.len, r.d1, r.d2, nullptr, 0.0, 0.0);
      else
        rowstats_kernel<RF_PATTERN_VARIANCE, 0, false><<<grid, kThreads, 0, st>>>(
            r.a, nullptr, r.rows, r.len, r.d1, r.d2, nullptr, 0.0, 0.0);
      break;
    case RF_PATTERN_SUM_SUM:
      if (per_warp)
        rowstats_kernel<RF_PATTERN_SUM_SUM, 0, true><<<grid, kThreads, 0, st>>>(
            r.a, r.b, r.rows, r.len, r.d1, r.d2, nullptr, r.c, r.eps);
      else
        rowstats_kernel<RF_PATTERN_SUM_SUM, 0, false><<<grid, kThreads, 0, st>>>(
            r.a, r.b, r.rows, r.len, r.d1, r.d2, nullptr, r.c, r.eps);
      break;
    case RF_PATTERN_MOMENTS:
      switch (r.free_len) {
#define RF_MOM_CASE(F)                                                                           \
  case F:                                                                                        \
    if (per_warp)                                                                                \
      moments_kernel<F, true><<<grid, kThreads, 0, st>>>(r.a, r.b, r.rows, r.len, r.d1, r.d2, r.d3); \
    else                                                                                         \
      moments_kernel<F, false><<<grid, kThreads, 0, st>>>(r.a, r.b, r.rows, r.len, r.d1, r.d2, r.d3); \
    break;
        RF_MOM_CASE(1)
        RF_MOM_CASE(2)
        RF_MOM_CASE(3)
        RF_MOM_CASE(4)
        RF_MOM_CASE(5)
        RF_MOM_CASE(6)
        RF_MOM_CASE(7)
        RF_MOM_CASE(8)
#undef RF_MOM_CASE
        default: return cudaErrorNotSupported;
      }
      break;
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

}  // namespace rf
