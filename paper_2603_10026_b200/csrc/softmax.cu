// Safe softmax statistics (d1 = max x, d2 = sum exp(x - d1)) in ONE pass over
// x: the cascade of make_safe_softmax (proj/src/workloads.cpp:38-62) in the
// incremental form. Each thread streams its strided elements with the Eq.17
// element update (store-prev, correct by exp(d1' - d1) — golden
// corrections.txt — reduce); the per-thread partials are then combined with
// the Eq.16 merge (incr_push_child, proj/src/simulator.cpp:592-608) across
// the warp and the CTA. HBM-bound: x is read once, 16 B vector loads.
#include "rf_internal.h"

namespace rf {
namespace {

struct MS {
  float m, t;
};

__device__ __forceinline__ void ingest(MS& s, float x) {
  // incr_ingest_element: m' = m; m = max(m, x); t = t e^(m'-m) + e^(x-m)
  const float mn = fmaxf(s.m, x);
  s.t = s.t * __expf(s.m - mn) + __expf(x - mn);
  s.m = mn;
}

__device__ __forceinline__ MS merge(MS a, MS b) {
  const float mn = fmaxf(a.m, b.m);
  if (mn == -INFINITY) return a;
  MS r;
  r.t = a.t * __expf(a.m - mn) + b.t * __expf(b.m - mn);
  r.m = mn;
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT) softmax_rows_kernel(const float* __restrict__ x, int64_t n,
                                                          float* __restrict__ d1,
                                                          float* __restrict__ d2) {
  const float* xr = x + static_cast<int64_t>(blockIdx.x) * n;
  MS s{-INFINITY, 0.f};
  const bool vec = (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0);
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(xr);
    for (int64_t i = threadIdx.x; i < n / 4; i += NT) {
      float4 v = __ldg(x4 + i);
      ingest(s, v.x);
      ingest(s, v.y);
      ingest(s, v.z);
      ingest(s, v.w);
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += NT) ingest(s, __ldg(xr + i));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    MS o{__shfl_xor_sync(0xffffffffu, s.m, off), __shfl_xor_sync(0xffffffffu, s.t, off)};
    s = merge(s, o);
  }
  __shared__ MS part[NT / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    MS r = part[0];
    for (int w = 1; w < NT / 32; ++w) r = merge(r, part[w]);  // warp order
    d1[blockIdx.x] = r.m;
    d2[blockIdx.x] = r.t;
  }
}

}  // namespace

cudaError_t launch_softmax_rows(const float* x, int64_t rows, int64_t n, float* d1, float* d2,
                                cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  if (n <= 2048)
    softmax_rows_kernel<128><<<static_cast<unsigned>(rows), 128, 0, st>>>(x, n, d1, d2);
  else
    softmax_rows_kernel<512><<<static_cast<unsigned>(rows), 512, 0, st>>>(x, n, d1, d2);
  return cudaGetLastError();
}

}  // namespace rf
