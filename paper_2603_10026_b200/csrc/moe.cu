// MoE routing: softmax statistics + top-k over the experts of each token, in
// one pass — the reference cascade make_moe_routing
// (proj/src/workloads.cpp:124-169): d1 = max s, d2 = sum exp(s - d1),
// d3 = top-K' of s as (value, 1-based index), ties to the LOWEST index
// (topk_merge, proj/src/simulator.cpp:80-88; tests/test_workloads.cpp:210-224).
//
// One warp per token row. Each lane streams its experts (e = lane, lane + 32,
// ...) with the Eq.17 element update (d1 max, d2 corrected by exp(d1' - d1),
// d3 inserted into a sorted K'-list); the 32 lane states are then folded with
// the Eq.16 merge (incr_push_child): the (max, sum) combine and the top-k
// merge of two sorted lists, by butterfly shuffles. Index outputs are
// bit-exact: the order is total (value desc, index asc), so the result does
// not depend on the merge tree.
// Up to 256 experts the row is held in registers instead (8 per lane) and the
// top-K' is K' rounds of a warp argmax (routing.cuh): ~10x fewer instructions
// than the sorted-list merges, same results bit for bit.
#include "rf_internal.h"
#include "routing.cuh"

namespace rf {
namespace {


struct Cand {
  float v;
  int i;  // 1-based expert index; 0 = empty slot
};

// a ranks before b: larger value, then lower index (empty slots rank last)
__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  if (a.i == 0) return false;
  if (b.i == 0) return true;
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}

template <int K>
__device__ __forceinline__ void insert(Cand (&t)[K], Cand c) {
  // one pass of insertion into the sorted list (K <= 8, fully unrolled)
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (before(c, t[j])) {
      const Cand tmp = t[j];
      t[j] = c;
      c = tmp;
    }
  }
}

template <int K>
__global__ void moe_routing_kernel(const float* __restrict__ s, int64_t rows, int64_t experts,
                                   float* __restrict__ d1, float* __restrict__ d2,
                                   int2* __restrict__ topk) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float* sr = s + row * experts;
  float m = -INFINITY, t = 0.f;
  Cand tk[K];
#pragma unroll
  for (int j = 0; j < K; ++j) tk[j] = {0.f, 0};
  for (int64_t e = lane; e < experts; e += 32) {
    const float x = __ldg(sr + e);
    const float mn = fmaxf(m, x);
    t = t * __expf(m - mn) + __expf(x - mn);  // Eq.17: store-prev, correct, reduce
    m = mn;
    insert(tk, Cand{x, static_cast<int>(e) + 1});
  }
  // Eq.16 fold across lanes (butterfly: every lane ends with the full state)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, off);
    const float to = __shfl_xor_sync(0xffffffffu, t, off);
    const float mn = fmaxf(m, mo);
    if (mn != -INFINITY) {
      t = t * __expf(m - mn) + to * __expf(mo - mn);
      m = mn;
    }
    Cand other[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      other[j].v = __shfl_xor_sync(0xffffffffu, tk[j].v, off);
      other[j].i = __shfl_xor_sync(0xffffffffu, tk[j].i, off);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) insert(tk, other[j]);
  }
  if (lane == 0) {
    d1[row] = m;
    d2[row] = t;
  }
  if (lane < K) {
    Cand c = tk[0];
#pragma unroll
    for (int j = 1; j < K; ++j)
      if (lane == j) c = tk[j];
    topk[row * K + lane] = make_int2(__float_as_int(c.v), c.i);
  }
}

template <int K, int PER>
__global__ void __launch_bounds__(256) moe_routing_regs_kernel(const float* __restrict__ s, int64_t rows,
                                                               int experts, float* __restrict__ d1,
                                                               float* __restrict__ d2, int2* __restrict__ topk) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float* sr = s + row * experts;
  float x[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane + 32 * j;
    x[j] = e < experts ? __ldg(sr + e) : 0.f;
  }
  warp_route<PER, K>(x, experts, lane, d1 + row, d2 + row, topk + row * K);
}

template <int K>
cudaError_t launch_k(const float* s, int64_t rows, int64_t experts, float* d1, float* d2, int2* out,
                     cudaStream_t st) {
  const int warps = 8;
  dim3 grid(static_cast<unsigned>((rows + warps - 1) / warps));
  const int e = static_cast<int>(experts);
  if (experts <= 32) moe_routing_regs_kernel<K, 1><<<grid, warps * 32, 0, st>>>(s, rows, e, d1, d2, out);
  else if (experts <= 64) moe_routing_regs_kernel<K, 2><<<grid, warps * 32, 0, st>>>(s, rows, e, d1, d2, out);
  else if (experts <= 128) moe_routing_regs_kernel<K, 4><<<grid, warps * 32, 0, st>>>(s, rows, e, d1, d2, out);
  else if (experts <= 256) moe_routing_regs_kernel<K, 8><<<grid, warps * 32, 0, st>>>(s, rows, e, d1, d2, out);
  else moe_routing_kernel<K><<<grid, warps * 32, 0, st>>>(s, rows, experts, d1, d2, out);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_moe_routing(const float* s, int64_t rows, int64_t experts, int k, float* d1,
                               float* d2, void* topk, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  int2* out = static_cast<int2*>(topk);
  switch (k) {
#define RF_MOE_CASE(K) \
  case K: return launch_k<K>(s, rows, experts, d1, d2, out, st);
    RF_MOE_CASE(1)
    RF_MOE_CASE(2)
    RF_MOE_CASE(3)
    RF_MOE_CASE(4)
    RF_MOE_CASE(5)
    RF_MOE_CASE(6)
    RF_MOE_CASE(7)
    RF_MOE_CASE(8)
#undef RF_MOE_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace rf
