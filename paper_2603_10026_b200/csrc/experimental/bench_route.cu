// TEST-ONLY micro-benchmark (not part of librf_cuda): latency of one warp's
// routing cascade (routing.cuh warp_route: top-K' of 128 experts, 4 per lane)
// against a shuffle-butterfly argmax and the round-1 form (local 64-bit max +
// two redux.sync per round), in SM cycles per token with one warp per SM
// sub-partition busy — the router kernel's tail runs one token per warp.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I.. -o bench_route bench_route.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../routing.cuh"

using namespace rf;

// sorted heads: one redux.sync of the heads' value bits + a ballot per round,
// a second redux only on a value tie; the winner lane stores its record
template <int PER, int K>
__device__ __forceinline__ void route_ballot(const float (&x)[PER], int lane, int2* topk, float* d1) {
  uint64_t key[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) key[j] = route_key(x[j], lane + 32 * j + 1);
#pragma unroll
  for (int i = 0; i < PER; ++i)
#pragma unroll
    for (int j = i & 1; j + 1 < PER; j += 2) {
      const uint64_t a = key[j], b = key[j + 1];
      key[j] = a > b ? a : b;
      key[j + 1] = a > b ? b : a;
    }
  float m = -INFINITY;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t hi = static_cast<uint32_t>(key[0] >> 32);
    const uint32_t hmax = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t held = __ballot_sync(0xffffffffu, hi == hmax);
    int winner;
    if (__popc(held) == 1) {
      winner = __ffs(held) - 1;
    } else {
      const uint32_t lo = __reduce_max_sync(0xffffffffu, hi == hmax ? static_cast<uint32_t>(key[0]) : 0u);
      winner = __ffs(__ballot_sync(0xffffffffu, hi == hmax && static_cast<uint32_t>(key[0]) == lo)) - 1;
    }
    if (r == 0) m = route_value(static_cast<uint64_t>(hmax) << 32);
    if (lane == winner) {
      topk[r] = make_int2(__float_as_int(route_value(key[0])), route_index(key[0]));
#pragma unroll
      for (int j = 0; j + 1 < PER; ++j) key[j] = key[j + 1];
      key[PER - 1] = 0ull;
    }
  }
  if (lane == 0) *d1 = m;
}

// sorted heads + two redux per round (no ballot, no divergent store)
template <int PER, int K>
__device__ __forceinline__ void route_heads(const float (&x)[PER], int lane, int2* topk, float* d1) {
  uint64_t key[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) key[j] = route_key(x[j], lane + 32 * j + 1);
#pragma unroll
  for (int i = 0; i < PER; ++i)
#pragma unroll
    for (int j = i & 1; j + 1 < PER; j += 2) {
      const uint64_t a = key[j], b = key[j + 1];
      key[j] = a > b ? a : b;
      key[j + 1] = a > b ? b : a;
    }
  float m = -INFINITY;
  int2 rec = make_int2(0, 0);
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const uint32_t hi = static_cast<uint32_t>(key[0] >> 32);
    const uint32_t hmax = __reduce_max_sync(0xffffffffu, hi);
    const uint32_t lo = __reduce_max_sync(0xffffffffu, hi == hmax ? static_cast<uint32_t>(key[0]) : 0u);
    const uint64_t best = (static_cast<uint64_t>(hmax) << 32) | lo;
    const bool mine = key[0] == best;
#pragma unroll
    for (int j = 0; j + 1 < PER; ++j) key[j] = mine ? key[j + 1] : key[j];
    key[PER - 1] = mine ? 0ull : key[PER - 1];
    if (r == 0) m = route_value(best);
    if (lane == r) rec = make_int2(__float_as_int(route_value(best)), route_index(best));
  }
  if (lane < K) topk[lane] = rec;
  if (lane == 0) *d1 = m;
}

// sorted heads + a 64-bit shuffle butterfly per round
template <int PER, int K>
__device__ __forceinline__ void route_shfl(const float (&x)[PER], int lane, int2* topk, float* d1) {
  uint64_t key[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) key[j] = route_key(x[j], lane + 32 * j + 1);
#pragma unroll
  for (int i = 0; i < PER; ++i)
#pragma unroll
    for (int j = i & 1; j + 1 < PER; j += 2) {
      const uint64_t a = key[j], b = key[j + 1];
      key[j] = a > b ? a : b;
      key[j + 1] = a > b ? b : a;
    }
  float m = -INFINITY;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    uint64_t best = key[0];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, best, off);
      best = o > best ? o : best;
    }
    if (r == 0) m = route_value(best);
    if (key[0] == best) {
      topk[r] = make_int2(__float_as_int(route_value(best)), route_index(best));
#pragma unroll
      for (int j = 0; j + 1 < PER; ++j) key[j] = key[j + 1];
      key[PER - 1] = 0ull;
    }
  }
  if (lane == 0) *d1 = m;
}

template <int MODE>
__global__ void __launch_bounds__(512) route_bench(const float* __restrict__ s, int2* topk, float* d1, float* d2,
                                                   long long* cyc, int reps) {
  constexpr int PER = 4, K = 8;
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  float x[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) x[j] = s[w * 128 + lane + 32 * j];
  long long total = 0;
  for (int it = 0; it < reps; ++it) {
    __syncwarp();
    const long long t0 = clock64();
    if (MODE == 0) warp_route<PER, K>(x, 128, lane, d1 + w, d2 + w, topk + w * K);
    if (MODE == 1) route_ballot<PER, K>(x, lane, topk + w * K, d1 + w);
    if (MODE == 2) route_shfl<PER, K>(x, lane, topk + w * K, d1 + w);
    if (MODE == 3) route_heads<PER, K>(x, lane, topk + w * K, d1 + w);
    __syncwarp();
    const long long t1 = clock64();
    total += t1 - t0;
#pragma unroll
    for (int j = 0; j < PER; ++j) x[j] += 1e-3f * it;  // new data each rep
  }
  if (lane == 0) cyc[w] = total / reps;
}

int main() {
  const int warps = 148 * 16;
  float* s;
  int2* tk;
  float *d1, *d2;
  long long* cyc;
  cudaMalloc(&s, warps * 128 * sizeof(float));
  cudaMalloc(&tk, warps * 8 * sizeof(int2));
  cudaMalloc(&d1, warps * 4);
  cudaMalloc(&d2, warps * 4);
  cudaMalloc(&cyc, warps * sizeof(long long));
  float* h = new float[warps * 128];
  unsigned z = 1;
  for (int i = 0; i < warps * 128; ++i) {
    z = z * 1664525u + 1013904223u;
    h[i] = static_cast<float>(z >> 8) / 16777216.0f;
  }
  cudaMemcpy(s, h, warps * 128 * sizeof(float), cudaMemcpyHostToDevice);
  const char* names[4] = {"routing.cuh (sorted heads, 2 x redux; + d2)", "sorted heads, redux + ballot",
                          "sorted heads, 64-bit shuffle butterfly", "sorted heads, 2 x redux"};
  static long long hc[148 * 16];
  for (int threads : {128, 512}) {
    const int nw = 148 * threads / 32;
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) route_bench<0><<<148, threads>>>(s, tk, d1, d2, cyc, 64);
        if (mode == 1) route_bench<1><<<148, threads>>>(s, tk, d1, d2, cyc, 64);
        if (mode == 2) route_bench<2><<<148, threads>>>(s, tk, d1, d2, cyc, 64);
        if (mode == 3) route_bench<3><<<148, threads>>>(s, tk, d1, d2, cyc, 64);
      }
      if (cudaDeviceSynchronize() != cudaSuccess) return 1;
      cudaMemcpy(hc, cyc, nw * sizeof(long long), cudaMemcpyDeviceToHost);
      double sum = 0;
      for (int i = 0; i < nw; ++i) sum += hc[i];
      printf("%2d warps/SM  %-42s K'=8 of 128: %.0f cycles per token\n", threads / 32, names[mode], sum / nw);
    }
  }
  return 0;
}
