// microbenchmark: the softmax body of attn_sm100_2sm.cu in isolation (registers only)
#include <cstdio>
#include <cstdint>
#include "../paper_2603_10026_b200/csrc/sm100.cuh"  // nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I. tools/bench_softmax_body.cu
using namespace rf::sm100;
template <int POLY, bool PACK, bool SUM>  // POLY: pairs out of 8 on the FMA pipe
__global__ void k(float* out, int iters, float base) {
  float sv[32];
  for (int j = 0; j < 32; ++j) sv[j] = base * (threadIdx.x + j) * 1e-4f;
  uint32_t acc = 0; float lsum = 0.f;
  const uint64_t c12 = f2(1.4427f, 1.4427f), nmb2 = f2(-3.f, -3.f);
  for (int it = 0; it < iters; ++it) {
    float mx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) mx[j] = sv[j];
#pragma unroll
    for (int j = 4; j < 32; ++j) mx[j & 3] = fmaxf(mx[j & 3], sv[j]);
    const float tm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
    uint64_t a2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const uint64_t x2 = ffma2(f2(sv[2 * jj], sv[2 * jj + 1]), c12, nmb2);
      uint64_t p2;
      if ((jj & 7) < POLY) p2 = ex2_poly2(x2);
      else { float x0, x1; f2split(x2, x0, x1); p2 = f2(ex2_mufu(x0), ex2_mufu(x1)); }
      if (SUM) a2[jj & 3] = fadd2(a2[jj & 3], p2);
      float p0, p1; f2split(p2, p0, p1);
      if (PACK) acc ^= pack_bf16x2(p0, p1); else acc ^= __float_as_uint(p0) ^ __float_as_uint(p1);
    }
    float r0, r1; f2split(fadd2(fadd2(a2[0], a2[1]), fadd2(a2[2], a2[3])), r0, r1);
    lsum += r0 + r1 + tm;
    sv[it & 31] += 1e-7f;  // keep the loop live
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = lsum + acc;
}
template <int P, bool K, bool S> void run(const char* name, float* out) {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int iters = 2000, warps = 16;
  k<P, K, S><<<148, warps * 32>>>(out, iters, 1.f); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<P, K, S><<<148, warps * 32>>>(out, iters, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double el = 148.0 * warps * 32 * iters * 32;
  printf("%-40s %.1f elements/clk/SM\n", name, el / 148 / (ms * 1e-3 * clk * 1e3));
}
int main() {
  float* out; cudaMalloc(&out, 148 * 1024 * 4);
  run<0, true, true>("poly 0/8, pack, sum", out);
  run<2, true, true>("poly 2/8, pack, sum", out);
  run<3, true, true>("poly 3/8, pack, sum", out);
  run<4, true, true>("poly 4/8, pack, sum", out);
  run<8, true, true>("poly 8/8, pack, sum", out);
  run<0, false, true>("poly 0/8, no pack, sum", out);
  run<0, false, false>("poly 0/8, no pack, no sum", out);
  run<3, false, false>("poly 3/8, no pack, no sum", out);
}
