// microbenchmark: per-SM throughput of the softmax's instruction mix on B200
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pk(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t cvth2(float a, float b) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
template <int MODE>
__global__ void k(float* out, int iters) {
  float v[16]; uint64_t w[16]; uint32_t u[16];
  for (int i = 0; i < 16; ++i) { v[i] = threadIdx.x * 1e-3f + i; w[i] = (uint64_t)__float_as_uint(v[i]) | ((uint64_t)__float_as_uint(v[i]*2) << 32); u[i] = i; }
  const uint64_t c = 0x3f8000003f800000ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]);
      if (MODE == 1) w[i] = ffma2(w[i], c, w[i]);
      if (MODE == 2) u[i] = pk(v[i], __uint_as_float(u[i]));
      if (MODE == 3) v[i] = fmaf(v[i], 1.0001f, 0.5f);
      if (MODE == 4) { v[i] = fmaxf(fmaxf(v[i], v[(i+1)&15]), v[(i+2)&15]); }
      if (MODE == 5) u[i] = ex2h2(u[i]);   // 2 exps per lane
      if (MODE == 6) u[i] = ex2b2(u[i]);   // 2 exps per lane
      if (MODE == 7) u[i] = cvth2(v[i], __uint_as_float(u[i]));
    }
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += v[i] + (float)(w[i] & 0xff) + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float) * 4);
  const char* names[] = {"MUFU.EX2 (ex2.approx)", "FFMA2 (fma.rn.f32x2, 2 lanes)", "F2FP bf16x2 pack (2 lanes)", "FFMA", "FMNMX3",
                         "MUFU.EX2 f16x2 (2 exps/lane)", "MUFU.EX2 bf16x2 (2 exps/lane)", "F2FP f16x2 pack"};
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 8; ++mode) {
    for (int warps : {8, 16, 32}) {
      int iters = 4096;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&]() {
        switch (mode) {
          case 0: k<0><<<148, warps * 32>>>(out, iters); break;
          case 1: k<1><<<148, warps * 32>>>(out, iters); break;
          case 2: k<2><<<148, warps * 32>>>(out, iters); break;
          case 3: k<3><<<148, warps * 32>>>(out, iters); break;
          case 4: k<4><<<148, warps * 32>>>(out, iters); break;
          case 5: k<5><<<148, warps * 32>>>(out, iters); break;
          case 6: k<6><<<148, warps * 32>>>(out, iters); break;
          case 7: k<7><<<148, warps * 32>>>(out, iters); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = 148.0 * warps * 32 * iters * 16;  // thread-instructions
      double per_sm_clk = ops / 148 / (ms * 1e-3 * clk * 1e3);
      printf("%-32s warps/SM %2d: %.1f thread-instr/clk/SM\n", names[mode], warps, per_sm_clk);
    }
  }
}
