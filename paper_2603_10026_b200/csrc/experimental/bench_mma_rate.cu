// TEST-ONLY micro-benchmark (not part of librf_cuda): sustained issue rate of
// the 2-SM tcgen05 MMA groups the FP8 quant GEMM uses, with no loads, no
// quantiser and no epilogue — the tensor pipe's own ceiling for each operand
// form. One CTA pair per SM pair, every pair issuing R groups back to back.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I.. -o mma_rate bench_mma_rate.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../sm100.cuh"

using namespace rf::sm100;

struct Mode {
  const char* name;
  int kind;    // 0 = f8f6f4, 1 = f16 (bf16)
  int ts;      // A from TMEM
  int n;       // N per MMA
  int halves;  // MMAs per K sub-step (N halves)
  int m = 256; // pair M (128: 64 rows per CTA, the MLA kernel's form)
};

__device__ __forceinline__ void mma_f8_ts_2sm(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

struct Smem {
  uint8_t a[16384];
  uint8_t b[2][32768];
  uint64_t done;
  uint32_t tmem_base;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    rate_kernel(int kind, int ts, int n, int halves, int reps, long long* out, int m = 256) {
  extern __shared__ uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const bool leader = cluster_ctarank() == 0;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c3a3836u ^ (i * 2654435761u);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3a383634u ^ (i * 2246822519u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&s.done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (leader && threadIdx.x < 32) {
    const bool el = elect_one();
    const uint32_t id = kind == 0 ? idesc_f8(m, n) : idesc_f16(m, n, kFmtBF16, false, false);
    const int ksub = 4;  // 128 B of K per row: 4 x K=32 (fp8) or 4 x K=16 (bf16)
    const uint32_t acol = 448;           // TS: A operand columns (32 per K tile)
    long long t0 = clock64();
    if (el) {
      for (int r = 0; r < reps; ++r) {
        const uint32_t a = smem_u32(s.a), b = smem_u32(s.b[r & 1]);
        for (int h = 0; h < halves; ++h)
          for (int ks = 0; ks < ksub; ++ks) {
            const uint64_t bd = sdesc_kmajor_sw128(b + h * (n / 2) * 128 + ks * 32);
            if (kind == 0 && ts)
              mma_f8_ts_2sm(tmem + h * n, tmem + acol + ks * 8, bd, id, r | ks);
            else if (kind == 0)
              mma_f8_ss_2sm(tmem + h * n, sdesc_kmajor_sw128(a + ks * 32), bd, id, r | ks);
            else if (ts)
              mma_f16_ts_2sm(tmem + h * n, tmem + acol + ks * 8, bd, id, r | ks);
            else
              mma_f16_ss_2sm(tmem + h * n, sdesc_kmajor_sw128(a + ks * 32), bd, id, r | ks);
          }
      }
      mma_commit_2sm(&s.done);
    }
    __syncwarp();
    mbar_wait(&s.done, 0);
    const long long t1 = clock64();
    if (el) out[blockIdx.x >> 1] = t1 - t0;
  } else if (threadIdx.x < 32) {
    mbar_wait(&s.done, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) tmem_dealloc_2sm<512>(tmem);
}

// 1-SM forms (the attention kernel's S = Q K^T (SS, K-major B) and O += P V
// (TS, V MN-major)): one CTA per SM, M = 128.
__global__ void __launch_bounds__(128, 1)
    rate1_kernel(int ts, int mn_b, int n, int reps, long long* out, int mn_a = 0) {
  extern __shared__ uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(s.a)[i] = 0x3c3a3836u ^ (i * 2654435761u);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(s.b)[i] = 0x3a383634u ^ (i * 2246822519u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&s.done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (threadIdx.x < 32) {
    const bool el = elect_one();
    const uint32_t id = idesc_f16(128, n, kFmtBF16, mn_a != 0, mn_b != 0);
    long long t0 = clock64();
    if (el) {
      for (int r = 0; r < reps; ++r) {
        const uint32_t a = smem_u32(s.a), b = smem_u32(s.b[r & 1]);
        for (int ks = 0; ks < 8; ++ks) {  // K = 128 per group: 8 x K16
          // K-major B: 128 B rows, K16 = 32 B step inside the row, 2 row chunks of 64 K;
          // MN-major B (V): K16 = 16 rows of 128 B MN-chunks = 2048 B step
          const uint64_t bd = mn_b ? sdesc_mnmajor_sw128(b + ks * 2048, n * 128)
                                   : sdesc_kmajor_sw128(b + (ks >> 2) * (n * 128) + (ks & 3) * 32);
          if (ts)
            mma_f16_ts(tmem + 256, tmem + ks * 8, bd, id, r | ks);
          else
            mma_f16_ss(tmem + 256,
                       mn_a ? sdesc_mnmajor_sw128(a + ks * 2048, 128 * 128)
                            : sdesc_kmajor_sw128(a + (ks >> 2) * 16384 + (ks & 3) * 32),
                       bd, id, r | ks);
        }
      }
      mma_commit(&s.done);
    }
    __syncwarp();
    mbar_wait(&s.done, 0);
    const long long t1 = clock64();
    if (el) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main() {
  const Mode modes[] = {
      {"f8 SS N=256 x2 (qnt2)", 0, 0, 256, 2}, {"f8 TS N=224 x2 (qnt3)", 0, 1, 224, 2},
      {"f8 SS N=224 x2", 0, 0, 224, 2},        {"f8 TS N=256 x1", 0, 1, 256, 1},
      {"f8 SS N=256 x1", 0, 0, 256, 1},        {"f8 TS N=128 x2", 0, 1, 128, 2},
      {"bf16 SS N=256 x2", 1, 0, 256, 2},      {"bf16 TS N=224 x2", 1, 1, 224, 2},
      {"bf16 SS N=128 x1 (M=256)", 1, 0, 128, 1}, {"bf16 TS N=128 x1 (M=256)", 1, 1, 128, 1},
      {"bf16 SS N=256 x1 (M=256)", 1, 0, 256, 1}, {"bf16 SS N=128 x2 (M=256)", 1, 0, 128, 2},
      {"bf16 SS N=128 x1 (M=128, MLA S)", 1, 0, 128, 1, 128}, {"bf16 SS N=256 x1 (M=128, MLA PV)", 1, 0, 256, 1, 128},
      {"bf16 TS N=256 x1 (M=128)", 1, 1, 256, 1, 128},
  };
  const int pairs = 74, reps = 512;
  long long* out;
  cudaMalloc(&out, pairs * sizeof(long long));
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  for (const Mode& m : modes) {
    for (int it = 0; it < 2; ++it) rate_kernel<<<2 * pairs, 128, smem>>>(m.kind, m.ts, m.n, m.halves, reps, out, m.m);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", m.name, cudaGetErrorString(e));
      return 1;
    }
    long long h[74];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (long long v : h) {
      mx = v > mx ? v : mx;
      sum += v;
    }
    // floor per CTA: M = 128 rows per SM, 8192 (f8) / 4096 (bf16) MAC per clock per SM
    const double macs = (m.m / 2.0) * m.n * (m.kind == 0 ? 128.0 : 64.0) * m.halves;  // one 128-byte K tile, per CTA
    const double floor_cyc = macs / (m.kind == 0 ? 8192.0 : 4096.0);
    const double per = static_cast<double>(sum) / 74 / reps;
    printf("%-26s cycles per K tile: %7.1f (floor %6.1f) -> %.3f of peak (max-pair %.1f)\n", m.name, per,
           floor_cyc, floor_cyc / per, static_cast<double>(mx) / reps);
  }
  {
    struct M1 {
      const char* name;
      int ts, mn_b, n, mn_a;
    } m1[] = {{"bf16 1-SM SS N=128 A MN-major", 0, 0, 128, 1},
              {"bf16 1-SM SS N=128 B MN-major", 0, 1, 128, 0},
              {"bf16 1-SM SS N=128 A,B MN-major", 0, 1, 128, 1},{"bf16 1-SM SS N=128 (S=QK^T)", 0, 0, 128},
              {"bf16 1-SM TS N=128 MN-major B (PV)", 1, 1, 128},
              {"bf16 1-SM TS N=128 K-major B", 1, 0, 128},
              {"bf16 1-SM SS N=256", 0, 0, 256},
              {"bf16 1-SM TS N=64 K-major B", 1, 0, 64},
              {"bf16 1-SM SS N=64", 0, 0, 64},
              {"bf16 1-SM TS N=256 K-major B", 1, 0, 256},
              {"bf16 1-SM TS N=192 K-major B", 1, 0, 192}};
    long long* out1;
    cudaMalloc(&out1, 148 * sizeof(long long));
    const size_t smem1 = 160 * 1024;  // descriptors of the N = 256 / K = 128 case reach past Smem
    cudaFuncSetAttribute(rate1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem1));
    for (const M1& m : m1) {
      for (int it = 0; it < 2; ++it) rate1_kernel<<<148, 128, smem1>>>(m.ts, m.mn_b, m.n, reps, out1, m.mn_a);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("%s failed\n", m.name);
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, out1, sizeof h, cudaMemcpyDeviceToHost);
      double sum = 0;
      for (long long v : h) sum += v;
      const double floor_cyc = 128.0 * m.n * 128.0 / 4096.0;
      const double per = sum / 148 / reps;
      printf("%-36s cycles per K=128: %7.1f (floor %6.1f) -> %.3f of peak\n", m.name, per, floor_cyc,
             floor_cyc / per);
    }
  }
  return 0;
}
