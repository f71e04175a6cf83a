// TEST INFRASTRUCTURE: single-CTA probes of the sm100.cuh building blocks
// (TMA SWIZZLE_128B tiles -> UMMA descriptors -> tcgen05.mma -> TMEM ->
// tcgen05.ld), checked against torch.matmul by tests/test_gpu_umma_probe.py.
// Built as librf_probe.so, never linked into librf_cuda.
#include <cuda_bf16.h>

#include "../sm100.cuh"

using namespace rf;
using namespace rf::sm100;

namespace {

struct ProbeArgs {
  int mode;  // 0 bf16 SS K-major | 1 bf16 SS B MN-major | 2 bf16 TS | 3 e4m3 SS | 4 TS + B MN-major
  int n, k;
  const void* a_glob;  // for TS: A rows read by threads
  float* d;
};

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                 ProbeArgs p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // up to 32 KB
  uint8_t* sB = smem + 32768;       // up to 64 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base_s;
  const int warp = warp_id();
  const int n = p.n, k = p.k;
  const bool fp8 = p.mode == 3;
  const bool ts = p.mode == 2 || p.mode == 4;
  const bool bmn = p.mode == 1 || p.mode == 4;

  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  // ---- loads ----
  if (threadIdx.x == 0) {
    const int eb = fp8 ? 1 : 2;
    uint32_t bytes = (ts ? 0u : 128u * k * eb) + static_cast<uint32_t>(n) * k * eb;
    mbar_arrive_expect_tx(&bar_load, bytes);
    const int kchunk = fp8 ? 128 : 64;  // elements per 128 B row
    if (!ts)
      for (int kc = 0; kc < k / kchunk; ++kc) tma_load_2d(sA + kc * 16384, &tma_a, &bar_load, kc * kchunk, 0);
    if (!bmn) {
      for (int kc = 0; kc < k / kchunk; ++kc)
        tma_load_2d(sB + kc * n * 128, &tma_b, &bar_load, kc * kchunk, 0);
    } else {
      for (int nc = 0; nc < n / 64; ++nc) tma_load_2d(sB + nc * k * 128, &tma_b, &bar_load, nc * 64, 0);
    }
  }
  if (ts) {
    // Thread r writes A row r (bf16 pairs) into TMEM columns [256, 256 + k/2).
    const __nv_bfloat16* arow = static_cast<const __nv_bfloat16*>(p.a_glob) + threadIdx.x * k;
    const uint32_t lane_base = (warp * 32) << 16;
    for (int c0 = 0; c0 < k / 2; c0 += 16) {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        r[j] = pack_bf16x2(__bfloat162float(arow[2 * (c0 + j)]), __bfloat162float(arow[2 * (c0 + j) + 1]));
      tmem_st16(tmem + lane_base + 256 + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  // ---- MMA ----
  if (warp == 0) {
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    if (elect_one()) {
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
      if (fp8) {
        const uint32_t id = idesc_f8(128, n);
        for (int ks = 0; ks < k / 32; ++ks)
          mma_f8_ss(tmem, sdesc_kmajor_sw128(a_base + ks * 32), sdesc_kmajor_sw128(b_base + ks * 32), id, ks > 0);
      } else {
        const uint32_t id = idesc_f16(128, n, kFmtBF16, false, bmn);
        for (int ks = 0; ks < k / 16; ++ks) {
          const int kc = ks / 4, w = ks % 4;
          uint64_t bd = bmn ? sdesc_mnmajor_sw128(b_base + ks * 2048, k * 128)
                            : sdesc_kmajor_sw128(b_base + kc * n * 128 + w * 32);
          if (ts)
            mma_f16_ts(tmem, tmem + 256 + ks * 8, bd, id, ks > 0);
          else
            mma_f16_ss(tmem, sdesc_kmajor_sw128(a_base + kc * 16384 + w * 32), bd, id, ks > 0);
        }
      }
      mma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  // ---- epilogue: thread = row ----
  const int row = threadIdx.x;
  for (int c0 = 0; c0 < n; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((warp * 32) << 16) + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) p.d[row * n + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace

extern "C" int rf_probe_umma(int mode, const void* a, const void* b, float* d, int n, int k) {
  if (n % 64 || k % 64 || n > 256 || k > 128) return 1;
  CUtensorMap ta{}, tb{};
  const bool fp8 = mode == 3;
  const int eb = fp8 ? 1 : 2;
  const uint32_t kchunk = fp8 ? 128 : 64;
  {
    uint64_t dims[2] = {(uint64_t)k, 128}, str[1] = {(uint64_t)k * eb};
    uint32_t box[2] = {kchunk, 128};
    if (!make_tmap(&ta, a, 2, dims, str, box, eb)) return 2;
  }
  if (mode == 1 || mode == 4) {  // B stored [K][N]
    uint64_t dims[2] = {(uint64_t)n, (uint64_t)k}, str[1] = {(uint64_t)n * eb};
    uint32_t box[2] = {64, (uint32_t)k};
    if (!make_tmap(&tb, b, 2, dims, str, box, eb)) return 3;
  } else {  // B stored [N][K]
    uint64_t dims[2] = {(uint64_t)k, (uint64_t)n}, str[1] = {(uint64_t)k * eb};
    uint32_t box[2] = {kchunk, (uint32_t)n};
    if (!make_tmap(&tb, b, 2, dims, str, box, eb)) return 4;
  }
  ProbeArgs p{mode, n, k, a, d};
  const int smem = 98304 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(ta, tb, p);
  if (cudaGetLastError() != cudaSuccess) return 5;
  if (cudaDeviceSynchronize() != cudaSuccess) return 6;
  return 0;
}
