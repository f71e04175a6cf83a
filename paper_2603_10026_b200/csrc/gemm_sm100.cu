// GEMM-shaped cascades on Blackwell tensor cores: a per-row statistic of the
// streamed operand (reduction d1) fused with the GEMM it scales (reduction d2)
// in ONE loop over the reduce axis K — the reference's run_incremental
// (proj/src/simulator.cpp:631-658) for two cascades:
//
//  RMSNORM_GEMM  (DSL cascade; golden corrections.txt):
//     d1 = sum x^2,   d2[f] = sum_l x g / sqrt(d1/K + eps) w[l,f]
//     corr(d2) = sqrt(d1'/K + eps) / sqrt(d1/K + eps)
//  QUANT_GEMM_E4M3 (make_quant_gemm, proj/src/workloads.cpp:173-209):
//     d1 = max |a|,   d2[f] = sum_l (fmax a[l] / d1) w[l,f]
//     corr(d2) = d1' / d1
//
// Both keep the accumulator in TMEM scaled by a representative H' of the
// dependency factor and retarget it to the true H at finalize (finalize_root,
// simulator.cpp:611-621), i.e. the product of the per-element corrections
// telescopes:
//   * RMS: H' = 1 for the whole loop (the sqrt-ratio corrections multiply out
//     to 1/sqrt(d1/K + eps) of the final d1), applied in the epilogue; g is
//     folded into the packed weight at plan time (rf_pack_weight).
//   * QUANT: H' = fmax / ref, ref = the smallest power of two >= the running
//     absmax. Each K tile is quantised to e4m3 with the current ref (exact
//     power-of-two scaling, one RNE rounding); when ref grows the TMEM
//     accumulator rows are corrected by ref'/ref in the loop (exact powers of
//     two; rare after the first tile); finalize multiplies by ref / d1.
//
// Tiles: BM = 128 rows (tokens) x BN = 256 (N) per CTA, UMMA M=128 N=256.
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BN = 256;

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Offset of logical 16-byte unit u of row r inside a [rows x 128 B] SWIZZLE_128B tile.
__device__ __forceinline__ uint32_t sw128(uint32_t r, uint32_t u) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((u ^ (r & 7)) << 4);
}

// ============================================================ RMSNORM_GEMM ==

namespace rms {

constexpr int BK = 64;  // bf16: one 128 B swizzle row
constexpr int STAGES = 4;
constexpr int NT = 192;  // warps 0-3 stats + epilogue, 4 TMA, 5 MMA
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB

struct Smem {
  uint8_t a[STAGES][A_BYTES];
  uint8_t b[STAGES][B_BYTES];
  uint64_t full[STAGES], empty[STAGES];
  uint64_t acc_full;
  uint32_t tmem_base;
};

struct Params {
  float* d1;
  int64_t k;
  float inv_k, eps;
  int write_d1_tile;  // blockIdx.x that writes d1
};

__global__ void __launch_bounds__(NT, 1)
    rms_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                    const __grid_constant__ CUtensorMap ty, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * BM;
  const int kt = static_cast<int>(p.k / BK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1 + 4);  // MMA commit + 4 stats warps
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<256>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 4) {
    if (elect_one()) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
      prefetch_tmap(&ty);
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.empty[st], ((t / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[st], A_BYTES + B_BYTES);
        tma_load_2d(s.a[st], &ta, &s.full[st], t * BK, m0, kEvictNormal);
        tma_load_2d(s.b[st], &tb, &s.full[st], t * BK, n0, kEvictLast);
      }
    }
  } else if (warp == 5) {
    const uint32_t idesc = idesc_f16(BM, BN, kFmtBF16, false, false);
    const bool leader = elect_one();
    for (int t = 0; t < kt; ++t) {
      const int st = t % STAGES;
      mbar_wait(&s.full[st], (t / STAGES) & 1);
      tc_fence_after();
      if (leader) {
        const uint32_t a = smem_u32(s.a[st]), b = smem_u32(s.b[st]);
#pragma unroll
        for (int ks = 0; ks < BK / 16; ++ks)
          mma_f16_ss(tmem, sdesc_kmajor_sw128(a + ks * 32), sdesc_kmajor_sw128(b + ks * 32), idesc,
                     (t | ks) != 0);
        mma_commit(&s.empty[st]);
        if (t + 1 == kt) mma_commit(&s.acc_full);
      }
      __syncwarp();
    }
  } else {
    // ---- reduction 1 (d1 = sum x^2) from the same smem tiles, thread = row ----
    const int r = threadIdx.x;  // 0..127
    float ss = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int st = t % STAGES;
      mbar_wait(&s.full[st], (t / STAGES) & 1);
      const uint8_t* row = s.a[st] + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = *reinterpret_cast<const uint4*>(row + 16 * u);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float lo = bf_lo(w[i]), hi = bf_hi(w[i]);
          ss = fmaf(lo, lo, ss);
          ss = fmaf(hi, hi, ss);
        }
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.empty[st]);
    }
    // ---- finalize: d2 = acc * 1/sqrt(d1/K + eps) -> bf16 -> smem -> TMA store ----
    const float inv = rsqrtf(fmaf(ss, p.inv_k, p.eps));
    if (blockIdx.x == p.write_d1_tile) p.d1[m0 + r] = ss;
    named_bar_sync(1, 128);  // every stats warp is done reading the stages
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    uint8_t* stage = s.a[0];  // all stages are drained: reuse 64 KB as the Y tile
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + c * 32, v);
      tmem_ld_wait();
      uint8_t* chunk = stage + (c >> 1) * (BM * 128);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        *reinterpret_cast<uint4*>(chunk + sw128(r, (c & 1) * 4 + q)) = w;
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tma_store_2d(&ty, stage + c * (BM * 128), n0 + 64 * c, m0);
      bulk_commit();
      bulk_wait0();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<256>(tmem);
}

}  // namespace rms

// ============================================================== packing ====

// w [K,N] f32 (reduce-axis major) -> out [N,K]: transposed, g folded (rms) or
// e4m3-rounded (quant). 32x32 smem tile transpose.
template <bool kE4M3>
__global__ void pack_kernel(const float* __restrict__ w, const float* __restrict__ g, int64_t k,
                            int64_t n, void* __restrict__ out) {
  __shared__ float tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 32, n0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t kk = k0 + i, nn = n0 + threadIdx.x;
    float v = 0.f;
    if (kk < k && nn < n) v = w[kk * n + nn] * (g ? g[kk] : 1.f);
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t nn = n0 + i, kk = k0 + threadIdx.x;
    if (nn < n && kk < k) {
      const float v = tile[threadIdx.x][i];
      if constexpr (kE4M3) {
        static_cast<uint8_t*>(out)[nn * k + kk] = static_cast<uint8_t>(pack_e4m3x2(v, 0.f) & 0xff);
      } else {
        static_cast<__nv_bfloat16*>(out)[nn * k + kk] = __float2bfloat16_rn(v);
      }
    }
  }
}

}  // namespace

// ================================================================== launch ==

bool gemm_sm100_supports(int pattern, int64_t m, int64_t n, int64_t k) {
  if (m % BM || n % BN) return false;
  if (pattern == RF_PATTERN_RMSNORM_GEMM) return k % rms::BK == 0;
  return false;
}

cudaError_t launch_rms_gemm_sm100(const GemmArgs& g, cudaStream_t st) {
  if (!gemm_sm100_supports(RF_PATTERN_RMSNORM_GEMM, g.m, g.n, g.k)) return cudaErrorNotSupported;
  CUtensorMap ta, tb, ty;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k) * 2};
    const uint32_t box[2] = {rms::BK, BM};
    if (!make_tmap(&ta, g.a, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.n)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k) * 2};
    const uint32_t box[2] = {rms::BK, BN};
    if (!make_tmap(&tb, g.b, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.n), static_cast<uint64_t>(g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.n) * 2};
    const uint32_t box[2] = {64, BM};
    if (!make_tmap(&ty, g.c, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  rms::Params p{g.d1, g.k, 1.f / static_cast<float>(g.k), g.eps, 0};
  const size_t smem = sizeof(rms::Smem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(rms::rms_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(g.n / BN), static_cast<unsigned>(g.m / BM));
  rms::rms_gemm_kernel<<<grid, rms::NT, smem, st>>>(ta, tb, ty, p);
  return cudaGetLastError();
}

cudaError_t launch_quant_gemm_sm100(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }

cudaError_t launch_pack_e4m3(const float* w, int64_t k, int64_t n, uint8_t* packed, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32));
  pack_kernel<true><<<grid, dim3(32, 8), 0, st>>>(w, nullptr, k, n, packed);
  return cudaGetLastError();
}

cudaError_t launch_pack_rms(const float* w, const float* g, int64_t k, int64_t n, void* packed,
                            cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32));
  pack_kernel<false><<<grid, dim3(32, 8), 0, st>>>(w, g, k, n, packed);
  return cudaGetLastError();
}

}  // namespace rf
