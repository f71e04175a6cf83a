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

#include <cstdio>
#include <cstdlib>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

#ifdef RF_QNT_TRACE
// clock64 timeline of one CTA of the 2-SM quant kernel (probe build only,
// tools/trace_quant.py): slot = event * 64 + K step.
__device__ long long g_qnt_trace[2 * 4096];  // [CTA rank in the traced pair][event * 64 + K step]
__device__ int g_qnt_trace_cta;
#define QTRACE(ev, t)                                                                 \
  do {                                                                               \
    if ((blockIdx.x >> 1) == (g_qnt_trace_cta >> 1) && blockIdx.y == 0 && (t) < 64)  \
      g_qnt_trace[(blockIdx.x & 1) * 4096 + (ev) * 64 + (t)] = clock64();            \
  } while (0)
#else
#define QTRACE(ev, t) \
  do {                \
  } while (0)
#endif

constexpr int BM = 128;
constexpr int BN = 256;

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// Grouped rasterisation: CTAs walk column panels of `gn` N-tiles over all
// M-tiles, so a panel of the static weight (gn x BN x K) stays L2-resident
// while the activations stream, instead of re-reading the whole weight from
// HBM once per M-tile (the output stream would evict it).
// gn < 0: panels of -gn M-tiles instead, walking M fastest inside a panel and
// then every N tile: each activation panel is read from HBM once while the
// whole weight streams past it (L2-resident when it fits, evict-last).
__device__ __forceinline__ void tile_of(int b, int mt_count, int nt_count, int gn, int& mt,
                                        int& nt) {
  if (gn < 0) {
    const int gm = -gn;
    const int per_group = gm * nt_count;
    const int g = b / per_group;
    const int first_m = g * gm;
    const int height = min(gm, mt_count - first_m);
    const int w = b - g * per_group;
    nt = w / height;
    mt = first_m + w % height;
    return;
  }
  const int per_group = gn * mt_count;
  const int g = b / per_group;
  const int first_n = g * gn;
  const int width = min(gn, nt_count - first_n);
  const int w = b - g * per_group;
  mt = w / width;
  nt = first_n + w % width;
}

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
  int mt_count, nt_count, group_n;
  float* d2;            // layernorm: sum x^2 (d1 then holds sum x)
  const float* colsum;  // layernorm: column sums of the packed g*w
  int write_d4;         // layernorm: d4 requested
  // Multi-Segment (run_multisegment, simulator.cpp:660-687) as split-K: CTA
  // (tile, blockIdx.y = s) streams K slice s of k_slice elements from fresh
  // state and writes its raw partial state — the fp32 accumulator (H' = 1)
  // through `ty` (an fp32 map over [S * ws_rows, N]) and the slice's
  // statistics to ws_d1 / ws_d2 [S, ws_rows]; gemm_fold.cu folds the slices
  // in order. partial = 0: the single-segment loop (k_slice = k).
  int64_t k_slice;
  float* ws_d1;
  float* ws_d2;
  int64_t ws_rows;
  int partial;
};

// The raw fp32 accumulator of this warpgroup's 128 TMEM lanes (row r) x NCOLS
// columns -> smem staging, RND chunks of 32 columns (16 KB each) per round ->
// TMA store at (n0, row0). Called by the 128 statistics/epilogue threads.
template <int NCOLS, int RND>
__device__ __forceinline__ void store_acc_f32(uint32_t tmem_row, int r, uint8_t* stage_ptr,
                                              const CUtensorMap* tm, int n0, int row0) {
  const uint32_t stage = smem_u32(stage_ptr);
#pragma unroll 1
  for (int c0 = 0; c0 < NCOLS / 32; c0 += RND) {
#pragma unroll 1
    for (int c = 0; c < RND; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem_row + (c0 + c) * 32, v);
      tmem_ld_wait();
      const uint32_t chunk = stage + c * (BM * 128);
#pragma unroll
      for (int u = 0; u < 8; ++u) sts128(chunk + sw128(r, u), make_uint4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]));
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
      for (int c = 0; c < RND; ++c) tma_store_2d(tm, stage_ptr + c * (BM * 128), n0 + (c0 + c) * 32, row0);
      bulk_commit();
      bulk_wait_read0();
    }
    named_bar_sync(1, 128);
  }
}

__global__ void __launch_bounds__(NT, 1)
    rms_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                    const __grid_constant__ CUtensorMap ty, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  int mt, nt;
  tile_of(blockIdx.x, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const int n0 = nt * BN;
  const int m0 = mt * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);

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
        tma_load_2d(s.a[st], &ta, &s.full[st], k0 + t * BK, m0, kEvictNormal);
        tma_load_2d(s.b[st], &tb, &s.full[st], k0 + t * BK, n0, kEvictLast);
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
      const uint32_t row = smem_u32(s.a[st]) + (r >> 3) * 1024 + (r & 7) * 128;
      float ts[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // physical unit u ^ (r & 7): conflict-free across the 8 rows of a phase
        // (the sum of squares does not depend on the order within the row)
        const uint4 v = lds128(row + ((u ^ (r & 7)) << 4));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float lo = bf_lo(w[i]), hi = bf_hi(w[i]);
          ts[i] = fmaf(lo, lo, ts[i]);
          ts[i] = fmaf(hi, hi, ts[i]);
        }
      }
      ss += (ts[0] + ts[1]) + (ts[2] + ts[3]);  // per-tile partials: pairwise accumulation
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.empty[st]);
    }
    // ---- finalize: d2 = acc * 1/sqrt(d1/K + eps) -> bf16 -> smem -> TMA store ----
    const float inv = rsqrtf(fmaf(ss, p.inv_k, p.eps));
    named_bar_sync(1, 128);  // every stats warp is done reading the stages
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    const uint32_t stage = smem_u32(s.a[0]);  // all stages are drained: reuse 64 KB as the Y tile
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    if (p.partial) {  // slice partial state: raw accumulator + sum x^2 of the slice
      if (nt == 0) p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = ss;
      store_acc_f32<BN, 8>(tmem + lane_off, r, s.a[0], &ty, n0, static_cast<int>(blockIdx.y * p.ws_rows) + m0);
    } else {
    if (nt == 0) p.d1[m0 + r] = ss;
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + c * 32, v);
      tmem_ld_wait();
      const uint32_t chunk = stage + (c >> 1) * (BM * 128);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        sts128(chunk + sw128(r, (c & 1) * 4 + q), w);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tma_store_2d(&ty, s.a[0] + c * (BM * 128), n0 + 64 * c, m0);
      bulk_commit();
    }
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<256>(tmem);
}

}  // namespace rms

// ----------------------------------------------------- RMSNORM_GEMM, 2-SM --
//
// CTA pair (cluster of 2) on one 256 x 256 tile: tcgen05.mma.cta_group::2 with
// M = 256 issued by the leader; each CTA stages its own 128 rows of X and its
// half (128 N-rows) of W', so per-SM shared-memory traffic for B halves. The
// peer's tiles land on its local barrier (its statistics warps need them too)
// and a relay warp forwards that completion to the leader's barrier.

namespace rms2 {

constexpr int BK = 64;
constexpr int STAGES = 3;  // two CTA pairs per SM pair: one pair's epilogue overlaps the other's mainloop
constexpr int NT = 192;  // warps 0-3 stats + epilogue, 4 TMA, 5 MMA (leader) / relay (peer)
constexpr int A_BYTES = BM * BK * 2;  // 16 KB: this CTA's 128 rows
constexpr int B_BYTES = 128 * BK * 2; // 16 KB: this CTA's half of the 256 N-rows

struct Smem {
  uint8_t a[STAGES][A_BYTES];
  uint8_t b[STAGES][B_BYTES];
  uint64_t full[STAGES];       // leader: own tx + peer relay (count 2); peer: own tx (count 1)
  uint64_t empty[STAGES];      // MMA multicast commit + 4 stats warps
  uint64_t acc_full;
  uint32_t tmem_base;
};

// LN = false: RMSNORM_GEMM; LN = true: LAYERNORM_GEMM (the variance cascade
// d1 = sum x, d2 = sum x^2 from the same tiles; d3 = acc / sigma and
// d4 = (d1/K) / sigma * colsum in the epilogue — both corrections telescope).
template <bool LN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 2)
    rms_gemm_2sm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                        const __grid_constant__ CUtensorMap ty, const __grid_constant__ CUtensorMap ty4,
                        const rms::Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  int mt, nt;  // mt: 256-row pair tile
  tile_of(blockIdx.x >> 1, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const int n0 = nt * BN;
  const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM;  // this CTA's 128 rows
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], leader ? 2 : 1);
      mbar_init(&s.empty[i], 1 + 4);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc_2sm<256>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 4) {
    if (elect_one()) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
      prefetch_tmap(&ty);
      if (LN) prefetch_tmap(&ty4);
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.empty[st], ((t / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[st], A_BYTES + B_BYTES);
        tma_load_2d(s.a[st], &ta, &s.full[st], k0 + t * BK, m0, kEvictNormal);
        tma_load_2d(s.b[st], &tb, &s.full[st], k0 + t * BK, n0 + static_cast<int>(rank) * 128, kEvictLast);
      }
    }
  } else if (warp == 5) {
    if (leader) {
      const uint32_t idesc = idesc_f16(2 * BM, BN, kFmtBF16, false, false);
      const bool el = elect_one();
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.full[st], (t / STAGES) & 1);  // both halves landed
        tc_fence_after();
        if (el) {
          const uint32_t a = smem_u32(s.a[st]), b = smem_u32(s.b[st]);
#pragma unroll
          for (int ks = 0; ks < BK / 16; ++ks)
            mma_f16_ss_2sm(tmem, sdesc_kmajor_sw128(a + ks * 32), sdesc_kmajor_sw128(b + ks * 32),
                           idesc, (t | ks) != 0);
          mma_commit_2sm(&s.empty[st]);
          if (t + 1 == kt) mma_commit_2sm(&s.acc_full);
        }
        __syncwarp();
      }
    } else if (elect_one()) {
      // relay: this CTA's tiles have landed -> the leader's full barrier
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.full[st], (t / STAGES) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.full[st]), 0));
      }
    }
  } else {
    const int r = threadIdx.x;
    float ss = 0.f, sx = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int st = t % STAGES;
      mbar_wait(&s.full[st], (t / STAGES) & 1);
      const uint32_t row = smem_u32(s.a[st]) + (r >> 3) * 1024 + (r & 7) * 128;
      float ts[4] = {0.f, 0.f, 0.f, 0.f}, tx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 v = lds128(row + ((u ^ (r & 7)) << 4));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float lo = bf_lo(w[i]), hi = bf_hi(w[i]);
          ts[i] = fmaf(lo, lo, ts[i]);
          ts[i] = fmaf(hi, hi, ts[i]);
          if (LN) tx[i] += lo + hi;
        }
      }
      ss += (ts[0] + ts[1]) + (ts[2] + ts[3]);  // per-tile partials: pairwise accumulation
      if (LN) sx += (tx[0] + tx[1]) + (tx[2] + tx[3]);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.empty[st]);
    }
    float inv, mean = 0.f;
    if (p.partial) {  // slice partial state: statistics of the slice only
      if (nt == 0) {
        p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = LN ? sx : ss;
        if (LN) p.ws_d2[blockIdx.y * p.ws_rows + m0 + r] = ss;
      }
      inv = 0.f;
    } else if (LN) {
      mean = sx * p.inv_k;
      inv = rsqrtf(fmaf(ss, p.inv_k, -mean * mean) + p.eps);  // 1/sigma
      if (nt == 0) {
        p.d1[m0 + r] = sx;
        p.d2[m0 + r] = ss;
      }
    } else {
      inv = rsqrtf(fmaf(ss, p.inv_k, p.eps));
      if (nt == 0) p.d1[m0 + r] = ss;
    }
    named_bar_sync(1, 128);
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    const uint32_t stage = smem_u32(s.a[0]);  // drained: 64 KB of A stages for the Y tile
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    if (p.partial) {
      // raw accumulator (H' = 1) of the slice: 4 x 16 KB staged per round (the
      // drained A stages hold 48 KB with 3 stages)
      rms::store_acc_f32<BN, 2>(tmem + lane_off, r, s.a[0], &ty, n0, static_cast<int>(blockIdx.y * p.ws_rows) + m0);
    } else {
#pragma unroll
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + c * 32, v);
      tmem_ld_wait();
      const uint32_t chunk = stage + (c >> 1) * (BM * 128);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]) * inv, __uint_as_float(v[8 * q + 1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]) * inv, __uint_as_float(v[8 * q + 3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]) * inv, __uint_as_float(v[8 * q + 5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]) * inv, __uint_as_float(v[8 * q + 7]) * inv);
        sts128(chunk + sw128(r, (c & 1) * 4 + q), w);
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tma_store_2d_hint(&ty, s.a[0] + c * (BM * 128), n0 + 64 * c, m0, kEvictFirst);
      bulk_commit();
      bulk_wait_read0();
    }
    if (LN && p.write_d4) {
      // d4 = (d1/K) / sigma * colsum[f]: a rank-1 tile, staged the same way
      named_bar_sync(1, 128);  // staging area free again
      const float mi = mean * inv;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        const uint32_t chunk = stage + (c >> 1) * (BM * 128);
        const float* cs = p.colsum + n0 + c * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 c0 = __ldg(reinterpret_cast<const float4*>(cs + 8 * q));
          const float4 c1 = __ldg(reinterpret_cast<const float4*>(cs + 8 * q + 4));
          uint4 w;
          w.x = pack_bf16x2(mi * c0.x, mi * c0.y);
          w.y = pack_bf16x2(mi * c0.z, mi * c0.w);
          w.z = pack_bf16x2(mi * c1.x, mi * c1.y);
          w.w = pack_bf16x2(mi * c1.z, mi * c1.w);
          sts128(chunk + sw128(r, (c & 1) * 4 + q), w);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) tma_store_2d_hint(&ty4, s.a[0] + c * (BM * 128), n0 + 64 * c, m0, kEvictFirst);
        bulk_commit();
      }
    }
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 5) tmem_dealloc_2sm<256>(tmem);
}

}  // namespace rms2


// ========================================================= QUANT_GEMM_E4M3 ==

namespace qnt {

constexpr int BK = 128;   // e4m3: one 128 B swizzle row; the bf16 A tile is 2 chunks
constexpr int BNQ = 512;  // two N=256 MMAs per K step (amortises the in-loop quantiser)
constexpr int SA = 2, SW = 2, S8 = 2;
constexpr int NT = 192;   // warps 0-3 quantiser + epilogue, 4 TMA, 5 MMA
constexpr int ABF_BYTES = BM * BK * 2;  // 32 KB
constexpr int W_BYTES = BNQ * BK;       // 64 KB
constexpr int A8_BYTES = BM * BK;       // 16 KB

struct Smem {
  uint8_t abf[SA][ABF_BYTES];
  uint8_t w[SW][W_BYTES];
  uint8_t a8[S8][A8_BYTES];
  uint64_t abf_full[SA], abf_empty[SA], w_full[SW], w_empty[SW], a8_full[S8], a8_empty[S8];
  uint64_t acc_full;
  uint32_t tmem_base;
};

struct Params {
  float* d1;
  int* domain_flag;
  int64_t k;
  float fmax;
  int mt_count, nt_count, group_n;
  // Multi-Segment split-K (see rms::Params): slice s = blockIdx.y from fresh
  // state; partial = 1 writes acc * ref_s (the slice's accumulator in units of
  // fmax * a / 1, i.e. H' retargeted to 1) through `tc` over [S * ws_rows, N]
  // and the slice's absmax to ws_d1; gemm_fold.cu finishes c = sum / d1.
  int64_t k_slice;
  float* ws_d1;
  int64_t ws_rows;
  int partial;
};

__device__ __forceinline__ float pow2_ceil(float x) {
  if (!(x > 0.f)) return 0.f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x007fffffu) ? __uint_as_float((b & 0x7f800000u) + 0x00800000u) : x;
}

__device__ __forceinline__ uint32_t absmax_bf16x2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// 2 bf16 (packed) * scale -> 2 e4m3 (RNE, satfinite) in the low 16 bits.
__device__ __forceinline__ uint32_t quant_pair(uint32_t u, uint64_t scale2) {
  uint64_t x, y;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(u << 16), "r"(u & 0xffff0000u));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(y) : "l"(x), "l"(scale2));
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(y));
  return pack_e4m3x2(lo, hi);
}

__global__ void __launch_bounds__(NT, 1)
    quant_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tw,
                      const __grid_constant__ CUtensorMap tc, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  int mt, nt;
  tile_of(blockIdx.x, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const int n0 = nt * BNQ;
  const int m0 = mt * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);

  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&s.abf_full[i], 1);
      mbar_init(&s.abf_empty[i], 4);
    }
    for (int i = 0; i < SW; ++i) {
      mbar_init(&s.w_full[i], 1);
      mbar_init(&s.w_empty[i], 1);
    }
    for (int i = 0; i < S8; ++i) {
      mbar_init(&s.a8_full[i], 4);
      mbar_init(&s.a8_empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 4) {
    if (elect_one()) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tw);
      prefetch_tmap(&tc);
      for (int t = 0; t < kt; ++t) {
        const int sa = t % SA, sw = t % SW;
        mbar_wait(&s.abf_empty[sa], ((t / SA) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.abf_full[sa], ABF_BYTES);
        tma_load_2d(s.abf[sa], &ta, &s.abf_full[sa], k0 + t * BK, m0, kEvictFirst);
        tma_load_2d(s.abf[sa] + BM * 128, &ta, &s.abf_full[sa], k0 + t * BK + 64, m0, kEvictFirst);
        mbar_wait(&s.w_empty[sw], ((t / SW) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.w_full[sw], W_BYTES);
        tma_load_2d(s.w[sw], &tw, &s.w_full[sw], k0 + t * BK, n0, kEvictLast);
        tma_load_2d(s.w[sw] + 256 * 128, &tw, &s.w_full[sw], k0 + t * BK, n0 + 256, kEvictLast);
      }
    }
  } else if (warp == 5) {
    const uint32_t idesc = idesc_f8(BM, 256);
    const bool leader = elect_one();
    for (int t = 0; t < kt; ++t) {
      const int sw = t % SW, s8 = t % S8;
      mbar_wait(&s.w_full[sw], (t / SW) & 1);
      mbar_wait(&s.a8_full[s8], (t / S8) & 1);
      tc_fence_after();
      if (leader) {
        const uint32_t a = smem_u32(s.a8[s8]), b = smem_u32(s.w[sw]);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks)
            mma_f8_ss(tmem + h * 256, sdesc_kmajor_sw128(a + ks * 32),
                      sdesc_kmajor_sw128(b + h * 256 * 128 + ks * 32), idesc, (t | ks) != 0);
        mma_commit(&s.w_empty[sw]);
        mma_commit(&s.a8_empty[s8]);
        if (t + 1 == kt) mma_commit(&s.acc_full);
      }
      __syncwarp();
    }
  } else {
    // ---- reduction 1 (running absmax) + e4m3 quantisation of A, thread = row ----
    const int r = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float amax = 0.f, ref = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int sa = t % SA, s8 = t % S8;
      mbar_wait(&s.abf_full[sa], (t / SA) & 1);
      uint32_t x[64];  // logical K order: x[8c + 4*vv + i] covers K = 64c + 8vv + 2i .. +1
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 q = lds128(smem_u32(s.abf[sa]) + c * (BM * 128) + sw128(r, v));
          x[32 * c + 4 * v + 0] = q.x;
          x[32 * c + 4 * v + 1] = q.y;
          x[32 * c + 4 * v + 2] = q.z;
          x[32 * c + 4 * v + 3] = q.w;
        }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.abf_empty[sa]);
      uint32_t mx = absmax_bf16x2(x[0], x[1]);
#pragma unroll
      for (int i = 2; i < 64; ++i) mx = absmax_bf16x2(mx, x[i]);
      const float tile_max = fmaxf(__uint_as_float((mx << 16) & 0x7fffffffu),
                                   __uint_as_float(mx & 0x7fff0000u));
      amax = fmaxf(amax, tile_max);  // d1: store-prev (ref) / reduce
      const float nref = pow2_ceil(amax);
      // Eq.17 correction of the accumulator rows: corr = ref'/ref (powers of two)
      const bool changed = t > 0 && nref != ref;
      if (__any_sync(0xffffffffu, changed)) {
        const int sp = (t - 1) % S8;
        mbar_wait(&s.a8_empty[sp], ((t - 1) / S8) & 1);  // MMA of tile t-1 complete
        tc_fence_after();
        const float f = changed ? ref / nref : 1.f;
#pragma unroll 1
        for (int c = 0; c < 2 * 256 / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * f);
          tmem_st32(tmem + lane_off + c * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
      }
      ref = nref;
      // exact: fmax * 2^-e. While the running absmax is still 0 every element
      // seen is 0: H is not invertible and the guarded H' is the identity
      // (the reference's repair), so the tile contributes 0 — a scale of 0,
      // not fmax / 0 (0 * inf would poison the accumulator with NaN).
      const float sc = ref > 0.f ? p.fmax / ref : 0.f;
      uint64_t sc2;
      asm("mov.b64 %0, {%1, %1};" : "=l"(sc2) : "f"(sc));
      mbar_wait(&s.a8_empty[s8], ((t / S8) & 1) ^ 1);
      const uint32_t dst = smem_u32(s.a8[s8]);
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // logical 16-element unit u = K [16u, 16u+16)
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint32_t lo = quant_pair(x[8 * u + 2 * h], sc2);
          const uint32_t hi = quant_pair(x[8 * u + 2 * h + 1], sc2);
          w[h] = (lo & 0xffffu) | (hi << 16);
        }
        sts128(dst + sw128(r, u), make_uint4(w[0], w[1], w[2], w[3]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.a8_full[s8]);
    }
    // ---- finalize_root: retarget H'(ref) -> H(d1): c = acc * ref / d1 ----
    // (partial: the slice's state, retargeted to H' = 1: acc * ref)
    const float fin = p.partial ? ref : ref / amax;  // 0/0 -> NaN for an all-zero row (DomainError)
    if (p.partial) {
      if (nt == 0) p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = amax;
    } else {
      if (!(amax > 0.f)) atomicExch(p.domain_flag, 1);
      if (nt == 0) p.d1[m0 + r] = amax;
    }
    const int crow = p.partial ? static_cast<int>(blockIdx.y * p.ws_rows) + m0 : m0;
    named_bar_sync(1, 128);
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    const uint32_t stage = smem_u32(s.abf[0]);  // 192 KB of drained stages: C half-tile staging
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + lane_off + h * 256 + c * 32, v);
        tmem_ld_wait();
        const uint32_t chunk = stage + c * (BM * 128);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          sts128(chunk + sw128(r, u),
                 make_uint4(__float_as_uint(__uint_as_float(v[4 * u]) * fin),
                            __float_as_uint(__uint_as_float(v[4 * u + 1]) * fin),
                            __float_as_uint(__uint_as_float(v[4 * u + 2]) * fin),
                            __float_as_uint(__uint_as_float(v[4 * u + 3]) * fin)));
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          tma_store_2d(&tc, s.abf[0] + c * (BM * 128), n0 + h * 256 + 32 * c, crow);
        bulk_commit();
        bulk_wait_read0();
      }
      named_bar_sync(1, 128);
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

}  // namespace qnt

// ------------------------------------------------------ QUANT_GEMM, 2-SM --
//
// CTA pair on a 256 x 512 tile: each CTA quantises its own 128 rows of A into
// e4m3 (the in-loop correction stays CTA-local: each CTA rescales the TMEM
// rows it owns) and stages half of each 256-wide W block; the leader issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256, twice per K step). The peer
// relays "my W half landed and my A rows are quantised" for every K step.

namespace qnt2 {

using qnt::BK;
using qnt::BNQ;
// ring depths (A/B on cfg4, TFLOP/s): SA/SW/S8 = 3/3/2 2284, 2/3/2 2271,
// 2/3/3 2267, 2/4/2 2235, 3/2/3 2163
constexpr int SA = 3, SW = 3, S8 = 2;
constexpr int NT = 192;  // warps 0-3 quantiser + epilogue, 4 TMA, 5 MMA (leader) / relay (peer)
constexpr int ABF_BYTES = BM * BK * 2;  // 32 KB
constexpr int W_BYTES = 2 * 128 * BK;   // 32 KB: this CTA's halves of the two 256-row blocks
constexpr int A8_BYTES = BM * BK;       // 16 KB

struct Smem {
  uint8_t abf[SA][ABF_BYTES];
  uint8_t w[SW][W_BYTES];
  uint8_t a8[S8][A8_BYTES];
  uint64_t abf_full[SA], abf_empty[SA], w_full[SW], w_empty[SW], a8_full[S8], a8_empty[S8];
  uint64_t acc_full;
  uint32_t tmem_base;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    quant_gemm_2sm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tw,
                          const __grid_constant__ CUtensorMap tc, const qnt::Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  int mt, nt;
  tile_of(blockIdx.x >> 1, p.mt_count, p.nt_count, p.group_n, mt, nt);
  const int n0 = nt * BNQ;
  const int m0 = mt * 2 * BM + static_cast<int>(rank) * BM;
  const int kt = static_cast<int>(p.k_slice / BK);
  const int k0 = static_cast<int>(blockIdx.y * p.k_slice);
  if (threadIdx.x == 0) QTRACE(7, 2);

  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) {
      mbar_init(&s.abf_full[i], 1);
      mbar_init(&s.abf_empty[i], 4);
    }
    for (int i = 0; i < SW; ++i) {
      mbar_init(&s.w_full[i], 1);
      mbar_init(&s.w_empty[i], 1);
    }
    for (int i = 0; i < S8; ++i) {
      mbar_init(&s.a8_full[i], leader ? 4 + 1 : 4);  // leader: + peer relay
      mbar_init(&s.a8_empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  if (threadIdx.x == 0) QTRACE(7, 3);  // common origin of the pair's clocks

  if (warp == 4) {
    if (elect_one()) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tw);
      prefetch_tmap(&tc);
      for (int t = 0; t < kt; ++t) {
        const int sa = t % SA, sw = t % SW;
        mbar_wait(&s.abf_empty[sa], ((t / SA) & 1) ^ 1);
        QTRACE(5, t);
        mbar_arrive_expect_tx(&s.abf_full[sa], ABF_BYTES);
        tma_load_2d(s.abf[sa], &ta, &s.abf_full[sa], k0 + t * BK, m0, kEvictFirst);
        tma_load_2d(s.abf[sa] + BM * 128, &ta, &s.abf_full[sa], k0 + t * BK + 64, m0, kEvictFirst);
        mbar_wait(&s.w_empty[sw], ((t / SW) & 1) ^ 1);
        QTRACE(6, t);
        mbar_arrive_expect_tx(&s.w_full[sw], W_BYTES);
        for (int h = 0; h < 2; ++h)
          tma_load_2d(s.w[sw] + h * 128 * 128, &tw, &s.w_full[sw], k0 + t * BK,
                      n0 + 256 * h + 128 * static_cast<int>(rank), kEvictLast);
      }
    }
  } else if (warp == 5) {
    if (leader) {
      const uint32_t idesc = idesc_f8(2 * BM, 256);
      const bool el = elect_one();
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        mbar_wait(&s.w_full[sw], (t / SW) & 1);
        if (el) QTRACE(0, t);
        mbar_wait(&s.a8_full[s8], (t / S8) & 1);  // own A8 + peer (W half + A8) relay
        if (el) QTRACE(1, t);
        tc_fence_after();
        if (el) {
          const uint32_t a = smem_u32(s.a8[s8]), b = smem_u32(s.w[sw]);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int ks = 0; ks < BK / 32; ++ks)
              mma_f8_ss_2sm(tmem + h * 256, sdesc_kmajor_sw128(a + ks * 32),
                            sdesc_kmajor_sw128(b + h * 128 * 128 + ks * 32), idesc, (t | ks) != 0);
          mma_commit_2sm(&s.w_empty[sw]);
          mma_commit_2sm(&s.a8_empty[s8]);
          if (t + 1 == kt) mma_commit_2sm(&s.acc_full);
        }
        __syncwarp();
      }
    } else if (elect_one()) {
      for (int t = 0; t < kt; ++t) {
        const int sw = t % SW, s8 = t % S8;
        mbar_wait(&s.w_full[sw], (t / SW) & 1);
        mbar_wait(&s.a8_full[s8], (t / S8) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.a8_full[s8]), 0));
      }
    }
  } else {
    const int r = threadIdx.x;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float amax = 0.f, ref = 0.f;
    for (int t = 0; t < kt; ++t) {
      const int sa = t % SA, s8 = t % S8;
      mbar_wait(&s.abf_full[sa], (t / SA) & 1);
      if (threadIdx.x == 0) QTRACE(2, t);
      uint32_t x[64];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 q = lds128(smem_u32(s.abf[sa]) + c * (BM * 128) + sw128(r, v));
          x[32 * c + 4 * v + 0] = q.x;
          x[32 * c + 4 * v + 1] = q.y;
          x[32 * c + 4 * v + 2] = q.z;
          x[32 * c + 4 * v + 3] = q.w;
        }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.abf_empty[sa]);
      // tile absmax: 8 independent chains, then a 3-level tree (the quantiser
      // is on the MMA's critical path: a 63-long dependent chain costs ~300 cycles)
      uint32_t mc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mc[i] = qnt::absmax_bf16x2(x[i], x[i + 8]);
#pragma unroll
      for (int i = 16; i < 64; ++i) mc[i & 7] = qnt::absmax_bf16x2(mc[i & 7], x[i]);
#pragma unroll
      for (int w = 4; w > 0; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) mc[i] = qnt::absmax_bf16x2(mc[i], mc[i + w]);
      const uint32_t mx = mc[0];
      const float tile_max = fmaxf(__uint_as_float((mx << 16) & 0x7fffffffu),
                                   __uint_as_float(mx & 0x7fff0000u));
      amax = fmaxf(amax, tile_max);
      const float nref = qnt::pow2_ceil(amax);
      const bool changed = t > 0 && nref != ref;
      if (__any_sync(0xffffffffu, changed)) {
        const int sp = (t - 1) % S8;
        mbar_wait(&s.a8_empty[sp], ((t - 1) / S8) & 1);  // MMA of tile t-1 complete
        tc_fence_after();
        const float f = changed ? ref / nref : 1.f;
#pragma unroll 1
        for (int c = 0; c < 2 * 256 / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(tmem + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * f);
          tmem_st32(tmem + lane_off + c * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
      }
      ref = nref;
      const float sc = ref > 0.f ? p.fmax / ref : 0.f;  // see quant_gemm_kernel
      uint64_t sc2;
      asm("mov.b64 %0, {%1, %1};" : "=l"(sc2) : "f"(sc));
      mbar_wait(&s.a8_empty[s8], ((t / S8) & 1) ^ 1);
      if (threadIdx.x == 0) QTRACE(3, t);
      const uint32_t dst = smem_u32(s.a8[s8]);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint32_t lo = qnt::quant_pair(x[8 * u + 2 * h], sc2);
          const uint32_t hi = qnt::quant_pair(x[8 * u + 2 * h + 1], sc2);
          w[h] = (lo & 0xffffu) | (hi << 16);
        }
        sts128(dst + sw128(r, u), make_uint4(w[0], w[1], w[2], w[3]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (threadIdx.x == 0) QTRACE(4, t);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.a8_full[s8]);
    }
    const float fin = p.partial ? ref : ref / amax;
    if (p.partial) {
      if (nt == 0) p.ws_d1[blockIdx.y * p.ws_rows + m0 + r] = amax;
    } else {
      if (!(amax > 0.f)) atomicExch(p.domain_flag, 1);
      if (nt == 0) p.d1[m0 + r] = amax;
    }
    const int crow = p.partial ? static_cast<int>(blockIdx.y * p.ws_rows) + m0 : m0;
    named_bar_sync(1, 128);
    mbar_wait(&s.acc_full, 0);
    if (threadIdx.x == 0) QTRACE(7, 0);
    tc_fence_after();
    // C tile (128 rows x 512 fp32 columns = 16 chunks of 32 columns) through
    // two 64 KB staging areas of the drained rings: round r (4 chunks) fills
    // area r & 1 while the TMA store of round r - 1 drains the other, and the
    // next chunk's TMEM load is in flight while the current one is staged.
    uint8_t* const base = reinterpret_cast<uint8_t*>(&s);  // abf ring then w ring: 192 KB drained
    uint8_t* const area[2] = {base, base + 4 * (BM * 128)};
    uint32_t v[2][32];
    tmem_ld32(tmem + lane_off, v[0]);
#pragma unroll 1
    for (int rnd = 0; rnd < 4; ++rnd) {
      if (rnd >= 2) {  // round rnd - 2's store has finished reading this area
        if (threadIdx.x == 0) bulk_wait_read1();
        named_bar_sync(1, 128);
      }
      const uint32_t stage = smem_u32(area[rnd & 1]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = 4 * rnd + c;
        tmem_ld_wait();
        if (cc + 1 < 16) tmem_ld32(tmem + lane_off + (cc + 1) * 32, v[(c + 1) & 1]);
        const uint32_t chunk = stage + c * (BM * 128);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          sts128(chunk + sw128(r, u),
                 make_uint4(__float_as_uint(__uint_as_float(v[c & 1][4 * u]) * fin),
                            __float_as_uint(__uint_as_float(v[c & 1][4 * u + 1]) * fin),
                            __float_as_uint(__uint_as_float(v[c & 1][4 * u + 2]) * fin),
                            __float_as_uint(__uint_as_float(v[c & 1][4 * u + 3]) * fin)));
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          tma_store_2d_hint(&tc, area[rnd & 1] + c * (BM * 128), n0 + 128 * rnd + 32 * c, crow, kEvictFirst);
        bulk_commit();
      }
    }
    if (threadIdx.x == 0) bulk_wait0();
    if (threadIdx.x == 0) QTRACE(7, 1);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 5) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace qnt2


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
  if (pattern == RF_PATTERN_LAYERNORM_GEMM) return k % rms::BK == 0 && m % (2 * BM) == 0;
  if (pattern == RF_PATTERN_QUANT_GEMM_E4M3) return n % qnt::BNQ == 0 && k % qnt::BK == 0;
  return false;
}

// Rasterisation group (tile_of): default per kernel, RF_GEMM_GROUP overrides
// (tuning experiments only).
static int group_param(int dflt) {
  static const char* env = std::getenv("RF_GEMM_GROUP");
  return env ? std::atoi(env) : dflt;
}

static cudaError_t launch_rms_like(const GemmArgs& g, cudaStream_t st, bool ln) {
  if (!gemm_sm100_supports(ln ? RF_PATTERN_LAYERNORM_GEMM : RF_PATTERN_RMSNORM_GEMM, g.m, g.n, g.k))
    return cudaErrorNotSupported;
  const bool pair = g.m % (2 * BM) == 0;
  CUtensorMap ta, tb, ty, ty4;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k) * 2};
    const uint32_t box[2] = {rms::BK, BM};
    if (!make_tmap(&ta, g.a, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.n)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k) * 2};
    const uint32_t box[2] = {rms::BK, pair ? 128u : static_cast<uint32_t>(BN)};
    if (!make_tmap(&tb, g.b, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  const int64_t S = g.segments > 1 ? g.segments : 1;
  const int64_t k_slice = g.k / S;
  if (g.k % S || k_slice % rms::BK) return cudaErrorNotSupported;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.n), static_cast<uint64_t>(g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.n) * 2};
    const uint32_t box[2] = {64, BM};
    if (!make_tmap(&ty, g.c, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
    if (!make_tmap(&ty4, ln && g.c4 ? g.c4 : g.c, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  if (S > 1) {  // slice partials: the raw fp32 accumulators into the workspace
    const uint64_t dims[2] = {static_cast<uint64_t>(g.n), static_cast<uint64_t>((S - 1) * g.ws_rows + g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.n) * 4};
    const uint32_t box[2] = {32, BM};
    if (!make_tmap(&ty, g.ws, 2, dims, str, box, 4)) return cudaErrorInvalidValue;
  }
  cudaError_t e;
  if (pair) {  // 2-SM path
    rms::Params p{g.d1, g.k, 1.f / static_cast<float>(g.stat_len > 0 ? g.stat_len : g.k), g.eps, static_cast<int>(g.m / (2 * BM)),
                  static_cast<int>(g.n / BN), group_param(16), g.d2, g.colsum, g.c4 != nullptr,
                  k_slice, g.ws_d1, g.ws_d2, g.ws_rows, S > 1};
    const size_t smem = sizeof(rms2::Smem) + 1024;
    auto kern = ln ? rms2::rms_gemm_2sm_kernel<true> : rms2::rms_gemm_2sm_kernel<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>(2 * (g.n / BN) * (g.m / (2 * BM))), static_cast<unsigned>(S));
    kern<<<grid, rms2::NT, smem, st>>>(ta, tb, ty, ty4, p);
  } else {
    if (ln) return cudaErrorNotSupported;  // layernorm: 2-SM tiles only (M % 256)
    rms::Params p{g.d1, g.k, 1.f / static_cast<float>(g.stat_len > 0 ? g.stat_len : g.k), g.eps, static_cast<int>(g.m / BM),
                  static_cast<int>(g.n / BN), group_param(8), nullptr, nullptr, 0,
                  k_slice, g.ws_d1, nullptr, g.ws_rows, S > 1};
    const size_t smem = sizeof(rms::Smem) + 1024;
    e = cudaFuncSetAttribute(rms::rms_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>((g.n / BN) * (g.m / BM)), static_cast<unsigned>(S));
    rms::rms_gemm_kernel<<<grid, rms::NT, smem, st>>>(ta, tb, ty, p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  return launch_gemm_fold(ln ? RF_PATTERN_LAYERNORM_GEMM : RF_PATTERN_RMSNORM_GEMM, g, st);
}

cudaError_t launch_rms_gemm_sm100(const GemmArgs& g, cudaStream_t st) {
  return launch_rms_like(g, st, false);
}

cudaError_t launch_layernorm_gemm_sm100(const GemmArgs& g, cudaStream_t st) {
  return launch_rms_like(g, st, true);
}

cudaError_t launch_quant_gemm_sm100(const GemmArgs& g, cudaStream_t st) {
  if (!gemm_sm100_supports(RF_PATTERN_QUANT_GEMM_E4M3, g.m, g.n, g.k)) return cudaErrorNotSupported;
  CUtensorMap ta, tw, tc;
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.m)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k) * 2};
    const uint32_t box[2] = {64, BM};
    if (!make_tmap(&ta, g.a, 2, dims, str, box, 2)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {static_cast<uint64_t>(g.k), static_cast<uint64_t>(g.n)};
    const uint64_t str[1] = {static_cast<uint64_t>(g.k)};
    const uint32_t box[2] = {qnt::BK, g.m % (2 * BM) == 0 ? 128u : 256u};
    if (!make_tmap(&tw, g.b, 2, dims, str, box, 1)) return cudaErrorInvalidValue;
  }
  const int64_t S = g.segments > 1 ? g.segments : 1;
  const int64_t k_slice = g.k / S;
  if (g.k % S || k_slice % qnt::BK) return cudaErrorNotSupported;
  {
    const uint64_t rows = S > 1 ? static_cast<uint64_t>((S - 1) * g.ws_rows + g.m) : static_cast<uint64_t>(g.m);
    const uint64_t dims[2] = {static_cast<uint64_t>(g.n), rows};
    const uint64_t str[1] = {static_cast<uint64_t>(g.n) * 4};
    const uint32_t box[2] = {32, BM};
    if (!make_tmap(&tc, S > 1 ? static_cast<void*>(g.ws) : g.c, 2, dims, str, box, 4))
      return cudaErrorInvalidValue;
  }
  cudaError_t e;
  if (g.m % (2 * BM) == 0) {  // 2-SM path
    qnt::Params p{g.d1, g.domain_flag, g.k, g.fmax, static_cast<int>(g.m / (2 * BM)),
                  static_cast<int>(g.n / qnt::BNQ), group_param(8), k_slice, g.ws_d1, g.ws_rows, S > 1};
    const size_t smem = sizeof(qnt2::Smem) + 1024;
    e = cudaFuncSetAttribute(qnt2::quant_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>(2 * (g.n / qnt::BNQ) * (g.m / (2 * BM))), static_cast<unsigned>(S));
    qnt2::quant_gemm_2sm_kernel<<<grid, qnt2::NT, smem, st>>>(ta, tw, tc, p);
  } else {
    qnt::Params p{g.d1, g.domain_flag, g.k, g.fmax, static_cast<int>(g.m / BM),
                  static_cast<int>(g.n / qnt::BNQ), 4, k_slice, g.ws_d1, g.ws_rows, S > 1};
    const size_t smem = sizeof(qnt::Smem) + 1024;
    e = cudaFuncSetAttribute(qnt::quant_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>((g.n / qnt::BNQ) * (g.m / BM)), static_cast<unsigned>(S));
    qnt::quant_gemm_kernel<<<grid, qnt::NT, smem, st>>>(ta, tw, tc, p);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess || S == 1) return e;
  return launch_gemm_fold(RF_PATTERN_QUANT_GEMM_E4M3, g, st);
}

cudaError_t launch_pack_e4m3(const float* w, int64_t k, int64_t n, uint8_t* packed, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32));
  pack_kernel<true><<<grid, dim3(32, 8), 0, st>>>(w, nullptr, k, n, packed);
  return cudaGetLastError();
}

namespace {
// one warp per column n of the packed [N,K] bf16 weight: colsum[n] = sum_k W'[n,k]
__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ w, int64_t k, int64_t n,
                              float* __restrict__ out) {
  const int64_t col = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (col >= n) return;
  float acc = 0.f;
  for (int64_t i = threadIdx.x & 31; i < k; i += 32) acc += __bfloat162float(w[col * k + i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) out[col] = acc;
}
}  // namespace

cudaError_t launch_colsum(const void* packed, int64_t k, int64_t n, float* colsum, cudaStream_t st) {
  colsum_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(packed), k, n, colsum);
  return cudaGetLastError();
}

cudaError_t launch_pack_rms(const float* w, const float* g, int64_t k, int64_t n, void* packed,
                            cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((k + 31) / 32));
  pack_kernel<false><<<grid, dim3(32, 8), 0, st>>>(w, g, k, n, packed);
  return cudaGetLastError();
}

}  // namespace rf
