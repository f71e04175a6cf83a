// EXPERIMENTAL, not part of librf_cuda: measured slower than attn_sm100.cu on
// cfg2; kept for the record and the probe library's traces.
// bf16 safe-softmax -> GEMM attention: the 1-SM ping-pong kernel
// (attn_sm100.cu) on a CTA PAIR with 2-SM UMMA (cta_group::2), sm_100a.
//
// Same cascade and incremental form (the reference's incr_ingest_element,
// proj/src/simulator.cpp:566-589, over make_attention,
// proj/src/workloads.cpp:66-120; the reference tile plan of
// tests/golden/flash_attention_tile.txt). What changes is where the MMA
// operands come from:
//   * each CTA keeps TWO 128-row Q tiles (as in the 1-SM kernel, ping-pong);
//     the pair's S_k MMA is M = 256 (CTA 0's tile k + CTA 1's tile k);
//   * each CTA stages only HALF of every K tile (64 keys) and of every V tile
//     (64 head-dim columns): the M = 256 MMA reads the pair's halves, so per
//     SM the S MMA reads 4 KB (Q) + 2 KB (K) of shared memory per K-step
//     instead of 4 + 4, and the K/V TMA traffic into each SM halves. With
//     N = 128 SS MMAs the 1-SM kernel sits at the 128 B/clk shared-memory
//     port (Q + K per 64-cycle K-step, plus V and the TMA writes);
//   * the leader's elected thread issues every MMA; commits multicast to both
//     CTAs' barriers; the peer relays "my K/V half landed" and "my P_k is in
//     TMEM" to the leader's barriers (relaxed remote arrives).
// The softmax, the lazy exp(d1' - d1) correction (threshold 2^8) and the
// finalize retarget are the 1-SM kernel's (two-pass softmax, thread = row).
//
// Warps (384 threads): 0-3 / 4-7 softmax + epilogue for Q tile 0 / 1,
// 8 TMA, 9 MMA issuer (leader) / K-V + Q relay (peer), 10-11 P relays (peer).
#include <cuda_bf16.h>

#include "../rf_internal.h"
#include "../sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int D = 128;
constexpr int BM = 128;        // rows per Q tile
constexpr int BN = 128;        // keys per KV tile
constexpr int NSLOT = 8;       // ring of 16 KB half-tiles (K half or V half)
constexpr int NT = 384;
constexpr int kTmaWarp = 8, kMmaWarp = 9, kRelayWarp0 = 10;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr int Q_BYTES = BM * D * 2;        // 32 KB per Q tile
constexpr int HALF_BYTES = 16384;          // K half: 64 keys x 128 dims; V half: 128 keys x 64 dims
__device__ __forceinline__ constexpr bool kPolyPairs(int jj) { return (jj & 3) == 3; }

struct Smem {
  uint8_t q[2][Q_BYTES];
  uint8_t kv[NSLOT][HALF_BYTES];
  uint64_t bar_q;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2], pv_done[2];
  uint32_t tmem_base;
};

struct Params {
  int64_t sq, skv, slice_len, slice_begin, part_base, rows_total;
  float scale_log2;
  float scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int bh = blockIdx.y;
  // CTA r's tile k covers query rows unit*512 + (2k + r)*128 .. +127
  const int64_t unit_row0 = static_cast<int64_t>(blockIdx.x >> 1) * 4 * BM;
  const int64_t slice = p.slice_begin + blockIdx.z;
  const int64_t kv0 = slice * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / BN);

  if (threadIdx.x == 0) {
    mbar_init(&s.bar_q, leader ? 2 : 1);
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], leader ? 2 : 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s.s_full[k], 1);
      mbar_init(&s.p_full[k], leader ? 4 + 1 : 4);  // own softmax warps (+ the peer's relay)
      mbar_init(&s.pv_done[k], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;  // S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512)

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      mbar_arrive_expect_tx(&s.bar_q, 2 * Q_BYTES);
      for (int k = 0; k < 2; ++k) {
        const int32_t qy = static_cast<int32_t>(bh * p.sq + unit_row0 + (2 * k + rank) * BM);
        for (int c = 0; c < D / 64; ++c) tma_load_2d(s.q[k] + c * BM * 128, &tq, &s.bar_q, c * 64, qy, kEvictFirst);
      }
      const int32_t ky = static_cast<int32_t>(bh * p.skv + kv0);
      for (int j = 0; j < 2 * n_tiles; ++j) {  // item j: K_{j/2} half (even) or V_{j/2} half (odd)
        const int slot = j % NSLOT;
        mbar_wait(&s.kv_empty[slot], ((j / NSLOT) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.kv_full[slot], HALF_BYTES);
        const int32_t key0 = ky + (j >> 1) * BN;
        if ((j & 1) == 0) {  // K half: keys [64 r, 64 r + 64), all dims (2 swizzle chunks)
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(s.kv[slot] + c * 64 * 128, &tk, &s.kv_full[slot], c * 64,
                        key0 + 64 * static_cast<int>(rank), kEvictLast);
        } else {  // V half: all 128 keys, dims [64 r, 64 r + 64)
          tma_load_2d(s.kv[slot], &tv, &s.kv_full[slot], 64 * static_cast<int>(rank), key0, kEvictLast);
        }
      }
    }
  } else if (warp == kMmaWarp && leader) {
    // ------------------------------------------------------------ MMA ----
    const uint32_t id_s = idesc_f16(2 * BM, BN, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(2 * BM, D, kFmtBF16, false, true);
    const uint32_t tS[2] = {tmem + 0, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 384};
    const bool el = elect_one();
    auto wait_item = [&](int j) {
      mbar_wait(&s.kv_full[j % NSLOT], (j / NSLOT) & 1);  // both CTAs' halves landed
      tc_fence_after();
    };
    auto issue_s = [&](int k, int slot) {  // S_k = Q_k K^T (M = 256 over the pair)
      if (el) {
        const uint32_t qa = smem_u32(s.q[k]), kb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          mma_f16_ss_2sm(tS[k], sdesc_kmajor_sw128(qa + (ks >> 2) * (BM * 128) + (ks & 3) * 32),
                         sdesc_kmajor_sw128(kb + (ks >> 2) * (64 * 128) + (ks & 3) * 32), id_s, ks > 0);
        mma_commit_2sm(&s.s_full[k]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int k, int slot, bool acc, bool last) {  // O_k += P_k V (P from TMEM)
      if (el) {
        const uint32_t vb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          mma_f16_ts_2sm(tO[k], tS[k] + ks * 8, sdesc_mnmajor_sw128(vb + ks * 2048, 128 * 128), id_o,
                         acc || ks > 0);
        if (last) mma_commit_2sm(&s.pv_done[k]);
      }
      __syncwarp();
    };
    auto release = [&](int slot) {
      if (el) mma_commit_2sm(&s.kv_empty[slot]);
      __syncwarp();
    };
    mbar_wait(&s.bar_q, 0);
    wait_item(0);
    issue_s(0, 0);
    issue_s(1, 0);
    release(0);
    for (int i = 0; i < n_tiles; ++i) {
      const int jV = 2 * i + 1, jK = 2 * i + 2;
      const int sV = jV % NSLOT, sK = jK % NSLOT;
      const uint32_t ph = i & 1;
      const bool last = i + 1 == n_tiles;
      wait_item(jV);
      // tile 0: PV0_i then S0_{i+1}
      mbar_wait(&s.p_full[0], ph);  // both CTAs' P_0,i in TMEM
      tc_fence_after();
      issue_pv(0, sV, i > 0, last);
      if (!last) {
        wait_item(jK);
        issue_s(0, sK);
      }
      // tile 1: PV1_i then S1_{i+1}
      mbar_wait(&s.p_full[1], ph);
      tc_fence_after();
      issue_pv(1, sV, i > 0, last);
      release(sV);
      if (!last) {
        issue_s(1, sK);
        release(sK);
      }
    }
  } else if (warp == kMmaWarp) {
    // ---- peer: relay Q and every K/V half to the leader's barriers ----
    if (elect_one()) {
      mbar_wait(&s.bar_q, 0);
      mbar_arrive_cluster(mapa_shared(smem_u32(&s.bar_q), 0));
      for (int j = 0; j < 2 * n_tiles; ++j) {
        const int slot = j % NSLOT;
        mbar_wait(&s.kv_full[slot], (j / NSLOT) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.kv_full[slot]), 0));
      }
    }
  } else if (warp >= kRelayWarp0) {
    // ---- peer: relay "P_k,i is in TMEM" to the leader (one warp per Q tile) ----
    const int k = warp - kRelayWarp0;
    if (!leader && elect_one()) {
      for (int i = 0; i < n_tiles; ++i) {
        mbar_wait(&s.p_full[k], i & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.p_full[k]), 0));
      }
    }
  } else {
    // ----------------------------------- softmax / correction / epilogue --
    const int k = warp >> 2;  // Q tile
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tSk = tmem + k * 128 + lane_off;
    const uint32_t tOk = tmem + 256 + k * 128 + lane_off;
    const float c1 = p.scale_log2;
    float m_true = -INFINITY;  // d1: exact running max
    float m_ref = -INFINITY;   // reference max of the accumulators
    float l = 0.f;             // d2 relative to m_ref
    for (int i = 0; i < n_tiles; ++i) {
      mbar_wait(&s.s_full[k], i & 1);
      tc_fence_after();
      float tmax;
      {
        // pass 1 (reduction 1): d1 = max(d1, max_tile) over the 4 chunks in flight
        uint32_t sr[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tSk + c * 32, sr[c]);
        tmem_ld_wait();
        float mx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) mx[j] = __uint_as_float(sr[0][j]);
#pragma unroll
        for (int j = 8; j < BN; ++j) mx[j & 7] = fmaxf(mx[j & 7], __uint_as_float(sr[j >> 5][j & 31]));
        tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      }
      m_true = fmaxf(m_true, tmax * p.scale);
      // correction exp(d1' - d1): lazily re-base the accumulators
      const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
      float alpha = 1.f;
      if (need) {
        alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
        l *= alpha;
        m_ref = m_true;
      }
      // pass 2 (reductions 2 and 3): S re-read one 32-column chunk at a time
      // (the next in flight); P chunk c lands in columns [16c, 16c + 16)
      const uint64_t c12 = f2(c1, c1), nmb2 = f2(-m_ref * kLog2e, -m_ref * kLog2e);
      uint64_t acc2[4] = {0, 0, 0, 0};
      uint32_t sr[2][32];
      tmem_ld32(tSk, sr[0]);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld_wait();
        if (c + 1 < 4) tmem_ld32(tSk + (c + 1) * 32, sr[(c + 1) & 1]);
        uint32_t pk[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const uint64_t x2 = ffma2(f2(__uint_as_float(sr[c & 1][2 * jj]), __uint_as_float(sr[c & 1][2 * jj + 1])),
                                    c12, nmb2);
          uint64_t p2;
          if (kPolyPairs(jj)) {
            p2 = ex2_poly2(x2);
          } else {
            float x0, x1;
            f2split(x2, x0, x1);
            p2 = f2(ex2_mufu(x0), ex2_mufu(x1));
          }
          acc2[jj & 3] = fadd2(acc2[jj & 3], p2);
          float p0, p1;
          f2split(p2, p0, p1);
          pk[jj] = pack_bf16x2(p0, p1);
        }
        tmem_st16(tSk + 16 * c, pk);
      }
      const uint64_t s01 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
      float rs0, rs1;
      f2split(s01, rs0, rs1);
      l += rs0 + rs1;
      // O *= exp(d1' - d1): P V_k,i-1 has retired (S_k,i, issued after it, is complete)
      if (i > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tOk + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
          tmem_st32(tOk + c * 32, r);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.p_full[k]);
    }
    // ---- finalize (finalize_root): d2 re-based to the true d1, d3 = O / d2 ----
    const float l_true = l * ex2_mufu((m_ref - m_true) * kLog2e);
    const int64_t grow = static_cast<int64_t>(bh) * p.sq + unit_row0 + (2 * k + rank) * BM + row;
    const int64_t ps = slice - p.part_base;
    if (p.part_m == nullptr) {
      p.m[grow] = m_true;
      p.l[grow] = l_true;
    } else {
      p.part_m[ps * p.rows_total + grow] = m_true;
      p.part_l[ps * p.rows_total + grow] = l_true;
    }
    mbar_wait(&s.pv_done[k], 0);
    tc_fence_after();
    const float inv_l = 1.f / l;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tOk + c * 32, r);
      tmem_ld_wait();
      if (p.part_o == nullptr) {
        uint4* dst = reinterpret_cast<uint4*>(p.o + grow * D + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(r[8 * v + 0]) * inv_l, __uint_as_float(r[8 * v + 1]) * inv_l);
          w.y = pack_bf16x2(__uint_as_float(r[8 * v + 2]) * inv_l, __uint_as_float(r[8 * v + 3]) * inv_l);
          w.z = pack_bf16x2(__uint_as_float(r[8 * v + 4]) * inv_l, __uint_as_float(r[8 * v + 5]) * inv_l);
          w.w = pack_bf16x2(__uint_as_float(r[8 * v + 6]) * inv_l, __uint_as_float(r[8 * v + 7]) * inv_l);
          dst[v] = w;
        }
      } else {
        float4* dst = reinterpret_cast<float4*>(p.part_o + (ps * p.rows_total + grow) * D + c * 32);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          dst[v] = make_float4(__uint_as_float(r[4 * v]) * inv_l, __uint_as_float(r[4 * v + 1]) * inv_l,
                               __uint_as_float(r[4 * v + 2]) * inv_l, __uint_as_float(r[4 * v + 3]) * inv_l);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == kMmaWarp) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace

bool attention_sm100_pair_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments) {
  if (d != D || sq % (4 * BM) != 0 || segments < 1 || skv % segments != 0) return false;
  return (skv / segments) % BN == 0;
}

cudaError_t launch_attention_sm100_pair(const AttnArgs& a, cudaStream_t st) {
  if (a.dtype != RF_BF16 || !attention_sm100_pair_supports(a.sq, a.skv, a.d, a.segments))
    return cudaErrorNotSupported;
  CUtensorMap tq, tk, tv;
  const uint64_t qdims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(a.bh * a.sq)};
  const uint64_t kdims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(a.bh * a.skv)};
  const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
  const uint32_t qbox[2] = {64, 128}, kbox[2] = {64, 64}, vbox[2] = {64, 128};
  if (!make_tmap(&tq, a.q, 2, qdims, strides, qbox, 2) ||
      !make_tmap(&tk, a.k, 2, kdims, strides, kbox, 2) ||
      !make_tmap(&tv, a.v, 2, kdims, strides, vbox, 2))
    return cudaErrorInvalidValue;
  Params p{};
  p.sq = a.sq;
  p.skv = a.skv;
  p.slice_len = a.skv / a.segments;
  p.slice_begin = a.slice_begin;
  p.part_base = a.part_base;
  p.rows_total = a.rows_total;
  p.scale = a.scale;
  p.scale_log2 = a.scale * kLog2e;
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  const size_t smem = sizeof(Smem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(a.sq / (2 * BM)), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
  attn_pair_kernel<<<grid, NT, smem, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace rf
