// EXPERIMENTAL, not part of librf_cuda: measured slower than attn_sm100.cu on
// cfg2; kept for the record and the probe library's traces.
// bf16 safe-softmax -> GEMM attention on a CTA PAIR (2-SM UMMA, sm_100a).
//
// Same cascade and incremental form as attn_sm100.cu (the reference's
// incr_ingest_element, proj/src/simulator.cpp:566-589, over make_attention,
// proj/src/workloads.cpp:66-120), restructured so the tensor core never waits
// for the softmax of the tile it just produced:
//
//   * a cluster of 2 CTAs owns 256 query rows; each CTA keeps its 128-row Q
//     tile, and stages only HALF of every K tile (64 keys) and of every V tile
//     (64 head-dim columns): tcgen05.mma.cta_group::2 (M = 256) reads the
//     pair's halves, so per-SM shared-memory and L2 traffic for K/V halves;
//   * TMEM per CTA holds two S buffers + O (384 of 512 columns), so S_{i+1}
//     is computed while the softmax works on S_i; P_i (bf16) overwrites S
//     buffer i%2 and is consumed from TMEM by PV_i;
//   * leader MMA issue order: S_0, S_1, PV_0, S_2, PV_1, S_3, ...;
//   * softmax: 16 warps per CTA, four threads per row (32 key columns each,
//     4-deep latency hiding per sub-partition), partial max / sum exchanged
//     through shared memory; 3 in 8 exponentials on the FMA pipe; the lazy
//     exp(d1'-d1) correction of O (threshold 2^8) waits for PV_{i-1} only when
//     it actually rescales; d2'/d2 telescopes to 1/d2 at finalize.
//
// The peer's completions (its K/V halves landed, its P ready) are relayed to
// the leader's barriers by two relay warps (independent streams, so neither
// can serialise the other).
//
// Warps: 0-15 softmax (four threads per row: key columns 32 g .. 32 g + 31),
//        16 TMA, 17 MMA issuer (leader) / K-V + Q relay (peer), 18 P relay (peer).
#include <cuda_bf16.h>

#include "../rf_internal.h"
#include "../sm100.cuh"

#ifdef RF_ATTN_TRACE
// Test-only timeline of the first cluster: [rank*1024 + ...] (tools/trace_attention.py)
__device__ long long g_attn2_trace[4096];
#define RF_TRACE2(idx) \
  do { if ((blockIdx.x >> 1) == 0 && (blockIdx.y | blockIdx.z) == 0) g_attn2_trace[(idx)] = clock64(); } while (0)
#else
#define RF_TRACE2(idx) do {} while (0)
#endif

namespace rf {
namespace {

using namespace sm100;

constexpr int D = 128;
constexpr int BM = 128;     // query rows per CTA
constexpr int BN = 128;     // keys per KV tile
constexpr int NSLOT = 8;    // ring of 16 KB half-tiles (K half or V half)
constexpr int NG = 4;       // threads (column groups) per row in the softmax
constexpr int NSW = 4 * NG; // softmax warps
constexpr int kTmaWarp = NSW, kMmaWarp = NSW + 1, kRelayWarp = NSW + 2;
constexpr int NT = 32 * (NSW + 3);
constexpr int CW = BN / NG;  // key columns per softmax thread
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;
constexpr int HALF_BYTES = 16384;  // K half: 64 keys x 128 dims; V half: 128 keys x 64 dims
constexpr int Q_BYTES = BM * D * 2;

struct Smem {
  uint8_t q[Q_BYTES];
  uint8_t kv[NSLOT][HALF_BYTES];
  uint64_t bar_q;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2], pv_done, o_final;
  float xmax[2][NG][BM];  // [tile parity][column group][row]
  float xsum[NG][BM];
  uint32_t tmem_base;
};

struct Params {
  int64_t sq, skv, slice_len, slice_begin, part_base, rows_total;
  float scale_log2, scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
};

__device__ __forceinline__ constexpr bool poly_pair(int jj) { return (jj & 3) == 3; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    attn_2sm_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int bh = blockIdx.y;
  const int64_t q_row0 = static_cast<int64_t>(blockIdx.x >> 1) * 2 * BM + rank * BM;
  const int64_t slice = p.slice_begin + blockIdx.z;
  const int64_t kv0 = slice * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / BN);

  if (threadIdx.x == 0) {
    mbar_init(&s.bar_q, leader ? 2 : 1);
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], leader ? 2 : 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s.s_full[b], 1);
      mbar_init(&s.p_full[b], leader ? NSW + 1 : NSW);
    }
    mbar_init(&s.pv_done, 1);
    mbar_init(&s.o_final, 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;  // S buffers at cols 0 / 128, O at 256

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      const int32_t qy = static_cast<int32_t>(bh * p.sq + q_row0);
      mbar_arrive_expect_tx(&s.bar_q, Q_BYTES);
      for (int c = 0; c < D / 64; ++c)
        tma_load_2d(s.q + c * BM * 128, &tq, &s.bar_q, c * 64, qy, kEvictFirst);
      const int32_t ky = static_cast<int32_t>(bh * p.skv + kv0);
      for (int j = 0; j < 2 * n_tiles; ++j) {  // item j: K_{j/2} (even) or V_{j/2} (odd)
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
    const bool el = elect_one();
    auto wait_item = [&](int j) {
      mbar_wait(&s.kv_full[j % NSLOT], (j / NSLOT) & 1);
      tc_fence_after();
    };
    auto issue_s = [&](int i) {  // S_i = Q K_i^T into buffer i % 2
      const int j = 2 * i, slot = j % NSLOT;
      wait_item(j);
      if (el) {
        RF_TRACE2(2048 + 4 * i + 0);
        const uint32_t qa = smem_u32(s.q), kb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          mma_f16_ss_2sm(tmem + (i & 1) * 128,
                         sdesc_kmajor_sw128(qa + (ks >> 2) * (BM * 128) + (ks & 3) * 32),
                         sdesc_kmajor_sw128(kb + (ks >> 2) * (64 * 128) + (ks & 3) * 32), id_s, ks > 0);
        mma_commit_2sm(&s.s_full[i & 1]);
        mma_commit_2sm(&s.kv_empty[slot]);
      }
      __syncwarp();
    };
    mbar_wait(&s.bar_q, 0);
    issue_s(0);
    if (n_tiles > 1) issue_s(1);
    for (int i = 0; i < n_tiles; ++i) {
      mbar_wait(&s.p_full[i & 1], (i >> 1) & 1);  // both CTAs' P_i in TMEM
      const int j = 2 * i + 1, slot = j % NSLOT;
      wait_item(j);
      if (el) {
        RF_TRACE2(2048 + 4 * i + 1);
        const uint32_t vb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          mma_f16_ts_2sm(tmem + 256, tmem + (i & 1) * 128 + ks * 8,
                         sdesc_mnmajor_sw128(vb + ks * 2048, 128 * 128), id_o, i > 0 || ks > 0);
        mma_commit_2sm(&s.pv_done);
        mma_commit_2sm(&s.kv_empty[slot]);
        if (i + 1 == n_tiles) mma_commit_2sm(&s.o_final);
      }
      __syncwarp();
      if (i + 2 < n_tiles) issue_s(i + 2);  // buffer i % 2 is free once PV_i is issued
    }
  } else if (warp == kMmaWarp) {
    // ---- peer: relay Q and every K/V half-tile to the leader's barriers ----
    if (elect_one()) {
      mbar_wait(&s.bar_q, 0);
      mbar_arrive_cluster(mapa_shared(smem_u32(&s.bar_q), 0));
      for (int j = 0; j < 2 * n_tiles; ++j) {
        const int slot = j % NSLOT;
        mbar_wait(&s.kv_full[slot], (j / NSLOT) & 1);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.kv_full[slot]), 0));
      }
    }
  } else if (warp == kRelayWarp) {
    // ---- peer: relay P_i ready to the leader ----
    if (!leader && elect_one()) {
      for (int i = 0; i < n_tiles; ++i) {
        mbar_wait(&s.p_full[i & 1], (i >> 1) & 1);
        RF_TRACE2(3072 + i);
        mbar_arrive_cluster(mapa_shared(smem_u32(&s.p_full[i & 1]), 0));
      }
    }
  } else {
    // ----------------------------------- softmax / correction / epilogue --
    const int grp = warp >> 2;  // key columns [CW grp, CW grp + CW) of the row
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tO = tmem + 256 + lane_off;
    const float c1 = p.scale_log2;
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      const uint32_t tS = tmem + (i & 1) * 128 + lane_off;
      mbar_wait(&s.s_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 0) RF_TRACE2(rank * 1024 + 4 * i + 0);
      uint32_t sr[CW];
      tmem_ld32(tS + CW * grp, *reinterpret_cast<uint32_t(*)[32]>(sr));
      tmem_ld_wait();
#define SV(j) __uint_as_float(sr[(j)])
      float mx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) mx[j] = SV(j);
#pragma unroll
      for (int j = 4; j < CW; ++j) mx[j & 3] = fmaxf(mx[j & 3], SV(j));
      s.xmax[i & 1][grp][row] = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      tc_fence_before();  // our S loads complete before other groups overwrite with P
      named_bar_sync(1, 32 * NSW);
      tc_fence_after();
      float tmax = s.xmax[i & 1][0][row];
#pragma unroll
      for (int g = 1; g < NG; ++g) tmax = fmaxf(tmax, s.xmax[i & 1][g][row]);
      if (threadIdx.x == 0) RF_TRACE2(rank * 1024 + 4 * i + 1);
      m_true = fmaxf(m_true, tmax * p.scale);
      const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
      float alpha = 1.f;
      if (need) {
        alpha = ex2_mufu((m_ref - m_true) * kLog2e);
        l *= alpha;
        m_ref = m_true;
      }
      const uint64_t c12 = f2(c1, c1), nmb2 = f2(-m_ref * kLog2e, -m_ref * kLog2e);
      uint64_t acc2[4] = {0, 0, 0, 0};
      uint32_t pk[CW / 2];
#pragma unroll
      for (int jj = 0; jj < CW / 2; ++jj) {
        const uint64_t x2 = ffma2(f2(SV(2 * jj), SV(2 * jj + 1)), c12, nmb2);
        uint64_t p2;
        if (poly_pair(jj)) {
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
      tmem_st16(tS + (CW / 2) * grp, pk);
#undef SV
      const uint64_t s01 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
      float rs0, rs1;
      f2split(s01, rs0, rs1);
      l += rs0 + rs1;
      if (i > 0 && __any_sync(0xffffffffu, need)) {
        // PV_{i-1} must be complete before O is rescaled (it may still run:
        // S_i was issued before PV_{i-1}); in-order MMA bounds the phase.
        mbar_wait(&s.pv_done, (i - 1) & 1);
        tc_fence_after();
        uint32_t r[D / NG];
        const uint32_t addr = tO + (D / NG) * grp;
        tmem_ld32(addr, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < D / NG; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
        tmem_st32(addr, *reinterpret_cast<uint32_t(*)[32]>(r));
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (threadIdx.x == 0) RF_TRACE2(rank * 1024 + 4 * i + 2);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.p_full[i & 1]);
    }
    // ---- finalize (finalize_root) ----
    s.xsum[grp][row] = l;
    named_bar_sync(1, 32 * NSW);
    l = s.xsum[0][row];
#pragma unroll
    for (int g = 1; g < NG; ++g) l += s.xsum[g][row];
    const float l_true = l * ex2_mufu((m_ref - m_true) * kLog2e);
    const int64_t grow = static_cast<int64_t>(bh) * p.sq + q_row0 + row;
    const int64_t ps = slice - p.part_base;
    if (grp == 0) {
      if (p.part_m == nullptr) {
        p.m[grow] = m_true;
        p.l[grow] = l_true;
      } else {
        p.part_m[ps * p.rows_total + grow] = m_true;
        p.part_l[ps * p.rows_total + grow] = l_true;
      }
    }
    mbar_wait(&s.o_final, 0);
    tc_fence_after();
    const float inv_l = 1.f / l;
    {
      uint32_t r[32];
      const int col = (D / NG) * grp;
      tmem_ld32(tO + col, r);
      tmem_ld_wait();
      if (p.part_o == nullptr) {
        uint4* dst = reinterpret_cast<uint4*>(p.o + grow * D + col);
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
        float4* dst = reinterpret_cast<float4*>(p.part_o + (ps * p.rows_total + grow) * D + col);
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

bool attention_sm100_2sm_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments) {
  if (d != D || sq % (2 * BM) != 0 || segments < 1 || skv % segments != 0) return false;
  return (skv / segments) % BN == 0;
}

cudaError_t launch_attention_sm100_2sm(const AttnArgs& a, cudaStream_t st) {
  if (a.dtype != RF_BF16 || !attention_sm100_2sm_supports(a.sq, a.skv, a.d, a.segments))
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
  cudaError_t e = cudaFuncSetAttribute(attn_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(a.sq / BM), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
  attn_2sm_kernel<<<grid, NT, smem, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace rf
