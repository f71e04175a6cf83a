// MLA decode (multi-latent attention, absorbed form; the paper's MLA workload
// L1-L9: hn = 128 heads, latent hd = 512, rope ped = 64)
// as the attention cascade of make_attention (proj/src/workloads.cpp:66-120):
//   d1 = max P, d2 = sum e^(P - d1), d3 = sum e^(P - d1) / d2 V,
//   P = scale Q K^T with K = the 576-wide cache rows [c_kv | k_rope] and
//   V = their first 512 columns (c_kv) — one cache tensor serves both.
// All 128 heads of a batch share the cache, so a decode step is GEMM-shaped:
// S = Q (128 x 576) K^T, O += P V (N = 512).
//
// A (batch, KV slice) runs on a CTA PAIR issuing 2-SM MMAs
// (tcgen05.mma.cta_group::2, M = 128): CTA h owns heads [64h, 64h + 64) —
// its 64 Q rows stay in shared memory (9 x 8 KB, SWIZZLE_128B) — and, per
// 128-key cache tile,
//   * S = Q K^T (N = 128 keys, K = 576): CTA h stages keys [64h, 64h + 64)
//     of the tile (9 chunks of 64 columns), so the pair reads every cache
//     byte from HBM once;
//   * the 2-SM accumulator layout puts row r's keys [0, 64) in TMEM lane r
//     and keys [64, 128) in lane r + 64: the softmax thread of each lane owns
//     half a row; the two halves exchange their row max through shared
//     memory (no cross-CTA traffic in the loop);
//   * P (bf16) goes to shared memory (the MMA's A operand, 16 KB);
//   * O += P V as two N = 256 MMAs (V columns [0, 256) and [256, 512));
//     CTA h supplies V columns 256j + [128h, 128h + 128) of all 128 keys —
//     re-read from L2 (the pair's K stages just brought them in);
//     O is 64 rows x 512 per CTA = 256 TMEM columns (lane r: columns
//     256j + [0, 128), lane r + 64: 256j + [128, 256)).
// One 17-stage ring of 8 KB (9 K + 8 V stages = exactly one tile): tile
// i + 1's K stages load as soon as S_i has consumed tile i's, its V stages
// once P V_i has. The MMA warp issues S_{i+1} and P V_i as their inputs arrive
// (S_{i+1} runs under softmax i; S is double-buffered in TMEM).
// The d3 correction exp(d1' - d1) is lazy (only when the running max passes
// the reference by 2^8, after P V_{i-1} has retired); d2'/d2 telescopes to
// 1/d2 at finalize (finalize_root, proj/src/simulator.cpp:611-621), as in
// attn_sm100.cu. Multi-Segment: each KV slice writes its (m, l, O/l)
// partial state, merged in slice order by merge.cu (run_multisegment).
// Warps: 0-3 softmax + correction + epilogue, 4 TMA, 5 MMA (leader) / relay
// of the peer's TMA completions to the leader (192 threads).
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int HN = 128;        // heads per batch (2-SM UMMA M)
constexpr int HC = HN / 2;     // heads per CTA
constexpr int DQK = 576;       // cache row / query width
constexpr int DV = 512;        // value width (latent)
constexpr int NCH = DQK / 64;  // 64-column chunks per cache row
constexpr int TK = 128;        // keys per tile
constexpr int NKS = NCH;       // K stages per tile (this CTA's 64 keys x 64 columns)
constexpr int NVS = 8;         // V stages per tile (2 halves x 4 x 32 keys x 128 columns)
constexpr int NST = NKS + NVS; // ring stages = one tile
constexpr int STB = 8192;      // stage bytes
constexpr int NT = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Smem {
  uint8_t q[NCH][HC * 128];  // 9 x 8 KB
  uint8_t ring[NST][STB];    // 17 x 8 KB
  uint8_t p[2][HC * 128];    // P: keys [0, 64) and [64, 128), K-major SWIZZLE_128B
  float xm[2][HN];           // row-half exchange (max per tile, then l)
  uint64_t q_full, full[NST], empty[NST];
  uint64_t s_full[2], p_full, pv_done, o_full;
  uint32_t tmem_base;
};

struct Params {
  int64_t skv, slice_len, rows_total;
  float scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int h = static_cast<int>(cluster_ctarank());
  const bool leader = h == 0;
  const int b = blockIdx.y;      // batch
  const int slice = blockIdx.z;  // KV slice
  const int64_t kv0 = static_cast<int64_t>(slice) * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / TK);

  if (threadIdx.x == 0) {
    mbar_init(&s.q_full, leader ? 2 : 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&s.full[i], leader ? 2 : 1);  // leader: own TMA + the peer's relay
      mbar_init(&s.empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) mbar_init(&s.s_full[k], 1);
    mbar_init(&s.p_full, 8);  // 4 softmax warps of each CTA (leader's copy is the one used)
    mbar_init(&s.pv_done, 1);
    mbar_init(&s.o_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc_2sm<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + 64};
  const uint32_t tO = tmem + 256;  // + 128 j: V columns 256 j + ...

  if (warp == 4) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      mbar_arrive_expect_tx(&s.q_full, NCH * HC * 128);
      for (int c = 0; c < NCH; ++c) tma_load_2d(s.q[c], &tq, &s.q_full, c * 64, b * HN + h * HC, kEvictFirst);
      const int32_t y0 = static_cast<int32_t>(static_cast<int64_t>(b) * p.skv + kv0);
      for (int t = 0; t < n_tiles; ++t) {
        const uint32_t ph = (t & 1) ^ 1;
        const int32_t key0 = y0 + t * TK;
        for (int c = 0; c < NKS; ++c) {  // this CTA's 64 keys, all 576 columns (HBM)
          mbar_wait(&s.empty[c], ph);
          mbar_arrive_expect_tx(&s.full[c], STB);
          tma_load_2d(s.ring[c], &tk, &s.full[c], c * 64, key0 + h * 64, kEvictNormal);
        }
        for (int v = 0; v < NVS; ++v) {  // all 128 keys, V columns 256 j + [128 h, +128) (L2)
          const int st = NKS + v, j = v >> 2, kk = v & 3;
          mbar_wait(&s.empty[st], ph);
          mbar_arrive_expect_tx(&s.full[st], STB);
          const int c0 = 4 * j + 2 * h;
          tma_load_2d(s.ring[st], &tv, &s.full[st], c0 * 64, key0 + 32 * kk, kEvictFirst);
          tma_load_2d(s.ring[st] + STB / 2, &tv, &s.full[st], (c0 + 1) * 64, key0 + 32 * kk, kEvictFirst);
        }
      }
    }
  } else if (warp == 5) {
    if (leader) {
      // ---------------------------------------------------------- MMA ----
      const uint32_t id_s = idesc_f16(HN, TK, kFmtBF16, false, false);
      const uint32_t id_o = idesc_f16(HN, 256, kFmtBF16, false, true);
      const bool el = elect_one();
      auto issue_s = [&](int i) {  // S_i = Q K_i^T into S buffer i & 1
        for (int c = 0; c < NKS; ++c) {
          mbar_wait(&s.full[c], i & 1);
          tc_fence_after();
          if (el) {
            const uint32_t qa = smem_u32(s.q[c]), kb = smem_u32(s.ring[c]);
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              mma_f16_ss_2sm(tS[i & 1], sdesc_kmajor_sw128(qa + k4 * 32), sdesc_kmajor_sw128(kb + k4 * 32), id_s,
                             (c | k4) != 0);
            mma_commit_2sm(&s.empty[c]);
            if (c + 1 == NKS) mma_commit_2sm(&s.s_full[i & 1]);
          }
          __syncwarp();
        }
      };
      auto issue_pv = [&](int i) {  // O += P_i V_i
        mbar_wait(&s.p_full, i & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(s.p[0]);
        for (int v = 0; v < NVS; ++v) {
          const int st = NKS + v, j = v >> 2, kk = v & 3;
          mbar_wait(&s.full[st], i & 1);
          tc_fence_after();
          if (el) {
            const uint32_t vb = smem_u32(s.ring[st]);
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              mma_f16_ss_2sm(tO + 128 * j, sdesc_kmajor_sw128(pa + (kk >> 1) * (HC * 128) + (kk & 1) * 64 + ks * 32),
                             sdesc_mnmajor_sw128(vb + ks * 2048, STB / 2), id_o, (i | kk | ks) != 0);
            mma_commit_2sm(&s.empty[st]);
            if (v + 1 == NVS) {
              mma_commit_2sm(&s.pv_done);
              if (i + 1 == n_tiles) mma_commit_2sm(&s.o_full);
            }
          }
          __syncwarp();
        }
      };
      mbar_wait(&s.q_full, 0);
      if (n_tiles > 0) issue_s(0);
      // S_{i+1} (other S buffer, runs under softmax i) and P V_i in whichever
      // order their inputs arrive: the tensor pipe executes in issue order,
      // so a fixed S-first order would hold P V_i — and the V loads of tile
      // i + 1 behind it — until tile i + 1's first K stage has landed.
      for (int i = 0; i < n_tiles; ++i) {
        bool s_next = i + 1 >= n_tiles;
        for (;;) {
          int pick = 0;
          if (lane_id() == 0) {
            if (!s_next && mbar_try_wait(&s.full[0], (i + 1) & 1)) pick = 1;
            else if (mbar_try_wait(&s.p_full, i & 1)) pick = 2;
          }
          pick = __shfl_sync(0xffffffffu, pick, 0);
          if (pick == 1) {
            issue_s(i + 1);
            s_next = true;
          } else if (pick == 2) {
            issue_pv(i);
            break;
          }
        }
        if (!s_next) issue_s(i + 1);
      }
    } else if (elect_one()) {
      // relay: this CTA's TMA stages have landed -> the leader's barriers
      mbar_wait(&s.q_full, 0);
      mbar_arrive_cluster(mapa_shared(smem_u32(&s.q_full), 0));
      for (int t = 0; t < n_tiles; ++t)
        for (int st = 0; st < NST; ++st) {
          mbar_wait(&s.full[st], t & 1);
          mbar_arrive_cluster(mapa_shared(smem_u32(&s.full[st]), 0));
        }
    }
  } else {
    // -------------------------- softmax / correction / epilogue (lane = thread) --
    const int lane = threadIdx.x;  // TMEM lane: row lane % 64, keys / V columns half lane / 64
    const int row = lane & (HC - 1), half = lane >> 6;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float c1 = p.scale * kLog2e;
    const uint32_t p_row = smem_u32(s.p[half]) + (row >> 3) * 1024 + (row & 7) * 128;
    const uint32_t pfull_leader = mapa_shared(smem_u32(&s.p_full), 0);
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      const int bb = i & 1;
      mbar_wait(&s.s_full[bb], (i >> 1) & 1);
      tc_fence_after();
      uint32_t sv[2][32];
      tmem_ld32(tS[bb] + lane_off, sv[0]);
      tmem_ld32(tS[bb] + lane_off + 32, sv[1]);
      tmem_ld_wait();
      float mx = __uint_as_float(sv[0][0]);
#pragma unroll
      for (int j = 1; j < 64; ++j) mx = fmaxf(mx, __uint_as_float(sv[j >> 5][j & 31]));
      s.xm[bb][lane] = mx;
      named_bar_sync(1, 128);
      mx = fmaxf(mx, s.xm[bb][lane ^ 64]);
      m_true = fmaxf(m_true, mx * p.scale);
      const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;  // same in both halves
      float alpha = 1.f;
      if (need) {
        alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
        l *= alpha;
        m_ref = m_true;
      }
      const float nmb = -m_ref * kLog2e;
      uint32_t pk[32];
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float p0 = ex2_mufu(fmaf(__uint_as_float(sv[j >> 4][(2 * j) & 31]), c1, nmb));
        const float p1 = ex2_mufu(fmaf(__uint_as_float(sv[j >> 4][(2 * j + 1) & 31]), c1, nmb));
        rs += p0 + p1;
        pk[j] = pack_bf16x2(p0, p1);
      }
      l += rs;
      // P V_{i-1} has retired: the P buffer is free and O may be rescaled
      if (i > 0) {
        mbar_wait(&s.pv_done, (i - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, need)) {
#pragma unroll 1
          for (int c = 0; c < 256 / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tO + lane_off + c * 16, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st16(tO + lane_off + c * 16, r);
          }
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        sts128(p_row + ((u ^ (row & 7)) << 4), make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        if (leader) mbar_arrive(&s.p_full);
        else mbar_arrive_cluster(pfull_leader);
      }
    }
    // ---- finalize (finalize_root): d2 = the two halves' sums re-based to d1 ----
    named_bar_sync(1, 128);  // every half has read the last max exchange
    s.xm[0][lane] = l;
    named_bar_sync(1, 128);
    const float lo = s.xm[0][lane & 63], hi = s.xm[0][(lane & 63) + 64];
    const float l_ref = lo + hi;  // same operand order in both halves
    const float l_true = l_ref * ex2_mufu((m_ref - m_true) * kLog2e);
    const int64_t grow = static_cast<int64_t>(b) * HN + h * HC + row;
    if (half == 0) {
      if (p.part_m == nullptr) {
        p.m[grow] = m_true;
        p.l[grow] = l_true;
      } else {
        p.part_m[slice * p.rows_total + grow] = m_true;
        p.part_l[slice * p.rows_total + grow] = l_true;
      }
    }
    if (n_tiles > 0) {
      mbar_wait(&s.o_full, 0);
      tc_fence_after();
    }
    const float inv_l = 1.f / l_ref;
#pragma unroll 1
    for (int c = 0; c < 256 / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tO + lane_off + c * 32, r);
      tmem_ld_wait();
      const int col = 256 * (c >> 2) + 128 * half + 32 * (c & 3);
      if (p.part_o == nullptr) {
        uint4* dst = reinterpret_cast<uint4*>(p.o + grow * DV + col);
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
        float4* dst = reinterpret_cast<float4*>(p.part_o + (slice * p.rows_total + grow) * DV + col);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          dst[v] = make_float4(__uint_as_float(r[4 * v]) * inv_l, __uint_as_float(r[4 * v + 1]) * inv_l,
                               __uint_as_float(r[4 * v + 2]) * inv_l, __uint_as_float(r[4 * v + 3]) * inv_l);
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // no remote traffic into a CTA that has exited
  if (warp == 5) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace

bool mla_supports(int64_t heads, int64_t skv, int64_t dv, int64_t dqk, int64_t segments) {
  return heads == HN && dv == DV && dqk == DQK && segments >= 1 && skv % segments == 0 &&
         (skv / segments) % TK == 0 && skv / segments > 0;
}

// Slices launched: the reference's segments, each cut into c sub-slices of
// >= 256 keys until the grid (2 halves x bs x slices) fills the GPU.
int64_t mla_pick_splits(int64_t bs, int64_t skv, int64_t segments) {
  int64_t n = segments;
  const int64_t slice = skv / segments;
  for (int64_t c = 2; c <= 64 && 2 * bs * n < 148; c *= 2)
    if (slice % (c * TK) == 0 && slice / c >= 256) n = segments * c;
  return n;
}

cudaError_t launch_mla_decode(const MlaArgs& a, cudaStream_t st) {
  if (!mla_supports(HN, a.skv, DV, DQK, a.nslices)) return cudaErrorNotSupported;
  CUtensorMap tq, tk, tv;
  const uint64_t qdims[2] = {DQK, static_cast<uint64_t>(a.bs * HN)};
  const uint64_t kdims[2] = {DQK, static_cast<uint64_t>(a.bs * a.skv)};
  const uint64_t strides[1] = {DQK * 2};
  const uint32_t qbox[2] = {64, HC}, kbox[2] = {64, TK / 2}, vbox[2] = {64, 32};
  if (!make_tmap(&tq, a.q, 2, qdims, strides, qbox, 2) || !make_tmap(&tk, a.kv, 2, kdims, strides, kbox, 2) ||
      !make_tmap(&tv, a.kv, 2, kdims, strides, vbox, 2))
    return cudaErrorInvalidValue;
  Params p{};
  p.skv = a.skv;
  p.slice_len = a.skv / a.nslices;
  p.rows_total = a.rows_total;
  p.scale = a.scale;
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  const size_t smem = sizeof(Smem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(mla_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(2, static_cast<unsigned>(a.bs), static_cast<unsigned>(a.nslices));
  mla_decode_kernel<<<grid, NT, smem, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace rf
