// MLA decode (multi-latent attention, absorbed form; the paper's MLA workload
// L1-L9: hn = 128 heads, latent hd = 512, rope ped = 64)
// as the attention cascade of make_attention (proj/src/workloads.cpp:66-120):
//   d1 = max P, d2 = sum e^(P - d1), d3 = sum e^(P - d1) / d2 V,
//   P = scale Q K^T with K = the 576-wide cache rows [c_kv | k_rope] and
//   V = their first 512 columns (c_kv) — one cache tensor serves both.
// All 128 heads of a batch share the cache, so a decode step is GEMM-shaped:
// S = Q (128 x 576) K^T, O += P V (N = 512). Per CTA (one batch, one half of
// the 512 V columns, one KV slice):
//   * TMA (SWIZZLE_128B): Q once as 9 chunks of [128 x 64] (144 KB); cache
//     tiles of 32 keys as 9 chunks of [32 x 64] (36 KB) into a 2-slot ring;
//     the same smem tile is the K-major B of S and the MN-major B of P V.
//   * tcgen05.mma kind::f16: S = Q K^T (M = 128, N = 32, 36 K-steps) into a
//     double-buffered S in TMEM, so S_{i+1} runs while the softmax works on
//     S_i; P (bf16) overwrites S_i and is the TMEM A operand of
//     O += P V (M = 128, N = 256, K = 32) into the O accumulator (256 cols).
//   * the cascaded statistics d1, d2 in registers, thread = head row; the d3
//     correction exp(d1' - d1) applied to the TMEM accumulator lazily (only
//     when the running max passes the reference by 2^8, after P V_{i-1} has
//     retired), the d2'/d2 factor telescoped to 1/d2 at finalize
//     (finalize_root, proj/src/simulator.cpp:611-621) — as attn_sm100.cu.
//   * Multi-Segment: each KV slice writes its (m, l, O/l) partial state,
//     merged in slice order by merge.cu (run_multisegment semantics).
// Warps: 0-3 softmax + epilogue, 4 TMA, 5 MMA (192 threads).
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

#ifdef RF_MLA_TRACE
__device__ unsigned long long g_mla_trace[8 * 64];
#define MT_STAMP(t, i) do { if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0 && (t) < 64) { unsigned long long v_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_)); g_mla_trace[(t) * 8 + (i)] = v_; } } while (0)
#else
#define MT_STAMP(t, i) do {} while (0)
#endif

namespace rf {
namespace {

using namespace sm100;

constexpr int HN = 128;        // heads (rows, UMMA M)
constexpr int DQK = 576;       // cache row / query width
constexpr int DV = 512;        // value width (latent)
constexpr int DH = DV / 2;     // value columns per CTA
constexpr int TK = 32;         // keys per tile
constexpr int NCH = DQK / 64;  // 128 B swizzle chunks per row
constexpr int NSLOT = 2;
constexpr int NT = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Smem {
  uint8_t q[NCH][HN * 128];       // 9 x 16 KB
  uint8_t kv[NSLOT][NCH][TK * 128];  // 2 x 9 x 4 KB
  uint64_t q_full;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2];
  uint64_t pv_done, o_full;
  uint32_t tmem_base;
};

struct Params {
  int64_t skv, slice_len, rows_total;
  int bs;
  float scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
};

__global__ void __launch_bounds__(NT, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                      const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int half = blockIdx.x;   // V columns [256 half, +256)
  const int b = blockIdx.y;      // batch
  const int slice = blockIdx.z;  // KV slice
  const int64_t kv0 = static_cast<int64_t>(slice) * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / TK);

  if (threadIdx.x == 0) {
    mbar_init(&s.q_full, 1);
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s.s_full[k], 1);
      mbar_init(&s.p_full[k], 4);  // one arrival per softmax warp
    }
    mbar_init(&s.pv_done, 1);
    mbar_init(&s.o_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + 32};
  const uint32_t tO = tmem + 256;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tkv);
      mbar_arrive_expect_tx(&s.q_full, NCH * HN * 128);
      for (int c = 0; c < NCH; ++c) tma_load_2d(s.q[c], &tq, &s.q_full, c * 64, b * HN, kEvictFirst);
      const int32_t y0 = static_cast<int32_t>(static_cast<int64_t>(b) * p.skv + kv0);
      for (int t = 0; t < n_tiles; ++t) {
        const int slot = t % NSLOT;
        mbar_wait(&s.kv_empty[slot], ((t / NSLOT) & 1) ^ 1);
        MT_STAMP(t, 0);
        mbar_arrive_expect_tx(&s.kv_full[slot], NCH * TK * 128);
        for (int c = 0; c < NCH; ++c)
          tma_load_2d(s.kv[slot][c], &tkv, &s.kv_full[slot], c * 64, y0 + t * TK, kEvictNormal);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA ----
    const uint32_t id_s = idesc_f16(HN, TK, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(HN, DH, kFmtBF16, false, true);
    const bool leader = elect_one();
    auto issue_pv = [&](int j) {  // O += P_j V_j  (P in S buffer j & 1, V = cache tile j)
      const int slot = j % NSLOT;
      mbar_wait(&s.p_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      if (leader) MT_STAMP(j, 5);
      if (leader) {
        const uint32_t vb = smem_u32(s.kv[slot][4 * half]);
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks)
          mma_f16_ts(tO, tS[j & 1] + ks * 8, sdesc_mnmajor_sw128(vb + ks * 2048, TK * 128), id_o,
                     (j | ks) != 0);
        mma_commit(&s.kv_empty[slot]);
        mma_commit(&s.pv_done);
        if (j + 1 == n_tiles) mma_commit(&s.o_full);
        MT_STAMP(j, 6);
      }
      __syncwarp();
    };
    mbar_wait(&s.q_full, 0);
    // Issue order S_i, P V_i: the tensor pipe executes in issue order and the
    // issue blocks at its rate, so issuing S_{i+1} ahead of P V_i would hold
    // P V_i (and with it the release of cache slot i, which gates the load of
    // tile i + 2) behind K_{i+1}'s arrival — a load-latency-bound loop
    // (measured 2.1 us per tile vs 1.3 us in this order).
    for (int i = 0; i < n_tiles; ++i) {
      const int slot = i % NSLOT;
      mbar_wait(&s.kv_full[slot], (i / NSLOT) & 1);
      tc_fence_after();
      if (leader) MT_STAMP(i, 1);
      if (leader) {  // S_i = Q K_i^T into S buffer i & 1
        const uint32_t qa = smem_u32(s.q[0]), kb = smem_u32(s.kv[slot][0]);
#pragma unroll 4
        for (int ks = 0; ks < DQK / 16; ++ks) {
          const int c = ks >> 2;
          const uint32_t off = (ks & 3) * 32;
          mma_f16_ss(tS[i & 1], sdesc_kmajor_sw128(qa + c * HN * 128 + off),
                     sdesc_kmajor_sw128(kb + c * TK * 128 + off), id_s, ks > 0);
        }
        mma_commit(&s.s_full[i & 1]);
        MT_STAMP(i, 2);
      }
      __syncwarp();
      issue_pv(i);
    }
  } else {
    // ----------------------------------- softmax / correction / epilogue --
    const int row = threadIdx.x;  // head
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float c1 = p.scale * kLog2e;
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      const int bb = i & 1;
      mbar_wait(&s.s_full[bb], (i >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 0) MT_STAMP(i, 3);
      uint32_t sr[32];
      tmem_ld32(tS[bb] + lane_off, sr);
      tmem_ld_wait();
      float mx = __uint_as_float(sr[0]);
#pragma unroll
      for (int j = 1; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(sr[j]));
      m_true = fmaxf(m_true, mx * p.scale);
      const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
      float alpha = 1.f;
      if (need) {
        alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
        l *= alpha;
        m_ref = m_true;
      }
      if (i > 0 && __any_sync(0xffffffffu, need)) {
        // O *= exp(d1' - d1) once P V_{i-1} has retired (completions of pv_done
        // so far are i - 1 or i: P V_i needs this tile's P)
        mbar_wait(&s.pv_done, (i - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tO + lane_off + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
          tmem_st32(tO + lane_off + c * 32, r);
        }
      }
      const float nmb = -m_ref * kLog2e;
      uint32_t pk[16];
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float p0 = ex2_mufu(fmaf(__uint_as_float(sr[2 * j]), c1, nmb));
        const float p1 = ex2_mufu(fmaf(__uint_as_float(sr[2 * j + 1]), c1, nmb));
        rs += p0 + p1;
        pk[j] = pack_bf16x2(p0, p1);
      }
      l += rs;
      tmem_st16(tS[bb] + lane_off, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.p_full[bb]);
      if (threadIdx.x == 0) MT_STAMP(i, 4);
    }
    // ---- finalize (finalize_root): d2 re-based to the true d1, d3 = O / d2 ----
    const float l_true = l * ex2_mufu((m_ref - m_true) * kLog2e);
    const int64_t grow = static_cast<int64_t>(b) * HN + row;
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
    const float inv_l = 1.f / l;
#pragma unroll 1
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(tO + lane_off + c * 32, r);
      tmem_ld_wait();
      const int col = half * DH + c * 32;
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
  __syncthreads();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

}  // namespace

bool mla_supports(int64_t heads, int64_t skv, int64_t dv, int64_t dqk, int64_t segments) {
  return heads == HN && dv == DV && dqk == DQK && segments >= 1 && skv % segments == 0 &&
         (skv / segments) % TK == 0 && skv / segments > 0;
}

// Slices launched: the reference's segments, each cut into c sub-slices of
// >= 128 keys until the grid (2 halves x bs x slices) fills the GPU.
int64_t mla_pick_splits(int64_t bs, int64_t skv, int64_t segments) {
  int64_t n = segments;
  const int64_t slice = skv / segments;
  for (int64_t c = 2; c <= 64 && 2 * bs * n < 148; c *= 2)
    if (slice % (c * TK) == 0 && slice / c >= 128) n = segments * c;
  return n;
}

cudaError_t launch_mla_decode(const MlaArgs& a, cudaStream_t st) {
  if (!mla_supports(HN, a.skv, DV, DQK, a.nslices)) return cudaErrorNotSupported;
  CUtensorMap tq, tkv;
  const uint64_t qdims[2] = {DQK, static_cast<uint64_t>(a.bs * HN)};
  const uint64_t kdims[2] = {DQK, static_cast<uint64_t>(a.bs * a.skv)};
  const uint64_t strides[1] = {DQK * 2};
  const uint32_t qbox[2] = {64, HN}, kbox[2] = {64, TK};
  if (!make_tmap(&tq, a.q, 2, qdims, strides, qbox, 2) || !make_tmap(&tkv, a.kv, 2, kdims, strides, kbox, 2))
    return cudaErrorInvalidValue;
  Params p{};
  p.skv = a.skv;
  p.slice_len = a.skv / a.nslices;
  p.rows_total = a.rows_total;
  p.bs = static_cast<int>(a.bs);
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
  mla_decode_kernel<<<grid, NT, smem, st>>>(tq, tkv, p);
  return cudaGetLastError();
}

}  // namespace rf
