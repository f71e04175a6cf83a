// MLA decode (multi-latent attention, absorbed form; the paper's MLA workload
// L1-L9: hn = 128 heads, latent hd = 512, rope ped = 64)
// as the attention cascade of make_attention (proj/src/workloads.cpp:66-120):
//   d1 = max P, d2 = sum e^(P - d1), d3 = sum e^(P - d1) / d2 V,
//   P = scale Q K^T with K = the 576-wide cache rows [c_kv | k_rope] and
//   V = their first 512 columns (c_kv) — one cache tensor serves both.
// All 128 heads of a batch share the cache, so a decode step is GEMM-shaped:
// S = Q (128 x 576) K^T, O += P V (N = 512).
//
// TMEM holds 512 fp32 columns and O alone is 128 x 512, so a (batch, KV
// slice) runs on a CTA PAIR (thread-block cluster of 2) that splits both
// reductions by the cache's 64-column chunks: CTA h owns chunks
// {4h .. 4h+3} (+ the rope chunk 8 for h = 0):
//   * its Q chunks stay resident in shared memory (80 / 64 KB) and it streams
//     only its own chunks of each 64-key cache tile (40 / 32 KB per tile,
//     2-slot TMA ring, SWIZZLE_128B) — the pair reads every cache byte once;
//   * tcgen05.mma kind::f16 computes its PARTIAL S_h = Q_h K_h^T
//     (M = 128, N = 64 keys, 20 / 16 K-steps) into a double-buffered S in TMEM;
//   * the softmax warps (thread = head row) swap partial S tiles with the
//     peer through distributed shared memory: each stages its 64 fp32
//     partials in its own shared memory, one thread bulk-copies the 32 KB
//     tile into the peer's receive buffer (cp.async.bulk shared::cta ->
//     shared::cluster, completing on the peer's mbarrier: no release fence;
//     per-thread st.async was measured ~10x slower); S = S_0 + S_1 is then
//     bit-identical in both CTAs (operands added in the same order), and so
//     are d1, d2 and P;
//   * P (bf16) overwrites the S buffer and is the TMEM A operand of
//     O_h += P V_h (M = 128, N = 256, K = 64), V_h = the CTA's own 4 chunks
//     of the same smem tile as an MN-major B;
//   * the d3 correction exp(d1' - d1) is applied to the TMEM accumulator
//     lazily (only when the running max passes the reference by 2^8, after
//     P V_{i-1} has retired); d2'/d2 telescopes to 1/d2 at finalize
//     (finalize_root, proj/src/simulator.cpp:611-621) — as attn_sm100.cu;
//   * Multi-Segment: each KV slice writes its (m, l, O/l) partial state,
//     merged in slice order by merge.cu (run_multisegment semantics).
// MMA order: S_{i+1} and P V_i as their inputs arrive (S_{i+1} under softmax i).
// Warps: 0-3 softmax + exchange + epilogue, 4 TMA, 5 MMA (192 threads).
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

#ifdef RF_MLA_TRACE
__device__ unsigned long long g_mla_trace[2][64][8];
#define MT_STAMP(t, i) do { if ((blockIdx.y | blockIdx.z) == 0 && (t) < 64) { unsigned long long v_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_)); g_mla_trace[blockIdx.x][(t)][(i)] = v_; } } while (0)
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
constexpr int TK = 64;         // keys per tile
constexpr int MAXC = 5;        // chunks per CTA (h = 0: 0-3 + rope 8; h = 1: 4-7)
constexpr int NSLOT = 2;
constexpr int NT = 192;
constexpr int XB = HN * TK * 4; // exchange buffer bytes (one partial S tile, fp32)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Smem {
  uint8_t q[MAXC][HN * 128];          // 5 x 16 KB
  uint8_t kv[NSLOT][MAXC][TK * 128];  // 2 x 5 x 8 KB
  float xsend[HN * TK];               // this CTA's partial S, staged for the bulk copy
  float xrecv[HN * TK];               // the peer's partial S of the current tile
  uint64_t q_full;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2];
  uint64_t pv_done, o_full;
  uint64_t x_full;   // peer's partial landed (complete_tx)
  uint64_t x_empty;  // peer has consumed the partial we sent (remote arrivals)
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

__device__ __forceinline__ int chunk_of(int h, int j) { return h == 0 ? (j < 4 ? j : 8) : 4 + j; }

// Bulk copy (TMA engine) from this CTA's shared memory into the peer's,
// completing `bytes` on the peer's mbarrier.
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes,
                                                  uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src), "r"(bytes), "r"(bar_cluster)
      : "memory");
}

// float4 chunk q of row r at chunk q ^ (r & 15): conflict-free row-per-thread access
__device__ __forceinline__ int xoff(int r, int q) { return r * TK + 4 * (q ^ (r & 15)); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tkv,
                      const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int h = static_cast<int>(cluster_ctarank());  // = blockIdx.x: V columns [256 h, +256)
  const int nc = h == 0 ? 5 : 4;
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
    mbar_init(&s.x_full, 1);   // armed with expect_tx by this CTA each tile
    mbar_init(&s.x_empty, 4);  // the peer's 4 softmax warps
    fence_barrier_init();
    mbar_arrive_expect_tx(&s.x_full, XB);  // tile 0's incoming partial
  }
  if (warp == 5) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote traffic
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + TK};
  const uint32_t tO = tmem + 256;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tkv);
      mbar_arrive_expect_tx(&s.q_full, nc * HN * 128);
      for (int j = 0; j < nc; ++j)
        tma_load_2d(s.q[j], &tq, &s.q_full, chunk_of(h, j) * 64, b * HN, kEvictFirst);
      const int32_t y0 = static_cast<int32_t>(static_cast<int64_t>(b) * p.skv + kv0);
      for (int t = 0; t < n_tiles; ++t) {
        const int slot = t % NSLOT;
        mbar_wait(&s.kv_empty[slot], ((t / NSLOT) & 1) ^ 1);
        MT_STAMP(t, 0);
        mbar_arrive_expect_tx(&s.kv_full[slot], nc * TK * 128);
        for (int j = 0; j < nc; ++j)
          tma_load_2d(s.kv[slot][j], &tkv, &s.kv_full[slot], chunk_of(h, j) * 64, y0 + t * TK, kEvictFirst);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA ----
    const uint32_t id_s = idesc_f16(HN, TK, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(HN, DH, kFmtBF16, false, true);
    const bool leader = elect_one();
    auto issue_s = [&](int i) {  // partial S_i = Q_h K_h,i^T into S buffer i & 1
      const int slot = i % NSLOT;
      mbar_wait(&s.kv_full[slot], (i / NSLOT) & 1);
      tc_fence_after();
      if (leader) {
        const uint32_t qa = smem_u32(s.q[0]), kb = smem_u32(s.kv[slot][0]);
        for (int j = 0; j < nc; ++j)
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4)
            mma_f16_ss(tS[i & 1], sdesc_kmajor_sw128(qa + j * HN * 128 + k4 * 32),
                       sdesc_kmajor_sw128(kb + j * TK * 128 + k4 * 32), id_s, (j | k4) != 0);
        mma_commit(&s.s_full[i & 1]);
        MT_STAMP(i, 1);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int i) {  // O_h += P_i V_h,i  (V_h = this CTA's chunks 0-3 of tile i)
      const int slot = i % NSLOT;
      mbar_wait(&s.p_full[i & 1], (i >> 1) & 1);
      tc_fence_after();
      if (leader) {
        const uint32_t vb = smem_u32(s.kv[slot][0]);
#pragma unroll
        for (int ks = 0; ks < TK / 16; ++ks)
          mma_f16_ts(tO, tS[i & 1] + ks * 8, sdesc_mnmajor_sw128(vb + ks * 2048, TK * 128), id_o,
                     (i | ks) != 0);
        mma_commit(&s.kv_empty[slot]);
        mma_commit(&s.pv_done);
        if (i + 1 == n_tiles) mma_commit(&s.o_full);
        MT_STAMP(i, 2);
      }
      __syncwarp();
    };
    mbar_wait(&s.q_full, 0);
    if (n_tiles > 0) issue_s(0);
    // S_{i+1} (other S buffer, runs under softmax i) and P V_i in whichever
    // order their inputs arrive: the tensor pipe executes in issue order and
    // issue blocks at its rate, so a fixed S-first order would hold P V_i —
    // and with it the release of cache slot i, which gates the load of tile
    // i + 2 — behind tile i + 1's arrival.
    for (int i = 0; i < n_tiles; ++i) {
      bool s_next = i + 1 >= n_tiles;  // S_{i+1} issued (or none)
      for (;;) {
        int pick = 0;  // 1: S_{i+1}, 2: P V_i (lane 0 decides for the warp)
        if (lane_id() == 0) {
          if (!s_next && mbar_try_wait(&s.kv_full[(i + 1) % NSLOT], ((i + 1) / NSLOT) & 1)) pick = 1;
          else if (mbar_try_wait(&s.p_full[i & 1], (i >> 1) & 1)) pick = 2;
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
  } else {
    // ------------------- partial-S exchange / softmax / correction / epilogue --
    const int row = threadIdx.x;  // head
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float c1 = p.scale * kLog2e;
    const uint32_t peer = static_cast<uint32_t>(h ^ 1);
    const uint32_t xrecv_peer = mapa_shared(smem_u32(s.xrecv), peer);
    const uint32_t xfull_peer = mapa_shared(smem_u32(&s.x_full), peer);
    const uint32_t xempty_peer = mapa_shared(smem_u32(&s.x_empty), peer);
    float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      const int bb = i & 1;
      mbar_wait(&s.s_full[bb], (i >> 1) & 1);
      tc_fence_after();
      if (threadIdx.x == 0) MT_STAMP(i, 3);
      uint32_t sv[2][32];
      tmem_ld32(tS[bb] + lane_off, sv[0]);
      tmem_ld32(tS[bb] + lane_off + 32, sv[1]);
      tmem_ld_wait();
      // stage this CTA's partial row; one thread bulk-copies the tile into the
      // peer once the peer has consumed the previous one
      if (i > 0) {
        if (threadIdx.x == 0) bulk_wait_read0();  // previous copy has read xsend
        named_bar_sync(1, 128);
      }
#pragma unroll
      for (int q = 0; q < TK / 4; ++q)
        *reinterpret_cast<uint4*>(s.xsend + xoff(row, q)) =
            make_uint4(sv[q >> 3][(4 * q) & 31], sv[q >> 3][(4 * q + 1) & 31], sv[q >> 3][(4 * q + 2) & 31],
                       sv[q >> 3][(4 * q + 3) & 31]);
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
        if (i > 0) mbar_wait(&s.x_empty, (i - 1) & 1);
        MT_STAMP(i, 4);
        bulk_copy_to_peer(xrecv_peer, smem_u32(s.xsend), XB, xfull_peer);
        bulk_commit();
      }
      // receive the peer's partial row: S = S_0 + S_1 (operands in chunk order,
      // so both CTAs round identically)
      mbar_wait(&s.x_full, i & 1);
      if (threadIdx.x == 0) MT_STAMP(i, 5);
      float sx[TK];
#pragma unroll
      for (int q = 0; q < TK / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(s.xrecv + xoff(row, q));
        const float pv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float own = __uint_as_float(sv[q >> 3][(4 * q + e) & 31]);
          sx[4 * q + e] = h == 0 ? own + pv[e] : pv[e] + own;
        }
      }
      // the receive buffer is free again: re-arm it for the next tile, then
      // tell the peer (its next copy may land after this point)
      __syncwarp();
      if (threadIdx.x == 0 && i + 1 < n_tiles) mbar_arrive_expect_tx(&s.x_full, XB);
      if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(xempty_peer);
      float mx = sx[0];
#pragma unroll
      for (int j = 1; j < TK; ++j) mx = fmaxf(mx, sx[j]);
      m_true = fmaxf(m_true, mx * p.scale);
      const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
      float alpha = 1.f;
      if (need) {
        alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
        l *= alpha;
        m_ref = m_true;
      }
      if (i > 0 && __any_sync(0xffffffffu, need)) {
        // O *= exp(d1' - d1) once P V_{i-1} has retired (pv_done completions so
        // far are i - 1 or i: P V_i needs this tile's P)
        mbar_wait(&s.pv_done, (i - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < DH / 16; ++c) {
          uint32_t r[16];
          tmem_ld16(tO + lane_off + c * 16, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
          tmem_st16(tO + lane_off + c * 16, r);
        }
        tmem_st_wait();
      }
      const float nmb = -m_ref * kLog2e;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float p0 = ex2_mufu(fmaf(sx[32 * c + 2 * j], c1, nmb));
          const float p1 = ex2_mufu(fmaf(sx[32 * c + 2 * j + 1], c1, nmb));
          rs += p0 + p1;
          pk[j] = pack_bf16x2(p0, p1);
        }
        tmem_st16(tS[bb] + lane_off + 16 * c, pk);
      }
      l += rs;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&s.p_full[bb]);
      if (threadIdx.x == 0) MT_STAMP(i, 6);
    }
    if (threadIdx.x == 0) bulk_wait0();  // the last copy has left this CTA
    // ---- finalize (finalize_root): d2 re-based to the true d1, d3 = O / d2 ----
    const float l_true = l * ex2_mufu((m_ref - m_true) * kLog2e);
    const int64_t grow = static_cast<int64_t>(b) * HN + row;
    if (h == 0) {
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
      const int col = h * DH + c * 32;
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
  if (warp == 5) tmem_dealloc<512>(tmem);
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
