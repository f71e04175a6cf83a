// bf16 safe-softmax -> GEMM attention on Blackwell tensor cores (sm_100a),
// Q resident in TMEM and S double-buffered so the tensor core never waits on
// the softmax -> P V -> S chain.
//
// Same cascade, incremental form and tile plan as attn_sm100.cu (the
// reference's incr_ingest_element, proj/src/simulator.cpp:566-589, over
// make_attention's reductions, proj/src/workloads.cpp:66-120; RT = ST = 128,
// tests/golden/flash_attention_tile.txt). What changes is where the operands
// live:
//   * the Q tile (128 rows x D) is written into TMEM by the softmax threads
//     themselves (thread = row, straight from global memory) and is the A
//     operand of S = Q K^T (tcgen05.mma with A in TMEM): shared memory only
//     feeds K / V (64 B/clk of operand reads at N = 128 instead of 128), and
//     the 64 KB of Q staging becomes K/V ring depth;
//   * TMEM (512 columns at D = 128): Q0 [0, 64)  Q1 [64, 128)  (double-
//     buffered: the next unit's Q is written while this one runs)
//     S0 [128, 256)  S1 [256, 384)  O [384, 512). S is double-buffered, so the
//     MMA issue order is S_0, S_1, P V_0, S_2, P V_1, S_3, ...: S_{i+1} runs
//     while the softmax works on S_i, and P V_i only waits for P_i. P_i (bf16)
//     overwrites S_i's first 64 columns and is the A operand of P V_i;
//   * one Q tile per CTA, softmax by 8 warps: the two warps of a TMEM lane
//     quarter split each row's 128 keys (64 each) and exchange their partial
//     row max through shared memory (one 64-thread named barrier per tile);
//     the two partial sums are added once, at finalize.
// The d3 correction exp(d1' - d1) is lazy as in attn_sm100.cu (re-base only
// when the running max passes the reference by 2^8; it waits for P V_{i-1});
// d2'/d2 telescopes to 1/d2 at finalize (finalize_root,
// proj/src/simulator.cpp:611-621).
// Persistent: one CTA per SM walks the (Q tile, b*h, slice) units; the tile
// sequence (and the MMA issue order) runs on across units, so the next
// unit's first S MMAs overlap this unit's last P V and its epilogue.
// Warps: 0-7 softmax + correction + epilogue (warp w: lane quarter w & 3,
// key half w >> 2), 8 TMA producer, 9 MMA issuer (one elected lane) + TMEM owner.
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;      // rows per Q tile
constexpr int BN = 128;      // keys per KV tile
constexpr int NSLOT = 6;     // K/V ring slots (32 KB each at D = 128)
constexpr int NSW = 8;       // softmax warps
constexpr int NTHREADS = (NSW + 2) * 32;
constexpr int WTMA = NSW, WMMA = NSW + 1;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
__device__ __forceinline__ constexpr bool kPolyPairs(int jj) { return (jj & 3) == 3; }

template <int D>
struct Smem {
  static constexpr int kTile = BN * D * 2;  // one bf16 [128 x D] K or V tile
  static constexpr int kChunks = D / 64;    // 128 B swizzle chunks along D
  uint8_t kv[NSLOT][kTile];
  float xmax[2][2][BM];  // [tile parity][key half][row]: partial row max
  float xl[2][BM];       // [key half][row]: partial row sum at finalize
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t q_full[2], s_full[2], p_full[2], pv_bar, o_empty;
  uint32_t tmem_base;
};

struct Params {
  int64_t sq, skv, slice_len, slice_begin, part_base, rows_total;
  float scale_log2;  // softmax_scale * log2(e)
  float scale;
  const __nv_bfloat16* q;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
  int units_x, units_bh, units;  // work units: (Q tile, b*h, slice)
};

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_qt_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem<D>& s = *reinterpret_cast<Smem<D>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int lane = lane_id();
  const int n = static_cast<int>(p.slice_len / BN);  // tiles per unit
  const int nunits = p.units > static_cast<int>(blockIdx.x)
                         ? (p.units - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                               static_cast<int>(gridDim.x)
                         : 0;
  const int G = nunits * n;  // this CTA's tiles, in order
  auto unit_of = [&](int uc, int& bh, int64_t& q_row0, int64_t& slice) {
    const int u = static_cast<int>(blockIdx.x) + uc * static_cast<int>(gridDim.x);
    const int x = u % p.units_x;
    const int r = u / p.units_x;
    bh = r % p.units_bh;
    slice = p.slice_begin + r / p.units_bh;
    q_row0 = static_cast<int64_t>(x) * BM;
  };
  constexpr uint32_t kQ = 0, kS = D, kO = D + 2 * BN;  // TMEM column bases

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s.q_full[k], NSW);  // every softmax warp wrote its part of Q
      mbar_init(&s.s_full[k], 1);
      mbar_init(&s.p_full[k], NSW);
    }
    mbar_init(&s.pv_bar, 1);
    mbar_init(&s.o_empty, NSW);
    fence_barrier_init();
  }
  if (warp == WMMA) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == WTMA) {
    // ---------------------------------------------------------------- TMA --
    // ring items in the MMA's consumption order: K_0, K_1, then V_g, K_{g+2}
    if (elect_one()) {
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      int t = 0;
      auto put = [&](bool v, int g) {
        int bh;
        int64_t q_row0, slice;
        unit_of(g / n, bh, q_row0, slice);
        const int32_t y = static_cast<int32_t>(bh * p.skv + slice * p.slice_len + (g % n) * BN);
        const int slot = t % NSLOT;
        mbar_wait(&s.kv_empty[slot], ((t / NSLOT) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.kv_full[slot], Smem<D>::kTile);
        for (int c = 0; c < Smem<D>::kChunks; ++c)
          tma_load_2d(s.kv[slot] + c * BN * 128, v ? &tv : &tk, &s.kv_full[slot], c * 64, y, kEvictLast);
        ++t;
      };
      if (G > 0) put(false, 0);
      if (G > 1) put(false, 1);
      for (int g = 0; g < G; ++g) {
        put(true, g);
        if (g + 2 < G) put(false, g + 2);
      }
    }
  } else if (warp == WMMA) {
    // ---------------------------------------------------------------- MMA --
    const uint32_t id_s = idesc_f16(BM, BN, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(BM, D, kFmtBF16, false, true);
    const bool leader = elect_one();
    int t = 0;
    auto take = [&]() {
      const int slot = t % NSLOT;
      mbar_wait(&s.kv_full[slot], (t / NSLOT) & 1);
      tc_fence_after();
      ++t;
      return slot;
    };
    auto issue_s = [&](int g) {  // S_g = Q K_g^T into S buffer g & 1
      const int uc = g / n;
      if (g % n == 0) {
        mbar_wait(&s.q_full[uc & 1], (uc >> 1) & 1);
        tc_fence_after();
      }
      const int slot = take();
      if (leader) {
        const uint32_t kb = smem_u32(s.kv[slot]);
        const uint32_t tq = tmem + kQ + (uc & 1) * (D / 2);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * (BN * 128) + (ks & 3) * 32;
          mma_f16_ts(tmem + kS + (g & 1) * BN, tq + ks * 8, sdesc_kmajor_sw128(kb + off), id_s, ks > 0);
        }
        mma_commit(&s.s_full[g & 1]);
        mma_commit(&s.kv_empty[slot]);
      }
      __syncwarp();
    };
    if (G > 0) issue_s(0);
    if (G > 1) issue_s(1);
    for (int g = 0; g < G; ++g) {
      const int uc = g / n, i = g % n;
      mbar_wait(&s.p_full[g & 1], (g >> 1) & 1);
      if (i == 0 && uc > 0) mbar_wait(&s.o_empty, (uc - 1) & 1);  // previous unit's O read
      tc_fence_after();
      const int slot = take();
      if (leader) {  // O += P_g V_g
        const uint32_t vb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          mma_f16_ts(tmem + kO, tmem + kS + (g & 1) * BN + ks * 8,
                     sdesc_mnmajor_sw128(vb + ks * 2048, BN * 128), id_o, i > 0 || ks > 0);
        mma_commit(&s.pv_bar);
        mma_commit(&s.kv_empty[slot]);
      }
      __syncwarp();
      if (g + 2 < G) issue_s(g + 2);
    }
  } else {
    // ------------------------------- softmax / correction / epilogue --------
    const int q = warp & 3, h = warp >> 2;
    const int row = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const float c1 = p.scale_log2;
    // Q of unit uc -> TMEM Q buffer uc & 1: this thread's row, key-half h of
    // the D columns (D / 4 TMEM columns of bf16 pairs)
    auto write_q = [&](int uc) {
      if (uc >= nunits) return;
      int bh;
      int64_t q_row0, slice;
      unit_of(uc, bh, q_row0, slice);
      const uint4* src = reinterpret_cast<const uint4*>(p.q + (bh * p.sq + q_row0 + row) * D + h * (D / 2));
      const uint32_t dst = tmem + lane_off + kQ + (uc & 1) * (D / 2) + h * (D / 4);
      if constexpr (D == 128) {
        uint32_t r[32];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint4 w = __ldg(src + v);
          r[4 * v] = w.x; r[4 * v + 1] = w.y; r[4 * v + 2] = w.z; r[4 * v + 3] = w.w;
        }
        tmem_st32(dst, r);
      } else {
        uint32_t r[16];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint4 w = __ldg(src + v);
          r[4 * v] = w.x; r[4 * v + 1] = w.y; r[4 * v + 2] = w.z; r[4 * v + 3] = w.w;
        }
        tmem_st16(dst, r);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.q_full[uc & 1]);
    };
    write_q(0);
    write_q(1);
    for (int uc = 0; uc < nunits; ++uc) {
      if (uc > 0) write_q(uc + 1);  // the buffer of unit uc - 1, whose S MMAs have all completed
      int bh;
      int64_t q_row0, slice;
      unit_of(uc, bh, q_row0, slice);
      float m_true = -INFINITY;  // d1: exact running max
      float m_ref = -INFINITY;   // reference max of the accumulators
      float l = 0.f;             // this half's d2 relative to m_ref
      for (int i = 0; i < n; ++i) {
        const int g = uc * n + i;
        const uint32_t tS = tmem + lane_off + kS + (g & 1) * BN;
        mbar_wait(&s.s_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sr[2][32];
        tmem_ld32(tS + 64 * h, sr[0]);
        tmem_ld32(tS + 64 * h + 32, sr[1]);
        tmem_ld_wait();
        // reduction 1: row max over this half's 64 keys, then the other half's
        float mx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) mx[j] = __uint_as_float(sr[0][j]);
#pragma unroll
        for (int j = 8; j < 64; ++j) mx[j & 7] = fmaxf(mx[j & 7], __uint_as_float(sr[j >> 5][j & 31]));
        const float pmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                 fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        s.xmax[g & 1][h][row] = pmax;
        named_bar_sync(2 + q, 64);  // both halves have read S_g and published their max
        const float tmax = fmaxf(pmax, s.xmax[g & 1][h ^ 1][row]);
        m_true = fmaxf(m_true, tmax * p.scale);
        // correction exp(d1' - d1): lazily re-base the accumulators (same
        // decision in both halves: the same max)
        const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
        float alpha = 1.f;
        if (need) {
          alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
          l *= alpha;
          m_ref = m_true;
        }
        // reductions 2 and 3: P = exp(S - d1) in bf16 into TMEM (keys [64h,
        // 64h + 64) -> columns [32h, 32h + 32) of the S buffer), row sum in fp32
        const uint64_t c12 = f2(c1, c1), nmb2 = f2(-m_ref * kLog2e, -m_ref * kLog2e);
        uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const uint64_t x2 = ffma2(f2(__uint_as_float(sr[c][2 * jj]), __uint_as_float(sr[c][2 * jj + 1])),
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
          tmem_st16(tS + 32 * h + 16 * c, pk);
        }
        const uint64_t s01 = fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3]));
        float rs0, rs1;
        f2split(s01, rs0, rs1);
        l += rs0 + rs1;
        // O *= exp(d1' - d1) once P V_{g-1} has retired (this half's D / 2 columns)
        if (i > 0 && __any_sync(0xffffffffu, need)) {
          mbar_wait(&s.pv_bar, (g - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            uint32_t r[32];
            const uint32_t ta = tmem + lane_off + kO + h * (D / 2) + c * 32;
            tmem_ld32(ta, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st32(ta, r);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.p_full[g & 1]);
      }
      // ---- finalize (finalize_root): d2 re-based to the true d1, d3 = O / d2 ----
      s.xl[h][row] = l;
      named_bar_sync(2 + q, 64);
      const float lsum = l + s.xl[h ^ 1][row];  // both halves relative to the same m_ref
      const float l_true = lsum * ex2_mufu((m_ref - m_true) * kLog2e);
      const int64_t grow = static_cast<int64_t>(bh) * p.sq + q_row0 + row;
      const int64_t ps = slice - p.part_base;
      if (h == 0) {
        if (p.part_m == nullptr) {
          p.m[grow] = m_true;
          p.l[grow] = l_true;
        } else {
          p.part_m[ps * p.rows_total + grow] = m_true;
          p.part_l[ps * p.rows_total + grow] = l_true;
        }
      }
      // the unit's last P V. S_{g_last} complete implies P V_{g_last - 2} is:
      // the barrier may still be one phase short of P V_{g_last - 1}, so wait
      // that phase first (a parity wait must never be two phases ahead)
      const int g_last = uc * n + n - 1;
      if (g_last > 0) mbar_wait(&s.pv_bar, (g_last - 1) & 1);
      mbar_wait(&s.pv_bar, g_last & 1);
      tc_fence_after();
      const float inv_l = 1.f / lsum;
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + kO + h * (D / 2) + c * 32, r);
        tmem_ld_wait();
        if (c + 1 == D / 64) {  // this half of O read: the next unit's P V may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.o_empty);
        }
        const int col = h * (D / 2) + c * 32;
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WMMA) tmem_dealloc<512>(tmem);
}

template <int D>
cudaError_t launch_qt(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tk, tv;
  const uint64_t kdims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(a.bh * a.skv)};
  const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
  const uint32_t box[2] = {64, 128};
  if (!make_tmap(&tk, a.k, 2, kdims, strides, box, 2) || !make_tmap(&tv, a.v, 2, kdims, strides, box, 2))
    return cudaErrorInvalidValue;
  Params p{};
  p.sq = a.sq;
  p.skv = a.skv;
  p.slice_len = a.skv / a.segments;
  p.slice_begin = a.slice_begin;
  p.part_base = a.part_base;
  p.rows_total = a.rows_total;
  p.scale = a.scale;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.q = static_cast<const __nv_bfloat16*>(a.q);
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  p.units_x = static_cast<int>(a.sq / BM);
  p.units_bh = static_cast<int>(a.bh);
  p.units = p.units_x * p.units_bh * static_cast<int>(a.nslices);
  const size_t smem = sizeof(Smem<D>) + 1024;
  auto kern = attn_qt_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dim3 grid(static_cast<unsigned>(p.units < sms ? p.units : sms));  // persistent: one CTA per SM
  kern<<<grid, NTHREADS, smem, st>>>(tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

bool attention_qt_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments) {
  if (d != 64 && d != 128) return false;
  if (sq % BM != 0) return false;
  if (segments < 1 || skv % segments != 0) return false;
  return (skv / segments) % BN == 0;
}

cudaError_t launch_attention_qt(const AttnArgs& a, cudaStream_t st) {
  if (a.dtype != RF_BF16 || !attention_qt_supports(a.sq, a.skv, a.d, a.segments))
    return cudaErrorNotSupported;
  return a.d == 128 ? launch_qt<128>(a, st) : launch_qt<64>(a, st);
}

}  // namespace rf
