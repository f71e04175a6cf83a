// bf16 safe-softmax -> GEMM attention on Blackwell tensor cores (sm_100a).
//
// The reference's fused loop for the attention cascade — incr_ingest_element
// (proj/src/simulator.cpp:566-589) over make_attention's reductions
// (proj/src/workloads.cpp:66-120), tiled as the reference's own tile plan
// (tests/golden/flash_attention_tile.txt: Q tile resident, K/V stage loop,
// reduce max -> corrected sum-exp -> corrected GEMM) — realised with:
//   * TMA (SWIZZLE_128B) K/V tiles into a 4-slot shared-memory ring,
//   * tcgen05.mma S = Q K^T and O += P V with fp32 accumulators in TMEM,
//     P (bf16) written back into TMEM over S and consumed as the A operand,
//   * the cascaded statistics (running max d1, rescaled sum-exp d2) in
//     registers, one thread per row,
//   * the d3 correction exp(d1' - d1) applied inside the loop to the TMEM
//     accumulator (see below); the d2'/d2 factor of the derived correction
//     exp(d1'-d1)*d2'/d2 telescopes over the loop to 1/d2(final) and is
//     applied once at finalize (finalize_root, simulator.cpp:611-621,
//     retargets the root's scaling the same way).
//
// CTA = 2 Q tiles x 128 rows (ping-pong), KV tiles of 128 keys; persistent
// (one CTA per SM walks the work units, see attn_sm100_kernel).
// Warp roles (320 threads, ~200 registers per thread):
//   warps 0-3  softmax + correction + epilogue for Q tile 0 (thread = row)
//   warps 4-7  the same for Q tile 1
//   warp 8     TMA producer          warp 9  MMA issuer (one elected lane) + TMEM owner
// TMEM (512 cols): S0 [0,128)  S1 [128,256)  O0 [256,256+D)  O1 [384,384+D);
// P_k (bf16 pairs) overwrites S_k cols [0,64) and is the A operand of P V.
//
// The correction O *= exp(d1' - d1) is applied by the softmax thread of the
// row itself: tcgen05.mma executes in issue order, so when S_k,i is complete
// PV_k,i-1 is too, and PV_k,i is only issued after the thread arrives on
// p_full. Rescaling is lazy: the accumulator keeps a reference max m_ref and
// is only re-based when the running max d1 exceeds it by more than 2^8 (the
// exponentials stay <= 256, far from overflow); O and d2 always share the same
// reference, so d3 = O / d2 is unchanged and d2 is re-based to the true d1 at
// finalize. d1 itself is the exact running max.
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

#ifdef RF_ATTN_TRACE
// Test-only timeline (tools/trace_attention.py): clock64 stamps of CTA (0,0,0).
__device__ long long g_attn_trace[4096];
#define RF_TRACE(idx) \
  do { if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0) g_attn_trace[(idx)] = clock64(); } while (0)
// effective SM clock of CTA 0 per launch: (clock64, globaltimer) at its start and end
__device__ long long g_attn_clk[64][4];
__device__ int g_attn_launch;
#define RF_CLK(slot)                                                                 \
  do {                                                                               \
    if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0 && threadIdx.x == 0) {            \
      long long g_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                         \
      const int l_ = g_attn_launch & 63;                                             \
      g_attn_clk[l_][2 * (slot)] = clock64();                                        \
      g_attn_clk[l_][2 * (slot) + 1] = g_;                                           \
      if ((slot) == 1) g_attn_launch = g_attn_launch + 1;                            \
    }                                                                                \
  } while (0)
#else
#define RF_CLK(slot) do {} while (0)
#define RF_TRACE(idx) do {} while (0)
#endif

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;       // rows per Q tile
constexpr int BN = 128;       // keys per KV tile
constexpr int NSLOT = 4;      // K/V ring slots (A/B on cfg2: 3 -> 1282, 4 -> 1323, 5 -> 1310 TFLOP/s)
constexpr int NTHREADS = 320;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// Pairs of exponentials evaluated by the FMA-pipe polynomial instead of MUFU.
__device__ __forceinline__ constexpr bool kPolyPairs(int jj) { return (jj & 3) == 3; }

template <int D>
struct Smem {
  static constexpr int kTile = BM * D * 2;  // one bf16 [128 x D] tile
  static constexpr int kChunks = D / 64;    // 128 B swizzle chunks along D
  uint8_t q[2][kTile];
  uint8_t kv[NSLOT][kTile];
  uint64_t q_full, q_empty;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2], pv_done[2], o_empty[2];
  uint32_t tmem_base;
};

struct Params {
  int64_t sq, skv, slice_len, slice_begin, part_base, rows_total;
  float scale_log2;  // softmax_scale * log2(e)
  float scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
  int units_x, units_bh, units;  // work units: (Q tile pair, b*h, slice)
};

// Persistent: one CTA per SM walks the work units u = blockIdx.x,
// blockIdx.x + gridDim.x, ... (unit = 2 Q tiles of one (b,h) and one KV
// slice). Barrier phases run on across units; the Q of unit u+1 is loaded as
// soon as the last S MMA of unit u has retired, and the epilogue of unit u
// (TMEM O -> global) overlaps the first S MMAs of unit u+1 (O_k is only
// overwritten by P V_k of the next unit after the epilogue released it).
template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem<D>& s = *reinterpret_cast<Smem<D>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  RF_CLK(0);
  const int warp = warp_id();
  const int n_tiles = static_cast<int>(p.slice_len / BN);
  auto unit_of = [&](int u, int& bh, int64_t& q_row0, int64_t& slice) {
    const int x = u % p.units_x;
    const int r = u / p.units_x;
    bh = r % p.units_bh;
    slice = p.slice_begin + r / p.units_bh;
    q_row0 = static_cast<int64_t>(x) * 2 * BM;
  };

  if (threadIdx.x == 0) {
    mbar_init(&s.q_full, 1);
    mbar_init(&s.q_empty, 1);
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s.s_full[k], 1);
      mbar_init(&s.p_full[k], 4);   // one arrival per softmax warp
      mbar_init(&s.pv_done[k], 1);
      mbar_init(&s.o_empty[k], 4);  // the tile's softmax warps have read O_k
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      int t = 0;  // K/V item counter across units
      int uc = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++uc) {
        int bh;
        int64_t q_row0, slice;
        unit_of(u, bh, q_row0, slice);
        mbar_wait(&s.q_empty, (uc & 1) ^ 1);
        const int32_t qy = static_cast<int32_t>(bh * p.sq + q_row0);
        mbar_arrive_expect_tx(&s.q_full, 2 * Smem<D>::kTile);
        for (int k = 0; k < 2; ++k)
          for (int c = 0; c < Smem<D>::kChunks; ++c)
            tma_load_2d(s.q[k] + c * BM * 128, &tq, &s.q_full, c * 64, qy + k * BM, kEvictFirst);
        const int32_t ky = static_cast<int32_t>(bh * p.skv + slice * p.slice_len);
        for (int j = 0; j < 2 * n_tiles; ++j, ++t) {
          const int slot = t % NSLOT;
          mbar_wait(&s.kv_empty[slot], ((t / NSLOT) & 1) ^ 1);
          RF_TRACE(1536 + (t & 511));
          mbar_arrive_expect_tx(&s.kv_full[slot], Smem<D>::kTile);
          const CUtensorMap* m = (j & 1) ? &tv : &tk;
          const int32_t y = ky + (j >> 1) * BN;
          for (int c = 0; c < Smem<D>::kChunks; ++c)
            tma_load_2d(s.kv[slot] + c * BN * 128, m, &s.kv_full[slot], c * 64, y, kEvictLast);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA ----
    const uint32_t id_s = idesc_f16(BM, BN, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(BM, D, kFmtBF16, false, true);
    const uint32_t tS[2] = {tmem + 0, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 384};
    const bool leader = elect_one();
    auto issue_s = [&](int k, int slot) {  // S_k = Q_k K^T
      if (leader) {
        const uint32_t qa = smem_u32(s.q[k]), kb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * (BM * 128) + (ks & 3) * 32;
          mma_f16_ss(tS[k], sdesc_kmajor_sw128(qa + off), sdesc_kmajor_sw128(kb + off), id_s,
                     ks > 0);
        }
        mma_commit(&s.s_full[k]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int k, int slot, bool acc, bool last) {  // O_k += P_k V
      if (leader) {
        const uint32_t vb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          mma_f16_ts(tO[k], tS[k] + ks * 8, sdesc_mnmajor_sw128(vb + ks * 2048, BN * 128), id_o,
                     acc || ks > 0);
        if (last) mma_commit(&s.pv_done[k]);
      }
      __syncwarp();
    };
    auto commit_to = [&](uint64_t* bar) {
      if (leader) mma_commit(bar);
      __syncwarp();
    };
    auto wait_kv = [&](int t) {
      mbar_wait(&s.kv_full[t % NSLOT], (t / NSLOT) & 1);
      tc_fence_after();
    };
    int t = 0;   // K/V item counter across units
    int g = 0;   // tile counter across units (s_full / p_full phases)
    int uc = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++uc) {
      mbar_wait(&s.q_full, uc & 1);
      wait_kv(t);
      tc_fence_after();
      if (leader && uc == 0) RF_TRACE(1024 + 0);
      issue_s(0, t % NSLOT);
      issue_s(1, t % NSLOT);
      if (n_tiles == 1) commit_to(&s.q_empty);  // last S of the unit
      commit_to(&s.kv_empty[t % NSLOT]);
      ++t;
      for (int i = 0; i < n_tiles; ++i, ++g) {
        const int tV = t, tK = t + 1;
        const uint32_t ph = g & 1;
        const bool last = i + 1 == n_tiles;
        wait_kv(tV);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          mbar_wait(&s.p_full[k], ph);
          if (i == 0 && uc > 0) mbar_wait(&s.o_empty[k], (uc - 1) & 1);  // previous unit's O_k read
          tc_fence_after();
          issue_pv(k, tV % NSLOT, i > 0, last);
          if (!last) {
            if (k == 0) wait_kv(tK);
            issue_s(k, tK % NSLOT);
            if (k == 1 && i + 2 == n_tiles) commit_to(&s.q_empty);  // last S of the unit
          }
        }
        commit_to(&s.kv_empty[tV % NSLOT]);
        if (!last) commit_to(&s.kv_empty[tK % NSLOT]);
        t += last ? 1 : 2;
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
    int g = 0;  // tile counter across units
    int uc = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++uc) {
      int bh;
      int64_t q_row0, slice;
      unit_of(u, bh, q_row0, slice);
      float m_true = -INFINITY;  // d1: exact running max
      float m_ref = -INFINITY;   // reference max of the accumulators
      float l = 0.f;             // d2 relative to m_ref
      for (int i = 0; i < n_tiles; ++i, ++g) {
        mbar_wait(&s.s_full[k], g & 1);
        tc_fence_after();
        if ((threadIdx.x & 127) == 0 && uc == 0) RF_TRACE(512 * k + 4 * i + 0);
        if (threadIdx.x == 0 && i == 0 && uc < 32) RF_TRACE(2048 + 2 * uc);  // unit start (softmax 0, S_0 ready)
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
        if ((threadIdx.x & 127) == 0 && uc == 0) RF_TRACE(512 * k + 4 * i + 3);
        m_true = fmaxf(m_true, tmax * p.scale);
        // correction exp(d1' - d1): lazily re-base the accumulators
        const bool need = (m_true - m_ref) * kLog2e > kRescaleThreshold;
        float alpha = 1.f;
        if (need) {
          alpha = ex2_mufu((m_ref - m_true) * kLog2e);  // 0 on the first tile
          l *= alpha;
          m_ref = m_true;
        }
        // pass 2 (reductions 2 and 3): S re-read from TMEM one 32-column chunk
        // at a time (chunk c + 1 in flight while c is exponentiated; P chunk c
        // lands in columns [16c, 16c + 16), never ahead of an unread S chunk).
        // P = exp(S - d1) in bf16 into TMEM, row sum in fp32; pairs packed
        // f32x2, one pair in four on the FMA pipe.
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
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tOk + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
            tmem_st32(tOk + c * 32, r);
          }
        }
        if ((threadIdx.x & 127) == 0 && uc == 0) RF_TRACE(512 * k + 4 * i + 1);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 127) == 0 && uc == 0) RF_TRACE(512 * k + 4 * i + 2);
        if (threadIdx.x == 0 && i + 1 == n_tiles && uc < 32) RF_TRACE(2048 + 2 * uc + 1);  // unit's last P released
        if ((threadIdx.x & 31) == 0) mbar_arrive(&s.p_full[k]);
      }
      // ---- finalize (finalize_root): d2 re-based to the true d1, d3 = O / d2 ----
      const float l_true = l * ex2_mufu((m_ref - m_true) * kLog2e);
      const int64_t grow = static_cast<int64_t>(bh) * p.sq + q_row0 + k * BM + row;
      const int64_t ps = slice - p.part_base;
      if (p.part_m == nullptr) {
        p.m[grow] = m_true;
        p.l[grow] = l_true;
      } else {
        p.part_m[ps * p.rows_total + grow] = m_true;
        p.part_l[ps * p.rows_total + grow] = l_true;
      }
      mbar_wait(&s.pv_done[k], uc & 1);
      tc_fence_after();
      const float inv_l = 1.f / l;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tOk + c * 32, r);
        tmem_ld_wait();
        if (c + 1 == D / 32) {  // O_k fully read: the next unit's P V_k may overwrite it
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(&s.o_empty[k]);
        }
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<512>(tmem);
  RF_CLK(1);
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tq, tk, tv;
  const uint64_t qdims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(a.bh * a.sq)};
  const uint64_t kdims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(a.bh * a.skv)};
  const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
  const uint32_t box[2] = {64, 128};
  if (!make_tmap(&tq, a.q, 2, qdims, strides, box, 2) ||
      !make_tmap(&tk, a.k, 2, kdims, strides, box, 2) ||
      !make_tmap(&tv, a.v, 2, kdims, strides, box, 2))
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
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  p.units_x = static_cast<int>(a.sq / (2 * BM));
  p.units_bh = static_cast<int>(a.bh);
  p.units = p.units_x * p.units_bh * static_cast<int>(a.nslices);
  const size_t smem = sizeof(Smem<D>) + 1024;
  auto kern = attn_sm100_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dim3 grid(static_cast<unsigned>(p.units < sms ? p.units : sms));  // persistent: one CTA per SM
  kern<<<grid, NTHREADS, smem, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

bool attention_sm100_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments) {
  if (d != 64 && d != 128) return false;
  if (sq % (2 * BM) != 0) return false;
  if (segments < 1 || skv % segments != 0) return false;
  return (skv / segments) % BN == 0;
}

cudaError_t launch_attention_sm100(const AttnArgs& a, cudaStream_t st) {
  if (a.dtype != RF_BF16 || !attention_sm100_supports(a.sq, a.skv, a.d, a.segments))
    return cudaErrorNotSupported;
  return a.d == 128 ? launch_d<128>(a, st) : launch_d<64>(a, st);
}

}  // namespace rf
