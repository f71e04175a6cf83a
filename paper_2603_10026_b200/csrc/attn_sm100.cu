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
//   * the d3 correction exp(d1' - d1) applied tile by tile to the TMEM
//     accumulator by a dedicated correction warpgroup; the d2'/d2 factor of
//     the derived correction exp(d1'-d1)*d2'/d2 telescopes over the loop to
//     1/d2(final) and is applied once at finalize (finalize_root,
//     simulator.cpp:611-621, retargets the root's scaling the same way).
//
// CTA = 2 Q tiles x 128 rows (ping-pong), KV tiles of 128 keys.
// Warp roles (512 threads):
//   warps 0-3  softmax for Q tile 0 (thread = row)
//   warps 4-7  softmax for Q tile 1
//   warps 8-11 correction (O *= alpha in TMEM) + epilogue (O / l -> global)
//   warp 12    TMA producer          warp 13  MMA issuer (one elected lane)
//   warp 14    TMEM allocator        warp 15  idle
// TMEM (512 cols): S0 [0,128)  S1 [128,256)  O0 [256,256+D)  O1 [384,384+D)
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;       // rows per Q tile
constexpr int BN = 128;       // keys per KV tile
constexpr int NSLOT = 4;      // K/V ring slots
constexpr int NTHREADS = 512;

template <int D>
struct Smem {
  static constexpr int kTile = BM * D * 2;  // one bf16 [128 x D] tile
  static constexpr int kChunks = D / 64;    // 128 B swizzle chunks along D
  uint8_t q[2][kTile];
  uint8_t kv[NSLOT][kTile];
  uint64_t bar_q;
  uint64_t kv_full[NSLOT], kv_empty[NSLOT];
  uint64_t s_full[2], p_full[2], sc_full[2], o_ready[2], pv_done[2], l_ready[2];
  float alpha[2][BM];
  float lfin[2][BM];
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
};

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_sm100_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem<D>& s = *reinterpret_cast<Smem<D>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int bh = blockIdx.y;
  const int64_t q_row0 = static_cast<int64_t>(blockIdx.x) * 2 * BM;  // within (b,h)
  const int64_t slice = p.slice_begin + blockIdx.z;
  const int64_t kv0 = slice * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / BN);

  if (threadIdx.x == 0) {
    mbar_init(&s.bar_q, 1);
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&s.kv_full[i], 1);
      mbar_init(&s.kv_empty[i], 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s.s_full[k], 1);
      mbar_init(&s.p_full[k], BM);
      mbar_init(&s.sc_full[k], BM);
      mbar_init(&s.o_ready[k], BM);
      mbar_init(&s.pv_done[k], 1);
      mbar_init(&s.l_ready[k], BM);
    }
    fence_barrier_init();
  }
  if (warp == 14) tmem_alloc<512>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + 128};
  const uint32_t tO[2] = {tmem + 256, tmem + 384};

  if (warp == 12) {
    // ------------------------------------------------------------ TMA ----
    if (elect_one()) {
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      prefetch_tmap(&tv);
      const int32_t qy = static_cast<int32_t>(bh * p.sq + q_row0);
      mbar_arrive_expect_tx(&s.bar_q, 2 * Smem<D>::kTile);
      for (int k = 0; k < 2; ++k)
        for (int c = 0; c < Smem<D>::kChunks; ++c)
          tma_load_2d(s.q[k] + c * BM * 128, &tq, &s.bar_q, c * 64, qy + k * BM, kEvictFirst);
      const int32_t ky = static_cast<int32_t>(bh * p.skv + kv0);
      for (int t = 0; t < 2 * n_tiles; ++t) {
        const int slot = t % NSLOT;
        const uint32_t ph = (t / NSLOT) & 1;
        mbar_wait(&s.kv_empty[slot], ph ^ 1);
        mbar_arrive_expect_tx(&s.kv_full[slot], Smem<D>::kTile);
        const CUtensorMap* m = (t & 1) ? &tv : &tk;
        const int32_t y = ky + (t >> 1) * BN;
        for (int c = 0; c < Smem<D>::kChunks; ++c)
          tma_load_2d(s.kv[slot] + c * BN * 128, m, &s.kv_full[slot], c * 64, y, kEvictLast);
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------ MMA ----
    const uint32_t id_s = idesc_f16(BM, BN, kFmtBF16, false, false);
    const uint32_t id_o = idesc_f16(BM, D, kFmtBF16, false, true);
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
    auto issue_pv = [&](int k, int slot, bool acc) {  // O_k += P_k V
      if (leader) {
        const uint32_t vb = smem_u32(s.kv[slot]);
#pragma unroll
        for (int ks = 0; ks < BN / 16; ++ks)
          mma_f16_ts(tO[k], tS[k] + ks * 8, sdesc_mnmajor_sw128(vb + ks * 2048, BN * 128), id_o,
                     acc || ks > 0);
        mma_commit(&s.pv_done[k]);
      }
      __syncwarp();
    };
    auto release = [&](int slot) {
      if (leader) mma_commit(&s.kv_empty[slot]);
      __syncwarp();
    };
    mbar_wait(&s.bar_q, 0);
    // prologue: S0_0, S1_0 on K_0 (ring index 0)
    mbar_wait(&s.kv_full[0], 0);
    tc_fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    release(0);
    for (int i = 0; i < n_tiles; ++i) {
      const int tV = 2 * i + 1, tK = 2 * i + 2;
      const int sV = tV % NSLOT, sK = tK % NSLOT;
      const uint32_t phV = (tV / NSLOT) & 1, phK = (tK / NSLOT) & 1;
      const uint32_t ph = i & 1;
      mbar_wait(&s.kv_full[sV], phV);
      // tile 0: PV0_i then S0_{i+1}
      mbar_wait(&s.p_full[0], ph);
      mbar_wait(&s.o_ready[0], ph);
      tc_fence_after();
      issue_pv(0, sV, i > 0);
      if (i + 1 < n_tiles) {
        mbar_wait(&s.kv_full[sK], phK);
        tc_fence_after();
        issue_s(0, sK);
      }
      // tile 1: PV1_i then S1_{i+1}
      mbar_wait(&s.p_full[1], ph);
      mbar_wait(&s.o_ready[1], ph);
      tc_fence_after();
      issue_pv(1, sV, i > 0);
      release(sV);
      if (i + 1 < n_tiles) {
        issue_s(1, sK);
        release(sK);
      }
    }
  } else if (warp < 8) {
    // -------------------------------------------------------- softmax ----
    const int k = warp >> 2;         // Q tile
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tSk = tS[k] + lane_off;
    const float c1 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int i = 0; i < n_tiles; ++i) {
      mbar_wait(&s.s_full[k], i & 1);
      tc_fence_after();
      // pass 1: reduction 1 (max) over the row of S
      float tmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tSk + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) tmax = fmaxf(tmax, __uint_as_float(r[j]));
      }
      const float m_new = fmaxf(m, tmax * p.scale);
      const float alpha = (i == 0) ? 1.f : exp2f((m - m_new) * 1.4426950408889634f);
      s.alpha[k][row] = alpha;
      mbar_arrive(&s.sc_full[k]);
      // pass 2: reduction 2 (sum exp, corrected by alpha) + P for reduction 3
      const float mb = m_new * 1.4426950408889634f;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tSk + c * 32, r);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float p0 = exp2f(fmaf(__uint_as_float(r[2 * j]), c1, -mb));
          const float p1 = exp2f(fmaf(__uint_as_float(r[2 * j + 1]), c1, -mb));
          rs += p0 + p1;
          pk[j] = pack_bf16x2(p0, p1);
        }
        tmem_st16(tSk + c * 16, pk);
      }
      l = l * alpha + rs;
      m = m_new;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&s.p_full[k]);
    }
    // finalize: publish l for the epilogue, write d1 / d2
    s.lfin[k][row] = l;
    mbar_arrive(&s.l_ready[k]);
    const int64_t grow = static_cast<int64_t>(bh) * p.sq + q_row0 + k * BM + row;
    if (p.part_m == nullptr) {
      p.m[grow] = m;
      p.l[grow] = l;
    } else {
      const int64_t ps = slice - p.part_base;
      p.part_m[ps * p.rows_total + grow] = m;
      p.part_l[ps * p.rows_total + grow] = l;
    }
  } else if (warp < 12) {
    // ----------------------------------------------------- correction ----
    const int row = threadIdx.x & 127;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    for (int i = 0; i < n_tiles; ++i) {
      for (int k = 0; k < 2; ++k) {
        mbar_wait(&s.sc_full[k], i & 1);
        if (i > 0) {
          const float a = s.alpha[k][row];
          mbar_wait(&s.pv_done[k], (i - 1) & 1);
          tc_fence_after();
          // exp(d1' - d1) == 1 exactly for every row of this warp: skip (bit-identical)
          if (__any_sync(0xffffffffu, a != 1.f)) {
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t r[32];
              const uint32_t addr = tO[k] + lane_off + c * 32;
              tmem_ld32(addr, r);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * a);
              tmem_st32(addr, r);
            }
            tmem_st_wait();
          }
          tc_fence_before();
        }
        mbar_arrive(&s.o_ready[k]);
      }
    }
    // epilogue: O / d2 -> global
    for (int k = 0; k < 2; ++k) {
      mbar_wait(&s.pv_done[k], (n_tiles - 1) & 1);
      mbar_wait(&s.l_ready[k], 0);
      tc_fence_after();
      const float inv_l = 1.f / s.lfin[k][row];
      const int64_t grow = static_cast<int64_t>(bh) * p.sq + q_row0 + k * BM + row;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO[k] + lane_off + c * 32, r);
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
          const int64_t ps = slice - p.part_base;
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
  if (warp == 14) tmem_dealloc<512>(tmem);
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
  const size_t smem = sizeof(Smem<D>) + 1024;
  auto kern = attn_sm100_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(a.sq / (2 * BM)), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
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
