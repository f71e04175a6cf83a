// bf16 decode attention (one query per (b,h), long KV) — the Multi-Segment
// strategy of the reference (run_multisegment, proj/src/simulator.cpp:660-687;
// FlashDecoding = tests/golden/flash_decoding_{scalar,tile}.txt) as an
// HBM-streaming kernel.
//
// grid = (slices, B*H). Each CTA streams one KV slice of one (b,h) through a
// shared-memory ring filled by 1-D TMA bulk copies (cp.async.bulk: K and V
// rows of consecutive keys are contiguous, so a 64-key stage is two 16 KB
// copies), and every compute warp keeps its own streaming state (m, l, o)
// updated with the Eq.17 element rule (store-prev, correct by exp(d1'-d1),
// reduce). Warp states are then folded in warp order with the Eq.16 merge
// (incr_push_child, simulator.cpp:592-608) and the slice's (m, l, O/l) is
// written as a partial (or as the final d1/d2/d3 when there is one slice).
// Slices are merged in slice order by merge.cu.
//
// Bound: HBM. Algorithmic bytes per (b,h) row: 2 * Skv * D * 2 (K and V read
// once) + Q/O; tensor cores are irrelevant at 1 FLOP/byte.
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

constexpr int D = 128;
constexpr int TK = 64;                 // keys per stage
constexpr int NSTAGE = 3;
constexpr int NCW = 8;                 // compute warps
constexpr int NT = (NCW + 1) * 32;     // + producer warp
constexpr int KPW = TK / NCW;          // keys per warp per stage (8)
constexpr int TILE_BYTES = TK * D * 2; // 16 KB

struct Smem {
  uint8_t k[NSTAGE][TILE_BYTES];
  uint8_t v[NSTAGE][TILE_BYTES];
  uint64_t full[NSTAGE], empty[NSTAGE];
  float wm[NCW], wl[NCW];
  float wo[NCW][D];
};

struct Params {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
  int64_t skv, slice_len, slice_begin, part_base, rows_total;
  float scale;
};

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

__global__ void __launch_bounds__(NT, 2) attn_decode_kernel(const Params p) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = warp_id(), lane = lane_id();
  const int64_t bh = blockIdx.y;
  const int64_t slice = p.slice_begin + blockIdx.x;
  const int64_t kv0 = slice * p.slice_len;
  const int n_tiles = static_cast<int>(p.slice_len / TK);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------------------------------------------------- producer --
    if (elect_one()) {
      const __nv_bfloat16* kb = p.k + (bh * p.skv + kv0) * D;
      const __nv_bfloat16* vb = p.v + (bh * p.skv + kv0) * D;
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % NSTAGE;
        mbar_wait(&s.empty[st], ((t / NSTAGE) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[st], 2 * TILE_BYTES);
        bulk_load(s.k[st], kb + static_cast<int64_t>(t) * TK * D, TILE_BYTES, &s.full[st]);
        bulk_load(s.v[st], vb + static_cast<int64_t>(t) * TK * D, TILE_BYTES, &s.full[st]);
      }
    }
    return;  // no block-wide barrier after this point includes the producer
  }

  // ----------------------------------------------------------- compute ----
  // q: half-warp h handles key 2*step + h; lane (lane & 15) owns dims [8j, 8j+8).
  const int j = lane & 15, h = lane >> 4;
  float qf[8];
  {
    const uint4 qv = *reinterpret_cast<const uint4*>(p.q + bh * D + 8 * j);
    const uint32_t w[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      qf[2 * i] = bf_lo(w[i]);
      qf[2 * i + 1] = bf_hi(w[i]);
    }
  }
  const float c1 = p.scale * 1.4426950408889634f;
  float m = -INFINITY, l = 0.f;  // natural-unit running max, sum
  float o[4] = {0.f, 0.f, 0.f, 0.f};  // dims [4*lane, 4*lane+4)
  for (int t = 0; t < n_tiles; ++t) {
    const int st = t % NSTAGE;
    mbar_wait(&s.full[st], (t / NSTAGE) & 1);
    const uint8_t* kt = s.k[st] + warp * KPW * D * 2;
    const uint8_t* vt = s.v[st] + warp * KPW * D * 2;
    // scores of this warp's 8 keys
    float sc[KPW];
#pragma unroll
    for (int step = 0; step < KPW / 2; ++step) {
      const uint4 kv = *reinterpret_cast<const uint4*>(kt + (2 * step + h) * D * 2 + 16 * j);
      const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc = fmaf(qf[2 * i], bf_lo(w[i]), acc);
        acc = fmaf(qf[2 * i + 1], bf_hi(w[i]), acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 8);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      sc[2 * step] = __shfl_sync(0xffffffffu, acc, 0);
      sc[2 * step + 1] = __shfl_sync(0xffffffffu, acc, 16);
    }
    // Eq.17 over the 8 keys: reduction 1 (max), 2 and 3 corrected by exp(d1'-d1)
    float tmax = sc[0];
#pragma unroll
    for (int i = 1; i < KPW; ++i) tmax = fmaxf(tmax, sc[i]);
    const float m_new = fmaxf(m, tmax * p.scale);
    const float mb = m_new * 1.4426950408889634f;
    const float alpha = exp2f(fmaf(m, 1.4426950408889634f, -mb));  // 0 on the first tile
    float pk[KPW], ps = 0.f;
#pragma unroll
    for (int i = 0; i < KPW; ++i) {
      pk[i] = exp2f(fmaf(sc[i], c1, -mb));
      ps += pk[i];
    }
    l = l * alpha + ps;
    m = m_new;
#pragma unroll
    for (int d = 0; d < 4; ++d) o[d] *= alpha;
#pragma unroll
    for (int i = 0; i < KPW; ++i) {
      const uint2 vv = *reinterpret_cast<const uint2*>(vt + i * D * 2 + 8 * lane);
      o[0] = fmaf(pk[i], bf_lo(vv.x), o[0]);
      o[1] = fmaf(pk[i], bf_hi(vv.x), o[1]);
      o[2] = fmaf(pk[i], bf_lo(vv.y), o[2]);
      o[3] = fmaf(pk[i], bf_hi(vv.y), o[3]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.empty[st]);
  }
  // ---- Eq.16 fold of the warp states, warp order ----
  if (lane == 0) {
    s.wm[warp] = m;
    s.wl[warp] = l;
  }
  *reinterpret_cast<float4*>(&s.wo[warp][4 * lane]) = make_float4(o[0], o[1], o[2], o[3]);
  asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32));
  if (warp == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < NCW; ++w) M = fmaxf(M, s.wm[w]);
    float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int w = 0; w < NCW; ++w) {
      const float a = __expf(s.wm[w] - M);
      L += s.wl[w] * a;
      const float4 ow = *reinterpret_cast<const float4*>(&s.wo[w][4 * lane]);
      acc[0] = fmaf(ow.x, a, acc[0]);
      acc[1] = fmaf(ow.y, a, acc[1]);
      acc[2] = fmaf(ow.z, a, acc[2]);
      acc[3] = fmaf(ow.w, a, acc[3]);
    }
    const float inv = 1.f / L;
    if (p.part_m == nullptr) {
      uint2 w;
      w.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
      w.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
      *reinterpret_cast<uint2*>(p.o + bh * D + 4 * lane) = w;
      if (lane == 0) {
        p.m[bh] = M;
        p.l[bh] = L;
      }
    } else {
      const int64_t ps = slice - p.part_base;
      *reinterpret_cast<float4*>(p.part_o + (ps * p.rows_total + bh) * D + 4 * lane) =
          make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
      if (lane == 0) {
        p.part_m[ps * p.rows_total + bh] = M;
        p.part_l[ps * p.rows_total + bh] = L;
      }
    }
  }
}

}  // namespace

cudaError_t launch_attention_decode(const AttnArgs& a, cudaStream_t st) {
  const int64_t slice = a.skv / a.segments;
  if (a.dtype != RF_BF16 || a.d != D || a.sq != 1 || slice % TK != 0)
    return launch_attention_f32(a, st);  // generic SIMT CUDA path for odd decode shapes
  Params p{};
  p.q = static_cast<const __nv_bfloat16*>(a.q);
  p.k = static_cast<const __nv_bfloat16*>(a.k);
  p.v = static_cast<const __nv_bfloat16*>(a.v);
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  p.skv = a.skv;
  p.slice_len = slice;
  p.slice_begin = a.slice_begin;
  p.part_base = a.part_base;
  p.rows_total = a.rows_total;
  p.scale = a.scale;
  const size_t smem = sizeof(Smem) + 128;
  cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(a.nslices), static_cast<unsigned>(a.bh));
  attn_decode_kernel<<<grid, NT, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace rf
