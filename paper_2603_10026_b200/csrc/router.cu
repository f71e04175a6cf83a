// MoE router: the expert-score GEMM s = X W (X [s, hd],
// W [hd, en]) followed by the routing cascade of make_moe_routing
// (proj/src/workloads.cpp:124-169): d1 = max s, d2 = sum exp(s - d1),
// d3 = top-K' of s (value, 1-based index), ties to the LOWEST index.
//
// The reference keeps the producer GEMM outside the cascade (its IR treats
// it as a producer, proj/src/scalar_ir.cpp:483-491); here it feeds the
// cascade without a round trip of the logits through HBM, in ONE launch:
//
//  router_kernel  tcgen05 split-K GEMM + routing. grid = (rows/128, splits),
//      all CTAs co-resident (cooperative launch, <= 148 CTAs, one per SM).
//      CTA (m, q) computes the fp32 partial scores of 128 tokens x en experts
//      over its K range: TMA (SWIZZLE_128B) stages X [128 x 64] and the packed
//      W^T [en x 64] tiles into a ring of up to 8 slots (192 KB), one elected
//      thread issues kind::f16 MMAs (M = 128, N = en) into TMEM, 4 epilogue
//      warps move the accumulator TMEM -> registers -> smem. Token slice q of
//      the row tile (128/splits tokens) is then owned by CTA q: every CTA
//      writes the other slices of its partial to L2 (coalesced rows), the
//      splits CTAs of a row tile meet on a counter in global memory, and each
//      folds its own slice's partials in split order (deterministic scores,
//      its own partial straight from shared memory) and routes those tokens
//      with one warp per token (routing.cuh: K' rounds of a total-order warp
//      argmax). The scores s may also be written out (for parity).
//      Split-K puts every SM on the HBM stream of X at the paper's shapes
//      (s = 2048 -> 16 row tiles only); splits = 1 (large s) skips the exchange.
//
// Bound: HBM (X is read once: 2 * s * hd bytes; the GEMM is 2 * en FLOP/B).
// Round 1 ran a 4-CTA cluster DSMEM fold + a PDL route kernel (two launches,
// DESIGN.md section 3.4 trace); the L2 exchange replaces both.
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "routing.cuh"
#include "sm100.cuh"

#ifdef RF_ROUTER_TRACE
__device__ unsigned long long g_router_trace[8 * 1024];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define RT_STAMP(i) do { if (threadIdx.x % 32 == 0) g_router_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (i)] = gtime(); } while (0)
__device__ unsigned long long g_route_trace[1024][3];  // unused since the single-launch form (kept for the ABI)
extern "C" int rf_router_trace_read(unsigned long long* gemm, unsigned long long* route) {
  cudaError_t e = cudaMemcpyFromSymbol(gemm, g_router_trace, sizeof(g_router_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(route, g_route_trace, sizeof(g_route_trace));
  return static_cast<int>(e);
}
#else
#define RT_STAMP(i) do {} while (0)
#endif

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;   // bf16: one 128 B swizzle row
constexpr int NT = 512;  // warps 0-3 epilogue, 4 TMA, 5 MMA; all 16 route (one token per warp at 8 splits)
constexpr int NW = NT / 32;
constexpr int kMaxSplits = 16;  // router_pick_splits' cap (the routing warps hold one partial per split)

template <int EN>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;  // 16 KB
  static constexpr int B_BYTES = EN * BK * 2;  // 4 .. 32 KB
  static constexpr int STAGES = (192 * 1024) / (A_BYTES + B_BYTES) < 8 ? (192 * 1024) / (A_BYTES + B_BYTES) : 8;
  static_assert(STAGES * (A_BYTES + B_BYTES) >= BM * (EN + 4) * 4, "epilogue staging fits the ring");
  uint8_t a[STAGES][A_BYTES];
  uint8_t b[STAGES][B_BYTES];
  uint64_t full[STAGES], empty[STAGES];
  uint64_t acc_full;
  uint32_t tmem_base;
};

__device__ __forceinline__ unsigned long long atom_add_release_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int EN, int K>
__global__ void __launch_bounds__(NT, 1)
    router_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                  float* __restrict__ part, unsigned long long* __restrict__ cnt, int64_t rows,
                  int64_t part_stride, int k_tiles_per_split, float* __restrict__ d1, float* __restrict__ d2,
                  int2* __restrict__ topk, float* __restrict__ scores) {
  constexpr int STAGES = Smem<EN>::STAGES;
  constexpr int kCols = EN < 32 ? 32 : EN;  // TMEM allocation: power of two >= 32
  constexpr int RS = EN + 4;                // staging row stride (floats): 16 B accesses at the 4-wavefront minimum
  constexpr int PER = EN / 32;              // experts per lane in routing: e = lane + 32 j
  extern __shared__ uint8_t smem_raw[];
  Smem<EN>& s = *reinterpret_cast<Smem<EN>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int split = blockIdx.y;
  const int splits = gridDim.y;
  const int kt0 = split * k_tiles_per_split;
  const int kt = k_tiles_per_split;
  if (threadIdx.x == 0) RT_STAMP(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    mbar_init(&s.acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<kCols>(&s.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  float* stage = reinterpret_cast<float*>(s.a[0]);
  // Token slice q = [q * per, (q + 1) * per) of the row tile belongs to CTA q.
  const int per = (BM + splits - 1) / splits;
  const int r0 = split * per;
  const int r1 = r0 + per < BM ? r0 + per : BM;

  if (warp == 4) {
    if (elect_one()) {
      prefetch_tmap(&tx);
      prefetch_tmap(&tw);
      for (int t = 0; t < kt; ++t) {
        const int st = t % STAGES;
        mbar_wait(&s.empty[st], ((t / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[st], Smem<EN>::A_BYTES + Smem<EN>::B_BYTES);
        tma_load_2d(s.a[st], &tx, &s.full[st], (kt0 + t) * BK, m0, kEvictFirst);
        tma_load_2d(s.b[st], &tw, &s.full[st], (kt0 + t) * BK, 0, kEvictLast);
      }
    }
  } else if (warp == 5) {
    const uint32_t idesc = idesc_f16(BM, EN, kFmtBF16, false, false);
    const bool leader = elect_one();
    for (int t = 0; t < kt; ++t) {
      const int st = t % STAGES;
      mbar_wait(&s.full[st], (t / STAGES) & 1);
      tc_fence_after();
      if (t == 0) RT_STAMP(2);
      if (t + 1 == kt) RT_STAMP(3);
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
  } else if (warp < 4) {
    // ---- epilogue: partial scores of this split, TMEM -> registers (thread =
    // token) -> the drained smem ring. ----
    const int r = threadIdx.x;  // 0..127 (TMEM lane = row)
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    if (threadIdx.x == 0) RT_STAMP(4);
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
#pragma unroll
    for (int c = 0; c < EN / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stage + r * RS + c * 32 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                        __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();  // the partial is staged; TMEM is no longer read
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<kCols>(tmem);
  }
  if (splits > 1) {
    // ---- the other slices of this partial -> L2 (a warp writes one token's
    // EN scores per instruction; bulk copies per row measured slower), then
    // meet the row tile's other CTAs. ----
    for (int rr = warp; rr < BM; rr += NW) {
      const int64_t row = m0 + rr;
      if (row >= rows) break;
      if (rr >= r0 && rr < r1) continue;
      float* dst = part + (static_cast<int64_t>(split) * part_stride + row) * EN;
#pragma unroll
      for (int c4 = lane; c4 < EN / 4; c4 += 32)
        __stcg(reinterpret_cast<float4*>(dst) + c4, *reinterpret_cast<const float4*>(stage + rr * RS + 4 * c4));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      RT_STAMP(5);
      // The counter only grows: each launch adds `splits` per row tile, so the
      // generation this CTA belongs to is old / splits (all CTAs of a launch
      // arrive before the next launch on the stream starts). The release add
      // publishes the CTA's stores (ordered before it by the barrier above).
      const unsigned long long old = atom_add_release_u64(cnt + blockIdx.x, 1ull);
      const unsigned long long target = old - old % splits + splits;
      while (ld_acquire_u64(cnt + blockIdx.x) < target) {
      }
      RT_STAMP(6);
    }
    __syncthreads();
  }
  // ---- routing of this CTA's token slice: one warp per token, the split
  // partials summed in split order (deterministic), own partial from smem. ----
  for (int rr = r0 + warp; rr < r1; rr += NW) {
    const int64_t row = m0 + rr;
    if (row >= rows) break;
    // the partials are summed in split order, CH splits' loads in flight at a
    // time (one L2 round trip per CH splits; CH * PER = 32 registers)
    constexpr int CH = 32 / PER;
    float x[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) x[j] = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < kMaxSplits; c0 += CH) {
      if (c0 >= splits) break;
      float v[CH][PER];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int sp = c0 + i;
        if (sp < splits) {
          const float* pr = sp == split ? stage + rr * RS : part + (static_cast<int64_t>(sp) * part_stride + row) * EN;
#pragma unroll
          for (int j = 0; j < PER; ++j) v[i][j] = sp == split ? pr[lane + 32 * j] : __ldcg(pr + lane + 32 * j);
        }
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        if (c0 + i < splits) {
#pragma unroll
          for (int j = 0; j < PER; ++j) x[j] += v[i][j];
        }
      }
    }
    if (scores != nullptr) {
#pragma unroll
      for (int j = 0; j < PER; ++j) scores[row * EN + lane + 32 * j] = x[j];
    }
#ifdef RF_ROUTER_TRACE
#pragma unroll
    for (int j = 0; j < PER; ++j) asm volatile("" ::"f"(x[j]));  // the stamp waits for the sums
    if (threadIdx.x == 0) RT_STAMP(1);  // slot 1 = warp 0's partials summed
#endif
    warp_route<PER, K>(x, EN, lane, d1 + row, d2 + row, topk + row * K);
  }
  if (threadIdx.x == 0) RT_STAMP(7);
}

template <int EN, int K>
cudaError_t launch_k(const RouterArgs& a, cudaStream_t st) {
  CUtensorMap tx, tw;
  const uint64_t xdims[2] = {static_cast<uint64_t>(a.hd), static_cast<uint64_t>(a.rows)};
  const uint64_t wdims[2] = {static_cast<uint64_t>(a.hd), static_cast<uint64_t>(EN)};
  const uint64_t strides[1] = {static_cast<uint64_t>(a.hd) * 2};
  const uint32_t xbox[2] = {BK, BM}, wbox[2] = {BK, static_cast<uint32_t>(EN)};
  if (!make_tmap(&tx, a.x, 2, xdims, strides, xbox, 2) || !make_tmap(&tw, a.w, 2, wdims, strides, wbox, 2))
    return cudaErrorInvalidValue;
  auto kern = router_kernel<EN, K>;
  const size_t smem = sizeof(Smem<EN>) + 1024;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((a.rows + BM - 1) / BM), static_cast<unsigned>(a.splits));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the split CTAs of a row tile wait for each other
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.splits > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tx, tw, a.part, a.cnt, a.rows, a.part_stride,
                            static_cast<int>(a.hd / BK / a.splits), a.d1, a.d2, static_cast<int2*>(a.topk),
                            a.scores);
}

template <int EN>
cudaError_t launch_en(const RouterArgs& a, cudaStream_t st) {
  switch (a.k) {
    case 1: return launch_k<EN, 1>(a, st);
    case 2: return launch_k<EN, 2>(a, st);
    case 3: return launch_k<EN, 3>(a, st);
    case 4: return launch_k<EN, 4>(a, st);
    case 5: return launch_k<EN, 5>(a, st);
    case 6: return launch_k<EN, 6>(a, st);
    case 7: return launch_k<EN, 7>(a, st);
    case 8: return launch_k<EN, 8>(a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

bool router_supports(int64_t rows, int64_t hd, int64_t experts, int64_t k) {
  (void)rows;
  return (experts == 32 || experts == 64 || experts == 128 || experts == 256) && hd % BK == 0 &&
         hd >= BK && k >= 1 && k <= 8 && k <= experts;
}

// Splits of the K axis: the fewest that give one full wave of CTAs (<= 148,
// one CTA per SM with a deep TMA ring), each with >= 8 K tiles; must divide
// hd / BK; at most kMaxSplits. Fewer splits = fewer partial scores through L2.
int64_t router_pick_splits(int64_t rows, int64_t hd) {
  const int64_t mt = (rows + BM - 1) / BM, kt = hd / BK;
  int64_t best = 1;
  for (int64_t s = 1; s <= kt; ++s) {
    if (kt % s != 0 || kt / s < 8 || mt * s > 148 || s > kMaxSplits) continue;
    best = s;
  }
  return best;
}

cudaError_t launch_router(const RouterArgs& a, cudaStream_t st) {
  switch (a.experts) {
    case 32: return launch_en<32>(a, st);
    case 64: return launch_en<64>(a, st);
    case 128: return launch_en<128>(a, st);
    case 256: return launch_en<256>(a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace rf
