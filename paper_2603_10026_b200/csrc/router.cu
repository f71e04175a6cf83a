// MoE router: the expert-score GEMM s = X W (X [s, hd],
// W [hd, en]) followed by the routing cascade of make_moe_routing
// (proj/src/workloads.cpp:124-169): d1 = max s, d2 = sum exp(s - d1),
// d3 = top-K' of s (value, 1-based index), ties to the LOWEST index.
//
// The reference keeps the producer GEMM outside the cascade (its IR treats
// it as a producer, proj/src/scalar_ir.cpp:483-491); here it feeds the
// cascade without a round trip of the logits through HBM:
//
//  router_gemm_kernel  tcgen05 split-K GEMM. grid = (rows/128, splits); CTA
//      (m, k) computes the fp32 partial scores of 128 tokens x en experts over
//      its K range: TMA (SWIZZLE_128B) stages X [128 x 64] and the packed
//      W^T [en x 64] tiles into a ring of up to 8 slots (192 KB), one elected thread issues
//      kind::f16 MMAs (M = 128, N = en) into TMEM, 4 epilogue warps move the
//      accumulator TMEM -> registers -> smem. The CTAs of up to 4
//      consecutive splits form a thread-block cluster and fold their staged
//      partials through distributed shared memory (split order), so only
//      splits/4 partials [groups, rows, en] go to L2 (coalesced rows).
//      Split-K puts every
//      SM on the HBM stream of X at the paper's shapes (s = 2048 -> 16 row
//      tiles only).
//  router_route_kernel warp per token (programmatic dependent launch): each
//      lane sums the split partials of its experts in split order (a fixed
//      order, so scores are deterministic), then runs the warp routing
//      cascade of routing.cuh (K' rounds of a total-order warp argmax). The
//      scores s may also be written out (the cascade's input, for parity).
//
// Bound: HBM (X is read once: 2 * s * hd bytes; the GEMM is 2 * en FLOP/B).
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
__device__ unsigned long long g_route_trace[1024][3];
extern "C" int rf_router_trace_read(unsigned long long* gemm, unsigned long long* route) {
  cudaError_t e = cudaMemcpyFromSymbol(gemm, g_router_trace, sizeof(g_router_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(route, g_route_trace, sizeof(g_route_trace));
  return static_cast<int>(e);
}
#define RR_STAMP(i) do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_route_trace[blockIdx.x][(i)] = gtime(); } while (0)
#else
#define RT_STAMP(i) do {} while (0)
#define RR_STAMP(i) do {} while (0)
#endif

namespace rf {
namespace {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;  // bf16: one 128 B swizzle row
constexpr int NT = 192;  // warps 0-3 epilogue, 4 TMA, 5 MMA

// CTAs of consecutive splits that pre-reduce their partials through DSMEM
// (a thread-block cluster along the split axis).
__host__ __device__ constexpr int router_cluster_size(int64_t splits) {
  return splits % 4 == 0 ? 4 : splits % 2 == 0 ? 2 : 1;
}

__device__ __forceinline__ float4 ld_shared_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

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

template <int EN>
__global__ void __launch_bounds__(NT, 1)
    router_gemm_kernel(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tw,
                       float* __restrict__ part, int64_t rows, int64_t part_stride,
                       int k_tiles_per_split, int cs) {
  constexpr int STAGES = Smem<EN>::STAGES;
  constexpr int kCols = EN < 32 ? 32 : EN;  // TMEM allocation: power of two >= 32
  extern __shared__ uint8_t smem_raw[];
  Smem<EN>& s = *reinterpret_cast<Smem<EN>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = warp_id();
  const int m0 = blockIdx.x * BM;
  const int split = blockIdx.y;
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
  if (threadIdx.x == 0) RT_STAMP(1);

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
  } else {
    // ---- epilogue: partial scores of this split. TMEM -> registers (thread
    // = token) -> the drained smem ring (row stride EN + 4 floats: 16 B
    // accesses at the 4-wavefront minimum) -> coalesced rows (a warp writes
    // one token's EN scores per instruction). ----
    const int r = threadIdx.x;  // 0..127 (TMEM lane = row)
    mbar_wait(&s.acc_full, 0);
    tc_fence_after();
    if (threadIdx.x == 0) RT_STAMP(4);
    constexpr int RS = EN + 4;
    float* stage = reinterpret_cast<float*>(s.a[0]);
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
  // ---- split pre-reduction inside the cluster (the cs CTAs of consecutive
  // splits of this row tile): CTA rank q folds rows [q*128/cs, (q+1)*128/cs)
  // of all cs staged partials in rank (= split) order through distributed
  // shared memory and writes one partial per cluster, coalesced. ----
  if (threadIdx.x == 0) RT_STAMP(6);
  cluster_sync();  // every CTA's staged partial is visible cluster-wide
  if (threadIdx.x == 0) RT_STAMP(7);
  if (warp < 4) {
    constexpr int RS = EN + 4;
    const uint32_t stage_u32 = smem_u32(s.a[0]);
    const int q = static_cast<int>(cluster_ctarank());
    const int rows_per = BM / cs;
    const int lane = threadIdx.x & 31;
    float* dst0 = part + static_cast<int64_t>(split / cs) * part_stride * EN;
    for (int i = warp; i < rows_per; i += 4) {
      const int rr = q * rows_per + i;
      const int64_t row = m0 + rr;
      if (row >= rows) break;
#pragma unroll
      for (int c4 = lane; c4 < EN / 4; c4 += 32) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t off = stage_u32 + static_cast<uint32_t>((rr * RS + 4 * c4) * 4);
        float4 v[4];
#pragma unroll
        for (int src = 0; src < 4; ++src)
          if (src < cs) v[src] = ld_shared_cluster_f4(mapa_shared(off, src));
#pragma unroll
        for (int src = 0; src < 4; ++src) {
          if (src < cs) {
            acc.x += v[src].x;
            acc.y += v[src].y;
            acc.z += v[src].z;
            acc.w += v[src].w;
          }
        }
        reinterpret_cast<float4*>(dst0 + row * EN)[c4] = acc;
      }
    }
  }
  cluster_sync();  // peers' staged partials stay alive until every fold is done
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) RT_STAMP(5);
  // the routing kernel (programmatic dependent) may be scheduled now
  asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 5) tmem_dealloc<kCols>(tmem);
}

// ---------------------------------------------------------------- routing --

template <int K, int EN>
__global__ void __launch_bounds__(256) router_route_kernel(const float* __restrict__ part, int splits,
                                                           int64_t rows, int64_t part_stride, float* __restrict__ d1,
                                                           float* __restrict__ d2, int2* __restrict__ topk,
                                                           float* __restrict__ scores) {
  RR_STAMP(0);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  RR_STAMP(1);
  constexpr int PER = EN / 32;  // experts per lane: e = lane + 32 j
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;
  float x[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) x[j] = 0.f;
#pragma unroll 8
  for (int sp = 0; sp < splits; ++sp) {  // split order: deterministic scores
    const float* pr = part + (static_cast<int64_t>(sp) * part_stride + row) * EN;
#pragma unroll
    for (int j = 0; j < PER; ++j) x[j] += __ldcg(pr + lane + 32 * j);
  }
  if (scores != nullptr) {
#pragma unroll
    for (int j = 0; j < PER; ++j) scores[row * EN + lane + 32 * j] = x[j];
  }
  warp_route<PER, K>(x, EN, lane, d1 + row, d2 + row, topk + row * K);
  RR_STAMP(2);
}

template <int EN>
cudaError_t launch_gemm(const RouterArgs& a, cudaStream_t st) {
  if (a.splits % router_cluster_size(a.splits) != 0) return cudaErrorInvalidValue;
  CUtensorMap tx, tw;
  const uint64_t xdims[2] = {static_cast<uint64_t>(a.hd), static_cast<uint64_t>(a.rows)};
  const uint64_t wdims[2] = {static_cast<uint64_t>(a.hd), static_cast<uint64_t>(EN)};
  const uint64_t strides[1] = {static_cast<uint64_t>(a.hd) * 2};
  const uint32_t xbox[2] = {BK, BM}, wbox[2] = {BK, static_cast<uint32_t>(EN)};
  if (!make_tmap(&tx, a.x, 2, xdims, strides, xbox, 2) || !make_tmap(&tw, a.w, 2, wdims, strides, wbox, 2))
    return cudaErrorInvalidValue;
  auto kern = router_gemm_kernel<EN>;
  const size_t smem = sizeof(Smem<EN>) + 1024;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int cs = router_cluster_size(a.splits);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((a.rows + BM - 1) / BM), static_cast<unsigned>(a.splits));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = static_cast<unsigned>(cs);
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tx, tw, a.part, a.rows, a.part_stride,
                            static_cast<int>(a.hd / BK / a.splits), cs);
}

template <int EN>
cudaError_t launch_route(const RouterArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((a.rows + 7) / 8));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int2* out = static_cast<int2*>(a.topk);
  const int sp = static_cast<int>(a.splits / router_cluster_size(a.splits));  // partials after the cluster fold
  switch (a.k) {
#define RF_ROUTE_CASE(K) \
  case K: return cudaLaunchKernelEx(&cfg, router_route_kernel<K, EN>, a.part, sp, a.rows, a.part_stride, a.d1, a.d2, out, a.scores);
    RF_ROUTE_CASE(1)
    RF_ROUTE_CASE(2)
    RF_ROUTE_CASE(3)
    RF_ROUTE_CASE(4)
    RF_ROUTE_CASE(5)
    RF_ROUTE_CASE(6)
    RF_ROUTE_CASE(7)
    RF_ROUTE_CASE(8)
#undef RF_ROUTE_CASE
    default: return cudaErrorNotSupported;
  }
}

template <int EN>
cudaError_t launch_en(const RouterArgs& a, cudaStream_t st) {
  cudaError_t e = launch_gemm<EN>(a, st);
  if (e != cudaSuccess) return e;
  return launch_route<EN>(a, st);
}

}  // namespace

bool router_supports(int64_t rows, int64_t hd, int64_t experts, int64_t k) {
  (void)rows;
  return (experts == 32 || experts == 64 || experts == 128 || experts == 256) && hd % BK == 0 &&
         hd >= BK && k >= 1 && k <= 8 && k <= experts;
}

// Splits of the K axis: the fewest that give one full wave of CTAs (<= 148,
// one CTA per SM with a deep TMA ring), each with >= 8 K tiles; must divide
// hd / BK. Fewer splits = fewer partial scores through L2.
int64_t router_pick_splits(int64_t rows, int64_t hd) {
  const int64_t mt = (rows + BM - 1) / BM, kt = hd / BK;
  int64_t best = 1;
  for (int64_t s = 1; s <= kt; ++s) {
    if (kt % s != 0 || kt / s < 8 || mt * s > 148) continue;
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
