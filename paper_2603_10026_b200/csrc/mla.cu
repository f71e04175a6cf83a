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

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "rf_internal.h"
#include "sm100.cuh"

// Timeline hooks (tools/trace_mla.py, built with -DRF_MLA_TRACE): globaltimer
// stamps of the first and the last cluster of the grid.
#ifdef RF_MLA_TRACE
__device__ unsigned long long g_mla_trace[2][2][64][8];
#define MT_STAMP(t, i)                                                                              \
  do {                                                                                              \
    const int c_ = (blockIdx.y | blockIdx.z) == 0 ? 0                                               \
                   : (blockIdx.y == gridDim.y - 1 && blockIdx.z == gridDim.z - 1) ? 1 : -1;         \
    if (c_ >= 0 && (t) < 64) {                                                                      \
      unsigned long long v_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));                                       \
      g_mla_trace[c_][blockIdx.x][(t)][(i)] = v_;                                                   \
    }                                                                                               \
  } while (0)
__device__ unsigned long long g_fold_trace[1024][3];
__device__ unsigned long long g_cta_end[256];
extern "C" int rf_mla_trace_read(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_mla_trace, sizeof(g_mla_trace)));
}
extern "C" int rf_mla_end_trace_read(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_cta_end, sizeof(g_cta_end)));
}
extern "C" int rf_mla_fold_trace_read(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_fold_trace, sizeof(g_fold_trace)));
}
#define FT_STAMP(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0 && blockIdx.y * 2 + blockIdx.x < 1024) {                     \
      unsigned long long v_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));                         \
      g_fold_trace[blockIdx.y * 2 + blockIdx.x][(i)] = v_;                            \
    }                                                                                 \
  } while (0)
#else
#define MT_STAMP(t, i) do {} while (0)
#define FT_STAMP(i) do {} while (0)
#endif

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
#ifndef MLA_NKR
#define MLA_NKR 9
#define MLA_NVR 6
#endif
#ifndef MLA_NP
#define MLA_NP 2
#endif
constexpr int NKR = MLA_NKR;   // K ring slots (1.4 tiles of K in flight)
constexpr int NVR = MLA_NVR;   // V ring slots
constexpr int STB = 8192;      // stage bytes
constexpr int NT = 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct Smem {
  uint8_t q[NCH][HC * 128];  // 9 x 8 KB
  uint8_t kr[NKR][STB];      // K ring
  uint8_t vr[NVR][STB];      // V ring
  uint8_t p[MLA_NP][2][HC * 128]; // P buffers: keys [0, 64) and [64, 128), K-major SW128
  float xm[2][HN];           // row-half exchange (max per tile, then l)
  uint64_t q_full, kfull[NKR], kempty[NKR], vfull[NVR], vempty[NVR];
  uint64_t q_empty, s_full[2], p_full[2], pv_done[2], o_full, o_empty;
  uint32_t tmem_base;
  int nfold;                          // batch segments of this CTA folded at the end (<= 2)
  int fold_b[2], fold_slot[2], fold_nseg[2];
};

constexpr int kMaxClusters = 74;  // CTA pairs resident on a 148-SM B200

struct Params {
  int64_t skv, rows_total;
  int tpb;        // 128-key tiles per batch
  int clusters;   // CTA pairs (= gridDim.y)
  int nslots;     // partial slots per batch (1: direct output)
  float scale;
  __nv_bfloat16* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
  unsigned long long* cnt;  // [bs, 2] arrivals per batch half (multiples of kCntStride between launches)
  // Range of CTA pair k: flattened tiles [cut[k], cut[k + 1]) of the (batch,
  // tile) sequence, every range non-empty (host: balanced_cuts).
  int64_t cut[kMaxClusters + 1];
};

// Range scheduling: the flattened (batch, tile) sequence is cut into
// `clusters` contiguous ranges, one per CTA pair; a range covers one or more
// batch segments, each of which writes a partial (m, l, O/l) state to slot
// (cluster - first cluster of that batch). The cuts are chosen on the host
// (balanced_cuts) to minimise the largest range cost, where a range costs its
// tiles plus `seg` tiles for every batch it switches to after its first: a
// switch inside a range pays a Q reload (72 KB; no second Q buffer fits) and
// one more epilogue. (Round 1 charged every batch START a fixed number of
// virtual tiles in a uniform cost space, which also discounted ranges that
// merely began at a batch start: their CTAs ended up to ~7 us early on L3.)

// Pair holding flattened tile x: the last k with cut[k] <= x.
__host__ __device__ __forceinline__ int cluster_of_tile(const int64_t* cut, int clusters, int64_t x) {
  int lo = 0, hi = clusters - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cut[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

struct Segment {
  int b, t0, t1, slot, nseg;  // nseg: segments (ranges) the batch is cut into
};
__device__ __forceinline__ void segment_slots(const Params& p, int k, Segment& sg) {
  const int64_t b = sg.b;
  const int k0 = cluster_of_tile(p.cut, p.clusters, b * p.tpb);
  sg.slot = k - k0;
  sg.nseg = cluster_of_tile(p.cut, p.clusters, (b + 1) * p.tpb - 1) - k0 + 1;
}
// Segment `i` of pair k's range (batch and tiles; slot / nseg by
// segment_slots, which only the epilogue needs); false when exhausted.
__device__ __forceinline__ bool segment(const Params& p, int k, int i, Segment& sg) {
  const int64_t x1 = p.cut[k + 1];
  int64_t x = p.cut[k];
  for (int j = 0; x < x1; ++j) {
    const int64_t b = x / p.tpb;
    const int64_t hi = x1 < (b + 1) * p.tpb ? x1 : (b + 1) * p.tpb;
    if (j == i) {
      sg.b = static_cast<int>(b);
      sg.t0 = static_cast<int>(x - b * p.tpb);
      sg.t1 = static_cast<int>(hi - b * p.tpb);
      return true;
    }
    x = hi;
  }
  return false;
}

// Fold of a batch's segment partials (the Multi-Segment merge,
// incr_push_child / acceptance.cpp:162-178 closed form, as fold.cuh, in slot
// order), inside the decode kernel: every CTA whose range cut a batch arrives
// on the batch half's counter once its partial is written; after its last
// segment it waits for the other segments of that batch and folds its share
// of the half's 64 heads (share = its slot of ns). All CTAs are co-resident
// (cooperative launch, one CTA per SM), so the wait cannot starve a producer.
// Round 1 ran this as a second kernel (programmatic dependent launch): its
// launch gap and serial drain cost ~5 us of the 45 us L3 step.
// Warp = one head row; lane = 4 float4 columns 512 B apart; two slots'
// (m, l, O) loads per round trip.
constexpr unsigned long long kCntStride = 128;  // > any slot count (<= kMaxClusters)

__device__ __forceinline__ unsigned long long atom_add_acq_rel_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// NR head rows per warp at once (all their loads in flight together).
template <int NR>
__device__ __forceinline__ void fold_rows(const Params& p, const int64_t (&grow)[NR], int ns, int c0) {
  float m[NR], L[NR];
  float4 acc[NR][4];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    m[q] = -INFINITY;
    L[q] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[q][i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int e0 = 0; e0 < ns; e0 += 2) {
    float ms[NR][2], ls[NR][2];
    float4 o[NR][2][4];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e = e0 + j < ns ? e0 + j : ns - 1;  // (duplicates are dropped below)
        ms[q][j] = __ldcg(p.part_m + e * p.rows_total + grow[q]);
        ls[q][j] = __ldcg(p.part_l + e * p.rows_total + grow[q]);
        const float4* src = reinterpret_cast<const float4*>(p.part_o + (e * p.rows_total + grow[q]) * DV) + c0;
#pragma unroll
        for (int i = 0; i < 4; ++i) o[q][j][i] = __ldcg(src + 32 * i);
      }
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      float mr = m[q];
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (e0 + j < ns) mr = fmaxf(mr, ms[q][j]);
      if (mr != m[q] && L[q] != 0.f) {  // re-base what is accumulated
        const float f = __expf(m[q] - mr);
        L[q] *= f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[q][i].x *= f;
          acc[q][i].y *= f;
          acc[q][i].z *= f;
          acc[q][i].w *= f;
        }
      }
      m[q] = mr;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float w = e0 + j < ns && ls[q][j] != 0.f ? ls[q][j] * __expf(ms[q][j] - m[q]) : 0.f;
        if (w == 0.f) continue;
        L[q] += w;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[q][i].x = fmaf(o[q][j][i].x, w, acc[q][i].x);
          acc[q][i].y = fmaf(o[q][j][i].y, w, acc[q][i].y);
          acc[q][i].z = fmaf(o[q][j][i].z, w, acc[q][i].z);
          acc[q][i].w = fmaf(o[q][j][i].w, w, acc[q][i].w);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const float inv = 1.f / L[q];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint2 v;
      v.x = pack_bf16x2(acc[q][i].x * inv, acc[q][i].y * inv);
      v.y = pack_bf16x2(acc[q][i].z * inv, acc[q][i].w * inv);
      *reinterpret_cast<uint2*>(p.o + grow[q] * DV + 4 * (c0 + 32 * i)) = v;
    }
    if (c0 == 0) {
      p.m[grow[q]] = m[q];
      p.l[grow[q]] = L[q];
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    mla_decode_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                      const __grid_constant__ CUtensorMap tv, const Params p) {
  // No alignment slack: the dynamic window starts 1024-aligned (no static
  // shared memory), and every byte counts.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int warp = warp_id();
  const int h = static_cast<int>(cluster_ctarank());
  const bool leader = h == 0;
  const int k = blockIdx.y;  // this pair's range of (batch, tile)
  if (threadIdx.x == 0) MT_STAMP(63, 0);

  if (warp == 0) {
    // full barriers: the leader's copy is armed with both CTAs' bytes and
    // completed by both CTAs' 2-SM TMA loads (the peer's copies are unused).
    // One lane per ring slot: ~40 serial inits took ~0.7 us of the start.
    const int i = threadIdx.x;
    if (i < NKR) {
      mbar_init(&s.kfull[i], 1);
      mbar_init(&s.kempty[i], 1);
    }
    if (i < NVR) {
      mbar_init(&s.vfull[i], 1);
      mbar_init(&s.vempty[i], 1);
    }
    if (i < 2) {
      mbar_init(&s.s_full[i], 1);
      mbar_init(&s.p_full[i], 8);  // 4 softmax warps of each CTA (the leader's copy is used)
      mbar_init(&s.pv_done[i], 1);
    }
    if (i == 31) {
      mbar_init(&s.q_full, 1);
      mbar_init(&s.q_empty, 1);
      mbar_init(&s.o_full, 1);
      mbar_init(&s.o_empty, 8);  // both CTAs' epilogues have drained their O
      s.nfold = 0;
    }
    fence_barrier_init();
    if (i == 0) MT_STAMP(63, 6);
  }
  unsigned long long fold_old[2] = {0, 0};  // thread 0: the counters before its arrivals
  if (warp == 5) tmem_alloc_2sm<512>(&s.tmem_base);
  if (threadIdx.x == 160) MT_STAMP(63, 7);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x == 0) MT_STAMP(63, 2);
  const uint32_t tmem = s.tmem_base;
  const uint32_t tS[2] = {tmem + 0, tmem + 64};
  const uint32_t tO = tmem + 256;  // + 128 j: V columns 256 j + ...
  Segment sg;

  if (warp == 4) {
    // ------------------------------------------------------ TMA: Q, K ----
    // 2-SM loads: bytes land in this CTA, completion on the leader's barrier
    if (elect_one()) {
      MT_STAMP(63, 4);
      prefetch_tmap(&tq);
      prefetch_tmap(&tk);
      MT_STAMP(63, 5);
      int g = 0, nq = 0, gt = 0, qb = -1;
      for (int si = 0; segment(p, k, si, sg); ++si) {
        if (sg.b != qb) {  // a new batch: its Q once the previous batch's S MMAs are done
          if (qb >= 0) mbar_wait(&s.q_empty, (nq - 1) & 1);
          if (qb < 0) MT_STAMP(63, 3);
          if (leader) mbar_arrive_expect_tx(&s.q_full, 2 * NCH * HC * 128);
          for (int c = 0; c < NCH; ++c)
            tma_load_2d_2sm(s.q[c], &tq, &s.q_full, c * 64, sg.b * HN + h * HC, kEvictFirst);
          qb = sg.b;
          ++nq;
        }
        const int32_t y0 = static_cast<int32_t>(static_cast<int64_t>(sg.b) * p.skv);
        for (int t = sg.t0; t < sg.t1; ++t, ++gt)
          for (int c = 0; c < NKS; ++c, ++g) {  // this CTA's 64 keys, all 576 columns (HBM)
            const int sl = g % NKR;
            mbar_wait(&s.kempty[sl], ((g / NKR) & 1) ^ 1);
            if (c == 0) MT_STAMP(gt, 0);
            if (c == NKS - 1) MT_STAMP(gt, 7);
            if (leader) mbar_arrive_expect_tx(&s.kfull[sl], 2 * STB);
            tma_load_2d_2sm(s.kr[sl], &tk, &s.kfull[sl], c * 64, y0 + t * TK + h * 64, kEvictNormal);
          }
      }
    }
  } else if (warp == 6) {
    // --------------------------------------------------------- TMA: V ----
    if (elect_one()) {
      prefetch_tmap(&tv);
      int g = 0, gt = 0;
      for (int si = 0; segment(p, k, si, sg); ++si) {
        const int32_t y0 = static_cast<int32_t>(static_cast<int64_t>(sg.b) * p.skv);
        for (int t = sg.t0; t < sg.t1; ++t, ++gt)
          for (int v = 0; v < NVS; ++v, ++g) {  // all 128 keys, V columns 256 j + [128 h, +128) (L2)
            const int sl = g % NVR, j = v >> 2, kk = v & 3;
            mbar_wait(&s.vempty[sl], ((g / NVR) & 1) ^ 1);
            if (v == 0) MT_STAMP(gt, 1);
            if (leader) mbar_arrive_expect_tx(&s.vfull[sl], 2 * STB);
            const int c0 = 4 * j + 2 * h;
            const int32_t y = y0 + t * TK + 32 * kk;
            tma_load_2d_2sm(s.vr[sl], &tv, &s.vfull[sl], c0 * 64, y, kEvictFirst);
            tma_load_2d_2sm(s.vr[sl] + STB / 2, &tv, &s.vfull[sl], (c0 + 1) * 64, y, kEvictFirst);
          }
      }
    }
  } else if (warp == 5) {
    if (leader) {
      // -------------------------------------------------------- MMA: S ----
      // S_t may start once softmax t-2 has released P_{t-2} (it has then
      // finished reading S buffer t & 1); P V runs from warp 7, so neither
      // chain waits behind the other's loads (the tensor pipe interleaves the
      // two warps' MMAs on separate accumulators).
      const uint32_t id_s = idesc_f16(HN, TK, kFmtBF16, false, false);
      const bool el = elect_one();
      int g = 0, gt = 0, nq = 0, qb = -1;
      for (int si = 0; segment(p, k, si, sg); ++si) {
        if (sg.b != qb) {
          if (qb >= 0) {
            if (el) mma_commit_2sm(&s.q_empty);  // the previous batch's S MMAs have read Q
            __syncwarp();
          }
          mbar_wait(&s.q_full, nq & 1);
          qb = sg.b;
          ++nq;
        }
        for (int t = sg.t0; t < sg.t1; ++t, ++gt) {
          if (gt >= 2) mbar_wait(&s.p_full[gt & 1], ((gt - 2) >> 1) & 1);
          for (int c = 0; c < NKS; ++c, ++g) {
            const int sl = g % NKR;
            mbar_wait(&s.kfull[sl], (g / NKR) & 1);
            tc_fence_after();
            if (el) {
              const uint32_t qa = smem_u32(s.q[c]), kb = smem_u32(s.kr[sl]);
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4)
                mma_f16_ss_2sm(tS[gt & 1], sdesc_kmajor_sw128(qa + k4 * 32), sdesc_kmajor_sw128(kb + k4 * 32),
                               id_s, (c | k4) != 0);
              mma_commit_2sm(&s.kempty[sl]);
              if (c + 1 == NKS) {
                mma_commit_2sm(&s.s_full[gt & 1]);
                MT_STAMP(gt, 2);
              }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == 7) {
    if (leader) {
      // ------------------------------------------------------ MMA: P V ----
      const uint32_t id_o = idesc_f16(HN, 256, kFmtBF16, false, true);
      const bool el = elect_one();
      int g = 0, gt = 0;
      for (int si = 0; segment(p, k, si, sg); ++si) {
        for (int t = sg.t0; t < sg.t1; ++t, ++gt) {
          mbar_wait(&s.p_full[gt & 1], (gt >> 1) & 1);
          const bool first = t == sg.t0;
          if (first && si > 0) mbar_wait(&s.o_empty, (si - 1) & 1);  // the previous segment's O drained
          tc_fence_after();
          if (el) MT_STAMP(gt, 3);
          const uint32_t pa = smem_u32(s.p[gt % MLA_NP][0]);
          for (int v = 0; v < NVS; ++v, ++g) {
            const int sl = g % NVR, j = v >> 2, kk = v & 3;
            mbar_wait(&s.vfull[sl], (g / NVR) & 1);
            tc_fence_after();
            if (el) {
              const uint32_t vb = smem_u32(s.vr[sl]);
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
                mma_f16_ss_2sm(tO + 128 * j,
                               sdesc_kmajor_sw128(pa + (kk >> 1) * (HC * 128) + (kk & 1) * 64 + ks * 32),
                               sdesc_mnmajor_sw128(vb + ks * 2048, STB / 2), id_o, !first || (kk | ks) != 0);
              mma_commit_2sm(&s.vempty[sl]);
              if (v + 1 == NVS) {
                MT_STAMP(gt, 4);
                mma_commit_2sm(&s.pv_done[gt & 1]);
                if (t + 1 == sg.t1) mma_commit_2sm(&s.o_full);
              }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp < 4) {
    // -------------------------- softmax / correction / epilogue (lane = thread) --
    const int lane = threadIdx.x;  // TMEM lane: row lane % 64, keys / V columns half lane / 64
    const int row = lane & (HC - 1), half = lane >> 6;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const float c1 = p.scale * kLog2e;
    const uint32_t p_row = smem_u32(s.p[0][half]) + (row >> 3) * 1024 + (row & 7) * 128;
    int gt = 0;
    for (int si = 0; segment(p, k, si, sg); ++si) {
      float m_true = -INFINITY, m_ref = -INFINITY, l = 0.f;
      for (int t = sg.t0; t < sg.t1; ++t, ++gt) {
        const int bb = gt & 1;
        mbar_wait(&s.s_full[bb], (gt >> 1) & 1);
        tc_fence_after();
        if (lane == 0) MT_STAMP(gt, 5);
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
        // P buffer gt & 1 is free once P V_{gt-2} has retired; O is rescaled
        // (rarely) once P V_{gt-1} has. pv_done[i] completes for the P V of
        // tiles with gt & 1 = i, and neither can run ahead: the next needs
        // this thread's P.
        const bool resc = t > sg.t0 && __any_sync(0xffffffffu, need);
        if (resc) {
          mbar_wait(&s.pv_done[(gt - 1) & 1], ((gt - 1) >> 1) & 1);
          tc_fence_after();
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
        if (MLA_NP == 2 && gt > 1) mbar_wait(&s.pv_done[gt & 1], ((gt - 2) >> 1) & 1);
        if (MLA_NP == 1 && gt > 0 && !resc) mbar_wait(&s.pv_done[(gt - 1) & 1], ((gt - 1) >> 1) & 1);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          sts128(p_row + (gt % MLA_NP) * (2 * HC * 128) + ((u ^ (row & 7)) << 4),
                 make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]));
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          if (leader) mbar_arrive(&s.p_full[gt & 1]);
          else mbar_arrive_cluster(mapa_shared(smem_u32(&s.p_full[gt & 1]), 0));
        }
        if (lane == 0) MT_STAMP(gt, 6);
      }
      // ---- finalize (finalize_root): d2 = the two halves' sums re-based to d1 ----
      named_bar_sync(1, 128);  // every half has read the last max exchange
      s.xm[0][lane] = l;
      named_bar_sync(1, 128);
      const float l_ref = s.xm[0][row] + s.xm[0][row + 64];  // same operand order in both halves
      named_bar_sync(1, 128);  // xm is free for the next segment
      const float l_true = l_ref * ex2_mufu((m_ref - m_true) * kLog2e);
      const int64_t grow = static_cast<int64_t>(sg.b) * HN + h * HC + row;
      segment_slots(p, k, sg);
      const bool direct = sg.nseg == 1;  // the whole batch is this segment: final outputs
      if (half == 0) {
        if (direct) {
          p.m[grow] = m_true;
          p.l[grow] = l_true;
        } else {
          p.part_m[sg.slot * p.rows_total + grow] = m_true;
          p.part_l[sg.slot * p.rows_total + grow] = l_true;
        }
      }
      mbar_wait(&s.o_full, si & 1);
      tc_fence_after();
      const float inv_l = 1.f / l_ref;
#pragma unroll 1
      for (int c = 0; c < 256 / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tO + lane_off + c * 32, r);
        tmem_ld_wait();
        if (c == 256 / 32 - 1) {  // O is in registers: the next segment's P V may overwrite it
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) {
            if (leader) mbar_arrive(&s.o_empty);
            else mbar_arrive_cluster(mapa_shared(smem_u32(&s.o_empty), 0));
          }
        }
        const int col = 256 * (c >> 2) + 128 * half + 32 * (c & 3);
        if (direct) {
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
          // through this warp's 4 KB of the (idle) P buffers: row-per-lane
          // float4 stores would touch 32 lines per instruction; re-read so
          // that 8 lanes cover one row's 128 B (4 whole lines per store)
          const uint32_t stg = smem_u32(s.p[0][0]) + warp * 4096;
          const int wr = lane & 31;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            sts128(stg + wr * 128 + ((q ^ (wr & 7)) << 4),
                   make_uint4(__float_as_uint(__uint_as_float(r[4 * q]) * inv_l),
                              __float_as_uint(__uint_as_float(r[4 * q + 1]) * inv_l),
                              __float_as_uint(__uint_as_float(r[4 * q + 2]) * inv_l),
                              __float_as_uint(__uint_as_float(r[4 * q + 3]) * inv_l)));
          __syncwarp();
          float* base = p.part_o + (sg.slot * p.rows_total + grow - wr) * DV + col;  // this warp's row 0
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = it * 4 + (wr >> 3), q = wr & 7;
            const uint4 v = lds128(stg + rr * 128 + ((q ^ (rr & 7)) << 4));
            stg128_hint(base + rr * DV + 4 * q, v, kEvictLast);  // kept in L2 for the fold
          }
          __syncwarp();
        }
      }
      if (!direct) {  // partial written: arrive on this batch half's counter (release; acquire for the fold)
        named_bar_sync(1, 128);
        if (lane == 0) {
          const int f = s.nfold++;
          if (f >= 2) __trap();  // only a range's first and last segments can be cut
          s.fold_b[f] = sg.b;
          s.fold_slot[f] = sg.slot;
          s.fold_nseg[f] = sg.nseg;
          fold_old[f] = atom_add_acq_rel_u64(p.cnt + 2 * sg.b + h, 1ull);
        }
      }
    }
  }
  if (threadIdx.x == 0) MT_STAMP(63, 1);
#ifdef RF_MLA_TRACE
  if (threadIdx.x == 0) {
    unsigned long long v_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));
    g_cta_end[blockIdx.y * 2 + blockIdx.x] = v_;
  }
#endif
  tc_fence_before();
  cluster_sync();  // no remote traffic into a CTA that has exited
  if (warp == 5) tmem_dealloc_2sm<512>(tmem);
  // ---- fold of the batches this CTA's range cut (heads [64 h, +64) of each) ----
  const int nfold = s.nfold;  // written by thread 0 before the cluster barrier
  for (int f = 0; f < nfold; ++f) {
    const int b = s.fold_b[f], slot = s.fold_slot[f], ns = s.fold_nseg[f];
    if (threadIdx.x == 0) {
      FT_STAMP(0);
      unsigned long long* c = p.cnt + 2 * b + h;
      const unsigned long long old = fold_old[f], target = old - old % kCntStride + ns;
      if (old + 1 == target) atomicAdd(c, kCntStride - ns);  // last arrival: pad to the next launch's base
      else
        while (ld_acquire_u64(c) < target) {
        }
      FT_STAMP(1);
    }
    __syncthreads();
    const int r0 = slot * HC / ns, r1 = (slot + 1) * HC / ns;
    const int64_t g0 = static_cast<int64_t>(b) * HN + h * HC;
    int r = r0 + warp;
    for (; r + NT / 32 < r1; r += 2 * (NT / 32)) {  // two rows per warp in flight
      const int64_t g[2] = {g0 + r, g0 + r + NT / 32};
      fold_rows<2>(p, g, ns, threadIdx.x & 31);
    }
    if (r < r1) {
      const int64_t g[1] = {g0 + r};
      fold_rows<1>(p, g, ns, threadIdx.x & 31);
    }
    if (threadIdx.x == 0) FT_STAMP(2);
  }
}

}  // namespace

bool mla_supports(int64_t heads, int64_t skv, int64_t dv, int64_t dqk, int64_t segments) {
  return heads == HN && dv == DV && dqk == DQK && segments >= 1 && skv > 0 && skv % TK == 0;
}

namespace {
// Virtual tiles charged for a batch switch inside a range (RF_MLA_SEG overrides, for A/B).
int64_t switch_cost() {
  static const int64_t v = [] {
    const char* e = std::getenv("RF_MLA_SEG");
    return e != nullptr ? static_cast<int64_t>(std::atoi(e)) : int64_t{4};
  }();
  return v;
}

// Greedy ranges of cost <= cap (a range's cost: its tiles + seg per batch it
// switches to after its first); returns the number of ranges, fills cut[]
// when given (at most `limit` ranges are written).
int64_t greedy_cuts(int64_t bs, int64_t tpb, int64_t seg, int64_t cap, int64_t limit, int64_t* cut) {
  const int64_t total = bs * tpb;
  int64_t x = 0, n = 0;
  while (x < total) {
    if (cut != nullptr && n < limit) cut[n] = x;
    ++n;
    int64_t cost = 0;
    bool first = true;
    while (x < total) {
      const int64_t end_b = (x / tpb + 1) * tpb;
      const int64_t extra = first ? 0 : seg;
      const int64_t take = std::min(end_b - x, cap - cost - extra);
      if (take <= 0) break;
      cost += extra + take;
      x += take;
      first = false;
      if (x < end_b) break;  // the range is full inside this batch
    }
  }
  if (cut != nullptr && n <= limit) cut[n] = total;
  return n;
}

// Cuts of the (batch, tile) sequence into at most k non-empty ranges
// minimising the largest range cost (binary search on the cap; the greedy
// fill is optimal for a given cap). Returns the number of ranges.
int64_t balanced_cuts(int64_t bs, int64_t tpb, int64_t k, int64_t* cut) {
  const int64_t seg = switch_cost(), total = bs * tpb;
  int64_t lo = (total + k - 1) / k, hi = total + seg * bs;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (greedy_cuts(bs, tpb, seg, mid, k, nullptr) <= k) hi = mid;
    else lo = mid + 1;
  }
  return greedy_cuts(bs, tpb, seg, lo, k, cut);
}

// Largest number of ranges a batch is cut into (the plan's partial slots).
int64_t slots_of(const int64_t* cut, int64_t clusters, int64_t bs, int64_t tpb) {
  int64_t n = 1;
  for (int64_t b = 0; b < bs; ++b)
    n = std::max<int64_t>(n, cluster_of_tile(cut, static_cast<int>(clusters), (b + 1) * tpb - 1) -
                                 cluster_of_tile(cut, static_cast<int>(clusters), b * tpb) + 1);
  return n;
}

// The balanced cuts over the most CTA pairs (<= one per SM pair, <= one per
// tile) that cut no batch into more than max_slots ranges (the plan's slots:
// a host-path chunk of few batches must not need more than the whole grid).
int64_t pick_cuts(int64_t bs, int64_t tpb, int64_t max_slots, int64_t* cut) {
  for (int64_t k = std::min<int64_t>(kMaxClusters, bs * tpb);; --k) {
    const int64_t n = balanced_cuts(bs, tpb, k, cut);
    if (k == 1 || slots_of(cut, n, bs, tpb) <= max_slots) return n;
  }
}
}  // namespace

// Partial slots per batch (the plan's split count): what range scheduling of
// the whole grid over the resident CTA pairs needs. KV segments of the
// reference are folded by the same closed form, so they need no slots of
// their own.
int64_t mla_pick_splits(int64_t bs, int64_t skv, int64_t segments) {
  (void)segments;
  const int64_t tpb = skv / TK;
  int64_t cut[kMaxClusters + 1];
  const int64_t n = pick_cuts(bs, tpb, INT64_MAX, cut);
  return slots_of(cut, n, bs, tpb);
}

cudaError_t launch_mla_decode(const MlaArgs& a, cudaStream_t st) {
  if (!mla_supports(HN, a.skv, DV, DQK, 1)) return cudaErrorNotSupported;
  CUtensorMap tq, tk, tv;
  const uint64_t qdims[2] = {DQK, static_cast<uint64_t>(a.bs * HN)};
  const uint64_t kdims[2] = {DQK, static_cast<uint64_t>(a.bs * a.skv)};
  const uint64_t strides[1] = {DQK * 2};
  const uint32_t qbox[2] = {64, HC}, kbox[2] = {64, TK / 2}, vbox[2] = {64, 32};
  if (!make_tmap(&tq, a.q, 2, qdims, strides, qbox, 2) || !make_tmap(&tk, a.kv, 2, kdims, strides, kbox, 2) ||
      !make_tmap(&tv, a.kv, 2, kdims, strides, vbox, 2))
    return cudaErrorInvalidValue;
  const int64_t tpb = a.skv / TK;
  Params p{};
  const int64_t clusters = pick_cuts(a.bs, tpb, a.nslices, p.cut);
  p.skv = a.skv;
  p.rows_total = a.rows_total;
  p.tpb = static_cast<int>(tpb);
  p.clusters = static_cast<int>(clusters);
  p.nslots = static_cast<int>(a.nslices);
  p.scale = a.scale;
  p.o = static_cast<__nv_bfloat16*>(a.o);
  p.m = a.m;
  p.l = a.l;
  p.part_m = a.part_m;
  p.part_l = a.part_l;
  p.part_o = a.part_o;
  p.cnt = a.cnt;
  const size_t smem = sizeof(Smem);
  static_assert(sizeof(Smem) <= 227 * 1024, "fits the opt-in shared memory of one CTA");
  cudaError_t e = cudaFuncSetAttribute(mla_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2, static_cast<unsigned>(clusters), 1);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the in-kernel fold waits on other pairs
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.nslices > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, mla_decode_kernel, tq, tk, tv, p);
}

}  // namespace rf
