// fp32 safe-softmax -> GEMM attention on the tensor cores (BASELINE config 1),
// one launch: the split-KV slices of a 128-row tile form a thread-block
// cluster and fold their (m, l, O) states inside the kernel.
//
// The cascade is the reference's attention workload
// (proj/src/workloads.cpp:66-120) run as run_multisegment
// (proj/src/simulator.cpp:660-687): every slice runs the incremental loop
// (incr_ingest_element, :566-589) from fresh state over its keys in tiles of
// 128 (tests/golden/flash_attention_tile.txt's RT = ST = 128), and the slice
// states fold in slice order (incr_push_child, :592-608; closed form and
// order in fold.cuh's arithmetic). The SIMT kernel (attn_f32.cu) spends most
// of cfg1 on shared-memory latency and a second (merge) launch; here both
// contractions are tcgen05 MMAs and the fold runs inside the cluster: after a
// cluster barrier every CTA bulk-copies each owner's block of its state into
// the owner's drained Q tiles (cp.async.bulk shared::cta -> shared::cluster,
// completing on the owner's mbarrier) and each owner folds its rows locally.
//
// fp32 accuracy (<= 1e-5 scaled error, north_star) with kind::tf32 MMAs: each
// operand x is split as x = hi + lo, hi = tf32(x) (cvt.rna), lo = x - hi
// (exact in fp32; the MMA reads its top 19 bits), and every product is
// hi*hi + hi*lo + lo*hi (3xTF32: the dropped lo*lo and the truncation of lo
// are ~2^-22 relative).
//   S  = Q K^T : A = Q (smem, K-major), B = K (smem, K-major), M=128 N=128 K=D
//   O += P V   : A = P (TMEM, written by the softmax threads), B = V^T (smem,
//                K-major: transposed while splitting), M=128 N=D K=128
// TMEM: S / P_hi [0,128), P_lo [128,256), O [256, 256 + D).
// Two threads per query row (TMEM lane, one per half of the columns) run the
// online softmax; O is kept unnormalised with the running max and rescaled in
// TMEM when it grows, and the slice state is (m, l, O / l) — the paper form
// the fold expects. Q and the first K / V tile land by TMA (K raw into the K
// hi tiles, V staged in the K lo tiles until it is transposed), then every
// thread splits its own row in place.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using namespace sm100;

#ifdef RF_TF32_TRACE
// globaltimer (ns) per CTA and event (probe build only, tools/trace_tf32.py)
__device__ unsigned long long g_tf32_trace[512][16];
#define TTRACE(ev)                                                                           \
  do {                                                                                       \
    if (threadIdx.x == 0) {                                                                  \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
      const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);       \
      if (cta_ < 512) g_tf32_trace[cta_][ev] = t_;                                           \
    }                                                                                        \
  } while (0)
#else
#define TTRACE(ev) \
  do {             \
  } while (0)
#endif

constexpr int BM = 128;   // query rows per CTA (UMMA M, TMEM lanes)
constexpr int BN = 128;   // keys per tile
constexpr int D = 64;     // head_dim (cfg1)
constexpr int NT = 256;   // 8 warps: warps w and w + 4 share TMEM lane quarter w (row halves)
constexpr uint32_t kFmtTF32 = 2;
constexpr int CH = BM * 128;            // one [128 rows x 128 B] SWIZZLE_128B chunk (16 KB)
constexpr uint32_t COL_P_LO = 128, COL_O = 256;

struct Smem {
  uint8_t q[2][D / 32][CH];             // [hi/lo][d chunk]: rows = queries, 32 fp32 of D each
  uint8_t k[2][D / 32][CH];             // rows = keys
  uint8_t vt[2][BN / 32][D * 128];      // [hi/lo][key chunk]: rows = d, 32 keys each
  float xchg[2][2][BM];                 // [max / sum][column half][row]
  uint64_t q_bar, ld_bar, mma_done, recv_bar;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t sw(uint32_t r, uint32_t u) {  // 16 B unit u of row r (SW128)
  return (r >> 3) * 1024 + (r & 7) * 128 + ((u ^ (r & 7)) << 4);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

// Row r of a [128 rows x 32 fp32] SWIZZLE_128B tile (as TMA lands it).
__device__ __forceinline__ void load_row(uint32_t tile, uint32_t r, float4 (&x)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint4 v = lds128(tile + sw(r, u));
    x[u] = make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
  }
}

// Split a row of 32 fp32 into hi / lo rows of SWIZZLE_128B tiles (hi may be
// the tile the row was read from: each thread rewrites only its own row).
__device__ __forceinline__ void split_row(const float4 (&x)[8], uint32_t hi_tile, uint32_t lo_tile, uint32_t r,
                                          float scale) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float v[4] = {x[u].x * scale, x[u].y * scale, x[u].z * scale, x[u].w * scale};
    float h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = tf32_hi(v[i]);
      l[i] = v[i] - h[i];
    }
    sts128(hi_tile + sw(r, u), make_uint4(__float_as_uint(h[0]), __float_as_uint(h[1]),
                                          __float_as_uint(h[2]), __float_as_uint(h[3])));
    sts128(lo_tile + sw(r, u), make_uint4(__float_as_uint(l[0]), __float_as_uint(l[1]),
                                          __float_as_uint(l[2]), __float_as_uint(l[3])));
  }
}

// V^T hi / lo from V row kr's D half h (32 fp32): element (d = 32 h + j, key
// kr) -> key chunk kr / 32, row d, 4-byte slot kr % 32 (a warp's 32 keys
// fill one 128 B row: conflict-free).
__device__ __forceinline__ void split_vt(const float4 (&xv)[8], Smem& s, int kr, int h) {
  const uint32_t kc = kr >> 5, ko = (kr & 31) * 4;
  const uint32_t vh = smem_u32(s.vt[0][kc]), vl = smem_u32(s.vt[1][kc]);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float v[4] = {xv[u].x, xv[u].y, xv[u].z, xv[u].w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t d = 32 * h + 4 * u + i;
      const uint32_t off = (d >> 3) * 1024 + (d & 7) * 128 + ((((ko >> 4) ^ (d & 7)) << 4) | (ko & 15));
      const float hv = tf32_hi(v[i]);
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(vh + off), "f"(hv) : "memory");
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(vl + off), "f"(v[i] - hv) : "memory");
    }
  }
}

// Bulk copy of `bytes` from this CTA's shared memory to a shared::cluster
// address, completing on a shared::cluster mbarrier (the receiver's).
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst_cluster), "r"(src), "r"(bytes), "r"(bar_cluster)
               : "memory");
}

// TMA of one 128-key tile: K (2 D halves) into the K hi tiles, V into the K
// lo tiles (staging; V^T is built from there before K is split).
__device__ __forceinline__ void load_kv(Smem& s, const CUtensorMap* tk, const CUtensorMap* tv, int64_t key0) {
  mbar_arrive_expect_tx(&s.ld_bar, 4 * CH);
  for (int hh = 0; hh < 2; ++hh) {
    tma_load_2d(s.k[0][hh], tk, &s.ld_bar, 32 * hh, static_cast<int32_t>(key0), kEvictLast);
    tma_load_2d(s.k[1][hh], tv, &s.ld_bar, 32 * hh, static_cast<int32_t>(key0), kEvictLast);
  }
}

__global__ void __launch_bounds__(NT, 1)
    attn_tf32_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t bh = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t slice = blockIdx.z;  // = rank in the cluster (cluster dims (1, 1, nslices))
  const int64_t slice_len = a.skv / a.nslices;
  const int64_t kv0 = slice * slice_len, kv1 = kv0 + slice_len;
  const float LOG2E = 1.4426950408889634f;
  TTRACE(0);

  if (tid == 0) {
    mbar_init(&s.q_bar, 1);
    mbar_init(&s.ld_bar, 1);
    mbar_init(&s.mma_done, 1);
    mbar_init(&s.recv_bar, 1);
    fence_barrier_init();
    // Q and the first K / V tile, all in flight at once. A ragged last row
    // tile (Sq % 128 != 0) reads the next head's rows or TMA zero fill past
    // the tensor: those rows are computed and never stored.
    mbar_arrive_expect_tx(&s.q_bar, 2 * CH);
    for (int hh = 0; hh < 2; ++hh)
      tma_load_2d(s.q[0][hh], &tq, &s.q_bar, 32 * hh, static_cast<int32_t>(bh * a.sq + row0), kEvictFirst);
    load_kv(s, &tk, &tv, bh * a.skv + kv0);
  }
  if (warp == 0) tmem_alloc<512>(&s.tmem_base);
  const int r = tid & (BM - 1), h = tid >> 7;  // thread (row / key r, D half h)
  uint32_t ld_phase = 0;
  tc_fence_before();
  __syncthreads();  // barriers initialised (and the TMEM base written) before anyone waits
  tc_fence_after();
  mbar_wait(&s.q_bar, 0);
  {
    float4 x[8];
    load_row(smem_u32(s.q[0][h]), r, x);
    split_row(x, smem_u32(s.q[0][h]), smem_u32(s.q[1][h]), r, a.scale);
  }
  TTRACE(1);
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t id_s = (1u << 4) | (kFmtTF32 << 7) | (kFmtTF32 << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);
  const uint32_t id_o = (1u << 4) | (kFmtTF32 << 7) | (kFmtTF32 << 10) | ((D >> 3) << 17) | ((BM >> 4) << 24);
  // softmax / epilogue split: warp w owns TMEM lane quarter w & 3 and column
  // half h of S (64 keys) and of O (32 of D)
  const uint32_t s_col = 64 * h, o_col = COL_O + (D / 2) * h;

  float m = -INFINITY, l = 0.f;
  uint32_t phase = 0;
  for (int64_t t0 = kv0; t0 < kv1; t0 += BN) {
    if (t0 != kv0 && tid == 0) load_kv(s, &tk, &tv, bh * a.skv + t0);  // previous tile's MMAs are done
    mbar_wait(&s.ld_bar, ld_phase);
    ld_phase ^= 1;
    float4 xv[8];
    {
      float4 x[8];
      load_row(smem_u32(s.k[1][h]), r, xv);  // V row r (staged in the K lo tiles), kept in registers
      load_row(smem_u32(s.k[0][h]), r, x);
      __syncthreads();  // V staging read by everybody before K lo overwrites it
      split_row(x, smem_u32(s.k[0][h]), smem_u32(s.k[1][h]), r, 1.f);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    TTRACE(2);
    const uint32_t tmem = s.tmem_base;
    // S = Qhi Khi + Qhi Klo + Qlo Khi  (K = D in steps of 8 fp32 = 32 B)
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < D / 8; ++ks) {
        const uint32_t c = ks >> 2, o = (ks & 3) * 32;
        const uint64_t qh = sdesc_kmajor_sw128(smem_u32(s.q[0][c]) + o), ql = sdesc_kmajor_sw128(smem_u32(s.q[1][c]) + o);
        const uint64_t kh = sdesc_kmajor_sw128(smem_u32(s.k[0][c]) + o), kl = sdesc_kmajor_sw128(smem_u32(s.k[1][c]) + o);
        mma_tf32_ss(tmem, qh, kh, id_s, ks != 0);
        mma_tf32_ss(tmem, qh, kl, id_s, 1);
        mma_tf32_ss(tmem, ql, kh, id_s, 1);
      }
      mma_commit(&s.mma_done);
    }
    split_vt(xv, s, r, h);  // V^T hi / lo while the S MMAs run (ordered before P V by the barriers below)
    fence_proxy_async_smem();
    mbar_wait(&s.mma_done, phase);
    phase ^= 1;
    tc_fence_after();
    TTRACE(3);
    // online softmax, the row's 128 scores split over the two warps of its
    // lane quarter (row max and sum exchanged in smem): pass 1 the max, pass 2
    // re-reads each 32-column chunk for the exponentials
    float tmax = -INFINITY;
    {
      uint32_t v0[32], v1[32];
      tmem_ld32(tmem + lane_off + s_col, v0);
      tmem_ld32(tmem + lane_off + s_col + 32, v1);
      tmem_ld_wait();
      float t2[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int j = 0; j < 32; ++j)
        t2[j & 3] = fmaxf(t2[j & 3], fmaxf(__uint_as_float(v0[j]), __uint_as_float(v1[j])));
      tmax = fmaxf(fmaxf(t2[0], t2[1]), fmaxf(t2[2], t2[3]));
    }
    s.xchg[0][h][r] = tmax;
    __syncthreads();
    tmax = fmaxf(s.xchg[0][0][r], s.xchg[0][1][r]);
    const float m_new = fmaxf(m, tmax);
    const float mb = m_new * LOG2E;
    const float alpha = l > 0.f ? exp2f((m - m_new) * LOG2E) : 0.f;
    float ps4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32], lo[32];
      tmem_ld32(tmem + lane_off + s_col + 32 * c, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float p = ex2_mufu(fmaf(__uint_as_float(v[j]), LOG2E, -mb));  // ex2.approx.ftz: ~2 ulp
        ps4[j & 3] += p;
        const float ph = tf32_hi(p);
        v[j] = __float_as_uint(ph);
        lo[j] = __float_as_uint(p - ph);
      }
      tmem_st32(tmem + lane_off + s_col + 32 * c, v);
      tmem_st32(tmem + lane_off + COL_P_LO + s_col + 32 * c, lo);
    }
    // O (unnormalised, running max) re-based to m_new; tcgen05.ld / st are
    // warp-collective, so the warp rescales together if any of its rows moved
    if (t0 != kv0 && __any_sync(0xffffffffu, alpha != 1.f)) {
      uint32_t o[32];
      tmem_ld32(tmem + lane_off + o_col, o);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
      tmem_st32(tmem + lane_off + o_col, o);
    }
    s.xchg[1][h][r] = (ps4[0] + ps4[1]) + (ps4[2] + ps4[3]);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    l = l * alpha + (s.xchg[1][0][r] + s.xchg[1][1][r]);
    m = m_new;
    TTRACE(4);
    // O += Phi Vhi + Phi Vlo + Plo Vhi  (K = 128 keys in steps of 8)
    if (tid == 0) {
#pragma unroll
      for (int ks = 0; ks < BN / 8; ++ks) {
        const uint32_t c = ks >> 2, o = (ks & 3) * 32;
        const uint64_t vh = sdesc_kmajor_sw128(smem_u32(s.vt[0][c]) + o), vl = sdesc_kmajor_sw128(smem_u32(s.vt[1][c]) + o);
        mma_tf32_ts(tmem + COL_O, tmem + 8 * ks, vh, id_o, (t0 != kv0) || ks != 0);
        mma_tf32_ts(tmem + COL_O, tmem + 8 * ks, vl, id_o, 1);
        mma_tf32_ts(tmem + COL_O, tmem + COL_P_LO + 8 * ks, vh, id_o, 1);
      }
      mma_commit(&s.mma_done);
    }
    mbar_wait(&s.mma_done, phase);  // P V done: S / P / V^T / K free for the next tile
    phase ^= 1;
    tc_fence_after();
    TTRACE(5);
  }

  // slice state (m, l, O / l) of this CTA's rows (warp w: D half h)
  const uint32_t tmem = s.tmem_base;
  const bool fold = a.nslices > 1;
  const float inv = 1.f / l;
  uint32_t o[32];
  tmem_ld32(tmem + lane_off + o_col, o);
  tmem_ld_wait();
  if (!fold) {  // one slice: the state is the result
    const int64_t grow = row0 + r;
    if (grow < a.sq) {
      const int64_t row = bh * a.sq + grow;
      float4* p = reinterpret_cast<float4*>(static_cast<float*>(a.o) + row * D + (D / 2) * h);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        p[j] = make_float4(__uint_as_float(o[4 * j]) * inv, __uint_as_float(o[4 * j + 1]) * inv,
                           __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
      if (h == 0) {
        a.m[row] = m;
        a.l[row] = l;
      }
    }
  } else {
    // Stage the state for the bulk push: row-major [128][D] in the drained K
    // tiles (16-byte units of row r XOR-swizzled by r & 15: conflict-free
    // here, undone by the reader), then m[128], l[128]. The rows of each
    // owner (16 / 32 / 64 consecutive rows) are one contiguous block.
    float* so = reinterpret_cast<float*>(s.k);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int u = (D / 8) * h + j;  // 16-byte unit of the row
      *reinterpret_cast<float4*>(so + r * D + 4 * (u ^ (r & 15))) =
          make_float4(__uint_as_float(o[4 * j]) * inv, __uint_as_float(o[4 * j + 1]) * inv,
                      __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
    }
    if (h == 0) {
      so[BM * D + r] = m;
      so[BM * D + BM + r] = l;
    }
    fence_proxy_async_smem();  // generic stores -> the bulk copies' reads
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
  TTRACE(6);
  if (!fold) return;
  // In-cluster fold. CTA z owns rows [z * per, (z + 1) * per) of the tile.
  // After a cluster barrier (every CTA is past its MMAs, so every Q region is
  // free), each CTA pushes the owners' blocks of its slice state into their Q
  // region with bulk shared::cta -> shared::cluster copies that complete on
  // the owner's recv_bar; each owner then folds its rows locally, over all
  // slices in slice order with fold.cuh's arithmetic.
  const int ns = static_cast<int>(a.nslices);
  const int per = BM / ns;
  const uint32_t blk = static_cast<uint32_t>(per * D * 4), mlb = static_cast<uint32_t>(per * 4);
  const uint32_t recv = smem_u32(s.q), stage = smem_u32(s.k);
  // the own slice's block is read from the staging area in place (a bulk
  // copy to a shared::cluster address of the executing CTA is not allowed)
  if (tid == 0) mbar_arrive_expect_tx(&s.recv_bar, static_cast<uint32_t>(ns - 1) * (blk + 2 * mlb));
  cluster_sync();
  TTRACE(7);
  if (tid == 0) {
    const uint32_t me = static_cast<uint32_t>(slice);
    for (int z = 0; z < ns; ++z) {
      if (z == static_cast<int>(me)) continue;
      const uint32_t bar = mapa_shared(smem_u32(&s.recv_bar), z);
      const uint32_t dst = mapa_shared(recv, z);
      // [slot][per rows][D] O, then m[slot][per], then l[slot][per]
      bulk_s2c(dst + me * blk, stage + z * blk, blk, bar);
      bulk_s2c(dst + ns * blk + me * mlb, stage + BM * D * 4 + z * mlb, mlb, bar);
      bulk_s2c(dst + ns * blk + ns * mlb + me * mlb, stage + BM * D * 4 + BM * 4 + z * mlb, mlb, bar);
    }
    bulk_commit();
  }
  mbar_wait(&s.recv_bar, 0);
  const float* ro = reinterpret_cast<const float*>(s.q);
  const float* rm = ro + ns * per * D;
  const float* rl = rm + ns * per;
  const float* own = reinterpret_cast<const float*>(s.k);  // staging: [128][D], m[128], l[128]
  const int me = static_cast<int>(slice);
  for (int i = tid; i < per * (D / 4); i += NT) {
    const int lr = i / (D / 4), c4 = i % (D / 4);
    const int orow = me * per + lr;  // the own slice's row in the staging area
    float mm = -INFINITY;
    for (int j = 0; j < ns; ++j) mm = fmaxf(mm, j == me ? own[BM * D + orow] : rm[j * per + lr]);
    float ll = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < ns; ++j) {
      const float lj = j == me ? own[BM * D + BM + orow] : rl[j * per + lr];
      const float mj = j == me ? own[BM * D + orow] : rm[j * per + lr];
      if (lj != 0.f) {  // an empty slice contributes nothing whatever its staged O
        const float* src = j == me ? own + orow * D : ro + (j * per + lr) * D;
        const float4 oj = *reinterpret_cast<const float4*>(src + 4 * (c4 ^ (lr & 15)));
        const float w = lj * __expf(mj - mm);
        ll += w;
        acc.x = fmaf(oj.x, w, acc.x);
        acc.y = fmaf(oj.y, w, acc.y);
        acc.z = fmaf(oj.z, w, acc.z);
        acc.w = fmaf(oj.w, w, acc.w);
      }
    }
    const int64_t grow = row0 + static_cast<int64_t>(slice) * per + lr;
    if (grow < a.sq) {
      const int64_t row = bh * a.sq + grow;
      const float iv = 1.f / ll;
      reinterpret_cast<float4*>(static_cast<float*>(a.o) + row * D)[c4] =
          make_float4(acc.x * iv, acc.y * iv, acc.z * iv, acc.w * iv);
      if (c4 == 0) {
        a.m[row] = mm;
        a.l[row] = ll;
      }
    }
  }
  TTRACE(8);
  if (tid == 0) bulk_wait_read0();  // our outgoing copies have read the staging before we leave
}

}  // namespace

bool attention_tf32_supports(int64_t sq, int64_t skv, int64_t d, int64_t nslices) {
  return d == D && sq >= 1 && nslices >= 1 && nslices <= 8 && (BM % nslices) == 0 &&
         skv % nslices == 0 && (skv / nslices) % BN == 0;
}

cudaError_t launch_attention_tf32(const AttnArgs& a, cudaStream_t st) {
  if (!attention_tf32_supports(a.sq, a.skv, a.d, a.nslices) || a.dtype != RF_F32 || a.slice_begin != 0)
    return cudaErrorNotSupported;
  CUtensorMap tq, tk, tv;
  const uint32_t box[2] = {32, BM};
  const uint64_t str[1] = {D * 4};
  const uint64_t qd[2] = {D, static_cast<uint64_t>(a.bh * a.sq)};
  const uint64_t kd[2] = {D, static_cast<uint64_t>(a.bh * a.skv)};
  if (!make_tmap(&tq, a.q, 2, qd, str, box, 4) || !make_tmap(&tk, a.k, 2, kd, str, box, 4) ||
      !make_tmap(&tv, a.v, 2, kd, str, box, 4))
    return cudaErrorInvalidValue;
  const size_t smem = sizeof(Smem) + 1024;
  static std::atomic<uint64_t> attr_set{0};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(attn_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((a.sq + BM - 1) / BM), static_cast<unsigned>(a.bh),
                     static_cast<unsigned>(a.nslices));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = static_cast<unsigned>(a.nslices);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_tf32_kernel, tq, tk, tv, a);
}

}  // namespace rf
