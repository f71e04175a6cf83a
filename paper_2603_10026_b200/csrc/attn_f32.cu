// fp32 safe-softmax -> GEMM attention in the paper's incremental form (SIMT).
//
// Realises, per KV tile, the reference's element update incr_ingest_element
// (proj/src/simulator.cpp:566-589) for the attention cascade
// (proj/src/workloads.cpp:66-120), with the derived corrections
//   d2: exp(d1' - d1)            d3: exp(d1' - d1) * d2' / d2
// (golden corrections.txt; tests/golden/flash_attention_tile.txt:20-41 is the
// reference's own tile plan for this loop). The output accumulator is kept
// normalised every tile (paper form, not deferred), so each slice's state
// (m, l, O) is exactly the reference's exposed partial and slices merge with
// incr_push_child semantics.
//
// This path serves BASELINE config 1 (fp32, Sq=Skv=1024, D=64): small and
// latency-bound, so it is a SIMT kernel with split-KV for occupancy rather
// than a tensor-core kernel (fp32 parity at 1e-5 rules out single-pass TF32).
// Register tiling: a CTA owns 64 query rows x 64-key tiles; each thread
// computes a 4-row x 4-key block of S (float4 shared loads along D) and a
// 4-row x D/16 block of O whose columns are contiguous float4s, so the P V
// phase reads P and V as float4 too (3 shared wavefronts per 64 FMA). A row's
// 16 threads are one half-warp, so row statistics reduce with shuffles.
//
// Split-KV (run_multisegment, simulator.cpp:660-687): slice states go to the
// partial buffers and are folded in slice order by merge.cu (or across GPUs).
// The plan may cut each reference slice into c sub-slices to fill the GPU
// (cfg1: 8 slices x 2 -> 256 CTAs, 2 per SM); the fold's closed form
// (tests/acceptance.cpp:162-178) is the same sum over the finer slices.
// Two one-launch variants were measured slower on cfg1: the
// slices of a row tile as one thread-block cluster folding through DSMEM
// (only 15 8-CTA clusters are co-resident, 16 needed -> two waves; 25-31 us),
// and a last-arriving-CTA fold (threadfence + arrival counter; 22 us kernel
// vs 13 + a ~5 us merge launch).
#include <atomic>
#include <cuda_bf16.h>

#include "rf_internal.h"
#include "sm100.cuh"

namespace rf {
namespace {

using sm100::f2;
using sm100::f2split;
using sm100::ffma2;

constexpr int BM = 64;   // query rows per CTA
constexpr int BN = 64;   // keys per tile
constexpr int NT = 256;  // 16 x 16 threads: ty -> 4 rows, tx -> 4 keys / D/16 cols
constexpr int TR = 4;    // rows per thread
constexpr int TK = 4;    // keys per thread

__device__ __forceinline__ float load_f(const float* p) { return *p; }
__device__ __forceinline__ float load_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store_f(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_f(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ float hw_max(float v) {  // over the 16 lanes of a half-warp
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float hw_sum(float v) {
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float f4_at(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

template <int D>
constexpr size_t smem_floats() {
  return static_cast<size_t>(BM + 2 * BN) * (D + 4) + BM * (BN + 4);
}

template <int D, typename T>
__global__ void __launch_bounds__(NT, D <= 64 ? 2 : 1) attn_f32_kernel(AttnArgs a) {
  constexpr int DP = D + 4;  // padded rows (float4-aligned, conflict-free column reads)
  constexpr int TD = D / 16;  // O columns per thread
  // D >= 64: TD/4 float4s at columns c4*64 + 4*tx (P V reads P and V as
  // float4); D = 16/32: scalar columns tx + 16*c.
  constexpr bool VEC = D >= 64;
  constexpr int TD4 = VEC ? TD / 4 : 1;
  extern __shared__ __align__(16) float smem_f32[];
  float* sQ = smem_f32;              // [BM][DP]   (pre-scaled)
  float* sK = sQ + BM * DP;          // [BN][DP]
  float* sV = sK + BN * DP;          // [BN][DP]
  float* sP = sV + BN * DP;          // [BM][BN + 4]
  constexpr int PP = BN + 4;

  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t bh = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t slice = a.slice_begin + blockIdx.z;
  const int64_t slice_len = a.skv / a.segments;
  const int64_t kv0 = slice * slice_len, kv1 = kv0 + slice_len;
  const float LOG2E = 1.4426950408889634f;

  // tiles move as float4 chunks (D % 4 == 0): Q once, K/V double-buffered in
  // registers so the next tile's global loads overlap this tile's math
  constexpr int CH = D / 4;                       // float4 chunks per row
  constexpr int NQ = (BM * CH + NT - 1) / NT;     // chunks per thread (Q)
  constexpr int NKV = (BN * CH + NT - 1) / NT;    // chunks per thread (K or V)
  auto ld4 = [&](const T* base, int64_t row, int64_t nrows, int ch) -> float4 {
    if (row >= nrows) return make_float4(0.f, 0.f, 0.f, 0.f);
    const T* p = base + row * D + 4 * ch;
    if constexpr (sizeof(T) == 4) {
      return __ldg(reinterpret_cast<const float4*>(p));
    } else {
      return make_float4(load_f(p), load_f(p + 1), load_f(p + 2), load_f(p + 3));
    }
  };
  float4 kr[NKV], vr[NKV];
  auto fetch = [&](int64_t t0) {
#pragma unroll
    for (int u = 0; u < NKV; ++u) {
      const int idx = tid + u * NT;
      const int64_t key = t0 + idx / CH;
      const bool ok = idx < BN * CH;
      kr[u] = ok ? ld4(K + bh * a.skv * D, key, kv1, idx % CH) : make_float4(0.f, 0.f, 0.f, 0.f);
      vr[u] = ok ? ld4(V + bh * a.skv * D, key, kv1, idx % CH) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  {
    float4 qv[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int idx = tid + u * NT;
      qv[u] = idx < BM * CH ? ld4(Q + bh * a.sq * D, row0 + idx / CH, a.sq, idx % CH)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    fetch(kv0);  // first K/V tile in flight with Q
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int idx = tid + u * NT;
      if (idx < BM * CH) {
        float4 v = qv[u];
        v.x *= a.scale; v.y *= a.scale; v.z *= a.scale; v.w *= a.scale;
        *reinterpret_cast<float4*>(sQ + (idx / CH) * DP + 4 * (idx % CH)) = v;
      }
    }
  }

  // O column of this thread's c-th accumulator
  auto col_of = [&](int c) { return VEC ? (c >> 2) * 64 + 4 * tx + (c & 3) : tx + 16 * c; };
  float m[TR], l[TR], o[TR][TD];
  bool touched = false;
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int c = 0; c < TD; ++c) o[r][c] = 0.f;
  }

  for (int64_t t0 = kv0; t0 < kv1; t0 += BN) {
    __syncthreads();  // previous tile's sK / sV / sP reads are done
#pragma unroll
    for (int u = 0; u < NKV; ++u) {
      const int idx = tid + u * NT;
      if (idx < BN * CH) {
        *reinterpret_cast<float4*>(sK + (idx / CH) * DP + 4 * (idx % CH)) = kr[u];
        *reinterpret_cast<float4*>(sV + (idx / CH) * DP + 4 * (idx % CH)) = vr[u];
      }
    }
    __syncthreads();
    if (t0 + BN < kv1) fetch(t0 + BN);  // next tile in flight during this tile's math

    // S block: rows ty + 16 r, keys tx + 16 j. Packed FFMA2 over (even,
    // odd) d pairs: half the FMA instructions (the kernel is issue-bound)
    uint64_t s2[TR][TK];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < TK; ++j) s2[r][j] = 0ull;
#pragma unroll 4
    for (int dd = 0; dd < D; dd += 4) {
      float4 qv[TR], kv[TK];
#pragma unroll
      for (int r = 0; r < TR; ++r) qv[r] = *reinterpret_cast<const float4*>(sQ + (ty + 16 * r) * DP + dd);
#pragma unroll
      for (int j = 0; j < TK; ++j) kv[j] = *reinterpret_cast<const float4*>(sK + (tx + 16 * j) * DP + dd);
#pragma unroll
      for (int r = 0; r < TR; ++r)
#pragma unroll
        for (int j = 0; j < TK; ++j) {
          s2[r][j] = ffma2(f2(qv[r].x, qv[r].y), f2(kv[j].x, kv[j].y), s2[r][j]);
          s2[r][j] = ffma2(f2(qv[r].z, qv[r].w), f2(kv[j].z, kv[j].w), s2[r][j]);
        }
    }
    float s[TR][TK];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < TK; ++j) {
        float lo, hi;
        f2split(s2[r][j], lo, hi);
        s[r][j] = lo + hi;
      }
    float corr[TR], inv_l[TR];
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      // reduction 1 (max): store-prev, reduce
      float tmax = -INFINITY;
#pragma unroll
      for (int j = 0; j < TK; ++j) {
        if (t0 + tx + 16 * j >= kv1) s[r][j] = -INFINITY;
        tmax = fmaxf(tmax, s[r][j]);
      }
      tmax = hw_max(tmax);
      const float m_prev = m[r], l_prev = l[r];
      m[r] = fmaxf(m_prev, tmax);
      const float mb = m[r] * LOG2E;
      // reduction 2 (sum exp): correct by exp(d1' - d1), reduce
      float psum = 0.f;
#pragma unroll
      for (int j = 0; j < TK; ++j) {
        s[r][j] = exp2f(fmaf(s[r][j], LOG2E, -mb));
        psum += s[r][j];
      }
      psum = hw_sum(psum);
      const float alpha = touched ? exp2f((m_prev - m[r]) * LOG2E) : 0.f;
      l[r] = l_prev * alpha + psum;
      // reduction 3: correct by exp(d1' - d1) * d2' / d2, reduce with weights / d2
      inv_l[r] = 1.f / l[r];
      corr[r] = touched ? alpha * l_prev * inv_l[r] : 0.f;
#pragma unroll
      for (int j = 0; j < TK; ++j) sP[(ty + 16 * r) * PP + tx + 16 * j] = s[r][j];
    }
    touched = true;
    __syncwarp();  // a row's 16 threads are one half-warp
    float acc[TR][TD];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int c = 0; c < TD; ++c) acc[r][c] = 0.f;
if constexpr (VEC) {
    // column pairs (4 tx + 2i, +1) of P V as packed FFMA2
    uint64_t acc2[TR][TD / 2];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int c = 0; c < TD / 2; ++c) acc2[r][c] = 0ull;
#pragma unroll 2
    for (int kk = 0; kk < BN; kk += 4) {
      float4 pv[TR];
#pragma unroll
      for (int r = 0; r < TR; ++r) pv[r] = *reinterpret_cast<const float4*>(sP + (ty + 16 * r) * PP + kk);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float4 vv[TD4];
#pragma unroll
        for (int c4 = 0; c4 < TD4; ++c4)
          vv[c4] = *reinterpret_cast<const float4*>(sV + (kk + u) * DP + c4 * 64 + 4 * tx);
#pragma unroll
        for (int r = 0; r < TR; ++r) {
          const float pr = f4_at(pv[r], u);
          const uint64_t pp = f2(pr, pr);
#pragma unroll
          for (int c4 = 0; c4 < TD4; ++c4) {
            acc2[r][2 * c4] = ffma2(pp, f2(vv[c4].x, vv[c4].y), acc2[r][2 * c4]);
            acc2[r][2 * c4 + 1] = ffma2(pp, f2(vv[c4].z, vv[c4].w), acc2[r][2 * c4 + 1]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int c = 0; c < TD / 2; ++c) f2split(acc2[r][c], acc[r][2 * c], acc[r][2 * c + 1]);
    } else {
#pragma unroll 4
      for (int kk = 0; kk < BN; ++kk) {
        float pv[TR], vv[TD];
#pragma unroll
        for (int r = 0; r < TR; ++r) pv[r] = sP[(ty + 16 * r) * PP + kk];
#pragma unroll
        for (int c = 0; c < TD; ++c) vv[c] = sV[kk * DP + tx + 16 * c];
#pragma unroll
        for (int r = 0; r < TR; ++r)
#pragma unroll
          for (int c = 0; c < TD; ++c) acc[r][c] = fmaf(pv[r], vv[c], acc[r][c]);
      }
    }
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int c = 0; c < TD; ++c) o[r][c] = fmaf(o[r][c], corr[r], acc[r][c] * inv_l[r]);
  }

  // the slice merge (a programmatic dependent launch) may be scheduled now
  asm volatile("griddepcontrol.launch_dependents;");
  {
#pragma unroll
    for (int r = 0; r < TR; ++r) {
      const int64_t gr = row0 + ty + 16 * r;
      if (gr >= a.sq) continue;
      const int64_t row = bh * a.sq + gr;
      if (a.part_m == nullptr) {
        T* O = static_cast<T*>(a.o);
#pragma unroll
        for (int c = 0; c < TD; ++c) store_f(O + row * D + col_of(c), o[r][c]);
        if (tx == 0) {
          a.m[row] = m[r];
          a.l[row] = l[r];
        }
      } else {
        const int64_t ps = slice - a.part_base;
        float* po = a.part_o + (ps * a.rows_total + row) * D;
#pragma unroll
        for (int c = 0; c < TD; ++c) po[col_of(c)] = o[r][c];
        if (tx == 0) {
          a.part_m[ps * a.rows_total + row] = m[r];
          a.part_l[ps * a.rows_total + row] = l[r];
        }
      }
    }
  }
}

template <int D, typename T>
cudaError_t launch_t(const AttnArgs& a, cudaStream_t st) {
  auto k = attn_f32_kernel<D, T>;
  const size_t smem = sizeof(float) * smem_floats<D>();
  static std::atomic<uint64_t> attr_set{0};  // per device, per template instance
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  dim3 grid(static_cast<unsigned>((a.sq + BM - 1) / BM), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
  k<<<grid, NT, smem, st>>>(a);
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  return a.dtype == RF_BF16 ? launch_t<D, __nv_bfloat16>(a, st) : launch_t<D, float>(a, st);
}

}  // namespace

cudaError_t launch_attention_f32(const AttnArgs& a, cudaStream_t st) {
  switch (a.d) {
    case 16: return launch_d<16>(a, st);
    case 32: return launch_d<32>(a, st);
    case 64: return launch_d<64>(a, st);
    case 128: return launch_d<128>(a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace rf
