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
// incr_push_child semantics (merge.cu).
//
// This path serves BASELINE config 1 (fp32, Sq=Skv=1024, D=64): small and
// latency-bound, so it is a SIMT kernel with split-KV (segments) for
// occupancy rather than a tensor-core kernel (fp32 parity at 1e-5 rules out
// single-pass TF32). Register tiling: a CTA owns 64 query rows x 64-key tiles;
// each thread computes a 4-row x 4-key block of S and a 4-row x D/16 block of
// O (0.5 shared loads per FMA); a row's 16 threads are one half-warp, so the
// row statistics reduce with shuffles. Row = one reference cascade instance.
#include <cuda_bf16.h>

#include "rf_internal.h"

namespace rf {
namespace {

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

template <int D, typename T>
__global__ void __launch_bounds__(NT) attn_f32_kernel(AttnArgs a) {
  constexpr int DP = D + 4;  // padded rows (float4-aligned, conflict-free column reads)
  constexpr int TD = D / 16;  // O columns per thread
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
  {
    float4 qv[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int idx = tid + u * NT;
      qv[u] = idx < BM * CH ? ld4(Q + bh * a.sq * D, row0 + idx / CH, a.sq, idx % CH)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    }
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
  fetch(kv0);

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

    // S block: rows ty + 16 r, keys tx + 16 j
    float s[TR][TK];
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int j = 0; j < TK; ++j) s[r][j] = 0.f;
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
          s[r][j] = fmaf(qv[r].x, kv[j].x, s[r][j]);
          s[r][j] = fmaf(qv[r].y, kv[j].y, s[r][j]);
          s[r][j] = fmaf(qv[r].z, kv[j].z, s[r][j]);
          s[r][j] = fmaf(qv[r].w, kv[j].w, s[r][j]);
        }
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
#pragma unroll
    for (int r = 0; r < TR; ++r)
#pragma unroll
      for (int c = 0; c < TD; ++c) o[r][c] = fmaf(o[r][c], corr[r], acc[r][c] * inv_l[r]);
  }

#pragma unroll
  for (int r = 0; r < TR; ++r) {
    const int64_t gr = row0 + ty + 16 * r;
    if (gr >= a.sq) continue;
    const int64_t row = bh * a.sq + gr;
    if (a.part_m == nullptr) {
      T* O = static_cast<T*>(a.o);
#pragma unroll
      for (int c = 0; c < TD; ++c) store_f(O + row * D + tx + 16 * c, o[r][c]);
      if (tx == 0) {
        a.m[row] = m[r];
        a.l[row] = l[r];
      }
    } else {
      const int64_t ps = slice - a.part_base;
      float* po = a.part_o + (ps * a.rows_total + row) * D;
#pragma unroll
      for (int c = 0; c < TD; ++c) po[tx + 16 * c] = o[r][c];
      if (tx == 0) {
        a.part_m[ps * a.rows_total + row] = m[r];
        a.part_l[ps * a.rows_total + row] = l[r];
      }
    }
  }
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((a.sq + BM - 1) / BM), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
  const size_t smem = sizeof(float) * ((BM + 2 * BN) * (D + 4) + BM * (BN + 4));
  if (a.dtype == RF_BF16) {
    auto k = attn_f32_kernel<D, __nv_bfloat16>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, NT, smem, st>>>(a);
  } else {
    auto k = attn_f32_kernel<D, float>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, NT, smem, st>>>(a);
  }
  return cudaGetLastError();
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
