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
// latency-bound, so it is a plain SIMT kernel with split-KV (segments) for
// occupancy rather than a tensor-core kernel. Row = one reference cascade
// instance (one query of one (b,h)).
#include <cuda_bf16.h>

#include "rf_internal.h"

namespace rf {
namespace {

constexpr int BM = 32;   // query rows per CTA
constexpr int BN = 32;   // keys per tile
constexpr int NT = 128;  // threads: 4 per row

__device__ __forceinline__ float load_f(const float* p) { return *p; }
__device__ __forceinline__ float load_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void store_f(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_f(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <int D, typename T>
__global__ void __launch_bounds__(NT) attn_f32_kernel(AttnArgs a) {
  extern __shared__ float smem_f32[];
  float(*sQ)[D + 1] = reinterpret_cast<float(*)[D + 1]>(smem_f32);
  float(*sK)[D + 1] = reinterpret_cast<float(*)[D + 1]>(smem_f32 + BM * (D + 1));
  float(*sV)[D] = reinterpret_cast<float(*)[D]>(smem_f32 + (BM + BN) * (D + 1));
  float(*sP)[BN + 1] =
      reinterpret_cast<float(*)[BN + 1]>(smem_f32 + (BM + BN) * (D + 1) + BN * D);

  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);

  const int tid = threadIdx.x;
  const int r = tid >> 2;  // row within the tile
  const int qd = tid & 3;  // quad lane
  const int64_t bh = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t slice = a.slice_begin + blockIdx.z;
  const int64_t slice_len = a.skv / a.segments;
  const int64_t kv0 = slice * slice_len, kv1 = kv0 + slice_len;

  const float LOG2E = 1.4426950408889634f;
  for (int i = tid; i < BM * D; i += NT) {
    int rr = i / D, dd = i % D;
    int64_t gr = row0 + rr;
    sQ[rr][dd] = gr < a.sq ? load_f(Q + (bh * a.sq + gr) * D + dd) * a.scale : 0.f;
  }

  // Per-row streaming state (replicated across the quad).
  float m = -INFINITY, l = 0.f;
  bool touched = false;
  constexpr int NC = D / 4;
  float o[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) o[i] = 0.f;

  for (int64_t t0 = kv0; t0 < kv1; t0 += BN) {
    __syncthreads();  // previous tile's sK/sV/sP reads are done
    for (int i = tid; i < BN * D; i += NT) {
      int c = i / D, dd = i % D;
      int64_t gk = t0 + c;
      bool ok = gk < kv1;
      sK[c][dd] = ok ? load_f(K + (bh * a.skv + gk) * D + dd) : 0.f;
      sV[c][dd] = ok ? load_f(V + (bh * a.skv + gk) * D + dd) : 0.f;
    }
    __syncthreads();

    // S = (scale Q) K^T for this thread's 8 columns c = qd + 4j.
    float s[BN / 4];
#pragma unroll
    for (int j = 0; j < BN / 4; ++j) s[j] = 0.f;
#pragma unroll 8
    for (int dd = 0; dd < D; ++dd) {
      float qv = sQ[r][dd];
#pragma unroll
      for (int j = 0; j < BN / 4; ++j) s[j] = fmaf(qv, sK[qd + 4 * j][dd], s[j]);
    }
    // Reduction 1 (max): store-prev, reduce.
    float tmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < BN / 4; ++j) {
      bool ok = t0 + qd + 4 * j < kv1;
      if (!ok) s[j] = -INFINITY;
      tmax = fmaxf(tmax, s[j]);
    }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float m_prev = m, l_prev = l;
    m = fmaxf(m_prev, tmax);
    const float mb = m * LOG2E;
    // Reduction 2 (sum exp): correct by exp(d1' - d1), reduce.
    float psum = 0.f;
#pragma unroll
    for (int j = 0; j < BN / 4; ++j) {
      float p = exp2f(fmaf(s[j], LOG2E, -mb));
      s[j] = p;
      psum += p;
    }
    psum += __shfl_xor_sync(0xffffffffu, psum, 1);
    psum += __shfl_xor_sync(0xffffffffu, psum, 2);
    const float alpha = touched ? exp2f((m_prev - m) * LOG2E) : 0.f;
    l = l_prev * alpha + psum;
    // Reduction 3: correct by exp(d1' - d1) * d2' / d2, reduce with weights / d2.
    const float inv_l = 1.f / l;
    const float corr = touched ? alpha * l_prev * inv_l : 0.f;
    touched = true;
#pragma unroll
    for (int j = 0; j < BN / 4; ++j) sP[r][qd + 4 * j] = s[j];
    __syncwarp();  // a row's quad lives in one warp
    float acc[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = 0.f;
#pragma unroll 4
    for (int c = 0; c < BN; ++c) {
      float p = sP[r][c];
#pragma unroll
      for (int i = 0; i < NC; ++i) acc[i] = fmaf(p, sV[c][qd + 4 * i], acc[i]);
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) o[i] = fmaf(o[i], corr, acc[i] * inv_l);
  }

  const int64_t gr = row0 + r;
  if (gr >= a.sq) return;
  const int64_t row = bh * a.sq + gr;
  if (a.part_m == nullptr) {
    T* O = static_cast<T*>(a.o);
#pragma unroll
    for (int i = 0; i < NC; ++i) store_f(O + row * D + qd + 4 * i, o[i]);
    if (qd == 0) {
      a.m[row] = m;
      a.l[row] = l;
    }
  } else {
    const int64_t ps = slice - a.part_base;
    float* po = a.part_o + (ps * a.rows_total + row) * D;
#pragma unroll
    for (int i = 0; i < NC; ++i) po[qd + 4 * i] = o[i];
    if (qd == 0) {
      a.part_m[ps * a.rows_total + row] = m;
      a.part_l[ps * a.rows_total + row] = l;
    }
  }
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>((a.sq + BM - 1) / BM), static_cast<unsigned>(a.bh),
            static_cast<unsigned>(a.nslices));
  const size_t smem = sizeof(float) * ((BM + BN) * (D + 1) + BN * D + BM * (BN + 1));
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
