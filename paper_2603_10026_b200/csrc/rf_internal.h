// Internal declarations shared by the librf_cuda translation units.
// Not part of the ABI (see include/rf_cuda.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "rf_cuda.h"

namespace rf {

// Thread-local last-error text (rf_last_error).
void set_error(const std::string& msg);

#define RF_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t err__ = (expr);                                             \
    if (err__ != cudaSuccess) {                                             \
      ::rf::set_error(std::string(#expr) + ": " + cudaGetErrorString(err__)); \
      return RF_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

enum class Kernel {
  SoftmaxRows,        // softmax.cu
  AttentionF32,       // attn_f32.cu   (SIMT, paper form; partials, odd shapes)
  AttentionTf32,      // attn_tf32.cu  (3xTF32 tcgen05, in-cluster slice fold, cfg1)
  AttentionSm100,     // attn_sm100.cu (bf16 tcgen05/TMEM/TMA prefill, ping-pong Q tiles)
  AttentionDecode,    // attn_decode.cu (bf16 split-KV streaming, cfg3)
  QuantGemmSm100,     // gemm_sm100.cu (e4m3 kind::f8f6f4, cfg4)
  RmsGemmSm100,       // gemm_sm100.cu (bf16 kind::f16, cfg5)
  MoeRouting,         // moe.cu (softmax stats + top-k, bit-exact indices)
  LayerNormGemmSm100, // gemm_sm100.cu (bf16, 2-SM; variance cascade + GEMM)
  RowStats,           // rowstats.cu (variance / sum_sum / moments: HBM streaming)
  MoeRouter,          // router.cu (tcgen05 split-K router GEMM + routing cascade)
  MlaDecode,          // mla.cu (tcgen05 MLA decode, 128 heads share the latent cache)
  FusedRows,          // fused_seg.cu (run_fused: non-incremental level-1 segments, row patterns)
};

// run_fused (fused_seg.cu): on-chip buffer of one level-1 segment (one warp's
// registers) and the most segment partial states one CTA keeps in shared memory.
constexpr int64_t kSegMax = 1024;
constexpr int64_t kFusedSegsMax = 8192;
cudaError_t launch_fused_rows(int pattern, const float* a, const float* b, int64_t rows, int64_t n,
                              int64_t nseg, double c, double eps, float* d1, float* d2,
                              cudaStream_t st);

// MoE router (router.cu): scores = X W^T-packed, then the routing cascade.
struct RouterArgs {
  const void* x;        // [rows, hd] bf16
  const void* w;        // packed [experts, hd] bf16
  float* part;          // split partials [splits, part_stride, experts] (+ row offset)
  unsigned long long* cnt;  // per-row-tile arrival counters (zeroed at plan creation, only grow)
  int64_t rows, hd, experts, splits, part_stride;
  int k;                // K' (top-k size)
  float* d1;
  float* d2;
  void* topk;           // [rows, K'] {f32 value, i32 1-based index}
  float* scores;        // [rows, experts] f32 or null
};
cudaError_t launch_router(const RouterArgs& a, cudaStream_t st);

// MLA decode (mla.cu): 128 heads, cache rows [c_kv 512 | k_rope 64].
struct MlaArgs {
  const void* q;    // [bs, 128, 576] bf16
  const void* kv;   // [bs, skv, 576] bf16 (K = whole row, V = first 512)
  void* o;          // [bs, 128, 512] bf16 (nslices == 1)
  float* m;
  float* l;
  float* part_m;    // [nslices, rows_total] (nslices > 1)
  float* part_l;
  float* part_o;    // [nslices, rows_total, 512]
  unsigned long long* cnt;  // [bs, 2] arrival counters (zeroed at plan creation; multiples of 128 between launches)
  int64_t bs, skv, nslices, rows_total;
  float scale;
};
cudaError_t launch_mla_decode(const MlaArgs& a, cudaStream_t st);
bool mla_supports(int64_t heads, int64_t skv, int64_t dv, int64_t dqk, int64_t segments);
int64_t mla_pick_splits(int64_t bs, int64_t skv, int64_t segments);
bool router_supports(int64_t rows, int64_t hd, int64_t experts, int64_t k);
int64_t router_pick_splits(int64_t rows, int64_t hd);

// Row-statistics cascades (rowstats.cu): a = x | x1 | mass, b = - | x2 | pos.
struct RowStatsArgs {
  int pattern;  // RF_PATTERN_VARIANCE / SUM_SUM / MOMENTS
  const float* a;
  const float* b;
  int64_t rows, len, free_len;
  float* d1;
  float* d2;
  float* d3;
  double c, eps;  // sum_sum: sqrt(max(d1 - c, eps))
};
cudaError_t launch_rowstats(const RowStatsArgs& r, cudaStream_t st);

// ---- kernel launchers (stream-ordered; return cudaGetLastError()) ----------

// Safe softmax over rows (single pass, Eq.17 per element + Eq.16 merges).
cudaError_t launch_softmax_rows(const float* x, int64_t rows, int64_t n, float* d1,
                                float* d2, cudaStream_t st);

// fp32 attention, paper form. Slices [slice_begin, slice_begin+nslices) of a
// `segments`-way split of Skv. If part_* are null (segments == 1) the final
// O/m/l are written, else partials at slice index (s - part_base).
struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* m;
  float* l;
  float* part_m;
  float* part_l;
  float* part_o;
  int64_t bh, sq, skv, d;
  int64_t segments, slice_begin, nslices, part_base;
  int64_t rows_total;  // bh * sq (stride of the partial buffers)
  float scale;
  int dtype;
};
cudaError_t launch_attention_f32(const AttnArgs& a, cudaStream_t st);
// fp32 on tcgen05 (3xTF32) with the slice fold inside the kernel (one launch).
cudaError_t launch_attention_tf32(const AttnArgs& a, cudaStream_t st);
bool attention_tf32_supports(int64_t sq, int64_t skv, int64_t d, int64_t nslices);
cudaError_t launch_attention_decode(const AttnArgs& a, cudaStream_t st);
// Returns cudaErrorNotSupported when the shape has no tcgen05 instantiation.
cudaError_t launch_attention_sm100(const AttnArgs& a, cudaStream_t st);
bool attention_sm100_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments);
// experimental/attn_sm100_qt.cu (not in librf_cuda: Q in TMEM, measured slower)
cudaError_t launch_attention_qt(const AttnArgs& a, cudaStream_t st);
bool attention_qt_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments);
// experimental/attn_sm100_2sm.cu (probe library only; not in librf_cuda)
cudaError_t launch_attention_sm100_2sm(const AttnArgs& a, cudaStream_t st);
bool attention_sm100_2sm_supports(int64_t sq, int64_t skv, int64_t d, int64_t segments);

// Slice-ordered fold of partial (m, l, O) states (incr_push_child).
cudaError_t launch_attention_merge(const float* pm, const float* pl, const float* po,
                                   int64_t nslices, int64_t rows, int64_t stride, int64_t d,
                                   float* m, float* l, void* o, int out_dtype,
                                   cudaStream_t st);

cudaError_t launch_moe_routing(const float* s, int64_t rows, int64_t experts, int k, float* d1,
                               float* d2, void* topk, cudaStream_t st);

// GEMM patterns.
struct GemmArgs {
  const void* a;       // [M,K] bf16
  const void* b;       // packed [N,K] (e4m3 or bf16)
  float* d1;           // [M]
  float* d2;           // [M] (layernorm: sum x^2)
  void* c;             // [M,N] (f32 for quant, bf16 for rms / layernorm d3)
  void* c4;            // [M,N] bf16 (layernorm d4; may be null)
  const float* colsum; // [N] (layernorm: column sums of the packed g*w)
  int* domain_flag;    // device int, set to 1 on 0/0 at finalize
  int64_t m, n, k;
  int64_t stat_len;    // rms / layernorm: K of the statistics' means (0 = k)
  float fmax, eps;
  // Multi-Segment (segments > 1): split-K slice partials + ordered fold
  int64_t segments;    // S (1 = single segment)
  int64_t ws_rows;     // rows between slices in the workspace (the plan's M)
  float* ws;           // [S, ws_rows, N] f32 slice accumulators (this call's row offset applied)
  float* ws_d1;        // [S, ws_rows] slice statistic (sum x^2 | sum x | absmax)
  float* ws_d2;        // [S, ws_rows] layernorm: slice sum x^2
};
// Folds the S slice partials of a GEMM pattern in slice order (gemm_fold.cu).
cudaError_t launch_gemm_fold(int pattern, const GemmArgs& g, cudaStream_t st);
cudaError_t launch_quant_gemm_sm100(const GemmArgs& g, cudaStream_t st);
cudaError_t launch_rms_gemm_sm100(const GemmArgs& g, cudaStream_t st);
cudaError_t launch_layernorm_gemm_sm100(const GemmArgs& g, cudaStream_t st);
bool gemm_sm100_supports(int pattern, int64_t m, int64_t n, int64_t k);

// Weight packing (plan time).
cudaError_t launch_pack_e4m3(const float* w, int64_t k, int64_t n, uint8_t* packed,
                             cudaStream_t st);
cudaError_t launch_pack_rms(const float* w, const float* g, int64_t k, int64_t n,
                            void* packed_bf16, cudaStream_t st);
// column sums of a packed bf16 [N,K] weight -> colsum [N] f32
cudaError_t launch_colsum(const void* packed_bf16, int64_t k, int64_t n, float* colsum,
                          cudaStream_t st);

}  // namespace rf
