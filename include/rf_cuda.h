/* librf_cuda — C-ABI of the B200 (sm_100a) fused cascaded-reduction executors.
 *
 * Drop-in boundary for the reference's CPU fused-loop executors (RedFuser
 * artifact, /root/reference/proj). The reference has no FFI/plugin layer; its
 * operator API is C++:
 *
 *   ExecReport run_incremental(const FusedProgram&, const TreeConfig&, TensorStore&)
 *       proj/include/redfuse/simulator.hpp:76-77, proj/src/simulator.cpp:631-658
 *   ExecReport run_multisegment(const FusedProgram&, const TreeConfig&,
 *                               long long num_segments, TensorStore&)
 *       proj/include/redfuse/simulator.hpp:81-82, proj/src/simulator.cpp:660-687
 *   FusedProgram derive_fused(const CascadeSpec&, const ProbeConfig&)
 *       proj/include/redfuse/acrf.hpp:93-94 (plan time; stays on the host)
 *
 * This library replaces the *executors* (the per-element interpretive loop,
 * simulator.cpp:566-621) with one hand-written kernel per fusible pattern; the
 * host plan layer (C++ or the Python mirror) maps a FusedProgram / cascade
 * onto an rf_desc and calls rf_plan_create + rf_run. INTEGRATION.md shows the
 * reference-side binding.
 *
 * Conventions
 *  - Plain C types only; device pointers are `void*`, streams are the CUDA
 *    runtime handle passed as `void*` (cudaStream_t), 0 = legacy default.
 *  - Every call is stream-ordered and non-blocking unless it says otherwise.
 *    Plans are immutable after creation (one plan per device). A plan owns its
 *    split workspace and host-path staging, so rf_run / rf_run_host calls on
 *    ONE plan must be ordered (same stream or events); use one plan per
 *    stream for concurrent execution. (The MoE router's and MLA decode's
 *    kernels also keep arrival counters in the plan workspace; they rely on
 *    this ordering to tell one launch's arrivals from the next one's.)
 *  - No exceptions cross the boundary. Errors are rf_status codes that the
 *    host layer maps back onto the reference's exception types:
 *      RF_ERR_SHAPE        -> redfuse::ShapeMismatch          (simulator.hpp:17-19)
 *      RF_ERR_SEGMENTATION -> redfuse::IncompatibleSegmentation (simulator.hpp:21-23)
 *      RF_ERR_DOMAIN       -> redfuse::DomainError            (expr.hpp:29-31)
 *      RF_ERR_UNSUPPORTED  -> redfuse::NotFusable-like "no kernel for this pattern"
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns RF_ERR_CUDA.
 *
 * Outputs are named by reduction id like the reference's ExecReport.outputs
 * (simulator.hpp:49-61): io.d[0] is d1, io.d[1] is d2, io.d[2] is d3.
 */
#ifndef RF_CUDA_H
#define RF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RF_CUDA_ABI_VERSION 5

typedef enum rf_status {
  RF_OK = 0,
  RF_ERR_SHAPE = 1,        /* ShapeMismatch: dims/strides/pointers disagree with the desc */
  RF_ERR_SEGMENTATION = 2, /* IncompatibleSegmentation: segments do not divide L0 */
  RF_ERR_DOMAIN = 3,       /* DomainError at finalize (e.g. absmax == 0 -> 0/0) */
  RF_ERR_UNSUPPORTED = 4,  /* pattern / dtype / shape has no kernel */
  RF_ERR_CUDA = 5,         /* CUDA runtime/driver failure or no sm_100 device */
  RF_ERR_NCCL = 6,         /* reserved for the cross-GPU merge */
  RF_ERR_ARG = 7           /* null / malformed argument */
} rf_status;

/* Fusible cascade patterns with a kernel (plan layer matches FusedPrograms
 * onto these; see include/rf_host.hpp plan() and DESIGN.md). */
typedef enum rf_pattern {
  /* d1 = max x, d2 = sum exp(x - d1)          (make_safe_softmax, workloads.cpp:38-62) */
  RF_PATTERN_SAFE_SOFTMAX = 1,
  /* d1 = max P, d2 = sum e^(P-d1), d3 = sum e^(P-d1)/d2 V  with P = scale Q K^T
   *                                           (make_attention, workloads.cpp:66-120)   */
  RF_PATTERN_ATTENTION = 2,
  /* d1 = max|a|, d2[f] = sum (fmax a/d1) w[l,f], a quantised to e4m3 per K tile with
   * the running d1                            (make_quant_gemm, workloads.cpp:173-209) */
  RF_PATTERN_QUANT_GEMM_E4M3 = 3,
  /* d1 = sum x^2, d2[f] = sum x g / sqrt(d1/K + eps) w[l,f]   (DSL cascade) */
  RF_PATTERN_RMSNORM_GEMM = 4,
  /* d1 = max s, d2 = sum exp(s - d1), d3 = top-K' of s, ties to the lowest index
   *                                           (make_moe_routing, workloads.cpp:124-169) */
  RF_PATTERN_MOE_ROUTING = 5,
  /* LayerNorm statistics -> GEMM, the variance cascade (workloads.cpp:246-277) extended:
   * d1 = sum x, d2 = sum x^2, sigma = sqrt(d2/K - (d1/K)^2 + eps),
   * d3[f] = sum x g w[l,f] / sigma, d4[f] = sum (d1/K) g w[l,f] / sigma;
   * LayerNorm(x) . W = d3 - d4                    (DSL cascade) */
  RF_PATTERN_LAYERNORM_GEMM = 6,
  /* d1 = sum x, d2 = sum x^2                      (make_variance, workloads.cpp:246-277) */
  RF_PATTERN_VARIANCE = 7,
  /* d1 = sum x1^2, d2 = sum x1 x2 / sqrt(max(d1 - c, eps)), c = desc.offset
   *                                               (make_sum_sum, workloads.cpp:213-242)   */
  RF_PATTERN_SUM_SUM = 8,
  /* d1 = sum m, d2[f] = sum m p[l,f], d3[f] = sum m p[l,f]^2, free_len <= 8
   *                                               (data/moment_of_inertia.cascade)        */
  RF_PATTERN_MOMENTS = 9,
  /* MoE router: scores s = X W (the router GEMM; a producer of the
   * cascade input) feeding the MOE_ROUTING cascade: d1 = max s, d2 = sum exp(s - d1),
   * d3 = top-K' of s, ties to the lowest index. len = experts (32/64/128/256),
   * free_len = K' <= 8, producer_len = hd (the GEMM's reduce axis, % 64)      */
  RF_PATTERN_MOE_ROUTER = 10,
  /* MLA decode (absorbed multi-latent attention, the paper's L1-L9):
   * the ATTENTION cascade with P = scale q K^T over cache rows K = [c_kv | k_rope]
   * (producer_len = 576 wide) and V = c_kv (their first free_len = 512 columns);
   * heads = 128 queries per batch share the cache, rows = 1, len = Skv      */
  RF_PATTERN_MLA_DECODE = 11
} rf_pattern;

typedef enum rf_dtype { RF_F32 = 0, RF_BF16 = 1, RF_E4M3 = 2 } rf_dtype;

/* Pattern descriptor: the batched shape of one cascade family.
 * "row" = one reference cascade instance (one TensorStore in the reference). */
typedef struct rf_desc {
  int32_t pattern;   /* rf_pattern */
  int32_t dtype;     /* rf_dtype of the streamed inputs */
  int64_t batch;     /* attention: B            others: 1 */
  int64_t heads;     /* attention: H            others: 1 */
  int64_t rows;      /* attention: Sq (queries per (b,h)); GEMM patterns: M / T tokens;
                        softmax: number of rows */
  int64_t len;       /* L0 = reduce-axis length: Skv, K, or softmax n */
  int64_t free_len;  /* lanes of the free axis: head_dim D or N (softmax: 0) */
  int64_t segments;  /* Multi-Segment strategy S (run_multisegment); 1 = single segment */
  double fmax;       /* quant: FMAX (448 for e4m3) */
  double eps;        /* rmsnorm / layernorm / sum_sum: epsilon */
  double softmax_scale; /* attention: P = scale * Q K^T (reference stores Q pre-scaled: 1.0) */
  double offset;        /* sum_sum: c in sqrt(max(d1 - c, eps)) */
  int32_t tile_rows;    /* 0 = kernel default (reference pick_tile: 128) */
  int32_t tile_stream;  /* 0 = kernel default */
  int32_t device;       /* CUDA ordinal the plan is bound to */
  int32_t producer_len; /* MOE_ROUTER: hd, the reduce axis of the producer GEMM;
                           MLA_DECODE: the q / cache row width (576) (ABI v3;
                           was `reserved` in v2, same offset) */
  int64_t stat_len;     /* RMSNORM / LAYERNORM: the K of the statistics' means
                           d1/K, d2/K (0 = len). A host that zero-pads the reduce
                           axis to the kernel's K tile passes the cascade's own
                           L0 here (zeros add nothing to sum x, sum x^2). (ABI v4) */
  /* Fusion at level k, the non-incremental executor run_fused(prog, cfg, k, store)
   * (proj/src/simulator.cpp:485-559). 0 = the incremental
   * executors above. k >= 1: the reduction tree is tree[0..tree_depth-1] =
   * TreeConfig.levels[1..K] (L0 = len is implicit, tree[K-1] must be 1, every
   * width divides the one below it, 1 <= k <= K). Each level-1 segment of
   * len / tree[0] elements is buffered on chip and evaluated non-incrementally
   * with its own dependency values (fused_level1_segment, :430-457); the
   * segment partials are then corrected and folded in segment order (the
   * group combines of levels 2..k, :461-481, and the bridge to the final
   * dependency values, :510-536, are one closed-form fold — equal in exact
   * arithmetic). A segment longer than the pattern's on-chip buffer is
   * RF_ERR_UNSUPPORTED, as non-incremental fusion is only feasible for short
   * segments. `segments` must be 1. (ABI v5) */
  int32_t fuse_level;
  int32_t tree_depth;   /* K, 1..8 */
  int64_t tree[8];
} rf_desc;

/* Device buffers for one rf_run. Inputs by pattern:
 *   SAFE_SOFTMAX   in[0] = x [rows, len] f32
 *   ATTENTION      in[0] = Q [B,H,Sq,D], in[1] = K [B,H,Skv,D], in[2] = V [B,H,Skv,D]
 *                  (f32 or bf16, contiguous); d1 = m [B,H,Sq] f32, d2 = l f32,
 *                  d3 = O [B,H,Sq,D] (input dtype)
 *   QUANT_GEMM     in[0] = A [M,K] bf16, in[1] = packed W (rf_pack_weight, e4m3 [N,K]);
 *                  d1 = amax [M] f32, d2 = C [M,N] f32
 *   RMSNORM_GEMM   in[0] = X [T,K] bf16, in[1] = packed W (rf_pack_weight: g folded,
 *                  bf16 [N,K]); d1 = sum x^2 [T] f32, d2 = Y [T,N] bf16
 *   LAYERNORM_GEMM in[0] = X [T,K] bf16, in[1] = packed W (rf_pack_weight: bf16 [N,K] of
 *                  g*w followed by N f32 column sums); d1 = sum x [T] f32, d2 = sum x^2
 *                  [T] f32, d3 = [T,N] bf16, d4 = [T,N] bf16 (optional: may be null)
 *   MOE_ROUTING    in[0] = logits [rows, experts] f32 (len = experts, free_len = K' <= 8);
 *                  d1, d2 [rows] f32; d3 = [rows, K'] records {f32 value, i32 index}
 *                  (1-based expert index like OutputVal.topk; 0 = empty slot)
 *   MOE_ROUTER     in[0] = X [rows, hd] bf16, in[1] = packed W (rf_pack_weight: w [hd, en]
 *                  f32 -> bf16 [en, hd]); d1, d2, d3 as MOE_ROUTING; d4 = the scores s
 *                  [rows, en] f32 (optional: may be null)
 *   MLA_DECODE     in[0] = q [B, 128, 576] bf16, in[1] = cache [B, Skv, 576] bf16;
 *                  d1 = m [B, 128] f32, d2 = l f32, d3 = O [B, 128, 512] bf16
 *   VARIANCE       in[0] = x [rows, len] f32; d1, d2 [rows] f32
 *   SUM_SUM        in[0] = x1, in[1] = x2 [rows, len] f32; d1, d2 [rows] f32
 *   MOMENTS        in[0] = mass [rows, len] f32, in[1] = pos [rows, len, free_len] f32;
 *                  d1 [rows], d2, d3 [rows, free_len] f32                             */
typedef struct rf_io {
  const void* in[4];
  void* d[4];
} rf_io;

/* Host-memory variant of rf_io (the reference's TensorStore lives on the host):
 * same layouts and dtypes, host pointers (pinned memory gets full PCIe rate). */
typedef rf_io rf_host_io;

/* Split-KV partial states: one (m, l, O) per slice and row, slice-major:
 * m, l: [nslices, rows_total] f32, o: [nslices, rows_total, D] f32, where
 * rows_total = B*H*Sq. O is normalised by its own l (the paper form). */
typedef struct rf_partials {
  float* m;
  float* l;
  float* o;
  int64_t nslices;
} rf_partials;

typedef struct rf_plan rf_plan;

int rf_abi_version(void);
const char* rf_status_string(rf_status s);
/* Thread-local message of the last failing call on this thread ("" if none). */
const char* rf_last_error(void);

/* Validates the descriptor (shapes, S | L0, dtype support, device is sm_100),
 * picks the kernel and tile configuration, allocates the plan's persistent
 * workspace (segment partials) once. Blocking. */
rf_status rf_plan_create(const rf_desc* desc, rf_plan** out);
void rf_plan_destroy(rf_plan* plan);
/* Human-readable JSON: kernel name, tiles, grid, workspace bytes. */
rf_status rf_plan_describe(const rf_plan* plan, char* buf, size_t buflen);
/* Number of kernel launches one rf_run issues (for launch accounting). */
int64_t rf_plan_launches_per_run(const rf_plan* plan);
/* Byte sizes of every rf_io slot the plan reads (in[0..3]) and writes
 * (d[0..3]); 0 = slot unused. in[1] of the GEMM patterns is the packed weight
 * (rf_packed_bytes). Lets callers reject undersized buffers before rf_run
 * with the reference's ShapeMismatch (check_shapes, simulator.cpp:235-245)
 * instead of letting a kernel read out of bounds. (ABI v4) */
rf_status rf_plan_io_bytes(const rf_plan* plan, size_t in_bytes[4], size_t out_bytes[4]);

/* Plan-time weight packing for the GEMM patterns (outside any timed region):
 *   QUANT_GEMM:   w [K,N] f32 (reduce-axis major, the reference layout) ->
 *                 packed e4m3 [N,K] (RNE, satfinite; the static pre-rounded W)
 *   RMSNORM_GEMM: w [K,N] f32, g [K] f32 -> packed bf16 [N,K] of g[l]*w[l,f]
 *   LAYERNORM_GEMM: as RMSNORM_GEMM, followed by N f32 column sums of the packed
 *                 (bf16-rounded) g*w, at byte offset 2*N*K
 *   MOE_ROUTER:   w [hd, en] f32 -> packed bf16 [en, hd] (g unused)
 * `packed` must hold rf_packed_bytes(plan) bytes. Stream-ordered. */
rf_status rf_pack_weight(const rf_plan* plan, const void* w, const void* g, void* packed,
                         void* stream);
/* Bytes of the packed weight buffer for the plan's pattern (0 if none). */
size_t rf_packed_bytes(const rf_plan* plan);

/* Host-memory variant: uploads w (and g) from host memory, packs them into a
 * freshly allocated device buffer returned in *packed_dev (free it with
 * rf_buffer_free). Blocking. For host-side drop-in callers without CUDA. */
rf_status rf_pack_weight_host(const rf_plan* plan, const float* w, const float* g,
                              void** packed_dev);
void rf_buffer_free(void* dev_ptr);

/* The fused single-loop executor: run_incremental (segments == 1) or
 * run_multisegment (segments == S: S slice partials + in-order merge) over
 * every row of the batch. Stream-ordered, non-blocking. */
rf_status rf_run(const rf_plan* plan, const rf_io* io, void* stream);

/* End-to-end drop-in call on HOST buffers: H2D of the inputs, rf_run, D2H of
 * every output, pipelined in chunks over independent rows (copies overlap
 * kernels). Blocking: returns when the outputs are in host memory. The plan
 * owns the device staging buffers (allocated on first use). */
rf_status rf_run_host(rf_plan* plan, const rf_host_io* io);

/* Split-KV building blocks (attention only), for sharding the reduce axis
 * across CTAs or GPUs: compute the partial states of slices
 * [slice_begin, slice_begin + out->nslices) of a `segments`-way split. */
rf_status rf_run_partials(const rf_plan* plan, const rf_io* io, int64_t slice_begin,
                          rf_partials* out, void* stream);
/* Fold partial states in slice order (incr_push_child semantics,
 * simulator.cpp:592-608) and write d1/d2/d3 of io. */
rf_status rf_merge_partials(const rf_plan* plan, const rf_partials* in, const rf_io* io,
                            void* stream);

/* Reads (and clears) the plan's device-side domain flag after synchronising
 * the stream: RF_ERR_DOMAIN if any row hit a 0/0 at finalize since the last
 * check (reference: DomainError at finalize_root). Blocking. */
rf_status rf_check_domain(const rf_plan* plan, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RF_CUDA_H */
