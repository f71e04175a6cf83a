/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the fused cascaded-reduction
 * hot path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load this library, and only as the checker. The product path
 * (librf_cuda) never links or calls it.
 *
 * A plain-C restatement of the reference's CPU semantics (RedFuser artifact,
 * /root/reference/proj) for the patterns the CUDA kernels implement. Every
 * function cites the reference lines it restates. All arithmetic is float64
 * like the reference, except the explicitly named rounding emulations
 * (bf16 / e4m3 input rounding, the FP8 kernel's tile-wise quantisation), which
 * define "the reference evaluated on the same rounded inputs".
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by the reference itself (oracle/ref_driver.cpp ->
 * tests/golden/), so this restatement is pinned, not free-standing.
 */
#ifndef RF_ORACLE_H
#define RF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rounding helpers ---------------------------------------------------- */
/* float32 -> bf16 -> float32, round-to-nearest-even (NaN preserved). */
float rfo_round_bf16(float x);
/* float32 -> e4m3 (OCP FP8 E4M3FN), RNE, saturating to +-448, NaN -> NaN;
 * mirrors PTX cvt.rn.satfinite.e4m3x2.f32. Returns the value as float. */
float rfo_round_e4m3(float x);
void rfo_round_bf16_array(const double* in, double* out, int64_t n);
void rfo_round_e4m3_array(const double* in, double* out, int64_t n);

/* ---- safe softmax (proj/src/workloads.cpp:38-62) -------------------------- */
/* rows x n: d1 = max, d2 = sum exp(x - d1). */
void rfo_safe_softmax(const double* x, int64_t rows, int64_t n, double* d1, double* d2);

/* ---- attention ------------------------------------------------------------
 * Batched restatement of make_attention (proj/src/workloads.cpp:66-120) over
 * rows = (batch*heads*queries). q: [bh, sq, hd]; k, v: [bh, skv, hd].
 * P = q . K^T (fp64, the generator formula workloads.cpp:86-93) times
 * softmax_scale, then
 *   oracle form (workloads.cpp:101-118): m = max P, t = sum e^(P-m),
 *                                        O = sum e^(P-m)/t V
 * Outputs m, l: [bh*sq]; o: [bh*sq, hd].                                    */
void rfo_attention(const double* q, const double* k, const double* v, int64_t bh,
                   int64_t sq, int64_t skv, int64_t hd, double softmax_scale,
                   double* m, double* l, double* o, int threads);

/* The same rows through the reference's streaming executor semantics:
 * run_multisegment (proj/src/simulator.cpp:660-687) with `segments` equal
 * slices, each streamed by incr_ingest_element (566-589, Eq.17: store-prev,
 * correct by exp(d1'-d1) and exp(d1'-d1)*d2'/d2, reduce), merged in slice
 * order by incr_push_child (592-608, Eq.16). segments == 1 is run_incremental
 * on the flat tree (631-658). Throws nothing: returns -2 (IncompatibleSegmentation)
 * when segments does not divide skv.                                        */
int rfo_attention_incremental(const double* p, const double* v, int64_t rows,
                              int64_t kv, int64_t hd, int64_t segments, double* m,
                              double* l, double* o);

/* Associative combine of split-KV partial states (m_s, l_s, O_s), s in slice
 * order, into (m, l, O): incr_push_child semantics (simulator.cpp:592-608),
 * closed form of acceptance.cpp:162-178:
 *   m = max m_s;  l = sum l_s e^(m_s-m);  O = sum O_s e^(m_s-m) l_s / l.
 * part_m/part_l: [S, rows]; part_o: [S, rows, hd].                          */
void rfo_attention_merge(const double* part_m, const double* part_l,
                         const double* part_o, int64_t nslices, int64_t rows,
                         int64_t hd, double* m, double* l, double* o);

/* ---- per-token absmax -> FP8 quantise -> GEMM ------------------------------
 * Real-arithmetic oracle (make_quant_gemm, workloads.cpp:173-209):
 *   d1 = max|a|, c[f] = sum_l (fmax a[l]/d1) w[l,f]   (no rounding, no dequant)
 * a: [M, K] rows; w: [K, N] (reduce-axis major, the reference's layout).    */
void rfo_quant_gemm(const double* a, const double* w, int64_t M, int64_t K, int64_t N,
                    double fmax, double* d1, double* c, int threads);

/* The FP8 kernel's arithmetic restated (quant_gemm_sm100 in
 * paper_2603_10026_b200/csrc/gemm_sm100.cu). Per row, per K tile of width
 * tile_k: running absmax d1 (float32); H' reference ref = smallest power of
 * two >= d1; q_l = e4m3(fp32(a_l * fmax/ref)) (exact power-of-two scaling,
 * one RNE/satfinite rounding); acc = acc * ref'/ref + sum q_l w[l,f] (the
 * incremental form with corr = d1'/d1 evaluated on the H' proxy); finalize
 * c = acc * ref / d1 (finalize_root retarget, simulator.cpp:611-621).
 * w must already be e4m3-representable (static pre-rounded weight).
 * Rows whose absmax is 0 produce NaN (0/0), matching the reference's
 * DomainError at finalize_root.                                              */
void rfo_quant_gemm_e4m3(const double* a, const double* w, int64_t M, int64_t K,
                         int64_t N, double fmax, int64_t tile_k, double* d1, double* c,
                         int threads);

/* ---- RMSNorm statistics -> GEMM -------------------------------------------
 * The DSL cascade evaluated as run_unfused does
 * (simulator.cpp:377-421): d1 = sum x^2; y[f] = sum x g / sqrt(d1/K + eps) w[l,f]
 * x: [T, K]; g: [K]; w: [K, N].                                             */
void rfo_rmsnorm_gemm(const double* x, const double* g, const double* w, int64_t T,
                      int64_t K, int64_t N, double eps, double* d1, double* y,
                      int threads);

/* Incremental (streaming) form for one token: Eq.17 with
 * corr = sqrt(d1'/K + eps)/sqrt(d1/K + eps) (golden corrections.txt), used to
 * pin the restatement against the reference's run_incremental.              */
void rfo_rmsnorm_gemm_incremental(const double* x, const double* g, const double* w,
                                  int64_t K, int64_t N, double eps, double* d1,
                                  double* y);

/* ---- LayerNorm statistics -> GEMM -----------------------------------------
 * The 4-reduction DSL cascade, run_unfused order:
 *   d1 = sum x; d2 = sum x^2; sigma = sqrt(d2/K - (d1/K)^2 + eps)
 *   d3[f] = sum x g w[l,f] / sigma; d4[f] = sum (d1/K) g w[l,f] / sigma
 * (LayerNorm(x) @ W = d3 - d4). x: [T, K]; g: [K]; w: [K, N].               */
void rfo_layernorm_gemm(const double* x, const double* g, const double* w, int64_t T,
                        int64_t K, int64_t N, double eps, double* d1, double* d2, double* d3,
                        double* d4, int threads);

/* Incremental form for one token with the corrections derive_fused produces
 * (d3: sigma'/sigma; d4: (d1/d1') sigma'/sigma).                            */
void rfo_layernorm_gemm_incremental(const double* x, const double* g, const double* w,
                                    int64_t K, int64_t N, double eps, double* d1, double* d2,
                                    double* d3, double* d4);

/* ---- row statistics: the reference's remaining builtins ------------------- */
void rfo_variance(const double* x, int64_t rows, int64_t n, double* d1, double* d2);
void rfo_sum_sum(const double* x1, const double* x2, int64_t rows, int64_t n, double c,
                 double eps, double* d1, double* d2);
void rfo_moments(const double* mass, const double* pos, int64_t rows, int64_t n, int64_t F,
                 double* d1, double* d2, double* d3);

/* ---- MoE routing: softmax stats + top-k (workloads.cpp:124-169) -----------
 * Descending value, ties to the lowest index (test_workloads.cpp:210-224).
 * idx is 1-based like the reference's OutputVal.topk.                       */
void rfo_moe_routing(const double* s, int64_t rows, int64_t experts, int64_t k,
                     double* d1, double* d2, double* topk_val, int64_t* topk_idx);

/* ---- run_fused: fusion at level k (simulator.cpp:485-559) ----------------
 * The non-incremental executor on one row: the L0 elements are cut into
 * levels[1] level-1 segments, each evaluated with its OWN dependency values
 * (fused_level1_segment, :430-457); levels 2..k combine groups of children
 * corrected to the group's dependency values (fused_combine_group, :461-481);
 * the level-k partials are retargeted to the final values (the bridge,
 * :510-536) and folded plainly over levels k+1..K. levels[0] = L0,
 * levels[depth] = 1. pattern: 1 safe_softmax (a = x), 2 attention (a = P,
 * b = V [L0, hd]; d3 [hd]), 7 variance (a = x), 8 sum_sum (a = x1, b = x2,
 * c, eps). Returns -1 on a bad tree / level.                                  */
int rfo_fused_row(int pattern, const double* a, const double* b, int64_t hd, const int64_t* levels,
                  int depth, int k, double c, double eps, double* d1, double* d2, double* d3);

/* ---- parity metric (compare_reports, simulator.cpp:691-752) --------------- */
/* max over i of |x-y|/(1+max(|x|,|y|)); equal values (incl. matching infs)
 * count 0; NaN/inf mismatch is +inf. Returns the max, writes its index.     */
double rfo_scaled_max_err(const double* x, const double* y, int64_t n, int64_t* worst);

#ifdef __cplusplus
}
#endif
#endif /* RF_ORACLE_H */
