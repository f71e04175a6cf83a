// TEST INFRASTRUCTURE: the drop-in check. Runs the reference's own workloads
// (generators from proj/src/workloads.cpp, the RMSNorm DSL cascade) through
// BOTH the reference executors (run_incremental / run_multisegment) and the
// reference-side CUDA binding (integration/redfuse_cuda.cpp -> librf_cuda),
// and compares them with the reference's own compare_reports — values AND the
// load counters (input_load_delta / dep_root_delta must be 0).
// Built by oracle/Makefile into oracle/_ref/dropin_check; run on the GPU box
// by tests/test_gpu_dropin.py. Prints one JSON object per case.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include "../integration/redfuse_cuda.hpp"
#include "redfuse/workloads.hpp"

using namespace redfuse;

static int failures = 0;

// tol > 0: gate on compare_reports' scaled max error (fp32 paths).
// tol < 0: low-precision operands vs the UNROUNDED reference: gate on the RMS
// relative error of the last output (|tol|), report the scaled max error.
static void report(const std::string& name, const std::string& mode, const ExecReport& ref,
                   const ExecReport& cuda, double tol) {
  DiffReport d = compare_reports(cuda, ref, tol > 0 ? tol : 1e300);
  long long dl = 0, dd = 0;
  for (const auto& [k, v] : d.input_load_delta) dl += v < 0 ? -v : v;
  for (const auto& [k, v] : d.dep_root_delta) dd += v < 0 ? -v : v;
  double num = 0, den = 0;
  const auto& a = cuda.outputs.back().v;
  const auto& b = ref.outputs.back().v;
  for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  const double rms = den > 0 ? std::sqrt(num / den) : std::sqrt(num);
  const bool ok = (tol > 0 ? d.pass : rms <= -tol) && dl == 0 && dd == 0;
  if (!ok) ++failures;
  std::printf(
      "{\"case\": \"%s\", \"mode\": \"%s\", \"max_rel_err\": %.3e, \"rms_rel_err\": %.3e, "
      "\"gate\": \"%s %.1e\", \"worst\": \"%s\", \"input_load_delta\": %lld, \"dep_root_delta\": "
      "%lld, \"pass\": %s}\n",
      name.c_str(), mode.c_str(), d.max_rel_err, rms, tol > 0 ? "max_rel" : "rms_rel",
      tol > 0 ? tol : -tol, d.worst.c_str(), dl, dd, ok ? "true" : "false");
}

static void check_workload(const std::string& name, const Workload& w, double tol,
                           std::initializer_list<long long> segs, int seeds) {
  FusedProgram prog = derive_fused(w.spec);
  const long long l0 = w.spec.axis_len();
  for (int seed = 100; seed < 100 + seeds; ++seed) {
    for (const TreeConfig& cfg : {TreeConfig{{l0, 1}}, TreeConfig{{l0, l0 / 8, 1}}}) {
      TensorStore a = w.generate(seed), b = w.generate(seed);
      report(name + "/s" + std::to_string(seed) + "/L" + std::to_string(cfg.depth()), "incremental",
             run_incremental(prog, cfg, a), run_cuda(prog, cfg, b), tol);
      for (long long s : segs) {
        TensorStore c = w.generate(seed), d = w.generate(seed);
        report(name + "/s" + std::to_string(seed), "multi:" + std::to_string(s),
               run_multisegment(prog, cfg, s, c), run_cuda_multisegment(prog, cfg, s, d), tol);
      }
    }
  }
}

// run_fused (fusion at level k, simulator.cpp:485-559) against
// redfuse::run_cuda_fused at every level of each tree (levels[1..K]).
static void check_fused(const std::string& name, const Workload& w, double tol,
                        std::initializer_list<std::vector<long long>> trees, int seeds) {
  FusedProgram prog = derive_fused(w.spec);
  const long long l0 = w.spec.axis_len();
  for (int seed = 100; seed < 100 + seeds; ++seed)
    for (const auto& t : trees) {
      std::vector<long long> levels{l0};
      std::string tag;
      for (long long x : t) {
        levels.push_back(x);
        tag += "-" + std::to_string(x);
      }
      for (int k = 1; k <= static_cast<int>(t.size()); ++k) {
        TensorStore a = w.generate(seed), b = w.generate(seed);
        report(name + "/s" + std::to_string(seed) + "/tree" + tag, "fused@" + std::to_string(k),
               run_fused(prog, TreeConfig{levels}, k, a), run_cuda_fused(prog, TreeConfig{levels}, k, b), tol);
      }
    }
}

// A DSL cascade with uniform(-1, 1) inputs (the reference CLI's generator).
Workload dsl_workload(const std::string& name, const std::string& dsl) {
  CascadeSpec spec = parse_cascade(dsl);
  Workload w;
  w.name = name;
  w.spec = spec;
  w.generate = [spec](std::uint64_t seed) {
    TensorStore st;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (const auto& in : spec.inputs) {
      std::vector<double> v(in.len * (in.free_len > 0 ? in.free_len : 1));
      for (auto& x : v) x = u(rng);
      st.define(in.name, in.len, in.free_len, v);
    }
    return st;
  };
  return w;
}

int main() {
  // fp32 paths: the north_star's 1e-5
  check_workload("attention_256x64", make_attention(256, 64), 1e-5, {2, 4, 8}, 3);
  check_workload("attention_1024x64", make_attention(1024, 64), 1e-5, {8}, 1);
  check_workload("attention_128x128", make_attention(128, 128), 1e-5, {2}, 1);
  check_workload("safe_softmax_1024", make_safe_softmax(1024), 1e-5, {2, 4, 8}, 3);
  // bf16 / e4m3 operand paths: the reference here is evaluated on UNROUNDED
  // inputs, so the gap is the operands' rounding (e4m3: 3 mantissa bits); the
  // 2e-2 same-rounded-input gate is tests/test_gpu_gemm.py. Gated on RMS
  // relative error.
  check_workload("quant_gemm_512x256", make_quant_gemm(512, 256), -0.06, {}, 2);
  check_workload("rmsnorm_gemm_256x48",
                 dsl_workload("rmsnorm_gemm",
                              "cascade rmsnorm_gemm\ninput x len 256\ninput g len 256\n"
                              "input w len 256 free 48\nconst INVK = 0.00390625\nconst EPS = 1e-6\n"
                              "reduce 1 op sum\n    x[l] * x[l]\nreduce 2 op sum free 48\n"
                              "    x[l] * g[l] / sqrt(d1 * INVK + EPS) * w[l, f]\n"),
                 -0.02, {}, 2);
  {
    const std::string sig = "sqrt(d2 * INVK - d1 * INVK * d1 * INVK + EPS)";
    check_workload("layernorm_gemm_256x48",
                   dsl_workload("layernorm_gemm",
                                "cascade layernorm_gemm\ninput x len 256\ninput g len 256\n"
                                "input w len 256 free 48\nconst INVK = 0.00390625\n"
                                "const EPS = 1e-5\nreduce 1 op sum\n    x[l]\n"
                                "reduce 2 op sum\n    x[l] * x[l]\nreduce 3 op sum free 48\n"
                                "    x[l] * g[l] * w[l, f] / " + sig +
                                    "\nreduce 4 op sum free 48\n    d1 * INVK * g[l] * w[l, f] / " +
                                    sig + "\n"),
                   -0.02, {}, 2);
  }
  // MoE routing: top-k indices must match exactly (compare_reports' index check)
  check_workload("moe_routing_128x8", make_moe_routing(128, 8), 1e-5, {2, 4}, 3);
  check_workload("moe_routing_64x6", make_moe_routing(64, 6), 1e-5, {2}, 2);
  // the remaining builtins: row-statistics kernels (fp32 path)
  check_workload("variance_8192", builtin("variance"), 1e-5, {2, 8}, 3);
  check_workload("sum_sum_1024", builtin("sum_sum"), 1e-5, {2, 8}, 3);
  check_workload("moment_of_inertia_1024", builtin("moment_of_inertia"), 1e-5, {2, 8}, 3);
  // run_fused: level-1 segments evaluated non-incrementally on chip
  check_fused("attention_256x64", make_attention(256, 64), 1e-5, {{4, 1}, {16, 4, 1}, {128, 1}}, 2);
  check_fused("attention_128x128", make_attention(128, 128), 1e-5, {{2, 1}}, 1);
  check_fused("safe_softmax_1024", make_safe_softmax(1024), 1e-5, {{32, 4, 1}, {8, 1}, {1}}, 2);
  check_fused("variance_8192", builtin("variance"), 1e-5, {{16, 4, 1}, {64, 1}}, 2);
  check_fused("sum_sum_1024", builtin("sum_sum"), 1e-5, {{4, 1}, {32, 8, 1}}, 2);
  check_fused("quant_gemm_512x256", make_quant_gemm(512, 256), -0.06, {{4, 1}}, 1);
  check_fused("rmsnorm_gemm_256x48",
              dsl_workload("rmsnorm_gemm",
                           "cascade rmsnorm_gemm\ninput x len 256\ninput g len 256\n"
                           "input w len 256 free 48\nconst INVK = 0.00390625\nconst EPS = 1e-6\n"
                           "reduce 1 op sum\n    x[l] * x[l]\nreduce 2 op sum free 48\n"
                           "    x[l] * g[l] / sqrt(d1 * INVK + EPS) * w[l, f]\n"),
              -0.02, {{4, 1}, {2, 1}}, 1);
  // a level-1 segment longer than the on-chip buffer: NotFusable (non-incremental
  // fusion is only feasible for short segments)
  {
    Workload w = make_attention(256, 64);
    FusedProgram prog = derive_fused(w.spec);
    bool threw = false;
    try {
      TensorStore st = w.generate(1);
      run_cuda_fused(prog, TreeConfig{{256, 2, 1}}, 1, st);  // 128-key segments > the 64-key fp32 tile
    } catch (const NotFusable&) {
      threw = true;
    }
    if (!threw) ++failures;
    std::printf("{\"case\": \"attention_256x64/tree-2-1\", \"mode\": \"fused-too-long\", \"not_fusable\": %s}\n",
                threw ? "true" : "false");
  }
  // a cascade with no kernel: NotFusable from the binding (no CPU fallback)
  {
    Workload w = dsl_workload("prod_chain", "cascade prod_chain\ninput x len 64\n"
                                            "reduce 1 op prod\n    x[l]\nreduce 2 op sum\n    x[l] / d1\n");
    bool threw = false;
    try {
      FusedProgram prog = derive_fused(w.spec);
      TensorStore st = w.generate(1);
      run_cuda(prog, TreeConfig{{64, 1}}, st);
    } catch (const NotFusable&) {
      threw = true;
    }
    if (!threw) ++failures;
    std::printf("{\"case\": \"prod_chain\", \"mode\": \"no-kernel\", \"not_fusable\": %s}\n",
                threw ? "true" : "false");
  }
  // the batched drop-in: R reference rows in one librf_cuda run, each row's
  // report against the reference executor on that row's store
  auto check_batched = [&](const std::string& name, const Workload& w, double tol, int rows,
                           long long segs, bool share_static) {
    FusedProgram prog = derive_fused(w.spec);
    const long long l0 = w.spec.axis_len();
    std::vector<TensorStore> stores, refs;
    for (int r = 0; r < rows; ++r) {
      TensorStore st = w.generate(200 + r);
      if (share_static && r > 0)  // the GEMM weight (and gamma) are shared by the batch
        for (const char* nm : {"w", "g"})
          if (stores[0].has(nm)) {
            const auto& a = stores[0].array(nm);
            st.define(nm, a.len, a.free_len, a.data);
          }
      stores.push_back(st);
      refs.push_back(st);
    }
    TreeConfig cfg{{l0, 1}};
    std::vector<ExecReport> got = run_cuda_batched(prog, cfg, stores, segs);
    for (int r = 0; r < rows; ++r) {
      ExecReport want = segs == 1 ? run_incremental(prog, cfg, refs[r]) : run_multisegment(prog, cfg, segs, refs[r]);
      report(name + "/row" + std::to_string(r), "batched:" + std::to_string(segs), want, got[r], tol);
    }
  };
  check_batched("attention_256x64", make_attention(256, 64), 1e-5, 16, 1, false);
  check_batched("attention_256x64", make_attention(256, 64), 1e-5, 8, 4, false);
  check_batched("safe_softmax_1024", make_safe_softmax(1024), 1e-5, 32, 1, false);
  check_batched("moe_routing_128x8", make_moe_routing(128, 8), 1e-5, 32, 1, false);
  check_batched("quant_gemm_512x256", make_quant_gemm(512, 256), -0.06, 200, 1, true);
  check_batched("variance_8192", builtin("variance"), 1e-5, 8, 2, false);
  check_batched("sum_sum_1024", builtin("sum_sum"), 1e-5, 8, 1, false);
  check_batched("rmsnorm_gemm_256x48",
                dsl_workload("rmsnorm_gemm",
                             "cascade rmsnorm_gemm\ninput x len 256\ninput g len 256\n"
                             "input w len 256 free 48\nconst INVK = 0.00390625\nconst EPS = 1e-6\n"
                             "reduce 1 op sum\n    x[l] * x[l]\nreduce 2 op sum free 48\n"
                             "    x[l] * g[l] / sqrt(d1 * INVK + EPS) * w[l, f]\n"),
                -0.02, 130, 1, true);
  // a FusedProgram whose derived correction is not the kernel's closed form
  // (here: attention's d3 correction with the exponent's sign flipped) is
  // rejected at plan time (rfcuda::check_corrections), never run
  {
    Workload w = make_attention(256, 64);
    FusedProgram prog = derive_fused(w.spec);
    for (auto& d : prog.decomps)
      if (d.id == 3) d.corr = exp_of(dep_var(1) - dep_var(1, true)) * (dep_var(2, true) / dep_var(2));
    bool threw = false;
    try {
      TensorStore st = w.generate(1);
      run_cuda(prog, TreeConfig{{256, 1}}, st);
    } catch (const NotFusable&) {
      threw = true;
    }
    if (!threw) ++failures;
    std::printf("{\"case\": \"attention_bad_corr\", \"mode\": \"corr-pin\", \"not_fusable\": %s}\n",
                threw ? "true" : "false");
  }
  std::printf("{\"failures\": %d}\n", failures);
  return failures ? 1 : 0;
}
