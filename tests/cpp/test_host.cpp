// C++ host-layer tests (include/rf_host.hpp over librf_cuda), written after
// the reference's own tests/test_simulator.cpp and tests/test_cascade.cpp so
// that the drop-in reads like the original:  ./test_host cpu | gpu
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <random>
#include <string>

#include "rf_host.hpp"

using namespace rfcuda;

static int failures = 0, checks = 0;
#define CHECK(c)                                                           \
  do {                                                                     \
    ++checks;                                                              \
    if (!(c)) {                                                            \
      ++failures;                                                          \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    ++checks;                                                              \
    bool ok = false;                                                       \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const T&) {                                                   \
      ok = true;                                                           \
    } catch (...) {                                                        \
    }                                                                      \
    if (!ok) {                                                             \
      ++failures;                                                          \
      std::printf("  FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                      \
  } while (0)
#define TEST(name) static void name()
#define RUN(name)                       \
  do {                                  \
    std::printf("[ run ] %s\n", #name); \
    name();                             \
  } while (0)

static std::string softmax_dsl(long long n) {
  return "cascade safe_softmax\ninput x len " + std::to_string(n) +
         "\nreduce 1 op max\n    x[l]\nreduce 2 op sum\n    exp(x[l] - d1)\n";
}
static std::string attention_dsl(long long kv, long long hd) {
  return "cascade attention\ninput P len " + std::to_string(kv) + "\ninput V len " +
         std::to_string(kv) + " free " + std::to_string(hd) +
         "\nreduce 1 op max\n    P[l]\nreduce 2 op sum\n    exp(P[l] - d1)\nreduce 3 op sum free " +
         std::to_string(hd) + "\n    exp(P[l] - d1) / d2 * V[l, f]\n";
}
static std::string quant_dsl(long long k, long long n) {
  return "cascade quant_gemm\ninput a len " + std::to_string(k) + "\ninput w len " + std::to_string(k) +
         " free " + std::to_string(n) + "\nconst FMAX = 448.0\nreduce 1 op max\n    abs(a[l])\n"
         "reduce 2 op sum free " + std::to_string(n) + "\n    (FMAX * a[l] / d1) * w[l, f]\n";
}
static std::string rms_dsl(long long k, long long n) {
  return "cascade rmsnorm_gemm\ninput x len " + std::to_string(k) + "\ninput g len " +
         std::to_string(k) + "\ninput w len " + std::to_string(k) + " free " + std::to_string(n) +
         "\nconst K = " + std::to_string(k) + "\nconst EPS = 1e-6\nreduce 1 op sum\n    x[l] * x[l]\n"
         "reduce 2 op sum free " + std::to_string(n) + "\n    x[l] * g[l] / sqrt(d1 / K + EPS) * w[l, f]\n";
}
static std::string ln_dsl(long long k, long long n, bool w_first = true) {
  const std::string sig = "sqrt(d2 * INVK - d1 * INVK * d1 * INVK + EPS)";
  const std::string kk = std::to_string(k), nn = std::to_string(n);
  char invk[64];
  std::snprintf(invk, sizeof invk, "%.17g", 1.0 / static_cast<double>(k));
  return "cascade layernorm_gemm\ninput x len " + kk + "\ninput g len " + kk + "\ninput w len " + kk +
         " free " + nn + "\nconst INVK = " + invk + "\nconst EPS = 1e-5\nreduce 1 op sum\n    x[l]\n" +
         "reduce 2 op sum\n    x[l] * x[l]\nreduce 3 op sum free " + nn + "\n    " +
         (w_first ? "x[l] * g[l] * w[l, f] / " + sig : "x[l] * g[l] / " + sig + " * w[l, f]") +
         "\nreduce 4 op sum free " + nn + "\n    " +
         (w_first ? "d1 * INVK * g[l] * w[l, f] / " + sig : "d1 * INVK * g[l] / " + sig + " * w[l, f]") +
         "\n";
}
static std::vector<double> random_vec(std::size_t n, std::uint64_t seed, double lo, double hi) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> d(lo, hi);
  std::vector<double> v(n);
  for (auto& x : v) x = d(rng);
  return v;
}

// ---------------------------------------------------------------- CPU-only --

TEST(dsl_files_parse_and_match_kernels) {
  // proj/data/*.cascade contents
  CHECK(plan(softmax_dsl(1024)).pattern == RF_PATTERN_SAFE_SOFTMAX);
  Program a = plan(attention_dsl(256, 64));
  CHECK(a.pattern == RF_PATTERN_ATTENTION && a.x == "P" && a.v == "V" && a.free_len == 64);
  Program q = plan(quant_dsl(512, 256));
  CHECK(q.pattern == RF_PATTERN_QUANT_GEMM_E4M3 && q.fmax == 448.0 && q.w == "w");
  Program r = plan(rms_dsl(4096, 11008));
  CHECK(r.pattern == RF_PATTERN_RMSNORM_GEMM && r.eps == 1e-6 && r.g == "g");
  CHECK(std::fabs(r.inv_k * 4096 - 1.0) < 1e-15);
}

TEST(layernorm_gemm_matches) {
  for (bool wf : {true, false}) {
    Program p = plan(ln_dsl(4096, 11008, wf));
    CHECK(p.pattern == RF_PATTERN_LAYERNORM_GEMM && p.eps == 1e-5 && p.g == "g" && p.w == "w");
    CHECK(p.free_len == 11008 && std::fabs(p.inv_k * 4096 - 1.0) < 1e-15);
  }
  // a d4 that does not subtract the mean of the same statistic: not LayerNorm
  std::string bad = ln_dsl(64, 8);
  bad.replace(bad.rfind("d1 * INVK * g"), 13, "d2 * INVK * g");
  CHECK_THROWS_AS(plan(bad), NotFusable);
}

TEST(moe_routing_matches) {  // proj/data/moe_routing.cascade
  Program p = plan("cascade moe_routing\ninput s len 128\nreduce 1 op max\n    s[l]\nreduce 2 op sum\n"
                   "    exp(s[l] - d1)\nreduce 3 op topk 8\n    s[l]\n");
  CHECK(p.pattern == RF_PATTERN_MOE_ROUTING && p.free_len == 8 && p.x == "s");
}

TEST(row_statistics_builtins_match) {  // proj/data/{variance,sum_sum,moment_of_inertia}.cascade
  Program v = plan("cascade variance\ninput x len 8192\nreduce 1 op sum\n    x[l]\n"
                   "reduce 2 op sum\n    x[l] * x[l]\n");
  CHECK(v.pattern == RF_PATTERN_VARIANCE && v.x == "x");
  Program s = plan("cascade sum_sum\ninput x1 len 1024\ninput x2 len 1024\nconst EPS = 1e-12\n"
                   "reduce 1 op sum\n    x1[l] * x1[l]\nreduce 2 op sum\n"
                   "    x1[l] * x2[l] / sqrt(max(d1 - 10, EPS))\n");
  CHECK(s.pattern == RF_PATTERN_SUM_SUM && s.x == "x1" && s.v == "x2" && s.offset == 10.0 &&
        s.eps == 1e-12);
  Program m = plan("cascade moment_of_inertia\ninput mass len 1024\ninput pos len 1024 free 3\n"
                   "reduce 1 op sum\n    mass[l]\nreduce 2 op sum free 3\n    mass[l] * pos[l, f]\n"
                   "reduce 3 op sum free 3\n    mass[l] * pos[l, f] * pos[l, f]\n");
  CHECK(m.pattern == RF_PATTERN_MOMENTS && m.x == "mass" && m.v == "pos" && m.free_len == 3);
}

TEST(unsupported_cascades_are_not_fusable) {
  // cascades without a kernel: NotFusable, no CPU fallback
  CHECK_THROWS_AS(plan("cascade prod_chain\ninput x len 64\nreduce 1 op prod\n    x[l]\n"
                       "reduce 2 op sum\n    x[l] / d1\n"),
                  NotFusable);
  CHECK_THROWS_AS(plan("cascade v\ninput x len 8\ninput y len 8\nreduce 1 op sum\n    x[l]\n"
                       "reduce 2 op sum\n    x[l] * y[l]\n"),
                  NotFusable);  // not the variance shape
  CHECK_THROWS_AS(plan("cascade moe\ninput s len 8\nreduce 1 op max\n    s[l]\nreduce 2 op sum\n"
                       "    exp(s[l] - d1)\nreduce 3 op topk 9\n    s[l]\n"),
                  NotFusable);  // top-k > 8: no kernel
  // RMS statistic that is not the mean over L0
  CHECK_THROWS_AS(plan("cascade r\ninput x len 8\ninput g len 8\ninput w len 8 free 4\n"
                       "reduce 1 op sum\n    x[l] * x[l]\nreduce 2 op sum free 4\n"
                       "    x[l] * g[l] / sqrt(d1 / 3 + 0.1) * w[l, f]\n"),
                  NotFusable);
}

TEST(syntax_errors) {
  CHECK_THROWS_AS(parse_cascade("cascade x\ninput x len 0\n"), SyntaxError);
  CHECK_THROWS_AS(parse_cascade("cascade x\ninput x len 4\nreduce 1 op max\n"), SyntaxError);
  CHECK_THROWS_AS(parse_cascade("cascade x\ninput x len 4\nreduce 1 op max\n    x[l] + d1\n"),
                  SyntaxError);  // forward dependency
  CHECK_THROWS_AS(parse_cascade("cascade x\ninput x len 4\nreduce 1 op max\n    y[l]\n"), SyntaxError);
  CHECK_THROWS_AS(parse_cascade("cascade x\ninput x len 4\nreduce 1 op avg\n    x[l]\n"), SyntaxError);
}

TEST(compare_reports_flags_corruption_with_a_location) {
  ExecReport u, v;
  u.outputs = {{1, {3.0}, {}}, {2, {1.5}, {}}};
  v = u;
  DiffReport same = compare_reports(u, v, 1e-12);
  CHECK(same.pass && same.max_rel_err == 0.0);
  v.outputs[1].v[0] += 0.5;
  DiffReport diff = compare_reports(u, v, 1e-6);
  CHECK(!diff.pass);
  CHECK(diff.worst == "d2[0]");
  v = u;
  v.outputs[0].v[0] = std::nan("");
  CHECK(!compare_reports(u, v, 1.0).pass);
}

TEST(shape_checks) {
  Program p = plan(softmax_dsl(8));
  TensorStore st;
  st.define("x", 4, 0, std::vector<double>(4, 1.0));
  CHECK_THROWS_AS(run_incremental(p, TreeConfig{{8, 1}}, st), ShapeMismatch);
  TensorStore st2;
  CHECK_THROWS_AS(run_incremental(p, TreeConfig{{8, 1}}, st2), ShapeMismatch);
  TensorStore st3;
  st3.define("x", 8, 0, std::vector<double>(8, 1.0));
  CHECK_THROWS_AS(run_incremental(p, TreeConfig{{8, 3, 1}}, st3), ShapeMismatch);
  CHECK_THROWS_AS(st3.define("y", 4, 2, std::vector<double>(7, 0.0)), ShapeMismatch);
  Program q = plan(quant_dsl(16, 4));
  TensorStore st4;
  st4.define("a", 16, 0, random_vec(16, 7, -2, 2));
  st4.define("w", 16, 4, random_vec(64, 8, -1, 1));
  CHECK_THROWS_AS(run_multisegment(q, TreeConfig{{16, 4, 1}}, 3, st4), IncompatibleSegmentation);
}

// --------------------------------------------------------------------- GPU --

TEST(softmax_by_hand) {  // test_simulator.cpp:39-51
  Program p = plan(softmax_dsl(3));
  TensorStore st;
  st.define("x", 3, 0, {1, 2, 3});
  ExecReport r = run_incremental(p, TreeConfig{{3, 1}}, st);
  CHECK(r.outputs[0].v[0] == 3.0);
  const double t = std::exp(-2.0) + std::exp(-1.0) + 1.0;
  CHECK(std::fabs(r.outputs[1].v[0] - t) < 1e-6);
  CHECK(r.input_loads.at("x") == 3);  // fused: each element loaded once
  CHECK(r.dep_root_loads.at(1) == 1);
}

TEST(quant_trivia) {  // test_simulator.cpp:53-68
  Program q = plan(quant_dsl(1, 1));
  TensorStore st;
  st.define("a", 1, 0, {1.0});
  st.define("w", 1, 1, {2.0});
  ExecReport r = run_incremental(q, TreeConfig{{1, 1}}, st);
  CHECK(r.outputs[0].v[0] == 1.0);
  CHECK(r.outputs[1].v[0] == 896.0);
}

TEST(quant_zero_row_is_a_domain_error) {  // finalize_root fault propagation
  Program q = plan(quant_dsl(4, 2));
  TensorStore st;
  st.define("a", 4, 0, {0, 0, 0, 0});
  st.define("w", 4, 2, std::vector<double>(8, 1.0));
  CHECK_THROWS_AS(run_incremental(q, TreeConfig{{4, 1}}, st), DomainError);
}

static ExecReport attention_oracle(const TensorStore& st, long long kv, long long hd) {
  const auto& p = st.array("P").data;
  const auto& v = st.array("V").data;
  double m = p[0];
  for (double x : p) m = std::max(m, x);
  double t = 0;
  for (double x : p) t += std::exp(x - m);
  ExecReport r;
  r.outputs = {{1, {m}, {}}, {2, {t}, {}}, {3, std::vector<double>(hd, 0.0), {}}};
  for (long long l = 0; l < kv; ++l)
    for (long long f = 0; f < hd; ++f) r.outputs[2].v[f] += std::exp(p[l] - m) / t * v[l * hd + f];
  return r;
}

TEST(attention_incremental_and_multisegment_match_oracle) {
  const long long kv = 256, hd = 64;
  Program p = plan(attention_dsl(kv, hd));
  auto mk = [&] {
    TensorStore st;
    st.define("P", kv, 0, random_vec(kv, 3, -2, 2));
    st.define("V", kv, hd, random_vec(kv * hd, 4, -1, 1));
    return st;
  };
  TensorStore ref = mk();
  ExecReport want = attention_oracle(ref, kv, hd);
  for (const TreeConfig& cfg : {TreeConfig{{kv, 1}}, TreeConfig{{kv, kv / 8, 1}}}) {
    TensorStore st = mk();
    ExecReport inc = run_incremental(p, cfg, st);
    CHECK(compare_reports(inc, want, 1e-5).pass);
    CHECK(inc.input_loads.at("V") == kv * hd);
    CHECK(inc.peak_aux_slots.at(1) == 1 + 1 + hd);
    for (long long s : {2LL, 4LL, 8LL}) {
      TensorStore st2 = mk();
      CHECK(compare_reports(run_multisegment(p, cfg, s, st2), want, 1e-5).pass);
    }
  }
  TensorStore a = mk(), b = mk();  // multi:1 equals flat incremental exactly
  ExecReport i1 = run_incremental(p, TreeConfig{{kv, 1}}, a);
  ExecReport m1 = run_multisegment(p, TreeConfig{{kv, 1}}, 1, b);
  CHECK(compare_reports(i1, m1, 0.0).max_rel_err == 0.0);
}

TEST(softmax_weights_sum_to_one) {  // test_simulator.cpp:162-191
  Program p = plan(softmax_dsl(32));
  TensorStore st;
  st.define("x", 32, 0, random_vec(32, 11, -2, 2));
  ExecReport r = run_incremental(p, TreeConfig{{32, 8, 1}}, st);
  double m = r.outputs[0].v[0], t = r.outputs[1].v[0], sum = 0;
  for (double x : st.array("x").data) sum += std::exp(x - m) / t;
  CHECK(std::fabs(sum - 1.0) < 1e-5);
}

TEST(topk_reduction_ties_lowest_index) {  // test_simulator.cpp:254-271
  Program p = plan("cascade route\ninput g len 8\nreduce 1 op max\n    g[l]\nreduce 2 op sum\n"
                   "    exp(g[l] - d1)\nreduce 3 op topk 3\n    g[l]\n");
  TensorStore st;
  st.define("g", 8, 0, {0.3, 0.9, 0.9, -1.0, 0.5, 2.0, 0.1, 0.9});
  ExecReport r = run_incremental(p, TreeConfig{{8, 4, 1}}, st);
  CHECK(r.outputs[2].topk.size() == 3);
  CHECK(r.outputs[2].topk[0].second == 6 && r.outputs[2].topk[0].first == 2.0);
  CHECK(r.outputs[2].topk[1].second == 2 && std::fabs(r.outputs[2].topk[1].first - 0.9) < 1e-7);
  CHECK(r.outputs[2].topk[2].second == 3);
  CHECK(r.outputs[0].v[0] == 2.0);
}

static void rms_case(long long k, long long n, unsigned seed) {
  Program p = plan(rms_dsl(k, n));
  TensorStore st;
  st.define("x", k, 0, random_vec(k, seed, -1, 1));
  st.define("g", k, 0, random_vec(k, seed + 1, -1, 1));
  st.define("w", k, n, random_vec(k * n, seed + 2, -1, 1));
  ExecReport r = run_incremental(p, TreeConfig{{k, 1}}, st);
  const auto &x = st.array("x").data, &g = st.array("g").data, &w = st.array("w").data;
  double ss = 0;
  for (double v : x) ss += v * v;
  ExecReport want;
  want.outputs = {{1, {ss}, {}}, {2, std::vector<double>(n, 0.0), {}}};
  // the reference on the same rounded inputs: bf16 x and the bf16(g * w) the
  // kernel's packed weight holds
  using rfcuda::detail::from_bf16;
  using rfcuda::detail::to_bf16;
  double ssr = 0;
  for (double v : x) ssr += static_cast<double>(from_bf16(to_bf16(static_cast<float>(v)))) *
                            from_bf16(to_bf16(static_cast<float>(v)));
  want.outputs[0].v[0] = ssr;
  for (long long l = 0; l < k; ++l) {
    const double xr = from_bf16(to_bf16(static_cast<float>(x[l])));
    for (long long f = 0; f < n; ++f)
      want.outputs[1].v[f] += xr * from_bf16(to_bf16(static_cast<float>(g[l] * w[l * n + f]))) /
                              std::sqrt(ssr / k + 1e-6);
  }
  DiffReport d = compare_reports(r, want, 2e-2);  // north_star: 2e-2 on the same rounded inputs
  CHECK(d.pass);
  std::printf("  rmsnorm k=%lld scaled err vs the same-rounded reference: %.3g (%s)\n", k, d.max_rel_err,
              d.worst.c_str());
}

TEST(rmsnorm_gemm_matches_direct_loop) {
  rms_case(256, 48, 1);
  // K not a multiple of the kernel's 64-wide K tile: the host pads K with
  // zeros and must still normalise by the cascade's own mean d1 / L0
  rms_case(100, 48, 11);
  rms_case(4000, 40, 21);
}

static void ln_case(long long k, long long n, unsigned seed) {
  Program p = plan(ln_dsl(k, n));
  TensorStore st;
  st.define("x", k, 0, random_vec(k, seed, -1, 2));
  st.define("g", k, 0, random_vec(k, seed + 1, -1, 1));
  st.define("w", k, n, random_vec(k * n, seed + 2, -1, 1));
  ExecReport r = run_incremental(p, TreeConfig{{k, 1}}, st);
  const auto &x = st.array("x").data, &g = st.array("g").data, &w = st.array("w").data;
  // the reference on the same rounded inputs (bf16 x, bf16(g w)); sigma over
  // the cascade's own K even when the host zero-pads K to the 64-wide tile
  using rfcuda::detail::from_bf16;
  using rfcuda::detail::to_bf16;
  double s1 = 0, s2 = 0;
  for (double v : x) {
    const double xr = from_bf16(to_bf16(static_cast<float>(v)));
    s1 += xr, s2 += xr * xr;
  }
  const double sig = std::sqrt(s2 / k - (s1 / k) * (s1 / k) + 1e-5);
  ExecReport want;
  want.outputs = {{1, {s1}, {}}, {2, {s2}, {}}, {3, std::vector<double>(n, 0.0), {}},
                  {4, std::vector<double>(n, 0.0), {}}};
  for (long long l = 0; l < k; ++l) {
    const double xr = from_bf16(to_bf16(static_cast<float>(x[l])));
    for (long long f = 0; f < n; ++f) {
      const double gw = from_bf16(to_bf16(static_cast<float>(g[l] * w[l * n + f])));
      want.outputs[2].v[f] += xr * gw / sig;
      want.outputs[3].v[f] += s1 / k * gw / sig;
    }
  }
  DiffReport d = compare_reports(r, want, 2e-2);  // north_star: 2e-2 on the same rounded inputs
  CHECK(d.pass);
  std::printf("  layernorm k=%lld scaled err vs the same-rounded reference: %.3g (%s)\n", k, d.max_rel_err,
              d.worst.c_str());
}

TEST(layernorm_gemm_matches_direct_loop) {
  ln_case(256, 48, 4);
  // K % 64 != 0: zero-padded to the K tile, the means stay over the cascade's
  // own K (rf_desc.stat_len)
  ln_case(96, 8, 7);
  ln_case(1000, 40, 9);
}

// The corrections derive_fused derives for every builtin and the RMS / LN DSL
// cascades (tests/golden/corrections.txt, written by the reference itself:
// oracle/ref_driver.cpp golden) are exactly the kernels' closed forms
// (check_corrections: numeric_equiv, probe.cpp:15-42), and a tampered one is
// rejected with NotFusable.
static std::string g_golden_dir;

TEST(derived_corrections_are_the_kernels) {
  std::ifstream in(g_golden_dir + "/corrections.txt");
  CHECK(in.good());
  std::map<std::string, std::vector<std::pair<int, std::string>>> by_name;
  std::string line;
  while (std::getline(in, line)) {
    const auto a = line.find(' '), b = line.find(' ', a + 1);
    if (a == std::string::npos || b == std::string::npos) continue;
    const std::string name = line.substr(0, a);
    const int id = std::atoi(line.c_str() + a + 2);
    std::string corr = line.substr(b + 1);
    if (corr == "<identity>") corr.clear();
    by_name[name].emplace_back(id, corr);
  }
  const std::map<std::string, std::string> dsl = {
      {"safe_softmax", softmax_dsl(1024)},
      {"attention", attention_dsl(256, 64)},
      {"quant_gemm", quant_dsl(64, 32)},
      {"moe_routing", "cascade moe_routing\ninput s len 128\nreduce 1 op max\n    s[l]\nreduce 2 op sum\n"
                      "    exp(s[l] - d1)\nreduce 3 op topk 8\n    s[l]\n"},
      {"variance", "cascade variance\ninput x len 8192\nreduce 1 op sum\n    x[l]\n"
                   "reduce 2 op sum\n    x[l] * x[l]\n"},
      {"sum_sum", "cascade sum_sum\ninput x1 len 1024\ninput x2 len 1024\nconst EPS = 1e-12\n"
                  "reduce 1 op sum\n    x1[l] * x1[l]\nreduce 2 op sum\n"
                  "    x1[l] * x2[l] / sqrt(max(d1 - 10, EPS))\n"},
      {"moment_of_inertia", "cascade moment_of_inertia\ninput mass len 1024\ninput pos len 1024 free 3\n"
                            "reduce 1 op sum\n    mass[l]\nreduce 2 op sum free 3\n    mass[l] * pos[l, f]\n"
                            "reduce 3 op sum free 3\n    mass[l] * pos[l, f] * pos[l, f]\n"},
      {"rmsnorm_gemm", rms_dsl(64, 32)},
      {"layernorm_gemm", ln_dsl(64, 32)},
  };
  int pinned = 0;
  for (const auto& kv : by_name) {
    auto it = dsl.find(kv.first);
    CHECK(it != dsl.end());
    if (it == dsl.end()) continue;
    const Program p = plan(it->second);
    bool ok = true;
    try {
      check_corrections(p, kv.second);
    } catch (const NotFusable& e) {
      ok = false;
      std::printf("  %s: %s\n", kv.first.c_str(), e.what());
    }
    CHECK(ok);
    pinned += static_cast<int>(kv.second.size());
    // every non-identity correction, tampered, is rejected
    for (std::size_t i = 0; i < kv.second.size(); ++i) {
      auto bad = kv.second;
      if (bad[i].second.empty()) {
        bad[i].second = "d1_prev / d1";  // a correction where the kernel applies none
      } else {
        bad[i].second = "(" + bad[i].second + ") * 1.0001";
      }
      CHECK_THROWS_AS(check_corrections(p, bad), NotFusable);
    }
  }
  CHECK(pinned == 23);  // every reduction of the 9 cascades
  // the plan-layer entry with derived corrections
  const Program a = plan(parse_cascade(attention_dsl(256, 64)),
                         {{1, ""}, {2, "exp(d1_prev - d1)"}, {3, "exp(d1_prev - d1) * d2_prev / d2"}});
  CHECK(a.pattern == RF_PATTERN_ATTENTION);
  CHECK_THROWS_AS(plan(parse_cascade(attention_dsl(256, 64)),
                       {{1, ""}, {2, "exp(d1_prev - d1)"}, {3, "exp(d1 - d1_prev) * d2_prev / d2"}}),
                  NotFusable);
  // an RMS cascade with a different eps than its derived correction: rejected
  CHECK_THROWS_AS(plan(parse_cascade(rms_dsl(64, 32)),
                       {{1, ""}, {2, "sqrt(0.015625 * d1_prev + 1e-5) / sqrt(0.015625 * d1 + 1e-5)"}}),
                  NotFusable);
  std::printf("  %d derived corrections pinned to the kernels' closed forms\n", pinned);
}

// run_batched: R rows in one run equal R single-row runs (same kernels; the
// attention rows become (b,h) units of one launch).
TEST(batched_rows_match_single_rows) {
  {
    const long long kv = 512, hd = 64, R = 12;
    Program p = plan(attention_dsl(kv, hd));
    BatchedStore b;
    std::vector<double> P, V;
    std::vector<TensorStore> singles(R);
    for (long long r = 0; r < R; ++r) {
      auto pr = random_vec(kv, 40 + r, -3, 3), vr = random_vec(kv * hd, 80 + r, -1, 1);
      singles[r].define("P", kv, 0, pr);
      singles[r].define("V", kv, hd, vr);
      P.insert(P.end(), pr.begin(), pr.end());
      V.insert(V.end(), vr.begin(), vr.end());
    }
    b.define_rows("P", R, kv, 0, P);
    b.define_rows("V", R, kv, hd, V);
    for (long long segs : {1LL, 4LL}) {
      auto reps = run_batched(p, TreeConfig{{kv, 1}}, b, segs);
      CHECK(static_cast<long long>(reps.size()) == R);
      for (long long r = 0; r < R; ++r) {
        ExecReport one = run_multisegment(p, TreeConfig{{kv, 1}}, segs, singles[r]);
        CHECK(compare_reports(reps[r], one, 1e-6).pass);
        CHECK(reps[r].input_loads == one.input_loads);
      }
    }
  }
  {
    const long long k = 100, n = 40, R = 130;  // K padded, M spans two row tiles
    Program p = plan(rms_dsl(k, n));
    BatchedStore b;
    std::vector<double> X;
    const auto g = random_vec(k, 5, -1, 1), w = random_vec(k * n, 6, -1, 1);
    for (long long r = 0; r < R; ++r) {
      auto xr = random_vec(k, 300 + r, -1, 1);
      X.insert(X.end(), xr.begin(), xr.end());
    }
    b.define_rows("x", R, k, 0, X);
    b.define_shared("g", k, 0, g);
    b.define_shared("w", k, n, w);
    auto reps = run_batched(p, TreeConfig{{k, 1}}, b);
    CHECK(static_cast<long long>(reps.size()) == R);
    for (long long r : {0LL, 1LL, 127LL, 128LL, 129LL}) {
      TensorStore one;
      one.define("x", k, 0, std::vector<double>(X.begin() + r * k, X.begin() + (r + 1) * k));
      one.define("g", k, 0, g);
      one.define("w", k, n, w);
      ExecReport single = run_incremental(p, TreeConfig{{k, 1}}, one);
      // M = 256 runs the 2-SM tile, a single row the 1-SM one: the bf16 outputs
      // may differ by a rounding step
      CHECK(compare_reports(reps[r], single, 1e-2).pass);
      CHECK(std::fabs(reps[r].outputs[0].v[0] - single.outputs[0].v[0]) <= 1e-5 * single.outputs[0].v[0]);
    }
    // a per-row weight cannot be packed once: NotFusable
    BatchedStore bad;
    bad.define_rows("x", 2, k, 0, std::vector<double>(X.begin(), X.begin() + 2 * k));
    bad.define_shared("g", k, 0, g);
    std::vector<double> w2(w);
    w2.insert(w2.end(), w.begin(), w.end());
    bad.define_rows("w", 2, k, n, w2);
    CHECK_THROWS_AS(run_batched(p, TreeConfig{{k, 1}}, bad), NotFusable);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  {
    std::string self = argv[0];
    const auto slash = self.rfind('/');
    g_golden_dir = (slash == std::string::npos ? std::string(".") : self.substr(0, slash)) + "/../golden";
  }
  RUN(derived_corrections_are_the_kernels);
  RUN(dsl_files_parse_and_match_kernels);
  RUN(moe_routing_matches);
  RUN(layernorm_gemm_matches);
  RUN(row_statistics_builtins_match);
  RUN(unsupported_cascades_are_not_fusable);
  RUN(syntax_errors);
  RUN(compare_reports_flags_corruption_with_a_location);
  RUN(shape_checks);
  if (mode == "gpu") {
    RUN(softmax_by_hand);
    RUN(quant_trivia);
    RUN(quant_zero_row_is_a_domain_error);
    RUN(attention_incremental_and_multisegment_match_oracle);
    RUN(softmax_weights_sum_to_one);
    RUN(rmsnorm_gemm_matches_direct_loop);
    RUN(topk_reduction_ties_lowest_index);
    RUN(layernorm_gemm_matches_direct_loop);
    RUN(batched_rows_match_single_rows);
  }
  std::printf("%d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
