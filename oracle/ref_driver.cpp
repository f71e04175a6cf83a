// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product path.
//
// A driver over the *reference* library (RedFuser artifact, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/librefcore.a).
// Two jobs:
//
//   ref_driver golden <outdir>
//       Runs the reference's own generators, oracles and fused-loop executors
//       (run_incremental / run_multisegment / run_unfused) on small cases and
//       writes their inputs and outputs as golden fixtures (tests/golden/).
//       The oracle restatement (oracle/rf_oracle.c) and the CUDA kernels are
//       pinned against these.
//
//   ref_driver bench <pattern> <L0> <free> <rows> <threads> [segments] [budget_s]
//   ref_driver bench router <hd> <experts> <rows> <threads> <K'> [budget_s]
//       Times the reference's CPU fused loop (run_incremental, or
//       run_multisegment when segments > 1; proj/src/simulator.cpp:631-687) on
//       a bounded sample of rows of a BASELINE.json configuration, one row per
//       thread at a time (executors are pure; stores are per-row). With a
//       budget, threads stop taking new rows once budget_s has elapsed (rows is
//       then an upper bound). Prints one JSON object.  This is the `cpu_baseline` / `--impl reference` arm.
//
// Only reference *public API* is used (workloads.hpp, simulator.hpp, acrf.hpp).

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "redfuse/acrf.hpp"
#include "redfuse/cascade.hpp"
#include "redfuse/simulator.hpp"
#include "redfuse/workloads.hpp"

using namespace redfuse;

namespace {

// ---------------------------------------------------------------- fixtures --

// One golden case = <name>.json manifest + <name>.f64 blob (little-endian
// float64, arrays concatenated in manifest order).
struct Case {
  std::string name;
  std::vector<std::pair<std::string, std::vector<long long>>> shapes;
  std::vector<std::vector<double>> data;
  std::vector<std::pair<std::string, std::string>> meta;

  void add(const std::string& n, std::vector<long long> shape,
           std::vector<double> v) {
    shapes.emplace_back(n, std::move(shape));
    data.push_back(std::move(v));
  }
  void note(const std::string& k, const std::string& v) { meta.emplace_back(k, v); }

  void write(const std::string& dir) const {
    std::ofstream blob(dir + "/" + name + ".f64", std::ios::binary);
    std::ostringstream js;
    js << "{\n  \"case\": \"" << name << "\",\n  \"meta\": {";
    for (std::size_t i = 0; i < meta.size(); ++i)
      js << (i ? ", " : "") << "\"" << meta[i].first << "\": \"" << meta[i].second << "\"";
    js << "},\n  \"arrays\": [\n";
    long long off = 0;
    for (std::size_t i = 0; i < shapes.size(); ++i) {
      const auto& v = data[i];
      blob.write(reinterpret_cast<const char*>(v.data()),
                 static_cast<std::streamsize>(v.size() * sizeof(double)));
      js << "    {\"name\": \"" << shapes[i].first << "\", \"shape\": [";
      for (std::size_t d = 0; d < shapes[i].second.size(); ++d)
        js << (d ? ", " : "") << shapes[i].second[d];
      js << "], \"offset\": " << off << ", \"count\": " << v.size() << "}"
         << (i + 1 < shapes.size() ? "," : "") << "\n";
      off += static_cast<long long>(v.size());
    }
    js << "  ]\n}\n";
    std::ofstream(dir + "/" + name + ".json") << js.str();
  }
};

void add_store(Case& c, const TensorStore& st) {
  for (const auto& n : st.names()) {
    const auto& a = st.array(n);
    std::vector<long long> shape{a.len};
    if (a.free_len > 0) shape.push_back(a.free_len);
    c.add("in." + n, shape, a.data);
  }
}

void add_report(Case& c, const std::string& tag, const ExecReport& r) {
  for (const auto& o : r.outputs) {
    std::string base = tag + ".d" + std::to_string(o.id);
    if (!o.topk.empty()) {
      std::vector<double> vals, idx;
      for (const auto& [v, i] : o.topk) {
        vals.push_back(v);
        idx.push_back(static_cast<double>(i));
      }
      c.add(base + ".topk_val", {(long long)vals.size()}, vals);
      c.add(base + ".topk_idx", {(long long)idx.size()}, idx);
    } else {
      c.add(base, {(long long)o.v.size()}, o.v);
    }
  }
}

// Per-array uniform(-1,1) streams split off a run seed (the convention the
// reference CLI uses for DSL cascades; restated here, tools/redfuse.cpp:55-82).
std::uint64_t split_seed(std::uint64_t seed, const std::string& name) {
  std::uint64_t h = 1469598103934665603ull ^ seed;
  for (unsigned char ch : name) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

TensorStore dsl_inputs(const CascadeSpec& spec, std::uint64_t seed) {
  TensorStore st;
  for (const auto& in : spec.inputs) {
    std::mt19937_64 rng(split_seed(seed, in.name));
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    long long n = in.len * (in.free_len > 0 ? in.free_len : 1);
    std::vector<double> v(static_cast<std::size_t>(n));
    for (auto& x : v) x = uni(rng);
    st.define(in.name, in.len, in.free_len, std::move(v));
  }
  return st;
}

// RMSNorm statistics -> GEMM as a cascade in the reference DSL.
std::string rms_dsl(long long k, long long n, double eps) {
  std::ostringstream os;
  os.precision(17);
  os << "cascade rmsnorm_gemm\n"
     << "input x len " << k << "\ninput g len " << k << "\n"
     << "input w len " << k << " free " << n << "\n"
     << "const INVK = " << 1.0 / static_cast<double>(k) << "\n"
     << "const EPS = " << eps << "\n"
     << "reduce 1 op sum\n    x[l] * x[l]\n"
     << "reduce 2 op sum free " << n << "\n"
     << "    x[l] * g[l] / sqrt(d1 * INVK + EPS) * w[l, f]\n";
  return os.str();
}

// LayerNorm statistics -> GEMM: four reductions, two of them
// free-axis. d3 - d4 = LayerNorm(x) @ W (with g folded in).
std::string ln_dsl(long long k, long long n, double eps) {
  std::ostringstream os;
  os.precision(17);
  const std::string sig = "sqrt(d2 * INVK - d1 * INVK * d1 * INVK + EPS)";
  os << "cascade layernorm_gemm\n"
     << "input x len " << k << "\ninput g len " << k << "\n"
     << "input w len " << k << " free " << n << "\n"
     << "const INVK = " << 1.0 / static_cast<double>(k) << "\n"
     << "const EPS = " << eps << "\n"
     << "reduce 1 op sum\n    x[l]\n"
     << "reduce 2 op sum\n    x[l] * x[l]\n"
     << "reduce 3 op sum free " << n << "\n    x[l] * g[l] * w[l, f] / " << sig << "\n"
     << "reduce 4 op sum free " << n << "\n    d1 * INVK * g[l] * w[l, f] / " << sig << "\n";
  return os.str();
}

// run_fused (simulator.cpp:485-559) at every level k of each tree; a tree
// lists TreeConfig.levels[1..K] (L0 is prepended). Report "fused_<w1>-..-<wK>_k<k>".
template <class Gen>
void add_fused(Case& c, const FusedProgram& prog, long long l0, Gen gen,
               const std::vector<std::vector<long long>>& trees) {
  for (const auto& t : trees) {
    std::vector<long long> levels{l0};
    std::string tag;
    for (long long x : t) {
      levels.push_back(x);
      tag += (tag.empty() ? "" : "-") + std::to_string(x);
    }
    for (int k = 1; k <= static_cast<int>(t.size()); ++k) {
      TensorStore s2 = gen();
      add_report(c, "fused_" + tag + "_k" + std::to_string(k), run_fused(prog, TreeConfig{levels}, k, s2));
    }
  }
}

void golden_workload(const std::string& dir, const std::string& name,
                     const Workload& w, std::uint64_t seed,
                     const std::vector<long long>& segs,
                     const std::vector<std::vector<long long>>& trees = {}) {
  FusedProgram prog = derive_fused(w.spec);
  long long l0 = w.spec.axis_len();
  Case c;
  c.name = name;
  c.note("workload", w.name);
  c.note("seed", std::to_string(seed));
  c.note("source", "reference run: oracle/_ref/ref_driver golden");
  TensorStore st = w.generate(seed);
  add_store(c, st);
  add_report(c, "oracle", w.oracle(st));
  {
    TensorStore s2 = w.generate(seed);
    add_report(c, "incremental", run_incremental(prog, TreeConfig{{l0, 1}}, s2));
  }
  for (long long s : segs) {
    TensorStore s2 = w.generate(seed);
    add_report(c, "multi" + std::to_string(s),
               run_multisegment(prog, TreeConfig{{l0, 1}}, s, s2));
  }
  add_fused(c, prog, l0, [&] { return w.generate(seed); }, trees);
  c.write(dir);
}

int cmd_golden(const std::string& dir) {
  for (std::uint64_t seed : {100ull, 101ull})
    golden_workload(dir, "attention_256x64_s" + std::to_string(seed),
                    make_attention(256, 64), seed, {2, 4, 8}, {{4, 1}, {16, 4, 1}});
  golden_workload(dir, "attention_128x128_s7", make_attention(128, 128), 7, {2, 4}, {{2, 1}});
  for (std::uint64_t seed = 100; seed < 105; ++seed)
    golden_workload(dir, "safe_softmax_1024_s" + std::to_string(seed),
                    make_safe_softmax(1024), seed, {2, 4, 8}, {{32, 4, 1}, {8, 1}});
  golden_workload(dir, "quant_gemm_512x256_s100", make_quant_gemm(512, 256), 100,
                  {2, 4, 8}, {{4, 1}});
  for (std::uint64_t seed = 100; seed < 103; ++seed)
    golden_workload(dir, "quant_gemm_64x32_s" + std::to_string(seed),
                    make_quant_gemm(64, 32), seed, {2, 4, 8});
  golden_workload(dir, "variance_8192_s100", make_variance(8192), 100, {2, 8}, {{16, 4, 1}});
  golden_workload(dir, "sum_sum_1024_s100", make_sum_sum(1024), 100, {2, 8}, {{4, 1}, {32, 8, 1}});
  golden_workload(dir, "sum_sum_1024_s101", make_sum_sum(1024), 101, {2, 8}, {{4, 1}});
  golden_workload(dir, "variance_8192_s101", make_variance(8192), 101, {2, 8}, {{16, 4, 1}});
  golden_workload(dir, "moment_of_inertia_1024_s100", builtin("moment_of_inertia"), 100, {2, 8});
  golden_workload(dir, "moe_routing_128x8_s100", make_moe_routing(128, 8), 100, {2, 4});

  // RMSNorm / LayerNorm -> GEMM through the reference engine on the DSL spec
  // (no builtin: run_unfused is the oracle, as the reference CLI does).
  struct DslCase {
    std::string kind;
    long long k, n;
    std::uint64_t seed;
    double eps;
  };
  for (const DslCase& dc : std::vector<DslCase>{{"rmsnorm_gemm", 64, 32, 100, 1e-6},
                                                {"rmsnorm_gemm", 256, 48, 101, 1e-6},
                                                {"layernorm_gemm", 64, 32, 100, 1e-5},
                                                {"layernorm_gemm", 256, 48, 101, 1e-5}}) {
    const long long k = dc.k, n = dc.n;
    const std::uint64_t seed = dc.seed;
    const bool ln = dc.kind == "layernorm_gemm";
    CascadeSpec spec = parse_cascade(ln ? ln_dsl(k, n, dc.eps) : rms_dsl(k, n, dc.eps));
    FusedProgram prog = derive_fused(spec);
    Case c;
    c.name = dc.kind + "_" + std::to_string(k) + "x" + std::to_string(n) + "_s" +
             std::to_string(seed);
    c.note("workload", dc.kind + " (DSL)");
    c.note("eps", ln ? "1e-5" : "1e-6");
    const int last = ln ? 4 : 2;
    c.note("corr", prog.decomp(last).corr ? render(prog.decomp(last).corr) : "");
    TensorStore st = dsl_inputs(spec, seed);
    add_store(c, st);
    {
      TensorStore s2 = dsl_inputs(spec, seed);
      add_report(c, "oracle", run_unfused(spec, TreeConfig{{k, 1}}, s2));
    }
    {
      TensorStore s2 = dsl_inputs(spec, seed);
      add_report(c, "incremental", run_incremental(prog, TreeConfig{{k, 1}}, s2));
    }
    for (long long s : {2LL, 4LL}) {
      TensorStore s2 = dsl_inputs(spec, seed);
      add_report(c, "multi" + std::to_string(s),
                 run_multisegment(prog, TreeConfig{{k, 1}}, s, s2));
    }
    add_fused(c, prog, k, [&] { return dsl_inputs(spec, seed); },
              k == 256 ? std::vector<std::vector<long long>>{{4, 1}, {2, 1}}
                       : std::vector<std::vector<long long>>{{1}});
    c.write(dir);
  }

  // Derived correction terms, as strings, for the plan layer's pattern pins.
  {
    std::ofstream os(dir + "/corrections.txt");
    for (const auto& nm : builtin_names()) {
      FusedProgram p = derive_fused(builtin(nm).spec);
      for (const auto& d : p.decomps)
        os << nm << " d" << d.id << " " << (d.corr ? render(d.corr) : "<identity>")
           << "\n";
    }
    FusedProgram p = derive_fused(parse_cascade(rms_dsl(64, 32, 1e-6)));
    for (const auto& d : p.decomps)
      os << "rmsnorm_gemm d" << d.id << " " << (d.corr ? render(d.corr) : "<identity>")
         << "\n";
    FusedProgram q = derive_fused(parse_cascade(ln_dsl(64, 32, 1e-5)));
    for (const auto& d : q.decomps)
      os << "layernorm_gemm d" << d.id << " " << (d.corr ? render(d.corr) : "<identity>")
         << "\n";
  }
  std::printf("{\"golden\": \"%s\"}\n", dir.c_str());
  return 0;
}

// ------------------------------------------------------------------- bench --

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

struct RowJob {
  // Builds the per-row store (untimed) and returns the timed body's flops.
  virtual ~RowJob() = default;
  virtual TensorStore make(std::uint64_t seed) const = 0;
  virtual void run(TensorStore& st) const = 0;
  virtual double flops_per_row() const = 0;
};

struct AttentionJob : RowJob {
  long long kv, hd, segs;
  Workload w;
  FusedProgram prog;
  AttentionJob(long long kv_, long long hd_, long long s)
      : kv(kv_), hd(hd_), segs(s), w(make_attention(kv_, hd_)), prog(derive_fused(w.spec)) {}
  TensorStore make(std::uint64_t seed) const override { return w.generate(seed); }
  void run(TensorStore& st) const override {
    // The P row (q . K^T) is part of the fused op; the reference keeps it in
    // the generator (proj/src/workloads.cpp:86-93), so it is recomputed here
    // inside the timed region, then the cascade runs on it.
    const auto& q = st.array("Q").data;
    const auto& k = st.array("K").data;
    std::vector<double> p(static_cast<std::size_t>(kv));
    for (long long l = 0; l < kv; ++l) {
      double acc = 0;
      for (long long d = 0; d < hd; ++d) acc += q[d] * k[l * hd + d];
      p[l] = acc;
    }
    TensorStore row;
    row.define("P", kv, 0, std::move(p));
    row.define("V", kv, hd, st.array("V").data);
    ExecReport r = segs > 1 ? run_multisegment(prog, TreeConfig{{kv, 1}}, segs, row)
                            : run_incremental(prog, TreeConfig{{kv, 1}}, row);
    if (r.outputs.size() != 3) std::abort();
  }
  double flops_per_row() const override { return 4.0 * kv * hd; }
};

struct QuantJob : RowJob {
  long long k, n;
  Workload w;
  FusedProgram prog;
  QuantJob(long long k_, long long n_)
      : k(k_), n(n_), w(make_quant_gemm(k_, n_)), prog(derive_fused(w.spec)) {}
  TensorStore make(std::uint64_t seed) const override { return w.generate(seed); }
  void run(TensorStore& st) const override {
    ExecReport r = run_incremental(prog, TreeConfig{{k, 1}}, st);
    if (r.outputs.size() != 2) std::abort();
  }
  double flops_per_row() const override { return 2.0 * k * n; }
};

struct RmsJob : RowJob {
  long long k, n;
  CascadeSpec spec;
  FusedProgram prog;
  RmsJob(long long k_, long long n_)
      : k(k_), n(n_), spec(parse_cascade(rms_dsl(k_, n_, 1e-6))), prog(derive_fused(spec)) {}
  TensorStore make(std::uint64_t seed) const override { return dsl_inputs(spec, seed); }
  void run(TensorStore& st) const override {
    ExecReport r = run_incremental(prog, TreeConfig{{k, 1}}, st);
    if (r.outputs.size() != 2) std::abort();
  }
  double flops_per_row() const override { return 2.0 * k * n + 2.0 * k; }
};

struct LnJob : RowJob {
  long long k, n;
  CascadeSpec spec;
  FusedProgram prog;
  LnJob(long long k_, long long n_)
      : k(k_), n(n_), spec(parse_cascade(ln_dsl(k_, n_, 1e-5))), prog(derive_fused(spec)) {}
  TensorStore make(std::uint64_t seed) const override { return dsl_inputs(spec, seed); }
  void run(TensorStore& st) const override {
    ExecReport r = run_incremental(prog, TreeConfig{{k, 1}}, st);
    if (r.outputs.size() != 4) std::abort();
  }
  // the GEMM (d3); d4 is the rank-1 mean term, counted like the statistics
  double flops_per_row() const override { return 2.0 * k * n + 3.0 * k; }
};

struct SoftmaxJob : RowJob {
  long long n;
  Workload w;
  FusedProgram prog;
  explicit SoftmaxJob(long long n_) : n(n_), w(make_safe_softmax(n_)), prog(derive_fused(w.spec)) {}
  TensorStore make(std::uint64_t seed) const override { return w.generate(seed); }
  void run(TensorStore& st) const override {
    ExecReport r = run_incremental(prog, TreeConfig{{n, 1}}, st);
    if (r.outputs.size() != 2) std::abort();
  }
  double flops_per_row() const override { return 3.0 * n; }
};

// MoE router: the producer GEMM s = x W (hd -> en, the paper's routing
// module) recomputed per token inside the timed body like the
// attention P row, then the make_moe_routing cascade (workloads.cpp:124-169)
// through run_incremental.
struct RouterJob : RowJob {
  long long hd, en, k;
  Workload w;
  FusedProgram prog;
  std::vector<double> wt;  // [hd, en], shared by every token
  RouterJob(long long hd_, long long en_, long long k_)
      : hd(hd_), en(en_), k(k_), w(make_moe_routing(en_, k_)), prog(derive_fused(w.spec)) {
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    wt.resize(static_cast<std::size_t>(hd * en));
    for (double& x : wt) x = u(rng) / std::sqrt(static_cast<double>(hd));
  }
  TensorStore make(std::uint64_t seed) const override {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<double> x(static_cast<std::size_t>(hd));
    for (double& v : x) v = u(rng);
    TensorStore st;
    st.define("x", hd, 0, std::move(x));
    return st;
  }
  void run(TensorStore& st) const override {
    const auto& x = st.array("x").data;
    std::vector<double> sc(static_cast<std::size_t>(en), 0.0);
    for (long long l = 0; l < hd; ++l)
      for (long long e = 0; e < en; ++e) sc[e] += x[l] * wt[l * en + e];
    TensorStore row;
    row.define("s", en, 0, std::move(sc));
    ExecReport r = run_incremental(prog, TreeConfig{{en, 1}}, row);
    if (r.outputs.size() != 3) std::abort();
  }
  double flops_per_row() const override { return 2.0 * hd * en; }
};

int cmd_bench(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "bench <attention|quant|rms|ln|softmax> <L0> <free> <rows> <threads> [segments]\n"
                         "bench router <hd> <experts> <rows> <threads> <K'>\n");
    return 2;
  }
  std::string pat = argv[2];
  long long l0 = std::atoll(argv[3]), fr = std::atoll(argv[4]);
  long long rows = std::atoll(argv[5]);
  int threads = std::atoi(argv[6]);
  long long segs = argc > 7 ? std::atoll(argv[7]) : 1;
  double budget = argc > 8 ? std::atof(argv[8]) : 0.0;
  std::unique_ptr<RowJob> job;
  if (pat == "attention") job = std::make_unique<AttentionJob>(l0, fr, segs);
  else if (pat == "quant") job = std::make_unique<QuantJob>(l0, fr);
  else if (pat == "rms") job = std::make_unique<RmsJob>(l0, fr);
  else if (pat == "ln") job = std::make_unique<LnJob>(l0, fr);
  else if (pat == "softmax") job = std::make_unique<SoftmaxJob>(l0);
  else if (pat == "router") job = std::make_unique<RouterJob>(l0, fr, segs);  // hd, en, K'
  else return 2;
  if (threads < 1) threads = 1;
  if (rows < threads) rows = threads;

  std::atomic<long long> next{0}, done{0};
  std::vector<double> busy(static_cast<std::size_t>(threads), 0.0);
  double t0 = now_s();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (;;) {
        if (budget > 0 && now_s() - t0 > budget) break;
        long long r = next.fetch_add(1);
        if (r >= rows) break;
        TensorStore st = job->make(1000003ull * static_cast<std::uint64_t>(r) + 42);
        double a = now_s();
        job->run(st);
        busy[static_cast<std::size_t>(t)] += now_s() - a;
        done.fetch_add(1);
      }
    });
  }
  for (auto& th : pool) th.join();
  double wall = now_s() - t0;
  rows = done.load();
  double busy_sum = 0;
  for (double b : busy) busy_sum += b;
  // Throughput of the timed bodies on `threads` threads: rows / (busy / threads).
  double eff_s = busy_sum / threads;
  double flops = job->flops_per_row() * static_cast<double>(rows);
  std::printf(
      "{\"pattern\": \"%s\", \"L0\": %lld, \"free\": %lld, \"segments\": %lld, "
      "\"rows\": %lld, \"threads\": %d, \"wall_s\": %.6f, \"busy_s\": %.6f, "
      "\"s_per_row_thread\": %.6f, \"rows_per_s\": %.6f, \"flops\": %.6e, "
      "\"flop_per_s\": %.6e}\n",
      pat.c_str(), l0, fr, segs, rows, threads, wall, busy_sum, busy_sum / rows,
      rows / eff_s, flops, flops / eff_s);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 3 && std::string(argv[1]) == "golden") return cmd_golden(argv[2]);
  if (argc >= 2 && std::string(argv[1]) == "bench") return cmd_bench(argc, argv);
  std::fprintf(stderr, "usage: ref_driver golden <dir> | bench ...\n");
  return 2;
}
