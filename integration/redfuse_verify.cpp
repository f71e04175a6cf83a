// redfuse-verify: the reference CLI's `verify` command (proj/tools/redfuse.cpp
// cmd_verify, :226-312) with the CUDA executors added as modes — the "cuda mode
// in cmd_verify" of SURVEY §8 f2. The reference CLI itself needs CLI11, which
// this image lacks, so this is a standalone front end with the same flags,
// exit codes and JSON schema (version 1), built against the reference library
// and the reference-side binding (integration/redfuse_cuda.cpp).
//
//   redfuse-verify (--workload NAME | --spec FILE) [--levels a,b,..,1] [--k K]
//                  [--strategy single|multi:S] [--seeds N] [--seed S] [--tol T]
//                  [--modes m1,m2,..] [--json] [--out PATH]
//
// Modes: unfused, fused@k, incremental, multi:S (the reference's executors)
// and cuda, cuda-multi:S, cuda-fused@k (librf_cuda through redfuse::run_cuda*). Every mode is
// compared with the workload oracle by the reference's compare_reports.
// The cuda gate: fp32 patterns use max scaled error <= max(tol, 1e-5) (the
// north_star's fp32 bound); bf16/e4m3-operand patterns are compared against
// the UNROUNDED oracle, so they are gated on the RMS relative error of the
// last output (0.06 for e4m3, 0.02 for bf16) — the <= 2e-2 same-rounded-input
// gate lives in tests/test_gpu_gemm.py.
//
// Exit codes (as the reference): 0 pass, 1 usage/parse error, 2 not fusable
// (derive_fused, or no librf_cuda kernel for a requested cuda mode),
// 3 verification failure.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "redfuse/cascade.hpp"
#include "redfuse/workloads.hpp"
#include "redfuse_cuda.hpp"

using namespace redfuse;

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::string workload, spec, strategy = "single", out, modes;
  std::vector<long long> levels;
  int k = 0, seeds = 5;
  std::uint64_t seed = 42;
  double tol = 1e-6;
  bool json = false;
};

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> r;
  std::string cur;
  std::istringstream is(s);
  while (std::getline(is, cur, sep))
    if (!cur.empty()) r.push_back(cur);
  return r;
}

Args parse_args(int argc, char** argv) {
  Args a;
  if (const char* s = std::getenv("REDFUSE_SEED")) a.seed = std::strtoull(s, nullptr, 10);
  int i = 1;
  if (i < argc && std::string(argv[i]) == "verify") ++i;
  for (; i < argc; ++i) {
    const std::string f = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw Usage(f + " needs a value");
      return argv[++i];
    };
    if (f == "--workload") a.workload = val();
    else if (f == "--spec") a.spec = val();
    else if (f == "--levels")
      for (const auto& t : split(val(), ',')) a.levels.push_back(std::atoll(t.c_str()));
    else if (f == "--k") a.k = std::atoi(val().c_str());
    else if (f == "--strategy") a.strategy = val();
    else if (f == "--seeds") a.seeds = std::atoi(val().c_str());
    else if (f == "--seed") a.seed = std::strtoull(val().c_str(), nullptr, 10);
    else if (f == "--tol") a.tol = std::atof(val().c_str());
    else if (f == "--modes") a.modes = val();
    else if (f == "--out") a.out = val();
    else if (f == "--json") a.json = true;
    else throw Usage("unknown flag " + f);
  }
  if (a.workload.empty() == a.spec.empty()) throw Usage("exactly one of --workload or --spec is required");
  if (a.seeds < 1) throw Usage("--seeds must be >= 1");
  return a;
}

// Per-input random streams split off the run seed by an FNV-1a hash of the
// array name, uniform(-1, 1) — the reference CLI's convention for DSL specs
// (tools/redfuse.cpp:55-92), with run_unfused as the oracle.
std::uint64_t stream_seed(std::uint64_t seed, const std::string& name) {
  std::uint64_t h = 1469598103934665603ull ^ seed;
  for (unsigned char c : name) h = (h ^ c) * 1099511628211ull;
  return h;
}

Workload spec_workload(const CascadeSpec& spec) {
  Workload w;
  w.name = spec.name;
  w.spec = spec;
  w.generate = [spec](std::uint64_t seed) {
    TensorStore st;
    for (const auto& in : spec.inputs) {
      std::mt19937_64 rng(stream_seed(seed, in.name));
      std::uniform_real_distribution<double> u(-1.0, 1.0);
      std::vector<double> v(static_cast<std::size_t>(in.len * std::max(1LL, in.free_len)));
      for (auto& x : v) x = u(rng);
      st.define(in.name, in.len, in.free_len, std::move(v));
    }
    return st;
  };
  w.oracle = [spec](const TensorStore& st) {
    TensorStore copy = st;
    ExecReport r = run_unfused(spec, TreeConfig{{spec.axis_len(), 1}}, copy);
    r.strategy = "oracle";
    r.input_loads.clear();
    r.dep_root_loads.clear();
    r.peak_aux_slots.clear();
    return r;
  };
  return w;
}

long long segments_of(const std::string& s, const std::string& prefix) {
  const long long n = std::atoll(s.c_str() + prefix.size());
  if (n < 2) throw Usage(s + ": need S >= 2");
  return n;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char b[64];
  std::snprintf(b, sizeof b, "%.6g", v);
  return b;
}

struct Mode {
  std::string name;
  bool cuda = false;
  long long segments = 1;
  int fuse = 0;  // cuda-fused@k: run_cuda_fused at level k
  double max_rel = 0.0, rms_rel = 0.0;
  bool pass = true;
  std::string worst, note;
  std::vector<double> ms;  // cuda: wall ms per executor call
};

double rms_rel_last(const ExecReport& got, const ExecReport& want) {
  if (got.outputs.empty() || want.outputs.empty()) return 0.0;
  const auto& a = got.outputs.back().v;
  const auto& b = want.outputs.back().v;
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size() && i < b.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

int verify(const Args& a) {
  Workload w;
  if (!a.workload.empty()) {
    w = builtin(a.workload);
  } else {
    std::ifstream in(a.spec);
    if (!in.good()) throw Usage("cannot open " + a.spec);
    std::ostringstream os;
    os << in.rdbuf();
    w = spec_workload(parse_cascade(os.str()));
  }
  FusedProgram prog;
  try {
    prog = derive_fused(w.spec);
  } catch (const NotFusable& e) {
    std::cerr << "not fusable: " << e.what() << "\n";
    return 2;
  }
  TreeConfig tree;
  tree.levels = a.levels.empty() ? std::vector<long long>{w.spec.axis_len(), 1} : a.levels;
  if (!validate_tree(tree, w.spec.axis_len()).empty()) throw Usage("bad --levels");
  const int k = a.k == 0 ? tree.depth() : a.k;
  if (k < 1 || k > tree.depth()) throw Usage("--k must lie in 1.." + std::to_string(tree.depth()));
  const long long segs = a.strategy == "single" ? 4 : segments_of(a.strategy, "multi:");

  const std::string mode_list = a.modes.empty()
      ? "unfused,fused@" + std::to_string(k) + ",incremental,multi:" + std::to_string(segs) +
            ",cuda,cuda-multi:" + std::to_string(segs)
      : a.modes;
  std::vector<Mode> modes;
  for (const auto& m : split(mode_list, ',')) {
    Mode md;
    md.name = m;
    if (m == "cuda") md.cuda = true;
    else if (m.rfind("cuda-fused@", 0) == 0) {
      md.cuda = true;
      md.fuse = std::atoi(m.c_str() + 11);
      if (md.fuse < 1 || md.fuse > tree.depth()) throw Usage("cuda-fused@k: k must lie in 1.." + std::to_string(tree.depth()));
    }
    else if (m.rfind("cuda-multi:", 0) == 0) md.cuda = true, md.segments = segments_of(m, "cuda-multi:");
    else if (m.rfind("multi:", 0) == 0) md.segments = segments_of(m, "multi:");
    else if (m != "unfused" && m != "incremental" && m.rfind("fused@", 0) != 0)
      throw Usage("unknown mode " + m);
    modes.push_back(md);
  }

  CudaPattern pat;
  std::string no_kernel;
  const bool want_cuda = std::any_of(modes.begin(), modes.end(), [](const Mode& m) { return m.cuda; });
  if (want_cuda) {
    try {
      pat = cuda_pattern(prog);
    } catch (const NotFusable& e) {
      no_kernel = e.what();
    }
  }
  const double cuda_tol = pat.fp32 ? std::max(a.tol, 1e-5) : (pat.name == "quant_gemm_e4m3" ? 0.06 : 0.02);

  ExecReport last_incr;
  for (int s = 0; s < a.seeds; ++s) {
    const std::uint64_t seed = a.seed + static_cast<std::uint64_t>(s);
    const ExecReport want = w.oracle(w.generate(seed));
    for (auto& md : modes) {
      if (md.cuda && !no_kernel.empty()) {
        md.pass = false;
        md.note = "no librf_cuda kernel: " + no_kernel;
        continue;
      }
      TensorStore st = w.generate(seed);
      ExecReport got;
      const auto t0 = std::chrono::steady_clock::now();
      if (md.cuda) {
        try {
          got = md.fuse > 0 ? run_cuda_fused(prog, tree, md.fuse, st)
                : md.segments > 1 ? run_cuda_multisegment(prog, tree, md.segments, st)
                                  : run_cuda(prog, tree, st);
        } catch (const NotFusable& e) {
          md.pass = false;
          md.note = std::string("no librf_cuda kernel: ") + e.what();
          if (md.fuse == 0) no_kernel = e.what();  // a too-long fused segment is this mode's limit only
          continue;
        }
      } else if (md.name == "unfused") got = run_unfused(w.spec, tree, st);
      else if (md.name.rfind("fused@", 0) == 0) got = run_fused(prog, tree, std::atoi(md.name.c_str() + 6), st);
      else if (md.name == "incremental") got = last_incr = run_incremental(prog, tree, st);
      else got = run_multisegment(prog, tree, md.segments, st);
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (md.cuda) md.ms.push_back(ms);
      const double tol = md.cuda && pat.fp32 ? cuda_tol : md.cuda ? 1e300 : a.tol;
      DiffReport d = compare_reports(got, want, tol);
      bool ok = d.pass;
      if (md.cuda && !pat.fp32) {
        const double r = rms_rel_last(got, want);
        md.rms_rel = std::max(md.rms_rel, r);
        ok = ok && r <= cuda_tol;
      }
      md.max_rel = std::max(md.max_rel, d.max_rel_err);
      if (!ok && md.pass) md.worst = d.worst + " (seed " + std::to_string(seed) + ")";
      md.pass = md.pass && ok;
    }
  }
  bool all = true;
  for (const auto& md : modes) all = all && md.pass;

  std::ostringstream os;
  if (a.json) {
    os << "{\n  \"version\": 1,\n  \"command\": \"verify\",\n  \"workload\": " << jstr(w.name)
       << ",\n  \"levels\": [";
    for (std::size_t i = 0; i < tree.levels.size(); ++i) os << (i ? ", " : "") << tree.levels[i];
    os << "],\n  \"k\": " << k << ",\n  \"seeds\": " << a.seeds << ",\n  \"tolerance\": " << jnum(a.tol)
       << ",\n  \"pass\": " << (all ? "true" : "false") << ",\n  \"modes\": [";
    for (std::size_t i = 0; i < modes.size(); ++i) {
      const Mode& m = modes[i];
      os << (i ? "," : "") << "\n    {\"mode\": " << jstr(m.name) << ", \"max_rel_err\": " << jnum(m.max_rel)
         << ", \"pass\": " << (m.pass ? "true" : "false");
      if (!m.pass && !m.worst.empty()) os << ", \"worst\": " << jstr(m.worst);
      if (!m.note.empty()) os << ", \"note\": " << jstr(m.note);
      if (m.cuda && no_kernel.empty()) {
        std::vector<double> t = m.ms;
        std::sort(t.begin(), t.end());
        os << ", \"gate\": " << jstr(pat.fp32 ? "max_rel" : "rms_rel_last_output")
           << ", \"gate_tol\": " << jnum(cuda_tol);
        if (!pat.fp32) os << ", \"rms_rel_err\": " << jnum(m.rms_rel);
        os << ", \"gpu\": {\"pattern\": " << jstr(pat.name) << ", \"operands\": "
           << jstr(pat.fp32 ? "f32" : "bf16/e4m3") << ", \"ms_per_call_median\": "
           << jnum(t.empty() ? NAN : t[t.size() / 2])
           << ", \"timing\": \"wall clock around run_cuda: plan + H2D + kernels + D2H\"}";
      }
      os << "}";
    }
    os << "\n  ],\n  \"reductions\": [";
    for (std::size_t i = 0; i < prog.decomps.size(); ++i) {
      const auto& d = prog.decomps[i];
      os << (i ? "," : "") << "\n    {\"id\": " << d.id << ", \"op\": "
         << jstr(reduce_name(prog.spec.reduction(d.id).op)) << ", \"combine\": "
         << jstr(d.combine == MonoidOp::Add ? "add" : "mul") << ", \"G\": " << jstr(render(d.G))
         << ", \"H\": " << (d.h_identity ? "null" : jstr(render(d.H)))
         << ", \"correction\": " << (d.corr ? jstr(render(d.corr)) : "null")
         << ", \"log_transformed\": " << (d.prod_transformed ? "true" : "false") << "}";
    }
    os << "\n  ],\n  \"counters\": {\"input_loads\": {";
    bool first = true;
    for (const auto& [n, c] : last_incr.input_loads) os << (first ? "" : ", ") << jstr(n) << ": " << c, first = false;
    os << "}, \"dep_root_loads\": {";
    first = true;
    for (const auto& [id, c] : last_incr.dep_root_loads)
      os << (first ? "" : ", ") << "\"d" << id << "\": " << c, first = false;
    os << "}, \"peak_aux_slots\": {";
    first = true;
    for (const auto& [l, c] : last_incr.peak_aux_slots)
      os << (first ? "" : ", ") << "\"level" << l << "\": " << c, first = false;
    os << "}}\n}\n";
  } else {
    os << "verify " << w.name << ": levels [";
    for (std::size_t i = 0; i < tree.levels.size(); ++i) os << (i ? ", " : "") << tree.levels[i];
    os << "] k=" << k << " seeds=" << a.seeds << " tol=" << a.tol << "\n";
    for (const auto& m : modes) {
      char line[256];
      std::snprintf(line, sizeof line, "  %-14s max rel err %-10.4g %s", m.name.c_str(), m.max_rel,
                    m.pass ? "pass" : ("FAIL " + m.worst).c_str());
      os << line;
      if (m.cuda && no_kernel.empty()) {
        std::vector<double> t = m.ms;
        std::sort(t.begin(), t.end());
        os << "  [" << pat.name << (pat.fp32 ? "" : ", rms rel " + std::to_string(m.rms_rel)) << ", "
           << (t.empty() ? 0.0 : t[t.size() / 2]) << " ms/call]";
      }
      if (!m.note.empty()) os << "  (" << m.note << ")";
      os << "\n";
    }
    os << (all ? "PASS" : "FAIL") << "\n";
  }
  if (a.out.empty()) {
    std::cout << os.str();
  } else {
    std::ofstream f(a.out);
    if (!f.good()) throw Usage("cannot write " + a.out);
    f << os.str();
  }
  if (!no_kernel.empty()) {
    std::cerr << "not fusable on librf_cuda: " << no_kernel << "\n";
    return 2;
  }
  return all ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return verify(parse_args(argc, argv));
  } catch (const Usage& e) {
    std::cerr << "usage: " << e.what() << "\n";
    return 1;
  } catch (const SyntaxError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
