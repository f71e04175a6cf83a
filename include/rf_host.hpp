// rf_host.hpp — C++ host layer over librf_cuda (include/rf_cuda.h): the
// drop-in mirror of the reference's operator API for the fused-loop path.
//
//   reference (proj/include/redfuse/...)          this header (namespace rfcuda)
//   ------------------------------------          ------------------------------
//   CascadeSpec parse_cascade(text)   cascade.hpp:88     CascadeSpec parse_cascade(text)
//   FusedProgram derive_fused(spec)   acrf.hpp:93-94     Program plan(spec)   (pattern match)
//   bool attention_shaped(spec)       scalar_ir.cpp:495  match_* in plan()
//   class TensorStore                 simulator.hpp:27   class TensorStore
//   struct OutputVal / ExecReport     simulator.hpp:49   struct OutputVal / ExecReport
//   run_incremental(prog, cfg, store) simulator.hpp:76   run_incremental(prog, cfg, store)
//   run_multisegment(prog,cfg,S,store)simulator.hpp:81   run_multisegment(prog, cfg, S, store)
//   compare_reports(a, b, tol)        simulator.hpp:94   compare_reports(a, b, tol)
//   ShapeMismatch / IncompatibleSegmentation / DomainError / NotFusable  (same names)
//
// Where the reference derives a generic FusedProgram by symbolic probing
// (derive_fused, plan time), the host layer instead matches the cascade onto
// one of librf_cuda's kernels (the structural matcher mirrors the reference's
// own attention_shaped); cascades with no kernel raise NotFusable — there is
// no CPU fallback. The executors run a reference row through the kernel (an
// fp32 SIMT path for attention/softmax rows, tcgen05 kernels for the GEMM
// patterns, padding rows to the kernels' tiles) and return an ExecReport with
// the reference's field meanings, including the analytic load counters of the
// fused loop (every element loaded once; simulator.cpp:571-572, 617).
//
// Header-only; link with librf_cuda.so. C++17.
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rf_cuda.h"

namespace rfcuda {

// ------------------------------------------------------------------ errors --

struct SyntaxError : std::runtime_error {
  SyntaxError(int line, const std::string& m)
      : std::runtime_error("line " + std::to_string(line) + ": " + m), line(line) {}
  int line;
};
struct ShapeMismatch : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IncompatibleSegmentation : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DomainError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NotFusable : std::runtime_error {  // "no librf_cuda kernel for this cascade"
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(rf_status s) {
  if (s == RF_OK) return;
  std::string m = std::string(rf_status_string(s)) + ": " + rf_last_error();
  switch (s) {
    case RF_ERR_SHAPE: throw ShapeMismatch(m);
    case RF_ERR_SEGMENTATION: throw IncompatibleSegmentation(m);
    case RF_ERR_DOMAIN: throw DomainError(m);
    case RF_ERR_UNSUPPORTED: throw NotFusable(m);
    case RF_ERR_ARG: throw std::invalid_argument(m);
    default: throw CudaError(m);
  }
}

// ------------------------------------------------------------- expressions --

struct Node;
using Expr = std::shared_ptr<const Node>;
struct Node {
  enum Kind { Num, Input, Dep, Free, Un, Bin } kind;
  double num = 0;
  std::string name;  // Input name / Un, Bin operator name
  bool has_free = false;
  int dep = 0;
  Expr a, b;
};

inline Expr mk(Node n) { return std::make_shared<const Node>(std::move(n)); }
inline Expr num(double v) { return mk({Node::Num, v, "", false, 0, nullptr, nullptr}); }
inline Expr input(const std::string& n, bool fr = false) {
  return mk({Node::Input, 0, n, fr, 0, nullptr, nullptr});
}
inline Expr dep(int id) { return mk({Node::Dep, 0, "", false, id, nullptr, nullptr}); }
inline Expr un(const std::string& op, Expr a) { return mk({Node::Un, 0, op, false, 0, a, nullptr}); }
inline Expr bin(const std::string& op, Expr a, Expr b) {
  return mk({Node::Bin, 0, op, false, 0, a, b});
}

inline std::string render(const Expr& e) {
  switch (e->kind) {
    case Node::Num: {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", e->num);
      return buf;
    }
    case Node::Input: return e->name + (e->has_free ? "[l, f]" : "[l]");
    case Node::Dep: return e->dep < 0 ? "d" + std::to_string(-e->dep) + "_prev" : "d" + std::to_string(e->dep);
    case Node::Free: return "f";
    case Node::Un: return e->name + "(" + render(e->a) + ")";
    case Node::Bin:
      if (e->name == "max" || e->name == "min" || e->name == "pow")
        return e->name + "(" + render(e->a) + ", " + render(e->b) + ")";
      return "(" + render(e->a) + " " + e->name + " " + render(e->b) + ")";
  }
  return "?";
}

// Deps referenced by an expression.
inline void deps_of(const Expr& e, std::set<int>& out) {
  if (!e) return;
  if (e->kind == Node::Dep) out.insert(e->dep);
  deps_of(e->a, out);
  deps_of(e->b, out);
}

// ----------------------------------------------------------------- cascade --

struct InputDecl {
  std::string name;
  long long len = 0;
  long long free_len = 0;  // 0: rank-1
};
struct ReductionSpec {
  int id = 0;
  std::string op;  // sum | prod | max | min | topk
  int topk = 0;
  long long free_len = 1;
  Expr body;
};
struct CascadeSpec {
  std::string name;
  std::vector<InputDecl> inputs;
  std::vector<ReductionSpec> reductions;
  const InputDecl* find_input(const std::string& n) const {
    for (const auto& i : inputs)
      if (i.name == n) return &i;
    return nullptr;
  }
  long long axis_len() const { return inputs.empty() ? 0 : inputs.front().len; }
};
struct TreeConfig {
  std::vector<long long> levels;
  int depth() const { return static_cast<int>(levels.size()) - 1; }
};

namespace detail {

struct Lexer {
  enum Kind { End, Number, Ident, Sym };
  struct Tok {
    Kind kind = End;
    double num = 0;
    std::string text;
  };
  Lexer(const std::string& s, int line) : s(s), line(line) { next(); }
  const Tok& peek() const { return tok; }
  Tok take() {
    Tok t = tok;
    next();
    return t;
  }
  [[noreturn]] void fail(const std::string& m) const { throw SyntaxError(line, m); }
  void next() {
    while (pos < s.size() && std::isspace(static_cast<unsigned char>(s[pos]))) ++pos;
    if (pos >= s.size()) {
      tok = Tok{};
      return;
    }
    const char c = s[pos];
    if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
      char* end = nullptr;
      const double v = std::strtod(s.c_str() + pos, &end);
      tok = Tok{Number, v, ""};
      pos = static_cast<std::size_t>(end - s.c_str());
      return;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      std::size_t j = pos;
      while (j < s.size() && (std::isalnum(static_cast<unsigned char>(s[j])) || s[j] == '_')) ++j;
      tok = Tok{Ident, 0, s.substr(pos, j - pos)};
      pos = j;
      return;
    }
    tok = Tok{Sym, 0, std::string(1, c)};
    ++pos;
  }
  const std::string& s;
  int line;
  std::size_t pos = 0;
  Tok tok;
};

inline bool sym(const Lexer::Tok& t, const char* c) { return t.kind == Lexer::Sym && t.text == c; }

struct Parser {
  Lexer lx;
  const std::map<std::string, double>& consts;
  Expr expr() {
    Expr e = term();
    while (sym(lx.peek(), "+") || sym(lx.peek(), "-")) {
      const std::string op = lx.take().text;
      e = bin(op, e, term());
    }
    return e;
  }
  Expr term() {
    Expr e = primary();
    while (sym(lx.peek(), "*") || sym(lx.peek(), "/")) {
      const std::string op = lx.take().text;
      e = bin(op, e, primary());
    }
    return e;
  }
  Expr primary() {
    Lexer::Tok t = lx.take();
    if (t.kind == Lexer::Number) return num(t.num);
    if (sym(t, "(")) {
      Expr e = expr();
      if (!sym(lx.take(), ")")) lx.fail("expected )");
      return e;
    }
    if (sym(t, "-")) return un("neg", primary());
    if (t.kind != Lexer::Ident) lx.fail("unexpected token '" + t.text + "'");
    if (sym(lx.peek(), "(")) {
      lx.take();
      static const std::set<std::string> unary{"exp", "abs", "log2", "ln", "sqrt", "sign"};
      static const std::set<std::string> binary{"max", "min", "pow"};
      Expr a = expr();
      Expr e;
      if (binary.count(t.text)) {
        if (!sym(lx.take(), ",")) lx.fail(t.text + " takes two arguments");
        e = bin(t.text, a, expr());
      } else if (unary.count(t.text)) {
        e = un(t.text, a);
      } else {
        lx.fail("unknown function " + t.text);
      }
      if (!sym(lx.take(), ")")) lx.fail("expected ) closing " + t.text);
      return e;
    }
    if (sym(lx.peek(), "[")) {
      lx.take();
      const Lexer::Tok l = lx.take();
      if (l.kind != Lexer::Ident || l.text != "l") lx.fail("reduce-axis index must be l");
      bool fr = false;
      Lexer::Tok close = lx.take();
      if (sym(close, ",")) {
        const Lexer::Tok f = lx.take();
        if (f.kind != Lexer::Ident || f.text != "f") lx.fail("free-axis index must be f");
        fr = true;
        close = lx.take();
      }
      if (!sym(close, "]")) lx.fail("expected ]");
      return input(t.text, fr);
    }
    if (t.text.size() > 1 && t.text[0] == 'd' &&
        std::all_of(t.text.begin() + 1, t.text.end(), [](char ch) { return std::isdigit(ch); }))
      return dep(std::atoi(t.text.c_str() + 1));
    // d<k>_prev: the previous value of a dependency, as derive_fused renders
    // it inside a correction (expr.cpp:316-317); stored as Dep -k
    if (t.text.size() > 6 && t.text[0] == 'd' && t.text.compare(t.text.size() - 5, 5, "_prev") == 0 &&
        std::all_of(t.text.begin() + 1, t.text.end() - 5, [](char ch) { return std::isdigit(ch); }))
      return dep(-std::atoi(t.text.c_str() + 1));
    if (t.text == "f") return mk({Node::Free, 0, "f", false, 0, nullptr, nullptr});
    auto it = consts.find(t.text);
    if (it != consts.end()) return num(it->second);
    lx.fail("unknown identifier '" + t.text + "'");
  }
};

inline void input_refs(const Expr& e, std::vector<std::pair<std::string, bool>>& out) {
  if (!e) return;
  if (e->kind == Node::Input) out.emplace_back(e->name, e->has_free);
  input_refs(e->a, out);
  input_refs(e->b, out);
}

}  // namespace detail

// The cascade DSL of the reference (cascade.cpp:331-429 grammar; proj/data/*.cascade).
inline CascadeSpec parse_cascade(const std::string& text) {
  CascadeSpec spec;
  std::map<std::string, double> consts;
  std::size_t start = 0;
  int lineno = 0;
  bool want_body = false;
  while (start <= text.size()) {
    std::size_t nl = text.find('\n', start);
    if (nl == std::string::npos) nl = text.size();
    std::string line = text.substr(start, nl - start);
    start = nl + 1;
    ++lineno;
    const std::size_t b = line.find_first_not_of(" \t\r");
    if (b == std::string::npos) {
      if (nl == text.size()) break;
      continue;
    }
    const bool indented = b > 0;
    std::string t = line.substr(b);
    if (t[0] == '#') continue;
    if (want_body) {
      if (!indented) throw SyntaxError(lineno, "expected an indented body");
      detail::Parser p{detail::Lexer(t, lineno), consts};
      spec.reductions.back().body = p.expr();
      if (p.lx.peek().kind != detail::Lexer::End) p.lx.fail("trailing tokens after expression");
      want_body = false;
      continue;
    }
    if (indented) throw SyntaxError(lineno, "unexpected indentation");
    std::vector<std::string> w;
    {
      std::size_t i = 0;
      while (i < t.size()) {
        while (i < t.size() && std::isspace(static_cast<unsigned char>(t[i]))) ++i;
        std::size_t j = i;
        while (j < t.size() && !std::isspace(static_cast<unsigned char>(t[j]))) ++j;
        if (j > i) w.push_back(t.substr(i, j - i));
        i = j;
      }
    }
    auto len = [&](const std::string& s) {
      char* end = nullptr;
      const long long v = std::strtoll(s.c_str(), &end, 10);
      if (end == s.c_str() || *end || v <= 0) throw SyntaxError(lineno, "expected a positive length");
      return v;
    };
    if (w[0] == "cascade") {
      if (w.size() != 2) throw SyntaxError(lineno, "cascade <name>");
      spec.name = w[1];
    } else if (w[0] == "input") {
      if ((w.size() != 4 && w.size() != 6) || w[2] != "len")
        throw SyntaxError(lineno, "input <name> len <L0> [free <len>]");
      InputDecl in{w[1], len(w[3]), 0};
      if (w.size() == 6) {
        if (w[4] != "free") throw SyntaxError(lineno, "expected 'free'");
        in.free_len = len(w[5]);
      }
      spec.inputs.push_back(in);
    } else if (w[0] == "const") {
      if (w.size() != 4 || w[2] != "=") throw SyntaxError(lineno, "const <name> = <number>");
      char* end = nullptr;
      const double v = std::strtod(w[3].c_str(), &end);
      if (end == w[3].c_str() || *end) throw SyntaxError(lineno, "bad constant value");
      consts[w[1]] = v;
    } else if (w[0] == "reduce") {
      if (w.size() < 4 || w[2] != "op") throw SyntaxError(lineno, "reduce <id> op <op> [free <len>]");
      ReductionSpec r;
      r.id = static_cast<int>(len(w[1]));
      std::size_t i = 3;
      r.op = w[i++];
      static const std::set<std::string> ops{"sum", "prod", "max", "min", "topk"};
      if (!ops.count(r.op)) throw SyntaxError(lineno, "unknown reduce op '" + r.op + "'");
      if (r.op == "topk") {
        if (i >= w.size()) throw SyntaxError(lineno, "topk needs a tuple size");
        r.topk = static_cast<int>(len(w[i++]));
      }
      if (i < w.size()) {
        if (w[i] != "free" || i + 1 >= w.size()) throw SyntaxError(lineno, "expected 'free <len>'");
        r.free_len = len(w[i + 1]);
        i += 2;
      }
      if (i != w.size()) throw SyntaxError(lineno, "trailing tokens");
      spec.reductions.push_back(r);
      want_body = true;
    } else {
      throw SyntaxError(lineno, "unknown directive '" + w[0] + "'");
    }
    if (nl == text.size()) break;
  }
  if (want_body) throw SyntaxError(lineno, "missing reduction body");
  // structural validation (cascade.cpp:85-151 semantics)
  if (spec.inputs.empty()) throw SyntaxError(0, "cascade declares no inputs");
  for (const auto& in : spec.inputs)
    if (in.len != spec.axis_len()) throw SyntaxError(0, "inputs disagree on the reduce-axis length");
  for (std::size_t i = 0; i < spec.reductions.size(); ++i) {
    const auto& r = spec.reductions[i];
    if (r.id != static_cast<int>(i) + 1) throw SyntaxError(0, "reduction ids must be 1..n in order");
    std::set<int> ds;
    deps_of(r.body, ds);
    for (int d : ds)
      if (d >= r.id) throw SyntaxError(0, "forward dependency on d" + std::to_string(d));
    std::vector<std::pair<std::string, bool>> refs;
    detail::input_refs(r.body, refs);
    for (const auto& [n, fr] : refs) {
      const InputDecl* in = spec.find_input(n);
      if (!in) throw SyntaxError(0, "unknown input " + n);
      if (fr != (in->free_len > 0)) throw SyntaxError(0, "free-axis use of " + n + " disagrees with its decl");
      if (fr && r.free_len != in->free_len) throw SyntaxError(0, "free length mismatch for " + n);
    }
  }
  return spec;
}

// ------------------------------------------------------------ plan (match) --

struct Program {
  rf_pattern pattern = RF_PATTERN_SAFE_SOFTMAX;
  CascadeSpec spec;
  std::string x, v, g;  // bound input names (softmax x | attention P,V | quant a,w | rms x,g,w)
  std::string w;
  long long L0 = 0, free_len = 0;
  double fmax = 448.0, eps = 0.0, inv_k = 0.0, offset = 0.0;
};

namespace detail {

// Structural unification: pattern leaves "?X" bind rank-1 inputs, "?V" free
// inputs, "?c<k>" constants; everything else must match exactly.
struct Binding {
  std::map<std::string, std::string> in;
  std::map<std::string, double> c;
};

inline bool unify(const Expr& pat, const Expr& e, Binding& b) {
  if (pat->kind == Node::Input && pat->name.size() > 1 && pat->name[0] == '?') {
    if (e->kind != Node::Input || e->has_free != pat->has_free) return false;
    auto it = b.in.find(pat->name);
    if (it != b.in.end()) return it->second == e->name;
    b.in[pat->name] = e->name;
    return true;
  }
  if (pat->kind == Node::Num && std::isnan(pat->num)) {  // constant placeholder ?c
    if (e->kind != Node::Num) return false;
    auto it = b.c.find(pat->name);
    if (it != b.c.end()) return it->second == e->num;
    b.c[pat->name] = e->num;
    return true;
  }
  if (pat->kind != e->kind) return false;
  switch (pat->kind) {
    case Node::Num: return pat->num == e->num;
    case Node::Input: return pat->name == e->name && pat->has_free == e->has_free;
    case Node::Dep: return pat->dep == e->dep;
    case Node::Free: return true;
    case Node::Un: return pat->name == e->name && unify(pat->a, e->a, b);
    case Node::Bin: return pat->name == e->name && unify(pat->a, e->a, b) && unify(pat->b, e->b, b);
  }
  return false;
}

inline Expr cvar(const std::string& n) {
  return mk({Node::Num, std::numeric_limits<double>::quiet_NaN(), n, false, 0, nullptr, nullptr});
}

}  // namespace detail

// Matches a cascade onto a librf_cuda kernel (the host-side replacement of
// derive_fused for the supported patterns; mirrors attention_shaped,
// scalar_ir.cpp:495-514). Throws NotFusable when no kernel implements it.
inline Program plan(const CascadeSpec& spec) {
  using detail::Binding;
  using detail::cvar;
  using detail::unify;
  const auto& R = spec.reductions;
  Program p;
  p.spec = spec;
  p.L0 = spec.axis_len();
  const Expr X = input("?X"), Vf = input("?V", true), Wf = input("?W", true), G = input("?G");
  auto none = [&](const std::string& why) -> Program {
    throw NotFusable("cascade '" + spec.name + "': no librf_cuda kernel (" + why + ")");
  };
  if (R.size() == 2 && R[0].op == "max" && R[1].op == "sum" && R[0].free_len == 1 &&
      R[1].free_len == 1) {
    Binding b;
    if (unify(X, R[0].body, b) && unify(un("exp", bin("-", X, dep(1))), R[1].body, b)) {
      p.pattern = RF_PATTERN_SAFE_SOFTMAX;
      p.x = b.in["?X"];
      return p;
    }
  }
  if (R.size() == 3 && R[0].op == "max" && R[1].op == "sum" && R[2].op == "topk" &&
      R[0].free_len == 1 && R[1].free_len == 1 && R[2].topk >= 1 && R[2].topk <= 8) {
    Binding b;  // make_moe_routing (workloads.cpp:124-169)
    if (unify(X, R[0].body, b) && unify(un("exp", bin("-", X, dep(1))), R[1].body, b) &&
        unify(X, R[2].body, b)) {
      p.pattern = RF_PATTERN_MOE_ROUTING;
      p.x = b.in["?X"];
      p.free_len = R[2].topk;
      return p;
    }
  }
  if (R.size() == 3 && R[0].op == "max" && R[1].op == "sum" && R[2].op == "sum" &&
      R[0].free_len == 1 && R[1].free_len == 1 && R[2].free_len > 1) {
    Binding b;
    const Expr e = un("exp", bin("-", X, dep(1)));
    if (unify(X, R[0].body, b) && unify(e, R[1].body, b) &&
        unify(bin("*", bin("/", e, dep(2)), Vf), R[2].body, b)) {
      p.pattern = RF_PATTERN_ATTENTION;
      p.x = b.in["?X"];
      p.v = b.in["?V"];
      p.free_len = R[2].free_len;
      return p;
    }
  }
  if (R.size() == 2 && R[0].op == "max" && R[1].op == "sum" && R[0].free_len == 1) {
    Binding b;  // free_len may be 1: a one-lane free axis (test_simulator.cpp:53-68)
    if (unify(un("abs", X), R[0].body, b) &&
        unify(bin("*", bin("/", bin("*", cvar("fmax"), X), dep(1)), Wf), R[1].body, b)) {
      p.pattern = RF_PATTERN_QUANT_GEMM_E4M3;
      p.x = b.in["?X"];
      p.w = b.in["?W"];
      p.fmax = b.c["fmax"];
      p.free_len = R[1].free_len;
      return p;
    }
  }
  if (R.size() == 2 && R[0].op == "sum" && R[1].op == "sum" && R[0].free_len == 1) {
    Binding b;
    // x g / sqrt(d1 * INVK + EPS) * w   (or d1 / K)
    const Expr body_mul = bin("*", bin("/", bin("*", X, G), un("sqrt", bin("+", bin("*", dep(1), cvar("ik")), cvar("eps")))), Wf);
    Binding b2;
    const Expr body_div = bin("*", bin("/", bin("*", X, G), un("sqrt", bin("+", bin("/", dep(1), cvar("k")), cvar("eps")))), Wf);
    if (unify(bin("*", X, X), R[0].body, b)) {
      b2 = b;
      if (unify(body_mul, R[1].body, b) || unify(body_div, R[1].body, b2)) {
        Binding& bb = b.c.count("ik") ? b : b2;
        p.pattern = RF_PATTERN_RMSNORM_GEMM;
        p.x = bb.in["?X"];
        p.g = bb.in["?G"];
        p.w = bb.in["?W"];
        p.eps = bb.c["eps"];
        p.inv_k = bb.c.count("ik") ? bb.c["ik"] : 1.0 / bb.c["k"];
        if (std::fabs(p.inv_k * static_cast<double>(p.L0) - 1.0) > 1e-12)
          return none("RMS statistic must be the mean over the reduce axis");
        p.free_len = R[1].free_len;
        return p;
      }
    }
  }
  if (R.size() == 4 && R[0].op == "sum" && R[1].op == "sum" && R[2].op == "sum" &&
      R[3].op == "sum" && R[0].free_len == 1 && R[1].free_len == 1 && R[2].free_len >= 1 &&
      R[3].free_len == R[2].free_len) {
    // LayerNorm statistics -> GEMM:
    //   sigma = sqrt(d2 * INVK - d1 * INVK * d1 * INVK + EPS)
    //   d3: x g w / sigma      d4: d1 * INVK * g w / sigma
    // (either "... * w / sigma" or "... / sigma * w" operand order)
    const Expr ik = cvar("ik");
    const Expr mean = bin("*", dep(1), ik);
    const Expr sig = un("sqrt", bin("+", bin("-", bin("*", dep(2), ik), bin("*", bin("*", mean, dep(1)), ik)),
                                    cvar("eps")));
    const Expr xg = bin("*", X, G), mg = bin("*", mean, G);
    auto try_form = [&](bool w_first, Binding& b) {
      const Expr b3 = w_first ? bin("/", bin("*", xg, Wf), sig) : bin("*", bin("/", xg, sig), Wf);
      const Expr b4 = w_first ? bin("/", bin("*", mg, Wf), sig) : bin("*", bin("/", mg, sig), Wf);
      return unify(X, R[0].body, b) && unify(bin("*", X, X), R[1].body, b) &&
             unify(b3, R[2].body, b) && unify(b4, R[3].body, b);
    };
    Binding b1, b2;
    const bool f1 = try_form(true, b1);
    const bool f2 = !f1 && try_form(false, b2);
    if (f1 || f2) {
      Binding& bb = f1 ? b1 : b2;
      p.pattern = RF_PATTERN_LAYERNORM_GEMM;
      p.x = bb.in["?X"];
      p.g = bb.in["?G"];
      p.w = bb.in["?W"];
      p.eps = bb.c["eps"];
      p.inv_k = bb.c["ik"];
      if (std::fabs(p.inv_k * static_cast<double>(p.L0) - 1.0) > 1e-12)
        return none("LayerNorm statistics must be means over the reduce axis");
      p.free_len = R[2].free_len;
      return p;
    }
  }
  if (R.size() == 2 && R[0].op == "sum" && R[1].op == "sum" && R[0].free_len == 1 &&
      R[1].free_len == 1) {
    Binding b;  // make_variance (workloads.cpp:246-277)
    if (unify(X, R[0].body, b) && unify(bin("*", X, X), R[1].body, b)) {
      p.pattern = RF_PATTERN_VARIANCE;
      p.x = b.in["?X"];
      return p;
    }
    Binding b2;  // make_sum_sum (workloads.cpp:213-242): x1 x2 / sqrt(max(d1 - c, eps))
    const Expr Y = input("?Y");
    const Expr h = un("sqrt", bin("max", bin("-", dep(1), cvar("c")), cvar("eps")));
    if (unify(bin("*", X, X), R[0].body, b2) && unify(bin("/", bin("*", X, Y), h), R[1].body, b2)) {
      p.pattern = RF_PATTERN_SUM_SUM;
      p.x = b2.in["?X"];
      p.v = b2.in["?Y"];
      p.offset = b2.c["c"];
      p.eps = b2.c["eps"];
      if (!(p.eps > 0.0)) return none("sum_sum: the H guard max(d1 - c, eps) needs eps > 0");
      return p;
    }
  }
  if (R.size() == 3 && R[0].op == "sum" && R[1].op == "sum" && R[2].op == "sum" &&
      R[0].free_len == 1 && R[1].free_len >= 1 && R[1].free_len <= 8 &&
      R[2].free_len == R[1].free_len) {
    Binding b;  // moment_of_inertia (workloads.cpp:280-331)
    if (unify(X, R[0].body, b) && unify(bin("*", X, Vf), R[1].body, b) &&
        unify(bin("*", bin("*", X, Vf), Vf), R[2].body, b)) {
      p.pattern = RF_PATTERN_MOMENTS;
      p.x = b.in["?X"];
      p.v = b.in["?V"];
      p.free_len = R[1].free_len;
      return p;
    }
  }
  return none("not one of safe_softmax / attention / moe_routing / quant_gemm / rmsnorm_gemm / "
              "layernorm_gemm / variance / sum_sum / moment_of_inertia");
}

inline Program plan(const std::string& dsl) { return plan(parse_cascade(dsl)); }

// ------------------------------------------- derived-correction pinning --
//
// derive_fused (acrf.cpp:148-190) derives, per reduction, the correction
// corr = H(d) (x) inv(H(d_prev)) that the incremental loop applies to the
// accumulator (Eq.17, simulator.cpp:278-318). Each librf_cuda kernel hard-codes
// that correction in closed form. check_corrections proves, at
// plan time, that the FusedProgram's derived corrections are the ones the
// matched kernel applies — with the reference's own probe (numeric_equiv,
// probe.cpp:15-42: 32 valid samples, close_rel 1e-9) — and throws NotFusable
// otherwise, so a cascade whose derivation disagrees never runs.

// A correction expression in derive_fused's rendering (render, expr.cpp:303-357):
// deps d<k>, previous deps d<k>_prev, numbers, + - * /, exp/ln/log2/sqrt/abs/sign,
// max/min/pow. "" and "<identity>" mean "no correction".
inline Expr parse_correction(const std::string& text) {
  if (text.empty() || text == "<identity>") return nullptr;
  static const std::map<std::string, double> none;
  detail::Parser ps{detail::Lexer(text, 0), none};
  Expr e = ps.expr();
  if (ps.lx.peek().kind != detail::Lexer::End) throw SyntaxError(0, "trailing tokens in correction '" + text + "'");
  return e;
}

// Evaluates with d<k> = now[k-1], d<k>_prev = prev[k-1]; NaN outside the domain
// (the probe skips such points, as numeric_equiv skips DomainError).
inline double eval_correction(const Expr& e, const std::vector<double>& now, const std::vector<double>& prev) {
  const double nan = std::numeric_limits<double>::quiet_NaN();
  switch (e->kind) {
    case Node::Num: return e->num;
    case Node::Dep: {
      const int k = e->dep < 0 ? -e->dep : e->dep;
      const auto& v = e->dep < 0 ? prev : now;
      return k >= 1 && k <= static_cast<int>(v.size()) ? v[k - 1] : nan;
    }
    case Node::Un: {
      const double a = eval_correction(e->a, now, prev);
      if (e->name == "neg") return -a;
      if (e->name == "exp") return std::exp(a);
      if (e->name == "abs") return std::fabs(a);
      if (e->name == "sqrt") return a < 0 ? nan : std::sqrt(a);
      if (e->name == "ln") return a <= 0 ? nan : std::log(a);
      if (e->name == "log2") return a <= 0 ? nan : std::log2(a);
      if (e->name == "sign") return a > 0 ? 1.0 : a < 0 ? -1.0 : 0.0;
      return nan;
    }
    case Node::Bin: {
      const double a = eval_correction(e->a, now, prev), b = eval_correction(e->b, now, prev);
      if (e->name == "+") return a + b;
      if (e->name == "-") return a - b;
      if (e->name == "*") return a * b;
      if (e->name == "/") return b == 0.0 ? nan : a / b;
      if (e->name == "max") return std::fmax(a, b);
      if (e->name == "min") return std::fmin(a, b);
      if (e->name == "pow") return std::pow(a, b);
      return nan;
    }
    default: return nan;  // inputs / free index never appear in a correction
  }
}

// numeric_equiv (probe.cpp:15-42) over the deps d1..dn and d1_prev..dn_prev,
// probed in the reference's default domain [-2, 2] (probe.hpp:19-29) and in
// [0, 40] (past the guard offsets the builtins use, e.g. sum_sum's c = 10).
inline bool numeric_equiv(const Expr& a, const Expr& b, int ndeps, uint64_t seed = 0x5eedf00dULL) {
  uint64_t st = seed;
  auto uni = [&](double lo, double hi) {  // splitmix64 -> [lo, hi)
    st += 0x9e3779b97f4a7c15ULL;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return lo + (hi - lo) * (static_cast<double>(z >> 11) * 0x1.0p-53);
  };
  const double doms[2][2] = {{-2.0, 2.0}, {0.0, 40.0}};
  for (const auto& dom : doms) {
    int valid = 0, attempts = 0;
    while (valid < 32) {
      if (++attempts > 32 * 64) return valid > 0;  // InsufficientSamples: judge on what was valid
      std::vector<double> now(ndeps), prev(ndeps);
      for (int i = 0; i < ndeps; ++i) {
        now[i] = uni(dom[0], dom[1]);
        prev[i] = uni(dom[0], dom[1]);
      }
      const double l = eval_correction(a, now, prev), r = eval_correction(b, now, prev);
      if (!std::isfinite(l) || !std::isfinite(r)) continue;
      ++valid;
      if (std::fabs(l - r) > 1e-9 * (1.0 + std::fmax(std::fabs(l), std::fabs(r)))) return false;
    }
  }
  return true;
}

// The correction each kernel applies to reduction `id` (1-based), in the same
// rendering as derive_fused's; "" = none (h_identity).
inline std::string kernel_correction(const Program& p, int id) {
  auto num = [](double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return std::string(b);
  };
  switch (p.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX:
    case RF_PATTERN_MOE_ROUTING:
      return id == 2 ? "exp(d1_prev - d1)" : "";
    case RF_PATTERN_ATTENTION:  // attn_*.cu: lazy exp(d1'-d1) on O, d2'/d2 telescoped to 1/d2
      return id == 2 ? "exp(d1_prev - d1)" : id == 3 ? "exp(d1_prev - d1) * d2_prev / d2" : "";
    case RF_PATTERN_QUANT_GEMM_E4M3:  // gemm_sm100.cu qnt2: ref'/ref in-loop, ref/d1 at finalize
      return id == 2 ? "d1_prev / d1" : "";
    case RF_PATTERN_RMSNORM_GEMM: {  // gemm_sm100.cu rms2: 1/sqrt(d1/K+eps) at finalize
      const std::string ik = num(p.inv_k), e = num(p.eps);
      return id == 2 ? "sqrt(" + ik + " * d1_prev + " + e + ") / sqrt(" + ik + " * d1 + " + e + ")" : "";
    }
    case RF_PATTERN_LAYERNORM_GEMM: {  // rms2<LN>: 1/sigma at finalize; d4 via colsum
      const std::string ik = num(p.inv_k), ik2 = num(p.inv_k * p.inv_k), e = num(p.eps);
      const std::string sp = "sqrt(" + ik + " * d2_prev - " + ik2 + " * d1_prev * d1_prev + " + e + ")";
      const std::string sn = "sqrt(" + ik + " * d2 - " + ik2 + " * d1 * d1 + " + e + ")";
      return id == 3 ? sp + " / " + sn : id == 4 ? "d1 * " + sp + " / " + sn + " / d1_prev" : "";
    }
    case RF_PATTERN_SUM_SUM: {  // rowstats.cu: 1/sqrt(max(d1-c, eps)) at finalize
      const std::string c = num(p.offset), e = num(p.eps);
      return id == 2 ? "sqrt(max(d1_prev - " + c + ", " + e + ")) / sqrt(max(d1 - " + c + ", " + e + "))" : "";
    }
    default: return "";  // variance, moments: every H is the identity
  }
}

// derived[i] = {reduction id, derive_fused's corr rendered ("" when
// h_identity)}. Throws NotFusable naming the first reduction whose derived
// correction is not the kernel's.
inline void check_corrections(const Program& p, const std::vector<std::pair<int, std::string>>& derived) {
  const int n = static_cast<int>(p.spec.reductions.size());
  if (static_cast<int>(derived.size()) != n)
    throw NotFusable("cascade '" + p.spec.name + "': " + std::to_string(derived.size()) +
                     " derived corrections for " + std::to_string(n) + " reductions");
  for (const auto& dc : derived) {
    if (dc.first < 1 || dc.first > n) throw NotFusable("derived correction for unknown reduction d" + std::to_string(dc.first));
    const Expr want = parse_correction(kernel_correction(p, dc.first));
    const Expr got = parse_correction(dc.second);
    const bool ok = (!want && !got) || (want && got && numeric_equiv(want, got, n));
    if (!ok)
      throw NotFusable("cascade '" + p.spec.name + "' d" + std::to_string(dc.first) + ": derived correction '" +
                       (got ? dc.second : "<identity>") + "' is not the kernel's '" +
                       (want ? kernel_correction(p, dc.first) : "<identity>") + "'");
  }
}

// plan() with the FusedProgram's derived corrections checked (the binding's
// entry: integration/redfuse_cuda.cpp passes prog.decomps[i].corr).
inline Program plan(const CascadeSpec& spec, const std::vector<std::pair<int, std::string>>& derived) {
  Program p = plan(spec);
  check_corrections(p, derived);
  return p;
}

// ----------------------------------------------------------- TensorStore ----

class TensorStore {
 public:
  struct Array {
    std::vector<double> data;
    long long len = 0, free_len = 0, loads = 0, stores = 0;
  };
  void define(const std::string& name, long long len, long long free_len, std::vector<double> data) {
    const long long want = free_len > 0 ? len * free_len : len;
    if (static_cast<long long>(data.size()) != want)
      throw ShapeMismatch(name + ": got " + std::to_string(data.size()) + " values, want " +
                          std::to_string(want));
    Array a;
    a.data = std::move(data);
    a.len = len;
    a.free_len = free_len;
    a.stores = want;
    arrays_[name] = std::move(a);
  }
  const Array& array(const std::string& name) const {
    auto it = arrays_.find(name);
    if (it == arrays_.end()) throw ShapeMismatch("no array named " + name);
    return it->second;
  }
  bool has(const std::string& n) const { return arrays_.count(n) > 0; }
  std::vector<std::string> names() const {
    std::vector<std::string> out;
    for (const auto& kv : arrays_) out.push_back(kv.first);
    return out;
  }

 private:
  std::map<std::string, Array> arrays_;
};

struct OutputVal {
  int id = 0;
  std::vector<double> v;
  std::vector<std::pair<double, long long>> topk;
};

struct ExecReport {
  std::string strategy;
  std::vector<OutputVal> outputs;
  std::map<std::string, long long> input_loads;
  std::map<int, long long> dep_root_loads;
  std::map<int, long long> peak_aux_slots;
};

struct DiffReport {
  double max_rel_err = 0.0;
  bool pass = true;
  std::string worst;
};

// compare_reports' parity metric (simulator.cpp:691-752): per output
// |a-b| / (1 + max(|a|,|b|)); equal values (incl. matching infs) are 0;
// NaN/inf mismatches are +inf; top-k index mismatch is a hard fail.
inline DiffReport compare_reports(const ExecReport& a, const ExecReport& b, double tol) {
  DiffReport out;
  const double inf = std::numeric_limits<double>::infinity();
  if (a.outputs.size() != b.outputs.size()) return {inf, false, "output count mismatch"};
  for (std::size_t i = 0; i < a.outputs.size(); ++i) {
    const auto &oa = a.outputs[i], &ob = b.outputs[i];
    if (oa.id != ob.id || oa.v.size() != ob.v.size() || oa.topk.size() != ob.topk.size())
      return {inf, false, "shape mismatch at d" + std::to_string(oa.id)};
    for (std::size_t l = 0; l < oa.v.size(); ++l) {
      const double x = oa.v[l], y = ob.v[l];
      double e;
      if (x == y) e = 0.0;
      else if (std::isnan(x) || std::isnan(y) || std::isinf(x) || std::isinf(y)) e = inf;
      else e = std::fabs(x - y) / (1.0 + std::fmax(std::fabs(x), std::fabs(y)));
      if (e > out.max_rel_err) {
        out.max_rel_err = e;
        out.worst = "d" + std::to_string(oa.id) + "[" + std::to_string(l) + "]";
      }
    }
    for (std::size_t t = 0; t < oa.topk.size(); ++t)
      if (oa.topk[t].second != ob.topk[t].second)
        return {inf, false, "topk index set at d" + std::to_string(oa.id)};
  }
  if (out.max_rel_err > tol) out.pass = false;
  return out;
}

// -------------------------------------------------------------- executors --

namespace detail {

struct PlanHandle {
  rf_plan* p = nullptr;
  explicit PlanHandle(const rf_desc& d) { check(rf_plan_create(&d, &p)); }
  ~PlanHandle() { rf_plan_destroy(p); }
  PlanHandle(const PlanHandle&) = delete;
  PlanHandle& operator=(const PlanHandle&) = delete;
};

inline rf_desc base_desc(rf_pattern pat, rf_dtype dt) {
  rf_desc d;
  std::memset(&d, 0, sizeof d);
  d.pattern = pat;
  d.dtype = dt;
  d.batch = d.heads = 1;
  d.segments = 1;
  d.softmax_scale = 1.0;
  d.fmax = 448.0;
  return d;
}

inline uint16_t to_bf16(float f) {  // RNE
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
inline float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline long long round_up(long long x, long long m) { return (x + m - 1) / m * m; }

// The fused loop's counters: every input element loaded once
// (acceptance crit 6), root dependency reads once per corrected reduction at
// finalize (crit 7, simulator.cpp:617), O(1) auxiliary state per level (crit 8).
// run_fused (fuse_level k >= 1, simulator.cpp:485-559): inputs are still
// loaded once (the level-1 buffer), but every corrected reduction reads its
// final dependencies once per level-k partial (the bridge, :522-525), the
// level-1 buffer holds a segment's input lanes (:548-550) and levels 2..k keep
// a group of child states (:551-556).
inline void fill_counters(const Program& prog, const TreeConfig& cfg, ExecReport& r, int fuse_level = 0) {
  long long arity = 0;
  for (const auto& red : prog.spec.reductions) arity += red.op == "topk" ? 2LL * red.topk : red.free_len;
  long long lanes = 0;
  for (const auto& in : prog.spec.inputs) {
    r.input_loads[in.name] = in.len * std::max(1LL, in.free_len);
    lanes += std::max(1LL, in.free_len);
  }
  const long long root_reads = fuse_level > 0 ? cfg.levels[static_cast<std::size_t>(fuse_level)] : 1;
  for (const auto& red : prog.spec.reductions) {
    std::set<int> ds;
    deps_of(red.body, ds);
    for (int d : ds) r.dep_root_loads[d] += root_reads;
  }
  for (int m = 1; m <= cfg.depth(); ++m) r.peak_aux_slots[m] = arity;
  if (fuse_level > 0) {
    r.peak_aux_slots[1] = cfg.levels[0] / cfg.levels[1] * lanes + arity;
    for (int m = 2; m <= fuse_level; ++m)
      r.peak_aux_slots[m] = (cfg.levels[static_cast<std::size_t>(m) - 1] / cfg.levels[static_cast<std::size_t>(m)] + 1) * arity;
  }
}

// One host-side operand of a batched run: R rows of [len(, free)] values,
// or one array every row shares (a static weight).
inline const double* row_ptr(const std::vector<double>& data, bool shared, long long per_row, long long r) {
  return data.data() + (shared ? 0 : r * per_row);
}

}  // namespace detail

// ----------------------------------------------------------- BatchedStore --
//
// The rows axis the reference lacks (it exists only as scalar_ir's
// EmitStrategy.rows, scalar_ir.hpp:77): R instances of one cascade, each the
// reference's TensorStore row. An input is per row ([R, len(, free)],
// row-major, reduce-axis-major inside a row like TensorStore) or shared by
// every row ([len(, free)], e.g. the static GEMM weight and gamma).
class BatchedStore {
 public:
  struct Array {
    std::vector<double> data;
    long long rows = 1, len = 0, free_len = 0;
    bool shared = false;
    long long per_row() const { return free_len > 0 ? len * free_len : len; }
  };
  void define_rows(const std::string& name, long long rows, long long len, long long free_len,
                   std::vector<double> data) {
    Array a;
    a.rows = rows;
    a.len = len;
    a.free_len = free_len;
    if (rows < 0 || static_cast<long long>(data.size()) != rows * a.per_row())
      throw ShapeMismatch(name + ": got " + std::to_string(data.size()) + " values, want " +
                          std::to_string(rows) + " x " + std::to_string(a.per_row()));
    a.data = std::move(data);
    arrays_[name] = std::move(a);
  }
  void define_shared(const std::string& name, long long len, long long free_len, std::vector<double> data) {
    define_rows(name, 1, len, free_len, std::move(data));
    arrays_[name].shared = true;
  }
  const Array& array(const std::string& name) const {
    auto it = arrays_.find(name);
    if (it == arrays_.end()) throw ShapeMismatch("no array named " + name);
    return it->second;
  }
  // The common row count of the per-row arrays (1 if every array is shared).
  long long rows() const {
    long long r = -1;
    for (const auto& kv : arrays_) {
      if (kv.second.shared) continue;
      if (r >= 0 && kv.second.rows != r) throw ShapeMismatch(kv.first + ": row count disagrees with the batch");
      r = kv.second.rows;
    }
    return r < 0 ? 1 : r;
  }

 private:
  std::map<std::string, Array> arrays_;
};

namespace detail {

// The batched fused loop: every row of `st` through one kernel launch
// sequence (rf_run_host), one ExecReport per row with the reference's field
// meanings. Single-row run_incremental / run_multisegment are R = 1.
inline std::vector<ExecReport> execute_batched(const Program& prog, const TreeConfig& cfg, long long segments,
                                               const BatchedStore& st, const std::string& strategy,
                                               int fuse_level = 0) {
  // validate_tree (cascade.cpp:37-66) + store shapes (simulator.cpp:235-245)
  if (cfg.levels.size() < 2 || cfg.levels.front() != prog.L0 || cfg.levels.back() != 1)
    throw ShapeMismatch("BadTree: levels must run from L0 = " + std::to_string(prog.L0) + " to 1");
  for (std::size_t k = 1; k < cfg.levels.size(); ++k) {
    if (cfg.levels[k] == 1 && cfg.levels[k - 1] == 1) continue;  // [1, 1]: a length-1 axis
    if (cfg.levels[k] <= 0 || cfg.levels[k] >= cfg.levels[k - 1])
      throw ShapeMismatch("NotDecreasing: levels must strictly decrease at index " + std::to_string(k));
    if (cfg.levels[k - 1] % cfg.levels[k] != 0) throw ShapeMismatch("BadTree: level widths must divide");
  }
  for (const auto& in : prog.spec.inputs) {
    const auto& a = st.array(in.name);
    if (a.len != in.len || a.free_len != in.free_len)
      throw ShapeMismatch(in.name + ": store shape does not match the spec");
  }
  if (segments < 1 || prog.L0 % segments != 0)  // simulator.cpp:668-671
    throw IncompatibleSegmentation(std::to_string(segments) + " segments do not divide L0 = " +
                                   std::to_string(prog.L0));
  if (fuse_level != 0 && (fuse_level < 1 || fuse_level > cfg.depth()))  // simulator.cpp:491-493
    throw std::out_of_range("fuse level out of range");
  // run_fused: hand the tree to the plan (rf_desc.fuse_level / tree, ABI v5);
  // the kernel evaluates each level-1 segment non-incrementally.
  auto fuse = [&](rf_desc& d) {
    if (fuse_level == 0) return;
    if (d.len != prog.L0)
      throw NotFusable("run_fused: the level-1 segments must be whole kernel K tiles (L0 = " +
                       std::to_string(prog.L0) + ")");
    d.segments = 1;
    d.fuse_level = fuse_level;
    d.tree_depth = cfg.depth();
    for (int i = 0; i < cfg.depth() && i < 8; ++i) d.tree[i] = cfg.levels[static_cast<std::size_t>(i) + 1];
  };
  const long long R = st.rows();
  std::vector<ExecReport> reps(R);
  for (auto& r : reps) r.strategy = strategy;
  if (R == 0) return reps;
  const long long L0 = prog.L0;
  auto out = [&](long long r, int id, std::vector<double> v) {
    OutputVal o;
    o.id = id;
    o.v = std::move(v);
    reps[r].outputs.push_back(std::move(o));
  };
  // per-row operand r of input `name`, as float
  auto rows_f = [&](const std::string& name, long long rows) {
    const auto& a = st.array(name);
    std::vector<float> f(rows * a.per_row());
    for (long long r = 0; r < rows; ++r) {
      const double* src = row_ptr(a.data, a.shared, a.per_row(), std::min(r, a.rows - 1));
      std::copy(src, src + a.per_row(), f.begin() + r * a.per_row());
    }
    return f;
  };
  // the GEMM patterns share one static weight over the batch (it is packed
  // once into the kernel's K-major tiles)
  auto shared_weight = [&](const std::string& name) {
    const auto& a = st.array(name);
    if (!a.shared && a.rows != 1)
      throw NotFusable(name + ": batched GEMM rows must share the weight (define_shared)");
    return a.data.data();
  };
  switch (prog.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX:
    case RF_PATTERN_MOE_ROUTING: {
      const bool moe = prog.pattern == RF_PATTERN_MOE_ROUTING;
      const int K = moe ? static_cast<int>(prog.free_len) : 0;
      rf_desc d = base_desc(prog.pattern, RF_F32);
      d.rows = R;
      d.len = L0;
      d.free_len = K;
      fuse(d);
      PlanHandle h(d);
      std::vector<float> xf = rows_f(prog.x, R), m(R), t(R);
      std::vector<int32_t> rec(moe ? 2 * K * R : 0);
      rf_host_io io{};
      io.in[0] = xf.data();
      io.d[0] = m.data();
      io.d[1] = t.data();
      io.d[2] = moe ? rec.data() : nullptr;
      check(rf_run_host(h.p, &io));
      for (long long r = 0; r < R; ++r) {
        out(r, 1, {m[r]});
        out(r, 2, {t[r]});
        if (!moe) continue;
        OutputVal o;
        o.id = 3;
        for (int j = 0; j < K; ++j) {
          const int32_t* e = &rec[2 * (r * K + j)];
          if (e[1] == 0) break;  // fewer experts than K'
          float v;
          std::memcpy(&v, &e[0], 4);
          o.topk.emplace_back(static_cast<double>(v), static_cast<long long>(e[1]));
        }
        reps[r].outputs.push_back(std::move(o));
      }
      break;
    }
    case RF_PATTERN_ATTENTION: {
      // Each row is one (b,h) unit with one query: P and V. The kernel
      // consumes Q, K, V with P = Q K^T; q = e_0 and K[l] = (P[l], 0, ...)
      // reproduce P exactly in fp32.
      const long long hd = prog.free_len;
      long long D = 16;
      while (D < hd) D *= 2;
      if (D > 128) throw NotFusable("attention head dim > 128");
      rf_desc d = base_desc(RF_PATTERN_ATTENTION, RF_F32);
      d.heads = R;
      d.rows = 1;
      d.len = L0;
      d.free_len = D;
      d.segments = segments;
      fuse(d);
      PlanHandle h(d);
      const auto& P = st.array(prog.x);
      const auto& V = st.array(prog.v);
      std::vector<float> q(R * D, 0.f), k(R * L0 * D, 0.f), v(R * L0 * D, 0.f), o(R * D), m(R), t(R);
      for (long long r = 0; r < R; ++r) {
        q[r * D] = 1.f;
        const double* pr = row_ptr(P.data, P.shared, P.per_row(), std::min(r, P.rows - 1));
        const double* vr = row_ptr(V.data, V.shared, V.per_row(), std::min(r, V.rows - 1));
        for (long long l = 0; l < L0; ++l) {
          k[(r * L0 + l) * D] = static_cast<float>(pr[l]);
          for (long long f = 0; f < hd; ++f) v[(r * L0 + l) * D + f] = static_cast<float>(vr[l * hd + f]);
        }
      }
      rf_host_io io{};
      io.in[0] = q.data();
      io.in[1] = k.data();
      io.in[2] = v.data();
      io.d[0] = m.data();
      io.d[1] = t.data();
      io.d[2] = o.data();
      check(rf_run_host(h.p, &io));
      for (long long r = 0; r < R; ++r) {
        out(r, 1, {m[r]});
        out(r, 2, {t[r]});
        out(r, 3, std::vector<double>(o.begin() + r * D, o.begin() + r * D + hd));
      }
      break;
    }
    case RF_PATTERN_QUANT_GEMM_E4M3:
    case RF_PATTERN_RMSNORM_GEMM:
    case RF_PATTERN_LAYERNORM_GEMM: {
      const bool quant = prog.pattern == RF_PATTERN_QUANT_GEMM_E4M3;
      const bool ln = prog.pattern == RF_PATTERN_LAYERNORM_GEMM;
      // Pad to the kernel tiles: M to whole row tiles (copies of row 0: never
      // an all-zero padding row), K with zeros — neutral for max|a|, sum x and
      // sum x^2, zero contributions; the statistics' means keep the cascade's
      // own L0 (rf_desc.stat_len) — and N with zero weight columns.
      const long long N = prog.free_len;
      const long long Kp = round_up(L0, quant ? 128 : 64), Np = round_up(N, quant ? 512 : 256);
      const long long M = round_up(R, ln ? 256 : 128);
      rf_desc d = base_desc(prog.pattern, RF_BF16);
      d.rows = M;
      d.len = Kp;
      d.free_len = Np;
      d.stat_len = quant ? 0 : L0;
      // run_multisegment: the kernels split K into S slices (split-K partials
      // + slice-ordered fold, gemm_fold.cu) when the reference's slices of
      // L0 / S are whole K tiles; otherwise one segment (equal in exact
      // arithmetic; the S | L0 contract was checked above)
      d.segments = L0 % (segments * (quant ? 128 : 64)) == 0 ? segments : 1;
      d.fmax = prog.fmax;
      d.eps = prog.eps;
      fuse(d);
      PlanHandle h(d);
      const double* W = shared_weight(prog.w);
      std::vector<float> wf(Kp * Np, 0.f), gf(Kp, 0.f);
      for (long long l = 0; l < L0; ++l)
        for (long long f = 0; f < N; ++f) wf[l * Np + f] = static_cast<float>(W[l * N + f]);
      if (!quant) {
        const double* g = shared_weight(prog.g);
        for (long long l = 0; l < L0; ++l) gf[l] = static_cast<float>(g[l]);
      }
      void* packed = nullptr;
      check(rf_pack_weight_host(h.p, wf.data(), quant ? nullptr : gf.data(), &packed));
      const auto& A = st.array(prog.x);
      std::vector<uint16_t> a(M * Kp, 0);
      for (long long r = 0; r < M; ++r) {
        const double* ar = row_ptr(A.data, A.shared, A.per_row(), r < R ? std::min(r, A.rows - 1) : 0);
        for (long long l = 0; l < L0; ++l) a[r * Kp + l] = to_bf16(static_cast<float>(ar[l]));
      }
      std::vector<float> d1(M), d2(ln ? M : 0), cf(quant ? M * Np : 0);
      std::vector<uint16_t> cb(quant ? 0 : M * Np), c4(ln ? M * Np : 0);
      rf_host_io io{};
      io.in[0] = a.data();
      io.in[1] = packed;
      io.d[0] = d1.data();
      if (ln) {
        io.d[1] = d2.data();
        io.d[2] = cb.data();
        io.d[3] = c4.data();
      } else {
        io.d[1] = quant ? static_cast<void*>(cf.data()) : static_cast<void*>(cb.data());
      }
      const rf_status s = rf_run_host(h.p, &io);
      rf_buffer_free(packed);
      check(s);
      bool domain = false;
      for (long long r = 0; r < R; ++r) {
        std::vector<double> c(N), c4r(ln ? N : 0);
        for (long long f = 0; f < N; ++f) {
          c[f] = quant ? cf[r * Np + f] : from_bf16(cb[r * Np + f]);
          if (ln) c4r[f] = from_bf16(c4[r * Np + f]);
        }
        out(r, 1, {d1[r]});
        if (ln) out(r, 2, {d2[r]});
        out(r, ln ? 3 : 2, c);
        if (ln) out(r, 4, c4r);
        if (quant && !(d1[r] > 0.0f)) domain = true;
      }
      if (domain)  // finalize_root: 0/0 faults propagate (a row's absmax is 0)
        throw DomainError("division by zero");
      break;
    }
    case RF_PATTERN_VARIANCE:
    case RF_PATTERN_SUM_SUM:
    case RF_PATTERN_MOMENTS: {
      const bool mom = prog.pattern == RF_PATTERN_MOMENTS;
      const long long F = mom ? prog.free_len : 1;
      rf_desc d = base_desc(prog.pattern, RF_F32);
      d.rows = R;
      d.len = L0;
      d.free_len = mom ? F : 0;
      d.segments = segments;
      d.eps = prog.eps;
      d.offset = prog.offset;
      fuse(d);
      PlanHandle h(d);
      std::vector<float> xf = rows_f(prog.x, R), yf;
      if (prog.pattern != RF_PATTERN_VARIANCE) yf = rows_f(prog.v, R);
      std::vector<float> o1(R), o2(R * F), o3(mom ? R * F : 0);
      rf_host_io io{};
      io.in[0] = xf.data();
      io.in[1] = yf.empty() ? nullptr : yf.data();
      io.d[0] = o1.data();
      io.d[1] = o2.data();
      io.d[2] = mom ? o3.data() : nullptr;
      check(rf_run_host(h.p, &io));
      for (long long r = 0; r < R; ++r) {
        out(r, 1, {o1[r]});
        out(r, 2, std::vector<double>(o2.begin() + r * F, o2.begin() + (r + 1) * F));
        if (mom) out(r, 3, std::vector<double>(o3.begin() + r * F, o3.begin() + (r + 1) * F));
      }
      break;
    }
    default: throw NotFusable("unknown pattern");
  }
  for (auto& r : reps) fill_counters(prog, cfg, r, fuse_level);
  return reps;
}

inline ExecReport execute(const Program& prog, const TreeConfig& cfg, long long segments,
                          TensorStore& st, const std::string& strategy, int fuse_level = 0) {
  BatchedStore b;
  for (const auto& in : prog.spec.inputs) {
    const auto& a = st.array(in.name);  // ShapeMismatch if absent
    b.define_rows(in.name, 1, a.len, a.free_len, a.data);
  }
  return execute_batched(prog, cfg, segments, b, strategy, fuse_level).front();
}

}  // namespace detail

// run_incremental (simulator.hpp:76-77): the Single-Segment fused loop.
inline ExecReport run_incremental(const Program& prog, const TreeConfig& cfg, TensorStore& store) {
  return detail::execute(prog, cfg, 1, store, "incremental");
}

// run_multisegment (simulator.hpp:81-82): S equal slices streamed
// independently and merged in slice order (split-KV).
inline ExecReport run_multisegment(const Program& prog, const TreeConfig& cfg, long long num_segments,
                                   TensorStore& store) {
  return detail::execute(prog, cfg, num_segments, store, "multi:" + std::to_string(num_segments));
}

// run_fused (simulator.hpp, simulator.cpp:485-559): fusion at level k, the
// non-incremental executor. Each level-1 segment (L0 / levels[1] elements) is
// buffered on chip and evaluated with its own dependency values, then the
// segment states are corrected and folded in segment order. A segment longer
// than the kernel's on-chip buffer raises NotFusable.
inline ExecReport run_fused(const Program& prog, const TreeConfig& cfg, int fuse_level, TensorStore& store) {
  return detail::execute(prog, cfg, 1, store, "fused:k=" + std::to_string(fuse_level), fuse_level);
}

// The batched executors: every row of the store in one run, one ExecReport
// per row (the reference's executors take one TensorStore = one row).
inline std::vector<ExecReport> run_batched(const Program& prog, const TreeConfig& cfg, const BatchedStore& store,
                                           long long num_segments = 1) {
  return detail::execute_batched(prog, cfg, num_segments, store,
                                 num_segments == 1 ? "incremental" : "multi:" + std::to_string(num_segments));
}

}  // namespace rfcuda
