// Reference-side binding: redfuse::run_cuda over librf_cuda (see redfuse_cuda.hpp).
// The cascade travels through the reference's own DSL serializer
// (cascade.hpp:93 serialize) into the host layer's parser + pattern matcher;
// the TensorStore arrays are handed over as-is and the ExecReport is returned
// with the reference's field meanings.
#include "redfuse_cuda.hpp"

#include <string>
#include <utility>
#include <vector>

#include "redfuse/cascade.hpp"
#include "redfuse/expr.hpp"
#include "rf_host.hpp"

namespace redfuse {
namespace {

// The FusedProgram's derived corrections (derive_fused, acrf.cpp:184-186) in
// the reference's own rendering, for the plan layer's pin against the kernel.
std::vector<std::pair<int, std::string>> derived_corrections(const FusedProgram& prog) {
  std::vector<std::pair<int, std::string>> out;
  for (const auto& d : prog.decomps) out.emplace_back(d.id, d.corr ? render(d.corr) : "");
  return out;
}

// Matches the cascade onto a kernel AND checks that every derived correction
// is numerically the kernel's closed form (rfcuda::check_corrections, the
// reference's numeric_equiv probe); either failure is NotFusable.
rfcuda::Program plan_checked(const FusedProgram& prog) {
  try {
    return rfcuda::plan(rfcuda::parse_cascade(serialize(prog.spec)), derived_corrections(prog));
  } catch (const rfcuda::NotFusable& e) {
    throw NotFusable(0, e.what());
  }
}

ExecReport to_reference(const rfcuda::ExecReport& r) {
  ExecReport out;
  out.strategy = "cuda:" + r.strategy;
  for (const auto& o : r.outputs) out.outputs.push_back(OutputVal{o.id, o.v, o.topk});
  out.input_loads = r.input_loads;
  out.dep_root_loads = r.dep_root_loads;
  out.peak_aux_slots = r.peak_aux_slots;
  return out;
}

ExecReport run(const FusedProgram& prog, const TreeConfig& cfg, long long segments,
               TensorStore& store, int fuse_level = 0) {
  rfcuda::Program p = plan_checked(prog);
  rfcuda::TensorStore st;
  for (const auto& in : prog.spec.inputs) {
    const auto& a = store.array(in.name);  // ShapeMismatch if absent
    st.define(in.name, a.len, a.free_len, a.data);
  }
  rfcuda::ExecReport r;
  try {
    r = fuse_level > 0 ? rfcuda::run_fused(p, rfcuda::TreeConfig{cfg.levels}, fuse_level, st)
        : segments == 1 ? rfcuda::run_incremental(p, rfcuda::TreeConfig{cfg.levels}, st)
                        : rfcuda::run_multisegment(p, rfcuda::TreeConfig{cfg.levels}, segments, st);
  } catch (const rfcuda::ShapeMismatch& e) {
    throw ShapeMismatch(e.what());
  } catch (const rfcuda::IncompatibleSegmentation& e) {
    throw IncompatibleSegmentation(e.what());
  } catch (const rfcuda::DomainError& e) {
    throw DomainError(e.what());
  } catch (const rfcuda::NotFusable& e) {
    throw NotFusable(0, e.what());
  }
  return to_reference(r);
}

}  // namespace

std::vector<ExecReport> run_cuda_batched(const FusedProgram& prog, const TreeConfig& cfg,
                                         std::vector<TensorStore>& stores, long long num_segments) {
  rfcuda::Program p = plan_checked(prog);
  std::vector<ExecReport> out;
  if (stores.empty()) return out;
  rfcuda::BatchedStore b;
  const long long R = static_cast<long long>(stores.size());
  for (const auto& in : prog.spec.inputs) {
    const auto& a0 = stores[0].array(in.name);  // ShapeMismatch if absent
    bool same = R > 1;
    for (long long r = 1; r < R && same; ++r) {
      const auto& ar = stores[r].array(in.name);
      same = ar.len == a0.len && ar.free_len == a0.free_len && ar.data == a0.data;
    }
    if (same) {
      b.define_shared(in.name, a0.len, a0.free_len, a0.data);
      continue;
    }
    std::vector<double> rows;
    rows.reserve(a0.data.size() * R);
    for (long long r = 0; r < R; ++r) {
      const auto& ar = stores[r].array(in.name);
      if (ar.len != a0.len || ar.free_len != a0.free_len)
        throw ShapeMismatch(in.name + ": batched rows disagree in shape");
      rows.insert(rows.end(), ar.data.begin(), ar.data.end());
    }
    b.define_rows(in.name, R, a0.len, a0.free_len, std::move(rows));
  }
  std::vector<rfcuda::ExecReport> reps;
  try {
    reps = rfcuda::run_batched(p, rfcuda::TreeConfig{cfg.levels}, b, num_segments);
  } catch (const rfcuda::ShapeMismatch& e) {
    throw ShapeMismatch(e.what());
  } catch (const rfcuda::IncompatibleSegmentation& e) {
    throw IncompatibleSegmentation(e.what());
  } catch (const rfcuda::DomainError& e) {
    throw DomainError(e.what());
  } catch (const rfcuda::NotFusable& e) {
    throw NotFusable(0, e.what());
  }
  for (const auto& r : reps) out.push_back(to_reference(r));
  return out;
}

CudaPattern cuda_pattern(const FusedProgram& prog) {
  rfcuda::Program p = plan_checked(prog);
  switch (p.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX: return {"safe_softmax", true};
    case RF_PATTERN_ATTENTION: return {"attention", true};
    case RF_PATTERN_MOE_ROUTING: return {"moe_routing", true};
    case RF_PATTERN_QUANT_GEMM_E4M3: return {"quant_gemm_e4m3", false};
    case RF_PATTERN_RMSNORM_GEMM: return {"rmsnorm_gemm", false};
    case RF_PATTERN_LAYERNORM_GEMM: return {"layernorm_gemm", false};
    case RF_PATTERN_VARIANCE: return {"variance", true};
    case RF_PATTERN_SUM_SUM: return {"sum_sum", true};
    case RF_PATTERN_MOMENTS: return {"moment_of_inertia", true};
  }
  throw NotFusable(0, "unknown librf_cuda pattern");
}

ExecReport run_cuda(const FusedProgram& prog, const TreeConfig& cfg, TensorStore& store) {
  return run(prog, cfg, 1, store);
}

ExecReport run_cuda_multisegment(const FusedProgram& prog, const TreeConfig& cfg,
                                 long long num_segments, TensorStore& store) {
  return run(prog, cfg, num_segments, store);
}

ExecReport run_cuda_fused(const FusedProgram& prog, const TreeConfig& cfg, int fuse_level,
                          TensorStore& store) {
  return run(prog, cfg, 1, store, fuse_level);
}

}  // namespace redfuse
