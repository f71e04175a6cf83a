// Reference-side binding (what a RedFuser maintainer adds to proj/): a CUDA
// executor with the exact signature of the reference's executors
// (proj/include/redfuse/simulator.hpp:76-82), backed by librf_cuda through
// the C++ host layer include/rf_host.hpp. See INTEGRATION.md.
#pragma once

#include <string>
#include <vector>

#include "redfuse/acrf.hpp"
#include "redfuse/simulator.hpp"

namespace redfuse {

// Same contract as run_incremental / run_multisegment; throws the reference's
// ShapeMismatch / IncompatibleSegmentation / DomainError, and NotFusable when
// librf_cuda has no kernel for the cascade (there is no CPU fallback).
ExecReport run_cuda(const FusedProgram& prog, const TreeConfig& cfg, TensorStore& store);
ExecReport run_cuda_multisegment(const FusedProgram& prog, const TreeConfig& cfg,
                                 long long num_segments, TensorStore& store);
// Same contract as run_fused (simulator.cpp:485-559): fusion at level k, the
// level-1 segments evaluated non-incrementally on chip. NotFusable when a
// segment exceeds the kernel's on-chip buffer;
// std::out_of_range for k outside 1..depth, as the reference.
ExecReport run_cuda_fused(const FusedProgram& prog, const TreeConfig& cfg, int fuse_level,
                          TensorStore& store);

// Batched drop-in (the rows axis the reference only has as scalar_ir's
// EmitStrategy.rows, scalar_ir.hpp:77): R cascade rows — one TensorStore
// each, as run_incremental takes them — in ONE librf_cuda run, one
// ExecReport per row. Inputs identical in every store (the static GEMM
// weight, gamma) are passed once; the GEMM patterns require that.
// num_segments > 1 is run_multisegment per row.
std::vector<ExecReport> run_cuda_batched(const FusedProgram& prog, const TreeConfig& cfg,
                                         std::vector<TensorStore>& stores, long long num_segments = 1);

// The librf_cuda pattern a cascade maps onto ("attention", "safe_softmax",
// "moe_routing", "quant_gemm_e4m3", "rmsnorm_gemm", "layernorm_gemm"), and
// whether its operands are fp32 (else bf16/e4m3). Throws NotFusable when no
// kernel implements the cascade.
struct CudaPattern {
  std::string name;
  bool fp32 = true;
};
CudaPattern cuda_pattern(const FusedProgram& prog);

}  // namespace redfuse
