"""B200-native (sm_100a) fused cascaded-reduction executors — a drop-in for
the RedFuser reference's CPU fused-loop executors (run_incremental /
run_multisegment, /root/reference/proj/src/simulator.cpp:566-687).

Compute lives in librf_cuda.so (hand-written CUDA, C-ABI in include/rf_cuda.h);
this package is the host-side mirror of the reference operator API.
"""
from .executors import (  # noqa: F401
    CudaError,
    Desc,
    DomainError,
    IncompatibleSegmentation,
    Plan,
    RedfuseError,
    ShapeMismatch,
    UnsupportedPattern,
    attention,
    layernorm_gemm,
    layernorm_gemm_plan,
    mla_decode,
    moe_router,
    moe_router_plan,
    moe_routing,
    moments,
    plan,
    quant_gemm,
    quant_gemm_plan,
    rmsnorm_gemm,
    rmsnorm_gemm_plan,
    safe_softmax,
    sum_sum,
    variance,
)

__all__ = [
    "attention",
    "safe_softmax",
    "quant_gemm",
    "rmsnorm_gemm",
    "layernorm_gemm",
    "moe_routing",
    "moe_router",
    "mla_decode",
    "variance",
    "sum_sum",
    "moments",
    "Plan",
    "Desc",
    "plan",
]
