// Multi-Segment combine: folds split-KV partial states (m_s, l_s, O_s) into
// the root in slice order (incr_push_child, proj/src/simulator.cpp:592-608;
// closed form and evaluation order in fold.cuh). One thread per (row, 4
// columns): a merge costs ~2 dependent memory round trips regardless of the
// slice count, and the evaluation order is fixed for a given slice count, so
// results do not depend on scheduling.
#include <cuda_bf16.h>

#include "fold.cuh"
#include "rf_internal.h"

namespace rf {
namespace {

template <typename TO, int R>
__global__ void __launch_bounds__(128) merge_kernel(const float* __restrict__ pm, const float* __restrict__ pl,
                                                    const float* __restrict__ po, int64_t nslices, int64_t rows,
                                                    int64_t stride, int64_t d, float* __restrict__ m_out,
                                                    float* __restrict__ l_out, TO* __restrict__ o_out) {
  // launched as a programmatic dependent of the split kernel: wait for its
  // grid (and memory) to complete before reading partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t cpr = d / 4;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = t / cpr;
  if (row >= rows) return;
  fold_chunk<TO, R>(pm, pl, po, nslices, stride, d, row, t - row * cpr, m_out, l_out, o_out);
}

}  // namespace

cudaError_t launch_attention_merge(const float* pm, const float* pl, const float* po,
                                   int64_t nslices, int64_t rows, int64_t stride, int64_t d,
                                   float* m, float* l, void* o, int out_dtype,
                                   cudaStream_t st) {
  if (d % 4 != 0) return cudaErrorNotSupported;
  const int64_t threads = rows * (d / 4);
  // Programmatic dependent launch: the merge grid is scheduled while the split
  // kernel drains (its launch latency overlaps that kernel's tail);
  // griddepcontrol.wait in the kernel orders the partial reads.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((threads + 127) / 128));
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kernel, auto* out) {
    return cudaLaunchKernelEx(&cfg, kernel, pm, pl, po, nslices, rows, stride, d, m, l, out);
  };
  if (out_dtype == RF_BF16) {
    auto* ob = static_cast<__nv_bfloat16*>(o);
    if (nslices <= 2) return go(merge_kernel<__nv_bfloat16, 2>, ob);
    if (nslices <= 4) return go(merge_kernel<__nv_bfloat16, 4>, ob);
    if (nslices <= 8) return go(merge_kernel<__nv_bfloat16, 8>, ob);
    return go(merge_kernel<__nv_bfloat16, 16>, ob);
  }
  auto* of = static_cast<float*>(o);
  if (nslices <= 2) return go(merge_kernel<float, 2>, of);
  if (nslices <= 4) return go(merge_kernel<float, 4>, of);
  if (nslices <= 8) return go(merge_kernel<float, 8>, of);
  return go(merge_kernel<float, 16>, of);
}

}  // namespace rf
