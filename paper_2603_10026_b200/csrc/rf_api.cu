// librf_cuda C-ABI: plan layer (descriptor validation, kernel + tile choice,
// workspace), stream-ordered dispatch, host-buffer end-to-end path.
//
// Reference interface replaced (see include/rf_cuda.h): run_incremental /
// run_multisegment (proj/include/redfuse/simulator.hpp:76-82). Error mapping
// mirrors the reference's exceptions: ShapeMismatch (check_shapes,
// proj/src/simulator.cpp:235-245), IncompatibleSegmentation
// (simulator.cpp:668-671), DomainError at finalize (simulator.cpp:611-621).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "rf_internal.h"

namespace rf {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace rf

using rf::set_error;

struct rf_plan {
  rf_desc d{};
  rf::Kernel kernel = rf::Kernel::SoftmaxRows;
  int64_t rows_total = 0;   // B*H*Sq (attention) / M (GEMM) / rows (softmax)
  int64_t nsplit = 1;       // slices actually launched (>= segments for decode)
  int64_t launches = 1;
  // Segment partial workspace (attention, nsplit > 1).
  float* ws_m = nullptr;
  float* ws_l = nullptr;
  float* ws_o = nullptr;
  unsigned long long* ws_cnt = nullptr;  // arrival counters (MLA decode's in-kernel fold)
  int* domain_flag = nullptr;
  // Host-path staging (rf_run_host), allocated on first use.
  bool staged = false;
  void* dev_in[4] = {nullptr, nullptr, nullptr, nullptr};
  void* dev_out[4] = {nullptr, nullptr, nullptr, nullptr};
  // rf_run_host: H2D, compute and D2H streams, and per-chunk events linking them
  static constexpr int kChunks = 16;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_in[kChunks] = {}, ev_done[kChunks] = {};
  std::string describe;
};

namespace {

size_t dtype_size(int dt) { return dt == RF_F32 ? 4 : dt == RF_BF16 ? 2 : 1; }

rf_status fail(rf_status s, const std::string& msg) {
  set_error(msg);
  return s;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Selects the plan's device for the duration of an entry point and restores
// the caller's device on every return path.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Patterns with a plan-time packed weight in in[1] (tcgen05 GEMM tiles of 128 rows).
bool is_gemm(int pattern) {
  return pattern == RF_PATTERN_QUANT_GEMM_E4M3 || pattern == RF_PATTERN_RMSNORM_GEMM ||
         pattern == RF_PATTERN_LAYERNORM_GEMM || pattern == RF_PATTERN_MOE_ROUTER;
}

// The packed weight's source w [k, n] (reduce-axis major): GEMM patterns
// w [K, N]; the MoE router's w [hd, experts].
void pack_dims(const rf_desc& d, int64_t& k, int64_t& n) {
  if (d.pattern == RF_PATTERN_MOE_ROUTER) {
    k = d.producer_len;
    n = d.len;
  } else {
    k = d.len;
    n = d.free_len;
  }
}

// Input/output byte sizes per pattern, for the host path and shape checks.
void io_sizes(const rf_plan* p, size_t in[4], size_t out[4]) {
  const rf_desc& d = p->d;
  for (int i = 0; i < 4; ++i) in[i] = 0;
  for (int i = 0; i < 4; ++i) out[i] = 0;
  const size_t es = dtype_size(d.dtype);
  switch (d.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX:
      in[0] = sizeof(float) * d.rows * d.len;
      out[0] = out[1] = sizeof(float) * d.rows;
      break;
    case RF_PATTERN_ATTENTION: {
      const int64_t bh = d.batch * d.heads;
      in[0] = es * bh * d.rows * d.free_len;
      in[1] = in[2] = es * bh * d.len * d.free_len;
      out[0] = out[1] = sizeof(float) * bh * d.rows;
      out[2] = es * bh * d.rows * d.free_len;
      break;
    }
    case RF_PATTERN_QUANT_GEMM_E4M3:
      in[0] = 2 * d.rows * d.len;
      out[0] = sizeof(float) * d.rows;
      out[1] = sizeof(float) * d.rows * d.free_len;
      break;
    case RF_PATTERN_RMSNORM_GEMM:
      in[0] = 2 * d.rows * d.len;
      out[0] = sizeof(float) * d.rows;
      out[1] = 2 * d.rows * d.free_len;
      break;
    case RF_PATTERN_LAYERNORM_GEMM:
      in[0] = 2 * d.rows * d.len;
      out[0] = out[1] = sizeof(float) * d.rows;
      out[2] = out[3] = 2 * d.rows * d.free_len;
      break;
    case RF_PATTERN_MOE_ROUTING:
      in[0] = sizeof(float) * d.rows * d.len;
      out[0] = out[1] = sizeof(float) * d.rows;
      out[2] = 8 * d.rows * d.free_len;
      break;
    case RF_PATTERN_MLA_DECODE:
      in[0] = 2 * d.batch * d.heads * d.producer_len;
      in[1] = 2 * d.batch * d.len * d.producer_len;
      out[0] = out[1] = sizeof(float) * d.batch * d.heads;
      out[2] = 2 * d.batch * d.heads * d.free_len;
      break;
    case RF_PATTERN_MOE_ROUTER:
      in[0] = 2 * d.rows * d.producer_len;
      out[0] = out[1] = sizeof(float) * d.rows;
      out[2] = 8 * d.rows * d.free_len;
      out[3] = sizeof(float) * d.rows * d.len;
      break;
    case RF_PATTERN_VARIANCE:
      in[0] = sizeof(float) * d.rows * d.len;
      out[0] = out[1] = sizeof(float) * d.rows;
      break;
    case RF_PATTERN_SUM_SUM:
      in[0] = in[1] = sizeof(float) * d.rows * d.len;
      out[0] = out[1] = sizeof(float) * d.rows;
      break;
    case RF_PATTERN_MOMENTS:
      in[0] = sizeof(float) * d.rows * d.len;
      in[1] = sizeof(float) * d.rows * d.len * d.free_len;
      out[0] = sizeof(float) * d.rows;
      out[1] = out[2] = sizeof(float) * d.rows * d.free_len;
      break;
  }
}

const char* kernel_name(rf::Kernel k) {
  switch (k) {
    case rf::Kernel::SoftmaxRows: return "softmax_rows (SIMT, single pass)";
    case rf::Kernel::AttentionF32: return "attention_f32 (SIMT, paper form)";
    case rf::Kernel::AttentionTf32: return "attention_tf32 (fp32 as 3xTF32 tcgen05, in-cluster slice fold)";
    case rf::Kernel::AttentionSm100: return "attention_sm100 (bf16 tcgen05/TMEM/TMA, ping-pong Q tiles)";
    case rf::Kernel::AttentionDecode: return "attention_decode (bf16 split-KV, TMA bulk)";
    case rf::Kernel::QuantGemmSm100: return "quant_gemm_sm100 (e4m3 tcgen05 kind::f8f6f4)";
    case rf::Kernel::RmsGemmSm100: return "rmsnorm_gemm_sm100 (bf16 tcgen05 kind::f16)";
    case rf::Kernel::MoeRouting: return "moe_routing (SIMT, warp per token, bit-exact top-k)";
    case rf::Kernel::LayerNormGemmSm100: return "layernorm_gemm_sm100 (bf16 tcgen05 cta_group::2)";
    case rf::Kernel::RowStats: return "rowstats (SIMT HBM streaming, fp64 accumulation)";
    case rf::Kernel::MoeRouter: return "moe_router (tcgen05 split-K router GEMM + L2 split exchange + routing cascade, one launch)";
    case rf::Kernel::MlaDecode: return "mla_decode (tcgen05, 128 heads x latent cache, split-KV folded in-kernel)";
    case rf::Kernel::FusedRows: return "fused_rows (run_fused: warp-buffered level-1 segments, SIMT)";
  }
  return "?";
}

// Row coordinates of the flattened [B*H*S, D] attention views fit the TMA
// kernels' 32-bit coordinates.
bool tma_rows_fit(const rf_desc& d) {
  return d.batch * d.heads * std::max<int64_t>(d.rows, d.len) < (int64_t{1} << 31);
}

// Decode split count: a multiple of `segments` dividing Skv with slices of at
// least 512 keys, aiming at >= 4 CTAs per SM worth of (row, slice) units.
int64_t pick_decode_splits(int64_t rows, int64_t skv, int64_t segments) {
  int64_t best = segments;
  for (int64_t s = segments; s <= skv; s += segments) {
    if (skv % s) continue;
    if (skv / s < 512 && s != segments) break;
    best = s;
    if (rows * s >= 148 * 4) break;
  }
  return best;
}

rf_status attention_run(const rf_plan* p, const rf_io* io, int64_t bh0, int64_t nbh,
                        cudaStream_t st) {
  const rf_desc& d = p->d;
  const size_t es = dtype_size(d.dtype);
  const int64_t q_off = bh0 * d.rows * d.free_len, kv_off = bh0 * d.len * d.free_len;
  rf::AttnArgs a{};
  a.q = static_cast<const char*>(io->in[0]) + q_off * es;
  a.k = static_cast<const char*>(io->in[1]) + kv_off * es;
  a.v = static_cast<const char*>(io->in[2]) + kv_off * es;
  a.o = static_cast<char*>(io->d[2]) + q_off * es;
  a.m = static_cast<float*>(io->d[0]) + bh0 * d.rows;
  a.l = static_cast<float*>(io->d[1]) + bh0 * d.rows;
  a.bh = nbh;
  a.sq = d.rows;
  a.skv = d.len;
  a.d = d.free_len;
  a.segments = p->nsplit;
  a.slice_begin = 0;
  a.nslices = p->nsplit;
  a.part_base = 0;
  a.rows_total = p->rows_total;
  a.scale = static_cast<float>(d.softmax_scale);
  a.dtype = d.dtype;
  if (p->nsplit > 1) {
    a.part_m = p->ws_m + bh0 * d.rows;
    a.part_l = p->ws_l + bh0 * d.rows;
    a.part_o = p->ws_o + bh0 * d.rows * d.free_len;
  }
  cudaError_t e;
  switch (p->kernel) {
    case rf::Kernel::AttentionSm100: e = rf::launch_attention_sm100(a, st); break;
    case rf::Kernel::AttentionDecode: e = rf::launch_attention_decode(a, st); break;
    case rf::Kernel::AttentionTf32: e = rf::launch_attention_tf32(a, st); break;
    default: e = rf::launch_attention_f32(a, st); break;
  }
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
  if (p->nsplit > 1 && p->kernel != rf::Kernel::AttentionTf32) {  // tf32: folded in-kernel
    e = rf::launch_attention_merge(a.part_m, a.part_l, a.part_o, p->nsplit, nbh * d.rows,
                                   p->rows_total, d.free_len, a.m, a.l, a.o, d.dtype, st);
    if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("merge launch: ") + cudaGetErrorString(e));
  }
  return RF_OK;
}

rf_status gemm_run(const rf_plan* p, const rf_io* io, int64_t m0, int64_t nm, cudaStream_t st) {
  const rf_desc& d = p->d;
  rf::GemmArgs g{};
  g.a = static_cast<const char*>(io->in[0]) + 2 * m0 * d.len;
  g.b = io->in[1];
  g.d1 = static_cast<float*>(io->d[0]) + m0;
  const size_t cs = d.pattern == RF_PATTERN_QUANT_GEMM_E4M3 ? 4 : 2;
  if (d.pattern == RF_PATTERN_LAYERNORM_GEMM) {
    g.d2 = static_cast<float*>(io->d[1]) + m0;
    g.c = static_cast<char*>(io->d[2]) + cs * m0 * d.free_len;
    g.c4 = io->d[3] ? static_cast<char*>(io->d[3]) + cs * m0 * d.free_len : nullptr;
    g.colsum = reinterpret_cast<const float*>(static_cast<const char*>(io->in[1]) +
                                              2 * d.free_len * d.len);
  } else {
    g.c = static_cast<char*>(io->d[1]) + cs * m0 * d.free_len;
  }
  g.domain_flag = p->domain_flag;
  g.m = nm;
  g.n = d.free_len;
  g.k = d.len;
  g.stat_len = d.stat_len > 0 ? d.stat_len : d.len;
  g.fmax = static_cast<float>(d.fmax);
  g.eps = static_cast<float>(d.eps);
  g.segments = d.segments;
  g.ws_rows = d.rows;
  if (d.segments > 1) {  // run_multisegment: slice partials + ordered fold (gemm_fold.cu)
    g.ws = p->ws_o + m0 * d.free_len;
    g.ws_d1 = p->ws_m + m0;
    g.ws_d2 = p->ws_l ? p->ws_l + m0 : nullptr;
  }
  cudaError_t e = d.pattern == RF_PATTERN_QUANT_GEMM_E4M3 ? rf::launch_quant_gemm_sm100(g, st)
                  : d.pattern == RF_PATTERN_LAYERNORM_GEMM  ? rf::launch_layernorm_gemm_sm100(g, st)
                                                            : rf::launch_rms_gemm_sm100(g, st);
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return RF_OK;
}

rf_status run_range(const rf_plan* p, const rf_io* io, int64_t u0, int64_t nu, cudaStream_t st) {
  if (p->kernel == rf::Kernel::FusedRows) {  // run_fused on the row patterns
    const rf_desc& d = p->d;
    cudaError_t e = rf::launch_fused_rows(
        d.pattern, static_cast<const float*>(io->in[0]) + u0 * d.len,
        d.pattern == RF_PATTERN_SUM_SUM ? static_cast<const float*>(io->in[1]) + u0 * d.len : nullptr, nu,
        d.len, d.tree[0], d.offset, d.eps, static_cast<float*>(io->d[0]) + u0,
        static_cast<float*>(io->d[1]) + u0, st);
    if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("fused_rows launch: ") + cudaGetErrorString(e));
    return RF_OK;
  }
  switch (p->d.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX: {
      cudaError_t e = rf::launch_softmax_rows(
          static_cast<const float*>(io->in[0]) + u0 * p->d.len, nu, p->d.len,
          static_cast<float*>(io->d[0]) + u0, static_cast<float*>(io->d[1]) + u0, st);
      if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("softmax launch: ") + cudaGetErrorString(e));
      return RF_OK;
    }
    case RF_PATTERN_ATTENTION: return attention_run(p, io, u0, nu, st);
    case RF_PATTERN_MOE_ROUTING: {
      cudaError_t e = rf::launch_moe_routing(
          static_cast<const float*>(io->in[0]) + u0 * p->d.len, nu, p->d.len,
          static_cast<int>(p->d.free_len), static_cast<float*>(io->d[0]) + u0,
          static_cast<float*>(io->d[1]) + u0, static_cast<char*>(io->d[2]) + 8 * u0 * p->d.free_len, st);
      if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("moe launch: ") + cudaGetErrorString(e));
      return RF_OK;
    }
    case RF_PATTERN_MLA_DECODE: {
      const rf_desc& d = p->d;
      const int64_t hn = d.heads;
      rf::MlaArgs a{};
      a.q = static_cast<const char*>(io->in[0]) + 2 * u0 * hn * d.producer_len;
      a.kv = static_cast<const char*>(io->in[1]) + 2 * u0 * d.len * d.producer_len;
      a.o = static_cast<char*>(io->d[2]) + 2 * u0 * hn * d.free_len;
      a.m = static_cast<float*>(io->d[0]) + u0 * hn;
      a.l = static_cast<float*>(io->d[1]) + u0 * hn;
      a.bs = nu;
      a.skv = d.len;
      a.nslices = p->nsplit;
      a.rows_total = p->rows_total;
      a.scale = static_cast<float>(d.softmax_scale);
      if (p->nsplit > 1) {  // segment partials, folded inside the kernel (arrival counters per batch half)
        a.part_m = p->ws_m + u0 * hn;
        a.part_l = p->ws_l + u0 * hn;
        a.part_o = p->ws_o + u0 * hn * d.free_len;
        a.cnt = p->ws_cnt + 2 * u0;
      }
      cudaError_t e = rf::launch_mla_decode(a, st);
      if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("mla launch: ") + cudaGetErrorString(e));
      return RF_OK;
    }
    case RF_PATTERN_MOE_ROUTER: {
      const rf_desc& d = p->d;
      rf::RouterArgs r{};
      r.x = static_cast<const char*>(io->in[0]) + 2 * u0 * d.producer_len;
      r.w = io->in[1];
      r.part = p->ws_m + u0 * d.len;
      r.cnt = reinterpret_cast<unsigned long long*>(p->ws_l) + u0 / 128;
      r.rows = nu;
      r.hd = d.producer_len;
      r.experts = d.len;
      r.splits = p->nsplit;
      r.part_stride = d.rows;
      r.k = static_cast<int>(d.free_len);
      r.d1 = static_cast<float*>(io->d[0]) + u0;
      r.d2 = static_cast<float*>(io->d[1]) + u0;
      r.topk = static_cast<char*>(io->d[2]) + 8 * u0 * d.free_len;
      r.scores = io->d[3] ? static_cast<float*>(io->d[3]) + u0 * d.len : nullptr;
      cudaError_t e = rf::launch_router(r, st);
      if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("router launch: ") + cudaGetErrorString(e));
      return RF_OK;
    }
    case RF_PATTERN_VARIANCE:
    case RF_PATTERN_SUM_SUM:
    case RF_PATTERN_MOMENTS: {
      const rf_desc& d = p->d;
      const int64_t fl = d.pattern == RF_PATTERN_MOMENTS ? d.free_len : 0;
      rf::RowStatsArgs r{};
      r.pattern = d.pattern;
      r.a = static_cast<const float*>(io->in[0]) + u0 * d.len;
      r.b = d.pattern == RF_PATTERN_VARIANCE ? nullptr
                                             : static_cast<const float*>(io->in[1]) + u0 * d.len * std::max<int64_t>(fl, 1);
      r.rows = nu;
      r.len = d.len;
      r.free_len = fl;
      r.d1 = static_cast<float*>(io->d[0]) + u0;
      r.d2 = static_cast<float*>(io->d[1]) + u0 * std::max<int64_t>(fl, 1);
      r.d3 = fl ? static_cast<float*>(io->d[2]) + u0 * fl : nullptr;
      r.c = d.offset;
      r.eps = d.eps;
      cudaError_t e = rf::launch_rowstats(r, st);
      if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("rowstats launch: ") + cudaGetErrorString(e));
      return RF_OK;
    }
    default: return gemm_run(p, io, u0, nu, st);
  }
}

// Independent units for chunking: (b,h) pairs for attention, rows otherwise.
int64_t units_of(const rf_plan* p) {
  if (p->d.pattern == RF_PATTERN_MLA_DECODE) return p->d.batch;  // heads share the batch's cache
  return p->d.pattern == RF_PATTERN_ATTENTION ? p->d.batch * p->d.heads : p->d.rows;
}

}  // namespace

extern "C" {

int rf_abi_version(void) { return RF_CUDA_ABI_VERSION; }

const char* rf_status_string(rf_status s) {
  switch (s) {
    case RF_OK: return "RF_OK";
    case RF_ERR_SHAPE: return "RF_ERR_SHAPE (ShapeMismatch)";
    case RF_ERR_SEGMENTATION: return "RF_ERR_SEGMENTATION (IncompatibleSegmentation)";
    case RF_ERR_DOMAIN: return "RF_ERR_DOMAIN (DomainError)";
    case RF_ERR_UNSUPPORTED: return "RF_ERR_UNSUPPORTED";
    case RF_ERR_CUDA: return "RF_ERR_CUDA";
    case RF_ERR_NCCL: return "RF_ERR_NCCL";
    case RF_ERR_ARG: return "RF_ERR_ARG";
  }
  return "RF_ERR_UNKNOWN";
}

const char* rf_last_error(void) { return rf::g_last_error.c_str(); }

rf_status rf_plan_create(const rf_desc* desc, rf_plan** out) {
  if (!desc || !out) return fail(RF_ERR_ARG, "null desc/out");
  *out = nullptr;
  const rf_desc& d = *desc;
  // ---- shape validation (check_shapes, simulator.cpp:235-245) ----
  if (d.rows < 0 || d.len < 1 || d.free_len < 0 || d.batch < 1 || d.heads < 1)
    return fail(RF_ERR_SHAPE, "non-positive extent in descriptor");
  if (d.stat_len < 0 || d.stat_len > d.len) return fail(RF_ERR_SHAPE, "stat_len must be in [0, len]");
  if (d.segments < 1 || d.len % d.segments != 0)  // simulator.cpp:668-671
    return fail(RF_ERR_SEGMENTATION, std::to_string(d.segments) +
                                         " segments do not divide L0 = " + std::to_string(d.len));
  // run_fused: the reduction tree (validate_tree, cascade.cpp:37-66) and the
  // fuse level (simulator.cpp:491-493)
  int64_t fused_seg = 0;
  if (d.fuse_level != 0) {
    if (d.segments != 1) return fail(RF_ERR_ARG, "run_fused: segments must be 1 (the tree gives the segments)");
    if (d.tree_depth < 1 || d.tree_depth > 8) return fail(RF_ERR_SHAPE, "BadTree: depth must be 1..8");
    int64_t below = d.len;
    for (int i = 0; i < d.tree_depth; ++i) {
      if (d.tree[i] < 1 || (d.tree[i] >= below && !(d.tree[i] == 1 && below == 1)))
        return fail(RF_ERR_SHAPE, "NotDecreasing: levels must strictly decrease at index " + std::to_string(i + 1));
      if (below % d.tree[i] != 0)
        return fail(RF_ERR_SHAPE, "DivisibilityViolation: level widths must divide the level below");
      below = d.tree[i];
    }
    if (below != 1) return fail(RF_ERR_SHAPE, "BadTree: the last level must be 1");
    if (d.fuse_level < 1 || d.fuse_level > d.tree_depth)
      return fail(RF_ERR_ARG, "fuse level out of range");
    fused_seg = d.len / d.tree[0];
  }
  rf_plan* p = new (std::nothrow) rf_plan();
  if (!p) return fail(RF_ERR_CUDA, "out of host memory");
  p->d = d;
  if (p->d.softmax_scale == 0.0) p->d.softmax_scale = 1.0;
  if (p->d.fmax == 0.0) p->d.fmax = 448.0;
  auto bail = [&](rf_status s, const std::string& m) {
    rf_plan_destroy(p);
    return fail(s, m);
  };

  // ---- device: sm_100 only (no fallback) ----
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return bail(RF_ERR_CUDA, "no CUDA device (librf_cuda has no CPU fallback)");
  if (d.device < 0 || d.device >= ndev) return bail(RF_ERR_ARG, "bad device ordinal");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, d.device) != cudaSuccess)
    return bail(RF_ERR_CUDA, "cudaGetDeviceProperties failed");
  if (prop.major != 10 || prop.minor != 0)
    return bail(RF_ERR_CUDA, "librf_cuda is built for sm_100a only; device is sm_" +
                                 std::to_string(prop.major) + std::to_string(prop.minor));
  DeviceGuard guard(d.device);

  // ---- kernel choice ----
  if (fused_seg > 0) {
    // run_fused: every level-1 segment must fit the pattern's on-chip buffer
    // (non-incremental evaluation); the segments then run
    // as the kernel's slices and fold in segment order.
    const int64_t L1 = d.tree[0];
    auto too_long = [&](int64_t cap, const char* what) {
      return bail(RF_ERR_UNSUPPORTED, "run_fused: level-1 segment of " + std::to_string(fused_seg) +
                                          " elements exceeds the on-chip buffer (" + what + ": " +
                                          std::to_string(cap) + ")");
    };
    switch (d.pattern) {
      case RF_PATTERN_SAFE_SOFTMAX:
      case RF_PATTERN_VARIANCE:
      case RF_PATTERN_SUM_SUM:
        if (d.dtype != RF_F32) return bail(RF_ERR_UNSUPPORTED, "run_fused rows: f32 inputs");
        if (d.pattern == RF_PATTERN_SUM_SUM && !(d.eps > 0.0))
          return bail(RF_ERR_ARG, "sum_sum: eps must be > 0 (max(d1 - c, eps) is the H guard)");
        if (fused_seg > rf::kSegMax) return too_long(rf::kSegMax, "one warp's registers");
        if (L1 > rf::kFusedSegsMax)
          return bail(RF_ERR_UNSUPPORTED, "run_fused rows: more than 8192 level-1 segments per row");
        p->kernel = rf::Kernel::FusedRows;
        p->rows_total = d.rows;
        break;
      case RF_PATTERN_ATTENTION:
        // one KV tile per segment: the tile's row max is reduced before any
        // exponential, so the segment is evaluated non-incrementally
        if (d.dtype == RF_BF16 && d.rows > 1) {
          if (fused_seg != 128 || !rf::attention_sm100_supports(d.rows, d.len, d.free_len, L1))
            return bail(RF_ERR_UNSUPPORTED, "run_fused bf16 attention: segments of exactly one 128-key "
                                            "tcgen05 tile, Sq % 256 == 0");
          p->kernel = rf::Kernel::AttentionSm100;
        } else if (d.dtype == RF_F32) {
          if (fused_seg > 64) return too_long(64, "one 64-key fp32 tile");
          if (d.free_len != 16 && d.free_len != 32 && d.free_len != 64 && d.free_len != 128)
            return bail(RF_ERR_UNSUPPORTED, "attention: head_dim must be 16/32/64/128");
          p->kernel = rf::Kernel::AttentionF32;
        } else {
          return bail(RF_ERR_UNSUPPORTED, "run_fused attention: f32, or bf16 prefill (Sq % 256 == 0)");
        }
        p->rows_total = d.batch * d.heads * d.rows;
        p->nsplit = L1;
        p->d.segments = L1;
        break;
      case RF_PATTERN_QUANT_GEMM_E4M3:
      case RF_PATTERN_RMSNORM_GEMM:
      case RF_PATTERN_LAYERNORM_GEMM: {
        // quant: one 128-wide K tile per segment (its absmax is taken before
        // any element is quantised); rms / layernorm: the accumulator carries
        // H' = 1 and the segment's 1/sigma is applied once to the segment's
        // sum, which is the non-incremental form for any segment length.
        const bool quant = d.pattern == RF_PATTERN_QUANT_GEMM_E4M3;
        if (d.dtype != RF_BF16) return bail(RF_ERR_UNSUPPORTED, "GEMM patterns take bf16 activations");
        if (!rf::gemm_sm100_supports(d.pattern, d.rows, d.free_len, d.len))
          return bail(RF_ERR_UNSUPPORTED, "GEMM shape has no tcgen05 tiling");
        if (quant ? fused_seg != 128 : fused_seg % 64 != 0)
          return bail(RF_ERR_UNSUPPORTED, quant ? "run_fused quant: segments of exactly one 128-wide K tile"
                                                : "run_fused rms / layernorm: segments of whole 64-wide K tiles");
        p->kernel = quant ? rf::Kernel::QuantGemmSm100
                    : d.pattern == RF_PATTERN_LAYERNORM_GEMM ? rf::Kernel::LayerNormGemmSm100
                                                             : rf::Kernel::RmsGemmSm100;
        p->rows_total = d.rows;
        p->d.segments = L1;
        break;
      }
      default:
        return bail(RF_ERR_UNSUPPORTED, "run_fused: no non-incremental kernel for this pattern");
    }
  } else
  switch (d.pattern) {
    case RF_PATTERN_SAFE_SOFTMAX:
      if (d.dtype != RF_F32) return bail(RF_ERR_UNSUPPORTED, "safe_softmax: f32 input only");
      p->kernel = rf::Kernel::SoftmaxRows;
      p->rows_total = d.rows;
      if (d.segments != 1) p->nsplit = 1;  // single pass; segment merges are in-CTA
      break;
    case RF_PATTERN_ATTENTION:
      if (d.dtype != RF_F32 && d.dtype != RF_BF16)
        return bail(RF_ERR_UNSUPPORTED, "attention: f32 or bf16 inputs");
      if (d.free_len != 16 && d.free_len != 32 && d.free_len != 64 && d.free_len != 128)
        return bail(RF_ERR_UNSUPPORTED, "attention: head_dim must be 16/32/64/128");
      p->rows_total = d.batch * d.heads * d.rows;
      p->nsplit = d.segments;
      // (tma_rows_fit: the TMA kernels address rows of the flattened
      // [B*H*S, D] views with 32-bit coordinates)
      if (d.dtype == RF_F32 && d.segments <= 8 && d.rows >= 128 && tma_rows_fit(d) &&
          rf::attention_tf32_supports(d.rows, d.len, d.free_len, d.segments) && !std::getenv("RF_ATTN_F32_SIMT")) {
        // tcgen05 (3xTF32): cut the reference slices into up to 8 sub-slices of
        // >= 128 keys (one cluster per 128-row tile) while the grid is below
        // one CTA per SM; the in-kernel fold is the same closed-form sum over
        // the finer slices. RF_ATTN_F32_SIMT=1 keeps the SIMT kernel (A/B only).
        p->kernel = rf::Kernel::AttentionTf32;
        const int64_t tiles = d.batch * d.heads * ((d.rows + 127) / 128);
        while (p->nsplit * 2 <= 8 && tiles * p->nsplit < 148 &&
               rf::attention_tf32_supports(d.rows, d.len, d.free_len, p->nsplit * 2))
          p->nsplit *= 2;
      } else if (d.dtype == RF_F32) {
        p->kernel = rf::Kernel::AttentionF32;
        // A grid too small to fill the GPU (cfg1: 16 row tiles x 8 slices):
        // cut every reference slice into c sub-slices of >= 64 keys, up to
        // two CTAs per SM. The slice-ordered fold's closed form is the same
        // sum over the finer slices (merge.cu); rf_run_partials keeps the
        // reference's slices.
        const int64_t tiles = d.batch * d.heads * ((d.rows + 63) / 64);
        const int64_t slice = d.len / d.segments;
        for (int64_t c = 2; c <= 16 && tiles * p->nsplit < 2 * 148; c *= 2)
          if (slice % c == 0 && slice / c >= 64) p->nsplit = d.segments * c;
      } else if (d.rows == 1) {
        p->kernel = rf::Kernel::AttentionDecode;
        p->nsplit = pick_decode_splits(d.batch * d.heads, d.len, d.segments);
      } else if (tma_rows_fit(d) && rf::attention_sm100_supports(d.rows, d.len, d.free_len, d.segments)) {
        p->kernel = rf::Kernel::AttentionSm100;
      } else {
        p->kernel = rf::Kernel::AttentionF32;  // SIMT CUDA path for odd shapes
      }
      break;
    case RF_PATTERN_QUANT_GEMM_E4M3:
    case RF_PATTERN_RMSNORM_GEMM:
    case RF_PATTERN_LAYERNORM_GEMM:
      if (d.dtype != RF_BF16) return bail(RF_ERR_UNSUPPORTED, "GEMM patterns take bf16 activations");
      // segments > 1 (run_multisegment): S | K was checked above; the kernels
      // stream the S K-slices from fresh state (split-K partials) and
      // gemm_fold.cu merges them in slice order.
      if (!rf::gemm_sm100_supports(d.pattern, d.rows, d.free_len, d.len))
        return bail(RF_ERR_UNSUPPORTED,
                    "GEMM shape has no tcgen05 tiling (quant: M%128, N%512, K%128; rms: M%128, "
                    "N%256, K%64; layernorm: M%256, N%256, K%64)");
      if (d.segments > 1 && (d.len / d.segments) % (d.pattern == RF_PATTERN_QUANT_GEMM_E4M3 ? 128 : 64))
        return bail(RF_ERR_UNSUPPORTED, "multi-segment GEMM: K / segments must be a multiple of the "
                                        "K tile (quant 128, rms / layernorm 64)");
      p->kernel = d.pattern == RF_PATTERN_QUANT_GEMM_E4M3 ? rf::Kernel::QuantGemmSm100
                  : d.pattern == RF_PATTERN_LAYERNORM_GEMM ? rf::Kernel::LayerNormGemmSm100
                                                           : rf::Kernel::RmsGemmSm100;
      p->rows_total = d.rows;
      break;
    case RF_PATTERN_MOE_ROUTING:
      if (d.dtype != RF_F32) return bail(RF_ERR_UNSUPPORTED, "moe_routing: f32 logits");
      if (d.free_len < 1 || d.free_len > 8)
        return bail(RF_ERR_UNSUPPORTED, "moe_routing: top-k size must be 1..8");
      p->kernel = rf::Kernel::MoeRouting;
      p->rows_total = d.rows;
      break;
    case RF_PATTERN_MLA_DECODE:
      if (d.dtype != RF_BF16) return bail(RF_ERR_UNSUPPORTED, "mla_decode: bf16 q / cache");
      if (d.rows != 1) return bail(RF_ERR_SHAPE, "mla_decode: one query per head (rows = 1)");
      if (!rf::mla_supports(d.heads, d.len, d.free_len, d.producer_len, d.segments))
        return bail(RF_ERR_UNSUPPORTED,
                    "mla_decode: heads 128, free_len 512, producer_len 576, (Skv / segments) % 128 == 0");
      p->kernel = rf::Kernel::MlaDecode;
      p->rows_total = d.batch * d.heads;
      p->nsplit = rf::mla_pick_splits(d.batch, d.len, d.segments);
      break;
    case RF_PATTERN_MOE_ROUTER:
      if (d.dtype != RF_BF16) return bail(RF_ERR_UNSUPPORTED, "moe_router: bf16 activations");
      if (!rf::router_supports(d.rows, d.producer_len, d.len, d.free_len))
        return bail(RF_ERR_UNSUPPORTED,
                    "moe_router: experts (len) must be 32/64/128/256, hd (producer_len) % 64, "
                    "1 <= K' (free_len) <= min(8, experts)");
      p->kernel = rf::Kernel::MoeRouter;
      p->rows_total = d.rows;
      p->nsplit = rf::router_pick_splits(d.rows, d.producer_len);
      break;
    case RF_PATTERN_VARIANCE:
    case RF_PATTERN_SUM_SUM:
    case RF_PATTERN_MOMENTS:
      if (d.dtype != RF_F32) return bail(RF_ERR_UNSUPPORTED, "row statistics: f32 inputs");
      if (d.pattern == RF_PATTERN_MOMENTS && (d.free_len < 1 || d.free_len > 8))
        return bail(RF_ERR_UNSUPPORTED, "moments: free_len must be 1..8");
      if (d.pattern == RF_PATTERN_SUM_SUM && !(d.eps > 0.0))
        return bail(RF_ERR_ARG, "sum_sum: eps must be > 0 (max(d1 - c, eps) is the H guard)");
      p->kernel = rf::Kernel::RowStats;
      p->rows_total = d.rows;
      break;
    default:
      return bail(RF_ERR_UNSUPPORTED, "unknown pattern");
  }
  if (is_gemm(p->d.pattern) && p->d.pattern != RF_PATTERN_MOE_ROUTER) p->nsplit = p->d.segments;
  p->launches = ((p->d.pattern == RF_PATTERN_ATTENTION && p->nsplit > 1 &&
                  p->kernel != rf::Kernel::AttentionTf32) ||
                 (is_gemm(p->d.pattern) && p->d.pattern != RF_PATTERN_MOE_ROUTER && p->nsplit > 1)) ? 2 : 1;

  // ---- persistent workspace ----
  if (cudaMalloc(&p->domain_flag, sizeof(int)) != cudaSuccess ||
      cudaMemset(p->domain_flag, 0, sizeof(int)) != cudaSuccess)
    return bail(RF_ERR_CUDA, "workspace allocation failed");
  if ((p->d.pattern == RF_PATTERN_ATTENTION || p->d.pattern == RF_PATTERN_MLA_DECODE) && p->nsplit > 1) {
    const size_t n = static_cast<size_t>(p->nsplit) * p->rows_total;
    if (cudaMalloc(&p->ws_m, n * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&p->ws_l, n * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&p->ws_o, n * p->d.free_len * sizeof(float)) != cudaSuccess)
      return bail(RF_ERR_CUDA, "segment workspace allocation failed");
    if (p->d.pattern == RF_PATTERN_MLA_DECODE) {  // two counters per batch (one per CTA of the pair)
      const size_t nc = static_cast<size_t>(2 * p->d.batch) * sizeof(unsigned long long);
      if (cudaMalloc(&p->ws_cnt, nc) != cudaSuccess || cudaMemset(p->ws_cnt, 0, nc) != cudaSuccess)
        return bail(RF_ERR_CUDA, "segment workspace allocation failed");
    }
  }
  if (is_gemm(p->d.pattern) && p->d.pattern != RF_PATTERN_MOE_ROUTER && p->nsplit > 1) {
    // Multi-Segment GEMM: [S, M, N] f32 slice accumulators + [S, M] statistics
    const size_t sm = static_cast<size_t>(p->nsplit) * p->d.rows;
    if (cudaMalloc(&p->ws_o, sm * p->d.free_len * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&p->ws_m, sm * sizeof(float)) != cudaSuccess ||
        (p->d.pattern == RF_PATTERN_LAYERNORM_GEMM && cudaMalloc(&p->ws_l, sm * sizeof(float)) != cudaSuccess))
      return bail(RF_ERR_CUDA, "multi-segment GEMM workspace allocation failed");
  }
  if (p->d.pattern == RF_PATTERN_MOE_ROUTER) {  // split-K partial scores (L2-resident)
    // + one arrival counter per 128-token row tile (the split CTAs of a tile meet on it)
    const size_t n = static_cast<size_t>(p->nsplit) * p->d.rows * p->d.len;
    const size_t nc = static_cast<size_t>((p->d.rows + 127) / 128 + 1) * sizeof(unsigned long long);
    if ((n && cudaMalloc(&p->ws_m, n * sizeof(float)) != cudaSuccess) || cudaMalloc(&p->ws_l, nc) != cudaSuccess ||
        cudaMemset(p->ws_l, 0, nc) != cudaSuccess)
      return bail(RF_ERR_CUDA, "router workspace allocation failed");
  }
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "{\"kernel\": \"%s\", \"pattern\": %d, \"dtype\": %d, \"rows_total\": %lld, "
                "\"L0\": %lld, \"free\": %lld, \"segments\": %lld, \"slices_launched\": %lld, "
                "\"launches_per_run\": %lld, \"fuse_level\": %d, \"device\": \"%s\"}",
                kernel_name(p->kernel), d.pattern, d.dtype, (long long)p->rows_total,
                (long long)d.len, (long long)d.free_len, (long long)p->d.segments,
                (long long)p->nsplit, (long long)p->launches, d.fuse_level, prop.name);
  p->describe = buf;
  *out = p;
  return RF_OK;
}

void rf_plan_destroy(rf_plan* p) {
  if (!p) return;
  cudaFree(p->ws_m);
  cudaFree(p->ws_l);
  cudaFree(p->ws_o);
  cudaFree(p->ws_cnt);
  cudaFree(p->domain_flag);
  for (void* b : p->dev_in) cudaFree(b);
  for (void* b : p->dev_out) cudaFree(b);
  for (cudaStream_t s : p->streams)
    if (s) cudaStreamDestroy(s);
  for (int c = 0; c < rf_plan::kChunks; ++c) {
    if (p->ev_in[c]) cudaEventDestroy(p->ev_in[c]);
    if (p->ev_done[c]) cudaEventDestroy(p->ev_done[c]);
  }
  delete p;
}

rf_status rf_plan_describe(const rf_plan* p, char* buf, size_t n) {
  if (!p || !buf || n == 0) return fail(RF_ERR_ARG, "null plan/buffer");
  std::snprintf(buf, n, "%s", p->describe.c_str());
  return p->describe.size() < n ? RF_OK : fail(RF_ERR_ARG, "buffer too small");
}

int64_t rf_plan_launches_per_run(const rf_plan* p) { return p ? p->launches : 0; }

rf_status rf_plan_io_bytes(const rf_plan* p, size_t in_bytes[4], size_t out_bytes[4]) {
  if (!p || !in_bytes || !out_bytes) return fail(RF_ERR_ARG, "null plan/arrays");
  io_sizes(p, in_bytes, out_bytes);
  if (is_gemm(p->d.pattern)) in_bytes[1] = rf_packed_bytes(p);
  return RF_OK;
}

rf_status rf_pack_weight(const rf_plan* p, const void* w, const void* g, void* packed,
                         void* stream) {
  if (!p || !w || !packed) return fail(RF_ERR_ARG, "null plan/w/packed");
  DeviceGuard guard(p->d.device);
  cudaError_t e;
  if (p->d.pattern == RF_PATTERN_QUANT_GEMM_E4M3) {
    e = rf::launch_pack_e4m3(static_cast<const float*>(w), p->d.len, p->d.free_len,
                             static_cast<uint8_t*>(packed), as_stream(stream));
  } else if (p->d.pattern == RF_PATTERN_RMSNORM_GEMM || p->d.pattern == RF_PATTERN_LAYERNORM_GEMM) {
    if (!g) return fail(RF_ERR_ARG, "rmsnorm/layernorm pack needs g");
    e = rf::launch_pack_rms(static_cast<const float*>(w), static_cast<const float*>(g), p->d.len,
                            p->d.free_len, packed, as_stream(stream));
    if (e == cudaSuccess && p->d.pattern == RF_PATTERN_LAYERNORM_GEMM)
      e = rf::launch_colsum(packed, p->d.len, p->d.free_len,
                            reinterpret_cast<float*>(static_cast<char*>(packed) +
                                                     2 * p->d.free_len * p->d.len),
                            as_stream(stream));
  } else if (p->d.pattern == RF_PATTERN_MOE_ROUTER) {
    e = rf::launch_pack_rms(static_cast<const float*>(w), nullptr, p->d.producer_len, p->d.len, packed,
                            as_stream(stream));
  } else {
    return fail(RF_ERR_UNSUPPORTED, "pattern has no packed weight");
  }
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("pack: ") + cudaGetErrorString(e));
  return RF_OK;
}

size_t rf_packed_bytes(const rf_plan* p) {
  if (!p) return 0;
  const size_t nk = static_cast<size_t>(p->d.len) * p->d.free_len;
  switch (p->d.pattern) {
    case RF_PATTERN_QUANT_GEMM_E4M3: return nk;
    case RF_PATTERN_RMSNORM_GEMM: return 2 * nk;
    case RF_PATTERN_LAYERNORM_GEMM: return 2 * nk + 4 * static_cast<size_t>(p->d.free_len);
    case RF_PATTERN_MOE_ROUTER: return 2 * static_cast<size_t>(p->d.producer_len) * p->d.len;
    default: return 0;
  }
}

rf_status rf_pack_weight_host(const rf_plan* p, const float* w, const float* g, void** packed) {
  if (!p || !w || !packed) return fail(RF_ERR_ARG, "null plan/w/packed");
  *packed = nullptr;
  const bool needs_g = p->d.pattern == RF_PATTERN_RMSNORM_GEMM || p->d.pattern == RF_PATTERN_LAYERNORM_GEMM;
  if (rf_packed_bytes(p) == 0) return fail(RF_ERR_UNSUPPORTED, "pattern has no packed weight");
  if (needs_g && !g) return fail(RF_ERR_ARG, "rmsnorm/layernorm pack needs g");
  int64_t wk = 0, wn = 0;
  pack_dims(p->d, wk, wn);
  DeviceGuard guard(p->d.device);
  const size_t kn = static_cast<size_t>(wk) * wn;
  float *dw = nullptr, *dg = nullptr;
  void* out = nullptr;
  RF_CUDA_TRY(cudaMalloc(&dw, kn * sizeof(float)));
  RF_CUDA_TRY(cudaMalloc(&out, rf_packed_bytes(p)));
  RF_CUDA_TRY(cudaMemcpy(dw, w, kn * sizeof(float), cudaMemcpyHostToDevice));
  if (g && needs_g) {
    RF_CUDA_TRY(cudaMalloc(&dg, wk * sizeof(float)));
    RF_CUDA_TRY(cudaMemcpy(dg, g, wk * sizeof(float), cudaMemcpyHostToDevice));
  }
  rf_status st = rf_pack_weight(p, dw, dg, out, nullptr);
  RF_CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(dw);
  cudaFree(dg);
  if (st != RF_OK) {
    cudaFree(out);
    return st;
  }
  *packed = out;
  return RF_OK;
}

void rf_buffer_free(void* dev_ptr) { cudaFree(dev_ptr); }

rf_status rf_run(const rf_plan* p, const rf_io* io, void* stream) {
  if (!p || !io) return fail(RF_ERR_ARG, "null plan/io");
  size_t in[4], out[4];
  io_sizes(p, in, out);
  for (int i = 0; i < 4; ++i)
    if (in[i] && !io->in[i]) return fail(RF_ERR_SHAPE, "missing input " + std::to_string(i));
  for (int i = 0; i < 3; ++i)  // d4 (layernorm; router scores) is optional
    if (out[i] && !io->d[i]) return fail(RF_ERR_SHAPE, "missing output d" + std::to_string(i + 1));
  if (is_gemm(p->d.pattern) && !io->in[1])
    return fail(RF_ERR_SHAPE, "missing packed weight in[1]");
  if (units_of(p) == 0 || p->d.rows == 0) return RF_OK;  // empty batch
  DeviceGuard guard(p->d.device);
  return run_range(p, io, 0, units_of(p), as_stream(stream));
}

rf_status rf_run_host(rf_plan* p, const rf_host_io* io) {
  if (!p || !io) return fail(RF_ERR_ARG, "null plan/io");
  size_t in[4], out[4];
  io_sizes(p, in, out);
  const bool gemm = is_gemm(p->d.pattern);
  DeviceGuard guard(p->d.device);
  if (!p->staged) {
    for (int i = 0; i < 4; ++i)
      if (in[i]) RF_CUDA_TRY(cudaMalloc(&p->dev_in[i], in[i]));
    for (int i = 0; i < 4; ++i)
      if (out[i]) RF_CUDA_TRY(cudaMalloc(&p->dev_out[i], out[i]));
    for (auto& s : p->streams) RF_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (int c = 0; c < rf_plan::kChunks; ++c) {
      RF_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_in[c], cudaEventDisableTiming));
      RF_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_done[c], cudaEventDisableTiming));
    }
    p->staged = true;
  }
  auto drain = [&](rf_status s) {
    for (cudaStream_t st : p->streams) cudaStreamSynchronize(st);
    return s;
  };
  for (int i = 0; i < 4; ++i)
    if (in[i] && !(gemm && i == 1) && !io->in[i]) return fail(RF_ERR_SHAPE, "missing input " + std::to_string(i));
  for (int i = 0; i < 3; ++i)
    if (out[i] && !io->d[i]) return fail(RF_ERR_SHAPE, "missing output d" + std::to_string(i + 1));
  if (gemm && !io->in[1]) return fail(RF_ERR_SHAPE, "missing packed weight in[1]");
  rf_io dio{};
  for (int i = 0; i < 4; ++i) dio.in[i] = p->dev_in[i];
  for (int i = 0; i < 4; ++i) dio.d[i] = io->d[i] ? p->dev_out[i] : nullptr;
  if (gemm) dio.in[1] = io->in[1];  // packed weight: plan-time resident device buffer
  const int64_t units = units_of(p);
  if (units == 0 || p->d.rows == 0) return RF_OK;  // empty batch
  // Chunking: up to 16 chunks over independent units. The H2D copies run back
  // to back on their own stream (the link's host-to-device direction never
  // waits on a download), each chunk's kernels on the compute stream once its
  // inputs landed (event), and its D2H on a third stream once they finished
  // (event): PCIe both ways and the kernels overlap. GEMM chunks are whole
  // 128-row tiles.
  const int64_t gran = p->d.pattern == RF_PATTERN_LAYERNORM_GEMM ? 256 : gemm ? 128 : 1;
  const int64_t nchunk = std::max<int64_t>(1, std::min<int64_t>(rf_plan::kChunks, units / gran));
  const int64_t per = ((units + nchunk - 1) / nchunk + gran - 1) / gran * gran;
  cudaStream_t s_in = p->streams[0], s_run = p->streams[1], s_out = p->streams[2];
  for (int64_t c = 0; c < nchunk; ++c) {
    const int64_t u0 = c * per, nu = std::min(per, units - u0);
    if (nu <= 0) break;
    cudaStream_t st = s_in;
    for (int i = 0; i < 4; ++i) {
      if (!in[i] || (gemm && i == 1)) continue;
      const size_t chunk = in[i] / units * nu, off = in[i] / units * u0;
      const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(p->dev_in[i]) + off,
                                            static_cast<const char*>(io->in[i]) + off, chunk,
                                            cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return drain(fail(RF_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e)));
    }
    RF_CUDA_TRY(cudaEventRecord(p->ev_in[c], s_in));
    RF_CUDA_TRY(cudaStreamWaitEvent(s_run, p->ev_in[c], 0));
    rf_status s = run_range(p, &dio, u0, nu, s_run);
    // an early return must not leave copies into the caller's host buffers in flight
    if (s != RF_OK) return drain(s);
    RF_CUDA_TRY(cudaEventRecord(p->ev_done[c], s_run));
    RF_CUDA_TRY(cudaStreamWaitEvent(s_out, p->ev_done[c], 0));
    for (int i = 0; i < 4; ++i) {
      if (!out[i] || !io->d[i]) continue;
      const size_t chunk = out[i] / units * nu, off = out[i] / units * u0;
      const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(io->d[i]) + off,
                                            static_cast<char*>(p->dev_out[i]) + off, chunk,
                                            cudaMemcpyDeviceToHost, s_out);
      if (e != cudaSuccess) return drain(fail(RF_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e)));
    }
  }
  for (cudaStream_t st : p->streams) RF_CUDA_TRY(cudaStreamSynchronize(st));
  return RF_OK;
}

rf_status rf_run_partials(const rf_plan* p, const rf_io* io, int64_t slice_begin,
                          rf_partials* outp, void* stream) {
  if (!p || !io || !outp) return fail(RF_ERR_ARG, "null argument");
  if (p->d.pattern != RF_PATTERN_ATTENTION) return fail(RF_ERR_UNSUPPORTED, "partials: attention only");
  if (slice_begin < 0 || outp->nslices < 1 || slice_begin + outp->nslices > p->d.segments)
    return fail(RF_ERR_SEGMENTATION, "slice range outside the plan's segments");
  const rf_desc& d = p->d;
  DeviceGuard guard(d.device);
  rf::AttnArgs a{};
  a.q = io->in[0];
  a.k = io->in[1];
  a.v = io->in[2];
  a.bh = d.batch * d.heads;
  a.sq = d.rows;
  a.skv = d.len;
  a.d = d.free_len;
  a.segments = d.segments;
  a.slice_begin = slice_begin;
  a.nslices = outp->nslices;
  a.part_base = slice_begin;
  a.rows_total = p->rows_total;
  a.part_m = outp->m;
  a.part_l = outp->l;
  a.part_o = outp->o;
  a.scale = static_cast<float>(d.softmax_scale);
  a.dtype = d.dtype;
  cudaError_t e;
  switch (p->kernel) {
    case rf::Kernel::AttentionSm100: e = rf::launch_attention_sm100(a, as_stream(stream)); break;
    case rf::Kernel::AttentionDecode: e = rf::launch_attention_decode(a, as_stream(stream)); break;
    default: e = rf::launch_attention_f32(a, as_stream(stream)); break;
  }
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("partials: ") + cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_merge_partials(const rf_plan* p, const rf_partials* in, const rf_io* io,
                            void* stream) {
  if (!p || !in || !io) return fail(RF_ERR_ARG, "null argument");
  if (p->d.pattern != RF_PATTERN_ATTENTION) return fail(RF_ERR_UNSUPPORTED, "merge: attention only");
  if (in->nslices < 1) return fail(RF_ERR_SEGMENTATION, "merge: no slices");
  if (!in->m || !in->l || !in->o || !io->d[0] || !io->d[1] || !io->d[2])
    return fail(RF_ERR_SHAPE, "merge: missing partial or output buffer");
  DeviceGuard guard(p->d.device);
  cudaError_t e = rf::launch_attention_merge(in->m, in->l, in->o, in->nslices, p->rows_total,
                                             p->rows_total, p->d.free_len,
                                             static_cast<float*>(io->d[0]),
                                             static_cast<float*>(io->d[1]), io->d[2], p->d.dtype,
                                             as_stream(stream));
  if (e != cudaSuccess) return fail(RF_ERR_CUDA, std::string("merge: ") + cudaGetErrorString(e));
  return RF_OK;
}

rf_status rf_check_domain(const rf_plan* p, void* stream) {
  if (!p) return fail(RF_ERR_ARG, "null plan");
  DeviceGuard guard(p->d.device);
  int flag = 0;
  RF_CUDA_TRY(cudaStreamSynchronize(as_stream(stream)));
  RF_CUDA_TRY(cudaMemcpy(&flag, p->domain_flag, sizeof(int), cudaMemcpyDeviceToHost));
  RF_CUDA_TRY(cudaMemset(p->domain_flag, 0, sizeof(int)));
  if (flag) return fail(RF_ERR_DOMAIN, "division by zero at finalize (a row's absmax is 0)");
  return RF_OK;
}

}  // extern "C"
