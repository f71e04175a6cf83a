// TEST-ONLY: the FP8 quant GEMM compiled with RF_QNT_TRACE, plus a reader for
// its clock64 timeline (tools/trace_quant.py). Built into librf_qtrace.so.
#include "../gemm_sm100.cu"
#include "../gemm_fold.cu"

extern "C" int rf_probe_qnt_trace(const void* a, const void* w, float* d1, float* c, int* flag,
                                  long long m, long long n, long long k, int cta, long long* out) {
  rf::GemmArgs g{};
  g.a = a; g.b = w; g.d1 = d1; g.c = c; g.domain_flag = flag;
  g.m = m; g.n = n; g.k = k; g.stat_len = k; g.fmax = 448.f; g.segments = 1; g.ws_rows = m;
  static long long zero[2 * 4096] = {0};
  cudaMemcpyToSymbol(rf::g_qnt_trace, zero, sizeof zero);
  cudaMemcpyToSymbol(rf::g_qnt_trace_cta, &cta, sizeof cta);
  if (rf::launch_quant_gemm_sm100(g, 0) != cudaSuccess) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpyFromSymbol(out, rf::g_qnt_trace, sizeof(long long) * 2 * 4096);
  return 0;
}
