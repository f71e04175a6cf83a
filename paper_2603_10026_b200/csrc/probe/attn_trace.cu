// TEST-ONLY: the attention kernel compiled with RF_ATTN_TRACE, plus a reader
// for its clock64 timeline (tools/trace_attention.py). Built into librf_probe.so.
#include "../attn_sm100.cu"

extern "C" int rf_probe_attn_trace(const void* q, const void* k, const void* v, void* o, float* m,
                                   float* l, long long bh, long long s, long long* out) {
  rf::AttnArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o; a.m = m; a.l = l;
  a.bh = bh; a.sq = s; a.skv = s; a.d = 128;
  a.segments = 1; a.slice_begin = 0; a.nslices = 1; a.part_base = 0; a.rows_total = bh * s;
  a.scale = 1.f; a.dtype = RF_BF16;
  long long zero[4096] = {0};
  cudaMemcpyToSymbol(g_attn_trace, zero, sizeof zero);
  if (rf::launch_attention_sm100(a, 0) != cudaSuccess) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpyFromSymbol(out, g_attn_trace, sizeof(long long) * 4096);
  return 0;
}


// Effective SM clock of CTA 0 over n back-to-back launches (cfg2 shape):
// out[i] = MHz of launch i (clock64 delta / globaltimer delta).
extern "C" int rf_probe_attn_clock(const void* q, const void* k, const void* v, void* o, float* m, float* l,
                                   long long bh, long long s, int n, double* out) {
  rf::AttnArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o; a.m = m; a.l = l;
  a.bh = bh; a.sq = s; a.skv = s; a.d = 128;
  a.segments = 1; a.slice_begin = 0; a.nslices = 1; a.part_base = 0; a.rows_total = bh * s;
  a.scale = 1.f; a.dtype = RF_BF16;
  int zero = 0;
  cudaMemcpyToSymbol(g_attn_launch, &zero, sizeof zero);
  for (int i = 0; i < n; ++i)
    if (rf::launch_attention_sm100(a, 0) != cudaSuccess) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  long long c[64][4];
  cudaMemcpyFromSymbol(c, g_attn_clk, sizeof c);
  for (int i = 0; i < n && i < 64; ++i)
    out[i] = static_cast<double>(c[i][2] - c[i][0]) / static_cast<double>(c[i][3] - c[i][1]) * 1e3;
  return 0;
}
