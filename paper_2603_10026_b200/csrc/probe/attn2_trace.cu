// TEST-ONLY: timeline reader for the traced 2-SM attention kernel.
#include "../experimental/attn_sm100_2sm.cu"

extern "C" int rf_probe_attn2_trace(const void* q, const void* k, const void* v, void* o, float* m,
                                    float* l, long long bh, long long s, long long* out) {
  rf::AttnArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o; a.m = m; a.l = l;
  a.bh = bh; a.sq = s; a.skv = s; a.d = 128;
  a.segments = 1; a.slice_begin = 0; a.nslices = 1; a.part_base = 0; a.rows_total = bh * s;
  a.scale = 1.f; a.dtype = RF_BF16;
  long long zero[4096] = {0};
  cudaMemcpyToSymbol(g_attn2_trace, zero, sizeof zero);
  if (rf::launch_attention_sm100_2sm(a, 0) != cudaSuccess) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpyFromSymbol(out, g_attn2_trace, sizeof(long long) * 4096);
  return 0;
}
