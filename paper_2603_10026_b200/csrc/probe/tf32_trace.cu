// TEST-ONLY: the fp32 tcgen05 attention kernel compiled with RF_TF32_TRACE
// plus a reader for its per-CTA globaltimer events (tools/trace_tf32.py).
#include "../attn_tf32.cu"

extern "C" int rf_probe_tf32_trace(const void* q, const void* k, const void* v, float* o, float* m, float* l,
                                   float* pm, float* pl, float* po, long long sq, long long skv, int nslices,
                                   float scale, unsigned long long* out) {
  rf::AttnArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o; a.m = m; a.l = l;
  a.part_m = pm; a.part_l = pl; a.part_o = po;
  a.bh = 1; a.sq = sq; a.skv = skv; a.d = 64; a.segments = nslices; a.nslices = nslices;
  a.rows_total = sq; a.scale = scale; a.dtype = RF_F32;
  static unsigned long long zero[512][16] = {};
  cudaMemcpyToSymbol(rf::g_tf32_trace, zero, sizeof zero);
  if (rf::launch_attention_tf32(a, 0) != cudaSuccess) return 1;
  if (cudaDeviceSynchronize() != cudaSuccess) return 2;
  cudaMemcpyFromSymbol(out, rf::g_tf32_trace, sizeof zero);
  return 0;
}
