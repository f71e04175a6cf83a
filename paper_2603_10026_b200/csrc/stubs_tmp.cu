#include "rf_internal.h"
namespace rf {
cudaError_t launch_attention_decode(const AttnArgs& a, cudaStream_t st) { return launch_attention_f32(a, st); }
cudaError_t launch_attention_sm100(const AttnArgs&, cudaStream_t) { return cudaErrorNotSupported; }
bool attention_sm100_supports(int64_t, int64_t, int64_t, int64_t) { return false; }
cudaError_t launch_quant_gemm_sm100(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_rms_gemm_sm100(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
bool gemm_sm100_supports(int, int64_t, int64_t, int64_t) { return false; }
cudaError_t launch_pack_e4m3(const float*, int64_t, int64_t, uint8_t*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_pack_rms(const float*, const float*, int64_t, int64_t, void*, cudaStream_t) { return cudaErrorNotSupported; }
}
