#include "rf_internal.h"
namespace rf {
cudaError_t launch_quant_gemm_sm100(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_rms_gemm_sm100(const GemmArgs&, cudaStream_t) { return cudaErrorNotSupported; }
bool gemm_sm100_supports(int, int64_t, int64_t, int64_t) { return false; }
cudaError_t launch_pack_e4m3(const float*, int64_t, int64_t, uint8_t*, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_pack_rms(const float*, const float*, int64_t, int64_t, void*, cudaStream_t) { return cudaErrorNotSupported; }
}
