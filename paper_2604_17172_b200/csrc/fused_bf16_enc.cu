// fused_bf16_enc.cu -- instantiates the fused kernels for bf16, encode/decode variant.
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_tables_bf16(const Plan &p, cudaStream_t st) { return launch_tables_t<kBF16>(p, st); }
cudaError_t launch_fused_bf16_enc(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kBF16, false>(p, B, st, max_ctas);
}
cudaError_t preload_bf16_enc() { return preload_t<kBF16, false>(); }
}  // namespace uzip
