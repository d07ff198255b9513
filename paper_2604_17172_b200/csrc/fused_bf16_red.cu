// fused_bf16_red.cu -- instantiates the fused kernels for bf16, reduce variant.
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_fused_bf16_red(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kBF16, true>(p, B, st, max_ctas);
}
cudaError_t preload_bf16_red() { return preload_t<kBF16, true>(); }
}  // namespace uzip
