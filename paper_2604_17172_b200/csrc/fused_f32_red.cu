// fused_f32_red.cu -- instantiates the fused kernels for f32, reduce variant.
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_fused_f32_red(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kF32, true>(p, B, st, max_ctas);
}
cudaError_t preload_f32_red() { return preload_t<kF32, true>(); }
}  // namespace uzip
