// fused_f32_enc.cu -- instantiates the fused kernels for f32, encode/decode variant.
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_tables_f32(const Plan &p, cudaStream_t st) { return launch_tables_t<kF32>(p, st); }
cudaError_t launch_fused_f32_enc(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kF32, false>(p, B, st, max_ctas);
}
cudaError_t preload_f32_enc() { return preload_t<kF32, false>(); }
}  // namespace uzip
