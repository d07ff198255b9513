// fused_e4m3_enc.cu -- instantiates the fused kernels for e4m3, encode/decode variant (no reductions, R22).
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_tables_e4m3(const Plan &p, cudaStream_t st) { return launch_tables_t<kE4M3>(p, st); }
cudaError_t launch_fused_e4m3_enc(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kE4M3, false>(p, B, st, max_ctas);
}
cudaError_t preload_e4m3_enc() { return preload_t<kE4M3, false>(); }
}  // namespace uzip
