// fused_e5m2_enc.cu -- instantiates the fused kernels for e5m2, encode/decode variant (no reductions, R22).
#include "fused_impl.cuh"

namespace uzip {
cudaError_t launch_tables_e5m2(const Plan &p, cudaStream_t st) { return launch_tables_t<kE5M2>(p, st); }
cudaError_t launch_fused_e5m2_enc(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  return launch_fused_b<kE5M2, false>(p, B, st, max_ctas);
}
cudaError_t preload_e5m2_enc() { return preload_t<kE5M2, false>(); }
}  // namespace uzip
