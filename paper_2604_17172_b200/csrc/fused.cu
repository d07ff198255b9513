// fused.cu -- dtype/variant dispatch of the fused kernels (instantiated in
// fused_<dtype>_<enc|red>.cu, see fused_impl.cuh for the kernels themselves).
#include "plan.h"
#include "uzip_internal.h"

namespace uzip {

cudaError_t launch_tables_bf16(const Plan &, cudaStream_t);
cudaError_t launch_tables_f16(const Plan &, cudaStream_t);
cudaError_t launch_tables_f32(const Plan &, cudaStream_t);
cudaError_t launch_tables_e4m3(const Plan &, cudaStream_t);
cudaError_t launch_tables_e5m2(const Plan &, cudaStream_t);
#define UZIP_DECL(n) cudaError_t launch_fused_##n(const Plan &, uint32_t, cudaStream_t, int);
UZIP_DECL(bf16_enc) UZIP_DECL(bf16_red) UZIP_DECL(f16_enc) UZIP_DECL(f16_red) UZIP_DECL(f32_enc) UZIP_DECL(f32_red)
UZIP_DECL(e4m3_enc) UZIP_DECL(e5m2_enc)
#undef UZIP_DECL
cudaError_t preload_bf16_enc();
cudaError_t preload_bf16_red();
cudaError_t preload_f16_enc();
cudaError_t preload_f16_red();
cudaError_t preload_f32_enc();
cudaError_t preload_f32_red();
cudaError_t preload_e4m3_enc();
cudaError_t preload_e5m2_enc();

// Wait (one thread) until every slot credit of the next fused launch has
// arrived; on timeout record the error (site 4) -- the fused kernel then aborts
// its encode / forward items instead of overwriting a slot still in use.
__global__ void k_credit(const CreditWait w) {
  if (threadIdx.x != 0) return;
  unsigned long long t0 = 0;
  for (uint32_t i = 0; i < w.n; ++i) {
    for (int spin = 0;; ++spin) {
      const unsigned long long v = ld_acquire_sys_u64(w.cr[i]);
      if (v >= (unsigned long long)(w.epoch[i] - 2)) break;
      if ((spin & 63) == 63) {
        if (ld_volatile_u32(w.err)) return;
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > w.timeout_ns) {
          if (atomicCAS(w.err, 0u, (uint32_t)UZIP_ERR_TIMEOUT) == 0u) {
            w.err[1] = 4;
            w.err[2] = w.epoch[i];
            w.err[3] = (uint32_t)(v >> 32);
            w.err[4] = (uint32_t)v;
            w.err[5] = (uint32_t)(uintptr_t)w.cr[i];
            w.err[6] = 0;
            __threadfence_system();
          }
          return;
        }
      }
      __nanosleep(64);
    }
  }
}

cudaError_t launch_credit_wait(const CreditWait &w, cudaStream_t st) {
  k_credit<<<1, 32, 0, st>>>(w);
  return cudaGetLastError();
}

cudaError_t preload_kernels() {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, k_credit) != cudaSuccess) return cudaGetLastError();
  cudaError_t (*fns[])() = {preload_bf16_enc, preload_bf16_red, preload_f16_enc, preload_f16_red,
                            preload_f32_enc,  preload_f32_red,  preload_e4m3_enc, preload_e5m2_enc};
  for (auto f : fns) {
    const cudaError_t e = f();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tables(int dtype, const Plan &p, cudaStream_t st) {
  if (p.ne == 0) return cudaSuccess;
  switch (dtype) {
    case kBF16: return launch_tables_bf16(p, st);
    case kF16: return launch_tables_f16(p, st);
    case kE4M3: return launch_tables_e4m3(p, st);
    case kE5M2: return launch_tables_e5m2(p, st);
    default: return launch_tables_f32(p, st);
  }
}

cudaError_t launch_fused(int dtype, const Plan &p, cudaStream_t st, int max_ctas) {
  uint32_t B = 4096;
  bool red = false;
  for (int j = 0; j < p.ne; ++j)
    if (!p.e[j].raw) B = p.e[j].g.B;
  for (int j = 0; j < p.nd_jobs; ++j) {
    if (!p.d[j].raw) B = p.d[j].g.B;
    red |= p.d[j].nsrc > 1;
  }
  switch (dtype) {
    case kBF16: return red ? launch_fused_bf16_red(p, B, st, max_ctas) : launch_fused_bf16_enc(p, B, st, max_ctas);
    case kF16: return red ? launch_fused_f16_red(p, B, st, max_ctas) : launch_fused_f16_enc(p, B, st, max_ctas);
    case kE4M3: return red ? cudaErrorNotSupported : launch_fused_e4m3_enc(p, B, st, max_ctas);
    case kE5M2: return red ? cudaErrorNotSupported : launch_fused_e5m2_enc(p, B, st, max_ctas);
    default: return red ? launch_fused_f32_red(p, B, st, max_ctas) : launch_fused_f32_enc(p, B, st, max_ctas);
  }
}

}  // namespace uzip
