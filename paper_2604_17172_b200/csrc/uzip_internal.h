// uzip_internal.h -- declarations shared by the CUDA translation units of libuzip.
#pragma once
#include <cuda_runtime.h>

#include "../../include/uzip.h"
#include "uzip_device.cuh"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges are free unless a profiler is attached

namespace uzip {

// NVTX range around one C-ABI call (host side: the enqueue, visible in nsys / ncu timelines).
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

cudaError_t launch_decompress(int dtype, const void *in, uint64_t in_bytes, void *out, uint64_t n, void *ws,
                              int32_t *d_status, cudaStream_t st, int max_ctas);

// Resolve codec params (defaults of DESIGN.md section 2) into a geometry; returns
// UZIP_OK or UZIP_ERR_INVALID_ARG for unsupported values.
uzip_status_t resolve_geom(int dtype, uint64_t n, const uzip_codec_params_t *p, StreamGeom *g);

// Whether a launch whose largest encode stream has n_chunks table chunks builds its tables with
// the k_hist + k_norm launches (true) or with T items inside k_fused (false): the codec call always
// uses T items, communication launches from kTableKernelChunks chunks on use the launches;
// UZIP_TABLE_KERNELS overrides (A/B of the single-kernel table build).
constexpr uint64_t kTableKernelChunks = 16;  // >= 128 MiB of 2-byte input per stream
bool table_kernels(uint64_t n_chunks, bool codec);

}  // namespace uzip
