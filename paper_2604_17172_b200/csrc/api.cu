// api.cu -- the C ABI of include/uzip.h: host-side argument checks and dispatch.
// No compute happens here; every data call enqueues kernels on the caller's stream.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "plan.h"
#include "uzip_internal.h"

using namespace uzip;

namespace uzip {

bool table_kernels(uint64_t n_chunks, bool codec) {
  // UZIP_TABLE_KERNELS=1 / 0 forces the two table launches / the T items.  By default the codec call
  // (uzip_compress) always builds its tables with T items inside its one k_fused launch (C1 4 MiB
  // compress: 25 vs 33 us; 1 GiB: 0.661 vs 0.666 ms), and communication launches do so for small
  // streams (< kTableKernelChunks chunks) only: large ones launch k_hist + k_norm ahead, which overlap
  // the slot-credit wait and spare every E item the table-flag poll (loopback 1 GiB P2P: 2.15 vs 2.37 ms).
  static const int v = getenv("UZIP_TABLE_KERNELS") ? atoi(getenv("UZIP_TABLE_KERNELS")) : -1;
  if (v >= 0) return v != 0;
  return !codec && n_chunks >= kTableKernelChunks;
}

uzip_status_t resolve_geom(int dtype, uint64_t n, const uzip_codec_params_t *p, StreamGeom *g) {
  if (dtype < 0 || dtype >= kNumDtypes) return UZIP_ERR_UNSUPPORTED_DTYPE;
  const uint32_t eb = group_bytes(dtype);  // input bytes per symbol
  uint32_t B = (p && p->block_symbols) ? p->block_symbols : 4096u;
  if (!gpu_block_ok(B)) return UZIP_ERR_INVALID_ARG;
  const bool global = p && p->global_table;
  uint32_t CB = (p && p->chunk_blocks) ? p->chunk_blocks : (uint32_t)((8u << 20) / (B * eb));
  if (CB == 0 || (!global && CB % kTileBlocks != 0)) return UZIP_ERR_INVALID_ARG;
  uint32_t S = (p && p->sample_symbols) ? p->sample_symbols : (uint32_t)((256u << 10) / eb);
  g->init(dtype, n, B, CB, S, global);
  return UZIP_OK;
}

}  // namespace uzip

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

extern "C" {

const char *uzip_status_string(uzip_status_t s) {
  switch (s) {
    case UZIP_OK: return "ok";
    case UZIP_ERR_INVALID_ARG: return "invalid argument";
    case UZIP_ERR_UNSUPPORTED_DTYPE: return "unsupported dtype";
    case UZIP_ERR_CAPACITY: return "output or workspace capacity too small";
    case UZIP_ERR_CORRUPT_STREAM: return "corrupt stream";
    case UZIP_ERR_SIZE_MISMATCH: return "stream size or dtype mismatch";
    case UZIP_ERR_CUDA: return "CUDA error";
    case UZIP_ERR_COMM: return "communicator error";
    case UZIP_ERR_TIMEOUT: return "peer flag timeout";
    case UZIP_ERR_NOT_IMPLEMENTED: return "not implemented";
  }
  return "unknown status";
}

const char *uzip_version(void) { return "uzip-b200 0.1 sm_100a"; }

size_t uzip_compress_bound(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params) {
  StreamGeom g;
  if (resolve_geom((int)dtype, count, params, &g) != UZIP_OK) return 0;
  return (size_t)g.total(g.n_blocks * (uint64_t)g.B);
}

size_t uzip_workspace_bytes(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params) {
  StreamGeom g;
  if (resolve_geom((int)dtype, count, params, &g) != UZIP_OK) return 0;
  return (size_t)(64 + EncWs::bytes(g.n_chunks, g.n_blocks, g.global));
}

uzip_status_t uzip_workspace_init(void *ws, size_t ws_bytes, void *stream) {
  if (!ws || ws_bytes < 64) return UZIP_ERR_INVALID_ARG;
  return cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream) == cudaSuccess ? UZIP_OK : UZIP_ERR_CUDA;
}

uzip_status_t uzip_compress(const void *in, size_t count, uzip_dtype_t dtype, void *out, size_t out_capacity,
                            uint64_t *d_out_bytes, void *ws, size_t ws_bytes, const uzip_codec_params_t *params,
                            void *stream) {
  NvtxRange nvtx_range("uzip_compress");
  StreamGeom g;
  uzip_status_t st = resolve_geom((int)dtype, count, params, &g);
  if (st != UZIP_OK) return st;
  if (!out || !ws || !aligned16(out) || !aligned16(ws)) return UZIP_ERR_INVALID_ARG;
  if (count > 0 && (!in || !aligned16(in))) return UZIP_ERR_INVALID_ARG;
  if (out_capacity < g.total(g.n_blocks * (uint64_t)g.B)) return UZIP_ERR_CAPACITY;
  if (ws_bytes < 64 + EncWs::bytes(g.n_chunks, g.n_blocks, g.global)) return UZIP_ERR_CAPACITY;
  // one encode job, one destination (the caller's stream buffer), no flags
  Plan p;
  memset(&p, 0, sizeof p);
  p.ag_job = -1;
  p.dtype = (int)dtype;
  uint8_t *w = static_cast<uint8_t *>(ws);
  p.ticket = reinterpret_cast<uint32_t *>(w + 16);
  p.err = reinterpret_cast<uint32_t *>(w + 24);
  p.timeout_ns = 10000000000ull;
  p.codec_call = 1;
  EncJob &J = p.e[0];
  J.in = static_cast<const uint8_t *>(in);
  J.g = g;
  J.ntiles = tiles_of(g);
  J.nd = 1;
  J.dst[0] = static_cast<uint8_t *>(out);
  J.d_out_bytes = d_out_bytes;
  EncWs::carve(w + 64, g.n_chunks, g.n_blocks, g.global, J);
  p.ne = 1;
  p.n_e_items = J.ntiles;
  p.epoch = reinterpret_cast<uint32_t *>(w + 28);
  cudaStream_t cs = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (table_kernels(J.g.n_chunks, true)) {  // forced by UZIP_TABLE_KERNELS=1: k_hist + k_norm launches
    e = launch_tables((int)dtype, p, cs);
    p.tables_ready = 1;
  } else {
    p.n_t_items = t_items_of(J);  // small streams: T items inside k_fused (one launch)
  }
  plan_flags(p);
  if (e == cudaSuccess) e = launch_fused((int)dtype, p, cs, 0);
  if (e != cudaSuccess) {
    fprintf(stderr, "uzip_compress: %s\n", cudaGetErrorString(e));
    return UZIP_ERR_CUDA;
  }
  return UZIP_OK;
}

uzip_status_t uzip_decompress(const void *in, size_t in_bytes, void *out, size_t count, uzip_dtype_t dtype,
                              int32_t *d_status, void *ws, size_t ws_bytes, void *stream) {
  NvtxRange nvtx_range("uzip_decompress");
  if ((int)dtype < 0 || (int)dtype >= kNumDtypes) return UZIP_ERR_UNSUPPORTED_DTYPE;
  if (!in || !ws || !d_status || !aligned16(in) || !aligned16(ws)) return UZIP_ERR_INVALID_ARG;
  if (count > 0 && (!out || !aligned16(out))) return UZIP_ERR_INVALID_ARG;
  if (ws_bytes < 64) return UZIP_ERR_CAPACITY;
  cudaError_t e =
      launch_decompress((int)dtype, in, in_bytes, out, count, ws, d_status, (cudaStream_t)stream, 0);
  if (e != cudaSuccess) {
    fprintf(stderr, "uzip_decompress: %s\n", cudaGetErrorString(e));
    return UZIP_ERR_CUDA;
  }
  return UZIP_OK;
}

}  // extern "C"
