// staged.cu -- the paper's staged compression pipeline as an ablation baseline.
//
// PAPER.md §2.1.2 describes DietGPU-style compression in three global-memory passes:
//   Step 1  split every float into exponent symbol + remaining bits and build ONE global
//           frequency table               -> k_stage_split + k_stage_table
//   Step 2  code each block independently into a temporary buffer
//                                                  -> k_stage_encode
//   Step 3  "merged into a single contiguous output buffer ... a third global memory write"
//                                       -> prefix scan (CUB) + k_stage_copy
// The fused kernel (fused_impl.cuh) removes Steps 1 and 3 as passes.  This file keeps
// them, on the same encoder (encode_block) and the same stream format, so the two can be compared
// on one GPU byte for byte: the output equals uzip_compress(global_table = 1) and the oracle's
// global-table stream.  `res_out` optionally redirects the residual plane (Step 1's "remaining
// bits") to a separate buffer and `split_done` is recorded after Step 1, so a caller can move that
// plane with the copy engine while Steps 2-3 run (the split-send of P:300-311 on copy engines).
#include <cub/device/device_scan.cuh>

#include "fused_impl.cuh"

namespace uzip {
namespace {

constexpr int kStageCtasPerSm = 8;

struct StageWs {  // carved from the caller's workspace
  uint32_t *hist;          // 256 global counts (zero between calls: k_stage_table resets them)
  uint4 *enc;              // 256 encode entries
  uint16_t *tab16;         // 256 frequencies
  uint8_t *sym;            // symbols, per block in the encoder's coding order (n_coded bytes)
  uint8_t *tmp;            // coded blocks, one B-byte slot each (Step 2's temporary buffer)
  unsigned long long *size, *off;  // per block
  void *cub;               // CUB scan scratch
  size_t cub_bytes;
  static uint64_t bytes(const StreamGeom &g, size_t cub_bytes) {
    const uint64_t nb = g.n_blocks ? g.n_blocks : 1;
    return 1024 + 4096 + 512 + round16(g.n_coded) + round16(nb * g.B) + 2 * round16(8 * nb) + round16(cub_bytes);
  }
  static StageWs carve(void *base, const StreamGeom &g, size_t cub_bytes) {
    StageWs w;
    uint8_t *p = static_cast<uint8_t *>(base);
    const uint64_t nb = g.n_blocks ? g.n_blocks : 1;
    w.hist = reinterpret_cast<uint32_t *>(p), p += 1024;
    w.enc = reinterpret_cast<uint4 *>(p), p += 4096;
    w.tab16 = reinterpret_cast<uint16_t *>(p), p += 512;
    w.sym = p, p += round16(g.n_coded);
    w.tmp = p, p += round16(nb * g.B);
    w.size = reinterpret_cast<unsigned long long *>(p), p += round16(8 * nb);
    w.off = reinterpret_cast<unsigned long long *>(p), p += round16(8 * nb);
    w.cub = p;
    w.cub_bytes = cub_bytes;
    return w;
  }
};

size_t cub_scan_bytes(uint64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                (int)(n ? n : 1));
  return b;
}

// Step 1: split every 16-byte vector of the coded region; symbols to ws.sym in coding
// order (row of round j at (R-1-j)*32 of its block, as split_block with REV), residual bytes to
// their plane(s); per-CTA shared histogram, flushed into the global table counts.
template <int DT, int B>
__global__ void __launch_bounds__(256) k_stage_split(const uint8_t *__restrict__ in, StreamGeom g, StageWs ws,
                                                     uint8_t *res0, uint8_t *res1) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  constexpr uint32_t kVec = VecTraits<DT>::kSym;
  const uint64_t nvec = g.n_coded / kVec;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 w = ldg_nc_v4(in + v * 16);
    const uint64_t el = v * kVec, b = el / B;
    const uint32_t e = (uint32_t)(el % B);
    uint8_t *sp = ws.sym + b * B + (uint32_t)(B - 32) - (e & ~31u) + (e & 31u);
    uint32_t s4[2];
    if (DT == kF32) {
      uint2 lo;
      uint32_t hi4;
      split4_f32(w, s4[0], lo, hi4);
      *reinterpret_cast<uint32_t *>(sp) = s4[0];
      *reinterpret_cast<uint2 *>(res0 + 2 * el) = lo;
      *reinterpret_cast<uint32_t *>(res1 + el) = hi4;
    } else {
      uint32_t q0, q1;
      if (DT == kBF16) {
        split4_bf16(w.x, w.y, s4[0], q0);
        split4_bf16(w.z, w.w, s4[1], q1);
      } else {
        split4_f16(w.x, w.y, s4[0], q0);
        split4_f16(w.z, w.w, s4[1], q1);
      }
      *reinterpret_cast<uint2 *>(sp) = make_uint2(s4[0], s4[1]);
      *reinterpret_cast<uint2 *>(res0 + el) = make_uint2(q0, q1);
    }
#pragma unroll
    for (int k = 0; k < (int)kVec; ++k) atomicAdd(&h[(s4[k >> 2] >> (8 * (k & 3))) & 0xFFu], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(ws.hist + threadIdx.x, h[threadIdx.x]);
}

// Step 1 (cont.): rule N1 over the global counts (R5); the table and chunk offset 0 go to the
// output; the counts are cleared for the next call.
__global__ void __launch_bounds__(256) k_stage_table(StageWs ws, uint8_t *out, StreamGeom g) {
  __shared__ unsigned long long red64[8];
  __shared__ uint32_t red32[8];
  const uint32_t cnt = ws.hist[threadIdx.x];
  norm_tables(cnt, ws.enc, ws.tab16, nullptr, red64, red32);
  ws.hist[threadIdx.x] = 0;
  reinterpret_cast<uint16_t *>(out + g.off_tab)[threadIdx.x] = ws.tab16[threadIdx.x];
  if (threadIdx.x == 0 && g.n_blocks) *reinterpret_cast<unsigned long long *>(out + g.off_coff) = 0ull;
}

// Step 2: one warp per block codes it (the fused kernel's encoder) into its B-byte
// slot of ws.tmp; stored-raw blocks (R13) hold their symbols in element order; directory entry
// and size per block.
template <int DT, int B>
__global__ void __launch_bounds__(256) k_stage_encode(StreamGeom g, StageWs ws, uint8_t *out) {
  __shared__ __align__(16) uint4 tab[256];
  __shared__ __align__(16) uint8_t bufs[kWarps][B + 256];
  tab[threadIdx.x] = ws.enc[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = warp_id();
  uint8_t *buf = bufs[warp];
  uint16_t *buf16 = reinterpret_cast<uint16_t *>(buf);
  EncJob J;  // the encoder's rare overflow path stores words straight to J.dst[0] + off_pay + off + 128
  J.nd = 1;
  J.dst[0] = ws.tmp - g.off_pay;
  for (uint64_t b = (uint64_t)blockIdx.x * kWarps + warp; b < g.n_blocks; b += (uint64_t)gridDim.x * kWarps) {
    const uint8_t *sb = ws.sym + b * B;
    for (uint32_t i = lane; i < (uint32_t)B / 16; i += 32)
      reinterpret_cast<uint4 *>(buf)[i] = reinterpret_cast<const uint4 *>(sb)[i];
    __syncwarp();
    uint32_t x = kL, K = 0;
    bool ovf = false;
    encode_block<DT, B, false>(J, g, 0, buf, tab, x, K, ovf);
    const uint32_t coded = (uint32_t)round16(128 + 2ull * K);
    const bool raw = coded >= (uint32_t)B;
    uint8_t *slot = ws.tmp + b * B;
    __syncwarp();
    if (raw) {  // element order = the coding-order rows reversed
      for (uint32_t i = lane; i < (uint32_t)B / 16; i += 32) {
        const uint32_t row = i / 2, half = i % 2;
        reinterpret_cast<uint4 *>(slot)[((B / 32 - 1 - row) * 2) + half] = reinterpret_cast<const uint4 *>(sb)[i];
      }
    } else if (ovf) {  // rare: words outran the consumed rows -- code again straight into the slot
      for (uint32_t i = lane; i < (uint32_t)B / 16; i += 32)
        reinterpret_cast<uint4 *>(buf)[i] = reinterpret_cast<const uint4 *>(sb)[i];
      __syncwarp();
      uint32_t x2 = kL, K2 = 0;
      bool o2 = false;
      encode_block<DT, B, true>(J, g, b * B, buf, tab, x2, K2, o2);
      reinterpret_cast<uint32_t *>(slot)[lane] = x2;
      for (uint32_t i = 2 * K + lane * 2; i < coded - 128; i += 64) *reinterpret_cast<uint16_t *>(slot + 128 + i) = 0;
    } else {
      if (lane < 8) buf16[K + lane] = 0;
      __syncwarp();
      reinterpret_cast<uint32_t *>(slot)[lane] = x;
      for (uint32_t i = lane; i < (coded - 128) / 16; i += 32)
        reinterpret_cast<uint4 *>(slot + 128)[i] = reinterpret_cast<const uint4 *>(buf)[i];
    }
    if (lane == 0) {
      ws.size[b] = raw ? (unsigned long long)B : coded;
      reinterpret_cast<uint32_t *>(out + g.off_dir)[b] = raw ? kRawBlock : K;
    }
    __syncwarp();
  }
}

// Step 3: copy every coded block from its slot to its scanned offset in the payload;
// the last block's warp writes the header, zero pads and the raw tail (finalize_stream).
template <int DT, int B>
__global__ void __launch_bounds__(256) k_stage_copy(const uint8_t *__restrict__ in, StreamGeom g, StageWs ws,
                                                    uint8_t *out, uint64_t *d_out_bytes) {
  const int lane = threadIdx.x & 31, warp = warp_id();
  const uint64_t nb = g.n_blocks;
  for (uint64_t b = (uint64_t)blockIdx.x * kWarps + warp; b < nb; b += (uint64_t)gridDim.x * kWarps) {
    const unsigned long long off = ws.off[b], size = ws.size[b];
    const uint4 *src = reinterpret_cast<const uint4 *>(ws.tmp + b * B);
    uint4 *dst = reinterpret_cast<uint4 *>(out + g.off_pay + off);
    for (uint32_t i = lane; i < size / 16; i += 32) dst[i] = src[i];
  }
  if (blockIdx.x == 0 && warp == 0) {
    EncJob J;
    memset(&J, 0, sizeof J);
    J.in = in;
    J.g = g;
    J.nd = 1;
    J.dst[0] = out;
    J.d_out_bytes = d_out_bytes;
    finalize_stream<DT>(J, nb ? ws.off[nb - 1] + ws.size[nb - 1] : 0ull);
  }
}

template <int DT, int B>
cudaError_t staged_t(const uint8_t *in, const StreamGeom &g, uint8_t *out, uint64_t *d_out_bytes, void *wsp,
                     uint8_t *res_out, cudaEvent_t split_done, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const StageWs ws = StageWs::carve(wsp, g, cub_scan_bytes(g.n_blocks));
  uint8_t *res0 = res_out ? res_out : out + g.off_res0;
  uint8_t *res1 = res_out ? res_out + (g.off_res1 - g.off_res0) : out + g.off_res1;
  const int grid = sms * kStageCtasPerSm;
  k_stage_split<DT, B><<<grid, 256, 0, st>>>(in, g, ws, res0, res1);
  if (split_done) cudaEventRecord(split_done, st);
  k_stage_table<<<1, 256, 0, st>>>(ws, out, g);
  if (g.n_blocks) {
    k_stage_encode<DT, B><<<(unsigned)((g.n_blocks + kWarps - 1) / kWarps), 256, 0, st>>>(g, ws, out);
    size_t cb = ws.cub_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(ws.cub, cb, ws.size, ws.off, (int)g.n_blocks, st);
    if (e != cudaSuccess) return e;
  }
  k_stage_copy<DT, B><<<(unsigned)std::max<uint64_t>(1, (g.n_blocks + kWarps - 1) / kWarps), 256, 0, st>>>(
      in, g, ws, out, d_out_bytes);
  return cudaGetLastError();
}

template <int DT>
cudaError_t staged_dt(const uint8_t *in, const StreamGeom &g, uint8_t *out, uint64_t *d_out_bytes, void *ws,
                      uint8_t *res_out, cudaEvent_t ev, cudaStream_t st) {
  switch (g.B) {
    case 1024: return staged_t<DT, 1024>(in, g, out, d_out_bytes, ws, res_out, ev, st);
    case 2048: return staged_t<DT, 2048>(in, g, out, d_out_bytes, ws, res_out, ev, st);
    default: return staged_t<DT, 4096>(in, g, out, d_out_bytes, ws, res_out, ev, st);
  }
}

uzip_status_t staged_geom(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params, StreamGeom *g) {
  if (!(dtype == UZIP_BF16 || dtype == UZIP_F16 || dtype == UZIP_F32)) return UZIP_ERR_UNSUPPORTED_DTYPE;
  uzip_codec_params_t p = params ? *params : uzip_codec_params_t{0, 0, 0, 0};
  p.global_table = 1;  // Step 1 builds one global table
  if (p.block_symbols > kMaxB) return UZIP_ERR_INVALID_ARG;  // the ablation pipeline: B <= 4096
  return resolve_geom((int)dtype, count, &p, g);
}

}  // namespace
}  // namespace uzip

using namespace uzip;

extern "C" {

size_t uzip_staged_workspace_bytes(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params) {
  StreamGeom g;
  if (staged_geom(count, dtype, params, &g) != UZIP_OK) return 0;
  return (size_t)StageWs::bytes(g, cub_scan_bytes(g.n_blocks));
}

uzip_status_t uzip_compress_staged(const void *in, size_t count, uzip_dtype_t dtype, void *out, size_t out_capacity,
                                   uint64_t *d_out_bytes, void *ws, size_t ws_bytes,
                                   const uzip_codec_params_t *params, void *res_out, void *split_done,
                                   void *stream) {
  StreamGeom g;
  uzip_status_t s = staged_geom(count, dtype, params, &g);
  if (s != UZIP_OK) return s;
  if (!out || !ws || (count && !in)) return UZIP_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(ws) |
       reinterpret_cast<uintptr_t>(res_out)) & 15u)
    return UZIP_ERR_INVALID_ARG;
  if (out_capacity < g.total(g.n_blocks * (uint64_t)g.B)) return UZIP_ERR_CAPACITY;
  if (ws_bytes < StageWs::bytes(g, cub_scan_bytes(g.n_blocks))) return UZIP_ERR_CAPACITY;
  const uint8_t *ip = static_cast<const uint8_t *>(in);
  uint8_t *op = static_cast<uint8_t *>(out), *rp = static_cast<uint8_t *>(res_out);
  cudaEvent_t ev = static_cast<cudaEvent_t>(split_done);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  switch (dtype) {
    case UZIP_BF16: e = staged_dt<kBF16>(ip, g, op, d_out_bytes, ws, rp, ev, st); break;
    case UZIP_F16: e = staged_dt<kF16>(ip, g, op, d_out_bytes, ws, rp, ev, st); break;
    default: e = staged_dt<kF32>(ip, g, op, d_out_bytes, ws, rp, ev, st); break;
  }
  return e == cudaSuccess ? UZIP_OK : UZIP_ERR_CUDA;
}

}  // extern "C"
