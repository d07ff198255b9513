// codec.cu -- k_decode, the stream-validating decoder behind uzip_decompress.
//
//   k_decode  a7+a8: header/section validation, per-chunk decode table,
//             warp-per-block table-driven rANS decode + join (P:391,
//             P:405-406).  Never reads or writes out of bounds on a corrupt
//             stream.
//
// The encoder (uzip_compress) is the E item of k_fused (fused.cu).
#include <cstdio>

#include "codec_dev.cuh"
#include "uzip_device.cuh"
#include "uzip_internal.h"

namespace uzip {

// ================================================================ k_decode
// Occupancy (the decoder is latency-bound on the table-lookup -> ALU -> word-fetch chain, so
// resident warps matter): a coded block is staged in smem only up to kStage bytes -- every
// realistic block is far below it (bf16 weights ~1.4 KB, f16 uniform ~2.8 KB) -- and a larger
// one (rare) or a raw block is decoded / joined straight from global memory.  With kStage =
// 3200 and 256-block segments a CTA needs 44 KB, so 5 CTAs (40 warps) fit per SM instead of 4.
// (Round 2: 3584 bytes for f16 / fp8 / fp32 at 4 CTAs -- 256 MiB U[-1,1] f16 decode 0.161 -> 0.151 ms,
// e4m3 0.179 -> 0.164 ms.)  bf16 blocks (8-bit exponent symbols, ~1.2-1.5 KB coded) stage up to 2176 bytes, so 6 CTAs (48 warps,
// 40 registers, no spills) fit: 1 GiB bf16 decode 0.578 -> 0.567 ms.  f16 and fp8 symbols carry
// fraction / second-exponent bits (coded blocks up to ~3.4 KB) and keep 3200 bytes at 5 CTAs; fp32's
// two residual planes need more registers (at 40 it spills), so it keeps 5 CTAs too.
#ifndef UZIP_DEC_MINB
#define UZIP_DEC_MINB 5
#endif
#ifndef UZIP_DEC_STAGE
#define UZIP_DEC_STAGE 3584  // f16 / fp8 / fp32 (4 CTAs): U[-1,1] f16 blocks (~2.7 KB, some larger) stay staged
#endif
#ifndef UZIP_DEC_MINB_EXP8
#define UZIP_DEC_MINB_EXP8 6
#endif
#ifndef UZIP_DEC_STAGE_EXP8
#define UZIP_DEC_STAGE_EXP8 2176
#endif
// bf16 warps decode two coded blocks at once, their rANS chains interleaved (decode_join_warp2): the
// decoder is latency-bound on its lookup -> renormalize -> word-fetch chain, and a second chain per
// warp hides it better than more warps can (48 registers): 1 GiB bf16 decode 0.565 -> 0.540 ms.  Raw,
// oversized or lone blocks take the one-chain path.  Staging 1488 bytes per block (W = bf16 N(0, 0.02)
// blocks code to 1408-1488 bytes; a larger one takes the one-chain path) fits 5 CTAs x 8 warps x 2 chains
// per SM (45.3 KB each; 1664 bytes held 4): 0.511 -> 0.501 ms.
#ifndef UZIP_DEC_PAIR
#define UZIP_DEC_PAIR 1
#endif
#ifndef UZIP_DEC_MINB_F32
#define UZIP_DEC_MINB_F32 4  // fp32 (two residual planes): 64 registers without spills (5 CTAs spilled)
#endif
#ifndef UZIP_DEC_PAIR_MINB
#define UZIP_DEC_PAIR_MINB 5  // register budget (48); smem holds 4 CTAs
#endif
#ifndef UZIP_DEC_PAIR_WIDE
#define UZIP_DEC_PAIR_WIDE 0  // A/B: f16 / e4m3 pairs too (3 CTAs: f16 U decode 0.156 vs 0.150 ms, e4m3 0.168 vs 0.163)
#endif
#ifndef UZIP_DEC_PAIR_STAGE_WIDE
#define UZIP_DEC_PAIR_STAGE_WIDE 2816
#endif
#ifndef UZIP_DEC_L2PF
#define UZIP_DEC_L2PF 0  // A/B: L2 prefetch of the next pair's payload
#endif
#ifndef UZIP_DEC_CARVEOUT
#define UZIP_DEC_CARVEOUT 0  // A/B: preferred shared-memory carveout (percent) of k_decode; 0 = driver default
#endif
#ifndef UZIP_DEC_PAIR_STAGE
#define UZIP_DEC_PAIR_STAGE 1488  // 5 CTAs x 8 warps x 2 chains (45.3 KB per CTA); 1664 held 4: 0.511 -> 0.501 ms
#endif
#ifndef UZIP_DEC_SEG
#define UZIP_DEC_SEG 256
#endif
template <int DT>
struct DecShared {
  static constexpr bool kExp8 = DT == kBF16;  // 8-bit exponent symbols, one residual plane
  // two blocks per warp (two staging areas): bf16; f16 / e4m3 (one residual byte per symbol, wider
  // symbols -> larger staging, 3 CTAs) under UZIP_DEC_PAIR_WIDE
  static constexpr bool kWidePair = UZIP_DEC_PAIR_WIDE && (DT == kF16 || DT == kE4M3);
  static constexpr bool kPair = (kExp8 || kWidePair) && UZIP_DEC_PAIR;
  static constexpr int kMinB = kPair ? UZIP_DEC_PAIR_MINB : kExp8 ? UZIP_DEC_MINB_EXP8
                              : DT == kF32 ? UZIP_DEC_MINB_F32 : UZIP_DEC_MINB;
  static constexpr int kTab = 4096 * 4;              // decode table
  static constexpr int kSeg = UZIP_DEC_SEG;          // blocks per segment (a multiple of 256)
  static constexpr int kOff = kSeg * 4;              // per-segment block offsets (relative to chunk)
  static constexpr int kStage = kWidePair ? UZIP_DEC_PAIR_STAGE_WIDE : kPair ? UZIP_DEC_PAIR_STAGE
                               : kExp8 ? UZIP_DEC_STAGE_EXP8 : UZIP_DEC_STAGE;  // per block
  static constexpr int kWarpBuf = kStage + 256;      // staged payload + 8-round symbol ring
  // one-chain decodes (raw neighbours, oversized or lone blocks) of pair launches stage into the whole
  // warp buffer (both pair areas, one ring at its end): blocks up to 3232 bytes stay in smem
  static constexpr int kStage1 = (kPair ? 2 : 1) * kWarpBuf - 256;
  static constexpr int kWarpBytes = kWarpBuf * (kPair ? 2 : 1);
  static constexpr int kBytes = kTab + kOff + kWarps * kWarpBytes;
  static_assert(kStage % 16 == 0 && kSeg % 256 == 0, "decoder smem layout");
};

__device__ __forceinline__ void set_err(CodecWs &ws, uint32_t code) { atomicCAS(ws.err, 0u, code); }

// a8: one warp decodes block b (payload at `off` within the payload section)
// and joins it with the residual plane into `out`.
template <int DT, int B>
__device__ void decode_block_t(const uint8_t *__restrict__ in, const StreamGeom &g, uint32_t d, uint64_t b,
                               unsigned long long off, uint32_t size, const uint32_t *dtab, uint8_t *pay,
                               uint8_t *ring, uint8_t *__restrict__ out, CodecWs &ws) {
  const int lane = threadIdx.x & 31;
  const uint8_t *src = in + g.off_pay + off;
  uint8_t *dst = out + b * (uint64_t)B * g.eb;
  bool ok = true;
  if (d == kRawBlock) {
    join_block<DT, B>(src, in, g, b, dst);  // raw symbols joined straight from the stream
  } else if (size <= (uint32_t)DecShared<DT>::kStage1) {
    stage_block(src, size / 16, pay);
    // (B <= 4096: a corrupt word index reaches at most 8 KiB below the payload, inside the window)
    ok = decode_join_warp<DT, B, UZIP_DEC_NOCLAMP != 0 && DT != kF32 && B <= 4096>(pay, d, dtab, ring, in, g, b, dst);
  } else {
    // rare: a coded block larger than the staging area is decoded in place from global memory
    // (word indices never leave [0, K), so even a corrupt stream is read in bounds)
    ok = decode_join_warp<DT, B>(src, d, dtab, ring, in, g, b, dst);
  }
  if (!ok && lane == 0) set_err(ws, UZIP_ERR_CORRUPT_STREAM);
  __syncwarp();
}

template <int DT>
__device__ void decode_block(const uint8_t *__restrict__ in, const StreamGeom &g, unsigned long long payload,
                             uint32_t d, uint64_t b, unsigned long long off, const uint32_t *dtab, uint8_t *pay,
                             uint8_t *ring, uint8_t *__restrict__ out, CodecWs &ws) {
  const int lane = threadIdx.x & 31;
  bool bad = false;
  const uint32_t size = block_size(d, g.B, bad);
  if (bad || off + size > payload) {
    if (lane == 0) set_err(ws, UZIP_ERR_CORRUPT_STREAM);
    return;
  }
  switch (g.B) {
    case 1024: decode_block_t<DT, 1024>(in, g, d, b, off, size, dtab, pay, ring, out, ws); break;
    case 2048: decode_block_t<DT, 2048>(in, g, d, b, off, size, dtab, pay, ring, out, ws); break;
    case 8192: decode_block_t<DT, 8192>(in, g, d, b, off, size, dtab, pay, ring, out, ws); break;
    case 16384: decode_block_t<DT, 16384>(in, g, d, b, off, size, dtab, pay, ring, out, ws); break;
    default: decode_block_t<DT, 4096>(in, g, d, b, off, size, dtab, pay, ring, out, ws); break;
  }
}

// Two coded, staged 4096-symbol blocks at once (DecShared::kPair); false = not eligible (raw, too large,
// or another block size), the caller then decodes them one by one.
template <int DT>
__device__ bool decode_pair(const uint8_t *__restrict__ in, const StreamGeom &g, unsigned long long payload,
                            uint32_t dA, uint64_t bA, unsigned long long offA, uint32_t dB, uint64_t bB,
                            unsigned long long offB, const uint32_t *dtab, uint8_t *pay, uint8_t *__restrict__ out,
                            CodecWs &ws) {
  using DS = DecShared<DT>;
  if constexpr (!DS::kPair) {
    return false;
  } else {
    bool bad = false;
    const uint32_t sA = block_size(dA, g.B, bad), sB = block_size(dB, g.B, bad);
    if (g.B != 4096 || bad || dA == kRawBlock || dB == kRawBlock || sA > (uint32_t)DS::kStage ||
        sB > (uint32_t)DS::kStage || offA + sA > payload || offB + sB > payload)
      return false;
    const int lane = threadIdx.x & 31;
    uint8_t *payB = pay + DS::kWarpBuf;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(pay), s1 = (uint32_t)__cvta_generic_to_shared(payB);
    const uint8_t *srcA = in + g.off_pay + offA, *srcB = in + g.off_pay + offB;
    for (uint32_t i = lane; i < sA / 16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + 16 * i), "l"(srcA + 16 * i) : "memory");
    for (uint32_t i = lane; i < sB / 16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s1 + 16 * i), "l"(srcB + 16 * i) : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    __syncwarp();
    bool okA, okB;
    decode_join_warp2<DT, 4096>(pay, dA, payB, dB, dtab, pay + DS::kStage, payB + DS::kStage, in, g, bA, bB,
                                out + bA * 4096ull * g.eb, out + bB * 4096ull * g.eb, okA, okB);
    if (!(okA && okB) && lane == 0) set_err(ws, UZIP_ERR_CORRUPT_STREAM);
    __syncwarp();
    return true;
  }
}

template <int DT>
__global__ void __launch_bounds__(256, DecShared<DT>::kMinB) k_decode(const uint8_t *__restrict__ in, uint64_t in_bytes,
                                                  uint8_t *__restrict__ out, uint64_t n, CodecWs ws,
                                                  int32_t *__restrict__ d_status) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t *dtab = reinterpret_cast<uint32_t *>(smem);
  using DS = DecShared<DT>;
  uint32_t *soff = reinterpret_cast<uint32_t *>(smem + DS::kTab);
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  uint8_t *pay = smem + DS::kTab + DS::kOff + warp * DS::kWarpBytes;
  uint8_t *ring = pay + DS::kStage1;  // the one-chain ring (pairs use their own two)

  __shared__ uint32_t s_red[kWarps];
  __shared__ uint32_t s_bad;
  __shared__ unsigned long long s_base;
  __shared__ unsigned long long s_b[kWarps], s_t[kWarps];

  // ---- header validation (every CTA, identical outcome)
  uint32_t code = 0;
  StreamGeom g;
  unsigned long long payload = 0;
  if (in_bytes < kHeaderBytes) {
    code = UZIP_ERR_CORRUPT_STREAM;
  } else {
    const uint4 *h4 = reinterpret_cast<const uint4 *>(in);
    uint4 a = h4[0], b = h4[1], c = h4[2], d = h4[3];
    const uint32_t h[16] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w};
    const uint32_t dt = (h[1] >> 16) & 0xFF, flags = h[1] >> 24;
    const uint64_t hn = h[2] | ((uint64_t)h[3] << 32);
    const uint32_t B = h[4], CB = h[5], S = h[6];
    payload = h[10] | ((unsigned long long)h[11] << 32);
    const uint64_t total = h[12] | ((uint64_t)h[13] << 32);
    if (h[0] != 0x31425A55u || (h[1] & 0xFFFF) != kVersion) code = UZIP_ERR_CORRUPT_STREAM;
    else if (dt != (uint32_t)DT || hn != n) code = UZIP_ERR_SIZE_MISMATCH;
    else if ((flags & ~1u) != 0 || (h[7] & 0xFFFFFF) != (kProbBits | (kLanes << 8) | (kLBits << 16)))
      code = UZIP_ERR_CORRUPT_STREAM;
    else if (!gpu_block_ok(B) || CB == 0 || payload > in_bytes)
      code = UZIP_ERR_CORRUPT_STREAM;
    else {
      g.init(DT, n, B, CB, S, flags & 1);
      if ((flags & 1) && g.CB != CB) code = UZIP_ERR_CORRUPT_STREAM;
      else if (h[8] != g.n_blocks || h[9] != g.n_chunks) code = UZIP_ERR_CORRUPT_STREAM;
      else if (total != g.total(payload) || total > in_bytes) code = UZIP_ERR_CORRUPT_STREAM;
    }
  }

  if (code == 0) {
    const uint32_t B = g.B;
    const uint64_t nb = g.n_blocks;
    const uint64_t per = (nb + gridDim.x - 1) / gridDim.x;
    const uint64_t cb0 = (uint64_t)blockIdx.x * per;
    const uint64_t cb1 = min(nb, cb0 + per);
    const uint32_t *dir = reinterpret_cast<const uint32_t *>(in + g.off_dir);
    const unsigned long long *coff = reinterpret_cast<const unsigned long long *>(in + g.off_coff);
    for (uint64_t s0 = cb0; s0 < cb1;) {
      const uint64_t c = chunk_of(g, s0);
      const uint64_t c_first = c * g.CB;
      const uint64_t c_end = min(nb, c_first + g.CB);
      const uint64_t chunk_stop = min(cb1, c_end);
      __syncthreads();
      if (tid == 0) s_bad = 0;
      // ---- a7: decode table of chunk c (the shared builder; warp 0's staging buffer is its scratch,
      // free until the bookkeeping barriers below have published the table)
      if (!build_dtab(reinterpret_cast<const uint16_t *>(in + g.off_tab + 512 * c), dtab, s_red,
                      reinterpret_cast<uint32_t *>(smem + DS::kTab + DS::kOff))) {
        set_err(ws, UZIP_ERR_CORRUPT_STREAM);
        break;  // uniform: every warp read the same table
      }
      // ---- chunk bookkeeping: bytes before s0 inside the chunk; the CTA that
      // owns the chunk's first block also checks chunk_off[c] + sum == next.
      {
        const bool owner = c_first >= cb0;
        const uint64_t scan_end = owner ? c_end : s0;
        unsigned long long before = 0, chunk_total = 0;
        for (uint64_t bb = c_first + tid; bb < scan_end; bb += 256) {
          bool bad = false;
          const uint32_t sz = block_size(dir[bb], B, bad);
          if (bad) s_bad = 1;
          chunk_total += sz;
          if (bb < s0) before += sz;
        }
        before = warp_sum_u64(before);
        chunk_total = warp_sum_u64(chunk_total);
        if (lane == 0) {
          s_b[warp] = before;
          s_t[warp] = chunk_total;
        }
        __syncthreads();
        if (tid == 0) {
          unsigned long long bsum = 0, tsum = 0;
          for (int w = 0; w < kWarps; ++w) {
            bsum += s_b[w];
            tsum += s_t[w];
          }
          if (owner) {
            const unsigned long long co = coff[c];
            const unsigned long long next = (c + 1 < g.n_chunks) ? coff[c + 1] : payload;
            if ((c == 0 && co != 0) || co + tsum != next || next > payload) s_bad = 1;
          }
          s_base = bsum;
        }
        __syncthreads();
      }
      if (s_bad) {
        set_err(ws, UZIP_ERR_CORRUPT_STREAM);
        break;
      }
      const unsigned long long cbase = coff[c];
      // ---- segments of <= 1024 blocks: exclusive scan of sizes, then decode
      for (uint64_t seg = s0; seg < chunk_stop; seg += DS::kSeg) {
        const uint64_t seg_end = min(chunk_stop, seg + (uint64_t)DS::kSeg);
        const unsigned long long run0 = s_base;
        unsigned long long run = run0;
        for (uint64_t bb0 = seg; bb0 < seg_end; bb0 += 256) {
          const uint64_t bb = bb0 + tid;
          uint32_t sz = 0;
          if (bb < seg_end) {
            bool bad = false;
            sz = block_size(dir[bb], B, bad);
          }
          uint32_t inc2 = sz;
          for (int o = 1; o < 32; o <<= 1) {
            uint32_t tt = __shfl_up_sync(0xFFFFFFFFu, inc2, o);
            if (lane >= o) inc2 += tt;
          }
          if (lane == 31) s_red[warp] = inc2;
          __syncthreads();
          uint32_t wo = 0, all = 0;
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) wo += s_red[w];
            all += s_red[w];
          }
          if (bb < seg_end) soff[bb - seg] = (uint32_t)(run - run0 + wo + inc2 - sz);
          run += all;
          __syncthreads();
        }
        // ---- a8: warp per block
        for (uint64_t b = seg + warp; b < seg_end; b += kWarps) {
          const unsigned long long off = cbase + run0 + soff[b - seg];
#if UZIP_DEC_L2PF
          // A/B: pull the next pair's payload (blocks b + 16 and b + 24; lanes 0-15 / 16-31, 128 B each)
          // into L2 while this pair decodes
          if (DS::kPair && b + 3 * kWarps + 1 < seg_end) {
            const uint64_t nb2 = b + (lane < 16 ? 2 : 3) * kWarps - seg;
            const unsigned long long o0 = soff[nb2], o1 = soff[nb2 + 1];
            const unsigned long long at = (unsigned long long)(lane & 15) * 128;
            if (at < o1 - o0) asm volatile("prefetch.global.L2 [%0];" ::"l"(in + g.off_pay + cbase + run0 + o0 + at));
          }
#endif
          if (DS::kPair && b + kWarps < seg_end &&
              decode_pair<DT>(in, g, payload, dir[b], b, off, dir[b + kWarps], b + kWarps,
                              cbase + run0 + soff[b + kWarps - seg], dtab, pay, out, ws)) {
            b += kWarps;
            continue;
          }
          decode_block<DT>(in, g, payload, dir[b], b, off, dtab, pay, ring, out, ws);
        }
        __syncthreads();
        if (tid == 0) s_base = run;
        __syncthreads();
      }
      s0 = chunk_stop;
    }
    // raw tail
    if (blockIdx.x == 0) {
      const uint64_t tail_bytes = g.tail_bytes();
      const uint8_t *src = in + g.off_tail(payload);
      uint8_t *dst = out + g.n_coded * g.eb;
      for (uint64_t i = tid; i < tail_bytes; i += 256) dst[i] = src[i];
    }
  } else if (tid == 0) {
    set_err(ws, code);
  }

  // ---- completion: the last CTA publishes the status and resets the words
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const uint32_t old = atomicAdd(ws.dec_arrive, 1u);
    if (old == gridDim.x - 1) {
      __threadfence();
      *d_status = (int32_t)atomicExch(ws.err, 0u);
      *ws.dec_arrive = 0;
    }
  }
}

// ================================================================ launchers
namespace {
constexpr int kMaxDev = 64;
int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDev ? dev : 0;
}
int sm_count() {
  static int n[kMaxDev] = {0};
  const int dev = cur_dev();
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
  return occ > 0 ? occ : 1;
}

template <int DT>
cudaError_t launch_decode_t(const void *in, uint64_t in_bytes, void *out, uint64_t n, void *ws_ptr,
                            int32_t *d_status, cudaStream_t st, int max_ctas, uint64_t est_blocks) {
  CodecWs ws = CodecWs::carve(ws_ptr);
  auto kern = k_decode<DT>;
  static bool attr[kMaxDev] = {false};  // per device
  const int dev = cur_dev();
  if (!attr[dev]) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DecShared<DT>::kBytes);
    if (e != cudaSuccess) return e;
#if UZIP_DEC_CARVEOUT
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, UZIP_DEC_CARVEOUT);
#endif
    attr[dev] = true;
  }
  int grid = sm_count() * occupancy(kern, 256, DecShared<DT>::kBytes);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  const uint64_t want = (est_blocks + kWarps - 1) / kWarps;  // >= one block per warp: one table build per 8 blocks
  if ((uint64_t)grid > want) grid = (int)(want ? want : 1);
  kern<<<grid, 256, DecShared<DT>::kBytes, st>>>((const uint8_t *)in, in_bytes, (uint8_t *)out, n, ws, d_status);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_decompress(int dtype, const void *in, uint64_t in_bytes, void *out, uint64_t n, void *ws,
                              int32_t *d_status, cudaStream_t st, int max_ctas) {
  // the block size is in the (device-side) header; size the grid for the default B = 4096 (a
  // B = 1024 stream then gets 4 blocks per warp, still plenty of CTAs once it is large)
  const uint64_t est_blocks = n / 4096;
  switch (dtype) {
    case kBF16: return launch_decode_t<kBF16>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    case kF16: return launch_decode_t<kF16>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    case kE4M3: return launch_decode_t<kE4M3>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    case kE5M2: return launch_decode_t<kE5M2>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    default: return launch_decode_t<kF32>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
  }
}

}  // namespace uzip
