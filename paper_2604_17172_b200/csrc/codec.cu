// codec.cu -- the single-GPU Uzip codec kernels for sm_100a.
//
//   k_table   a2+a3: sampled per-chunk histogram -> rule-N1 table ->
//             encode reciprocals; also resets k_encode's look-back state.
//   k_encode  a1+a4+a5: split (residual leaves at once), one warp
//             per 4096-symbol block, 32-lane interleaved rANS (P:161-165,
//             P:421-424), decoupled look-back over tile sizes so every block
//             is written once at its final offset (Step 3 removed).
//   k_decode  a7+a8: per-chunk decode table, warp-per-block decode + join.
//
// Output bytes are identical to the CPU oracle's (checked by tests/test_gpu_codec.py).
#include <cstdio>

#include "uzip_device.cuh"
#include "uzip_internal.h"

namespace uzip {

// ================================================================ k_table
// grid = (parts, n_chunks), 256 threads.  Part p of chunk c histograms sample
// symbols [p*16384, (p+1)*16384) of the chunk; the last part to arrive
// normalizes (rule N1, R5) and writes the 512-byte table into the stream and
// the encode entries into the workspace.
template <int DT>
__global__ void __launch_bounds__(256) k_table(const uint8_t *__restrict__ in, StreamGeom g,
                                               uint8_t *__restrict__ out, CodecWs ws) {
  __shared__ uint32_t hist[kWarps][256];
  __shared__ uint32_t cnt[256];
  __shared__ uint16_t f16[256];
  __shared__ unsigned long long red64[kWarps];
  __shared__ uint32_t red32[kWarps];
  __shared__ uint32_t s_last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t c = blockIdx.y, part = blockIdx.x;

  // Reset k_encode's look-back words and ticket for the launch that follows.
  {
    const uint64_t nt = g.n_tiles();
    const uint64_t nctas = (uint64_t)gridDim.x * gridDim.y;
    const uint64_t me = (uint64_t)blockIdx.y * gridDim.x + blockIdx.x;
    for (uint64_t t = me * 256 + tid; t < nt; t += nctas * 256) ws.tile_status[t] = 0ull;
    if (me == 0 && tid == 0) *ws.ticket = 0;
  }

  const uint32_t slen = g.sample_len(c);
  const uint32_t parts = (slen + kHistSymsPerCta - 1) / kHistSymsPerCta;
  if (part >= parts) return;

  for (int i = tid; i < kWarps * 256; i += 256) (&hist[0][0])[i] = 0;
  __syncthreads();

  const uint64_t first = (uint64_t)c * g.CB * g.B + (uint64_t)part * kHistSymsPerCta;
  const uint32_t len = min(kHistSymsPerCta, slen - part * kHistSymsPerCta);
  // symbols per 16-byte vector: 8 (2-byte types) or 4 (fp32)
  constexpr uint32_t kPer = (DT == kF32) ? 4 : 8;
  const uint8_t *base = in + first * elem_bytes(DT);
  for (uint32_t v = tid; v < len / kPer; v += 256) {
    uint4 w = ldg_nc_v4(base + (size_t)v * 16);
    uint32_t s_lo, s_hi;
    if (DT == kBF16) {
      uint32_t r;
      split4_bf16(w.x, w.y, s_lo, r);
      split4_bf16(w.z, w.w, s_hi, r);
    } else if (DT == kF16) {
      uint32_t r;
      split4_f16(w.x, w.y, s_lo, r);
      split4_f16(w.z, w.w, s_hi, r);
    } else {
      uint2 lo;
      uint32_t hi;
      split4_f32(w, s_lo, lo, hi);
      s_hi = 0;
    }
#pragma unroll
    for (int k = 0; k < (int)kPer; ++k) {
      uint32_t s = ((k < 4 ? s_lo : s_hi) >> (8 * (k & 3))) & 0xFFu;
      atomicAdd(&hist[warp][s], 1u);
    }
  }
  // sample lengths that are not a multiple of the vector width (custom S)
  for (uint32_t i = (len / kPer) * kPer + tid; i < len; i += 256) {
    uint32_t s;
    if (DT == kF32) s = (reinterpret_cast<const uint32_t *>(base)[i] >> 23) & 0xFFu;
    else if (DT == kBF16) s = (reinterpret_cast<const uint16_t *>(base)[i] >> 7) & 0xFFu;
    else s = reinterpret_cast<const uint16_t *>(base)[i] >> 8;
    atomicAdd(&hist[warp][s], 1u);
  }
  __syncthreads();
  {
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += hist[w][tid];
    if (sum) atomicAdd(&ws.counts[c * 256 + tid], sum);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&ws.arrive[c], 1u) == parts - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- this CTA is the last for chunk c: normalize (rule N1)
  cnt[tid] = ld_cg_u32(&ws.counts[c * 256 + tid]);
  ws.counts[c * 256 + tid] = 0;
  if (tid == 0) ws.arrive[c] = 0;
  __syncthreads();
  // total and argmax (lowest symbol on ties): key = cnt<<8 | (255 - s)
  unsigned long long key = ((unsigned long long)cnt[tid] << 8) | (255u - tid);
  unsigned long long tot = cnt[tid];
  for (int o = 16; o; o >>= 1) {
    unsigned long long ok = __shfl_xor_sync(0xFFFFFFFFu, key, o);
    key = ok > key ? ok : key;
    tot += __shfl_xor_sync(0xFFFFFFFFu, tot, o);
  }
  if (lane == 0) {
    red64[warp] = key;
    red32[warp] = (uint32_t)tot;
  }
  __syncthreads();
  unsigned long long best_key = 0, total = 0;
  for (int w = 0; w < kWarps; ++w) {
    best_key = red64[w] > best_key ? red64[w] : best_key;
    total += red32[w];
  }
  const uint32_t best = 255u - (uint32_t)(best_key & 0xFFu);
  uint32_t f;
  if (total == 0) f = kM / 256;
  else f = 1u + (uint32_t)(((unsigned long long)cnt[tid] * (kM - 256)) / total);
  __syncthreads();
  // sum of f
  uint32_t fs = f;
  for (int o = 16; o; o >>= 1) fs += __shfl_xor_sync(0xFFFFFFFFu, fs, o);
  if (lane == 0) red32[warp] = fs;
  __syncthreads();
  uint32_t fsum = 0;
  for (int w = 0; w < kWarps; ++w) fsum += red32[w];
  if (total != 0 && tid == (int)best) f += kM - fsum;
  f16[tid] = (uint16_t)f;
  __syncthreads();
  // exclusive prefix (cdf) over 256 symbols
  uint32_t incl = f;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) red32[warp] = incl;
  __syncthreads();
  uint32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += red32[w];
  const uint32_t cdf = woff + incl - f;
  ws.enc[c * 256 + tid] = make_enc_entry(f, cdf);
  // 512-byte serialized table of chunk c (u16 little-endian)
  if (tid < 32) {
    const uint4 *src = reinterpret_cast<const uint4 *>(f16);
    reinterpret_cast<uint4 *>(out + g.off_tab + 512ull * c)[tid] = src[tid];
  }
}

// ================================================================ k_encode
// Decoupled look-back status word: flag in bits 62..63, value below.
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Called by one full warp; returns the exclusive prefix of tile `t`.
__device__ unsigned long long lookback(unsigned long long *status, uint64_t t, unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) st_relaxed_u64(&status[0], kFlagInc | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&status[t], kFlagAgg | agg);
  unsigned long long excl = 0;
  int64_t base = (int64_t)t - 1;
  while (true) {
    const int64_t idx = base - lane;
    unsigned long long s = idx >= 0 ? ld_relaxed_u64(&status[idx]) : (kFlagInc | 0ull);
    const uint32_t flag = (uint32_t)(s >> 62);
    const uint32_t inc = __ballot_sync(0xFFFFFFFFu, flag == 2);
    const uint32_t notready = __ballot_sync(0xFFFFFFFFu, flag == 0);
    const int first_inc = inc ? __ffs(inc) - 1 : 31;
    const uint32_t needed = first_inc == 31 ? 0xFFFFFFFFu : ((2u << first_inc) - 1u);
    if (notready & needed) {
      __nanosleep(32);
      continue;
    }
    excl += warp_sum_u64(lane <= first_inc ? (s & kValMask) : 0ull);
    if (inc) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(&status[t], kFlagInc | (excl + agg));
  return excl;
}

template <int DT, int B>
struct EncCfg {
  static constexpr int kVec = (DT == kF32) ? 4 : 8;          // elements per 16-byte load
  static constexpr int kIters = B / (32 * kVec);              // loads per lane per block
  static constexpr int kBatch = kIters < 16 ? kIters : 16;     // loads in flight per batch
  static constexpr int kRounds = B / 32;
  static constexpr int kWarpSmem = 2 * B;                     // symbols + coded block
  static constexpr int kSmem = 4096 /*enc table*/ + kWarps * kWarpSmem;
};

// Writes the header (payload and total sizes known now), section pads and the raw tail.
template <int DT>
__device__ void finalize_stream(const uint8_t *in, const StreamGeom &g, uint8_t *out, unsigned long long payload,
                                uint64_t *d_out_bytes) {
  const int lane = threadIdx.x & 31;
  const uint64_t total = g.total(payload);
  if (lane == 0) {
    uint32_t h[16];
    for (int i = 0; i < 16; ++i) h[i] = 0;
    h[0] = 0x31425A55u;                                  // "UZB1"
    h[1] = kVersion | (g.dtype << 16) | ((g.global & 1u) << 24);
    h[2] = (uint32_t)g.n;
    h[3] = (uint32_t)(g.n >> 32);
    h[4] = g.B;
    h[5] = g.CB;
    h[6] = g.S;
    h[7] = kProbBits | (kLanes << 8) | (kLBits << 16);
    h[8] = (uint32_t)g.n_blocks;
    h[9] = (uint32_t)g.n_chunks;
    h[10] = (uint32_t)payload;
    h[11] = (uint32_t)(payload >> 32);
    h[12] = (uint32_t)total;
    h[13] = (uint32_t)(total >> 32);
    uint4 *o = reinterpret_cast<uint4 *>(out);
    for (int i = 0; i < 4; ++i) o[i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    // zero pads: after chunk_off (n_chunks odd) and after dir
    const uint64_t e1 = g.off_coff + 8 * g.n_chunks;
    for (uint64_t p = e1; p < g.off_dir; ++p) out[p] = 0;
    const uint64_t e2 = g.off_dir + 4 * g.n_blocks;
    for (uint64_t p = e2; p < g.off_pay; ++p) out[p] = 0;
    if (d_out_bytes) *d_out_bytes = total;
  }
  const uint64_t tail_bytes = (g.n - g.n_coded) * g.eb;
  const uint8_t *src = in + g.n_coded * g.eb;
  uint8_t *dst = out + g.off_tail(payload);
  for (uint64_t i = lane; i < tail_bytes; i += 32) dst[i] = src[i];
}

template <int DT, int B>
__global__ void __launch_bounds__(256, 2) k_encode(const uint8_t *__restrict__ in, StreamGeom g,
                                                  uint8_t *__restrict__ out, CodecWs ws,
                                                  uint64_t *__restrict__ d_out_bytes) {
  using C = EncCfg<DT, B>;
  extern __shared__ __align__(16) uint8_t smem[];
  uint4 *tab = reinterpret_cast<uint4 *>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t *sym = smem + 4096 + warp * C::kWarpSmem;          // B symbol bytes
  uint8_t *blk = sym + B;                                    // coded block (states + words)
  uint16_t *blk16 = reinterpret_cast<uint16_t *>(blk);
  uint32_t *blk32 = reinterpret_cast<uint32_t *>(blk);

  __shared__ uint32_t s_ticket;
  __shared__ uint32_t s_size[kWarps], s_k[kWarps];
  __shared__ unsigned long long s_prefix;

  const uint64_t n_tiles = g.n_tiles();
  if (n_tiles == 0) {  // no whole block: header + raw tail only
    if (blockIdx.x == 0 && warp == 0) finalize_stream<DT>(in, g, out, 0ull, d_out_bytes);
    return;
  }
  const uint32_t lt = lanemask_lt();
  int64_t loaded_chunk = -1;

  while (true) {
    if (tid == 0) s_ticket = atomicAdd(ws.ticket, 1u);
    __syncthreads();
    const uint64_t t = s_ticket;
    if (t >= n_tiles) break;
    const uint64_t b0 = t * kTileBlocks;
    const int64_t c = (int64_t)(b0 / g.CB);
    if (c != loaded_chunk) {
      for (int i = tid; i < 256; i += 256) tab[i] = ws.enc[c * 256 + i];
      loaded_chunk = c;
    }
    __syncthreads();

    const uint64_t b = b0 + warp;
    uint32_t K = 0, size = 0;
    if (b < g.n_blocks) {
      // ---- a1: load 16-byte vectors, split, residual straight out, symbols to smem
      const uint8_t *src = in + b * (uint64_t)B * elem_bytes(DT);
#pragma unroll
      for (int h = 0; h < C::kIters; h += C::kBatch) {
      uint4 v[C::kBatch];
#pragma unroll
      for (int i = 0; i < C::kBatch; ++i) v[i] = ldg_nc_v4(src + (size_t)(lane + 32 * (h + i)) * 16);
#pragma unroll
      for (int i = 0; i < C::kBatch; ++i) {
        const uint32_t e = (uint32_t)(lane + 32 * (h + i)) * C::kVec;   // element within block
        if (DT == kF32) {
          uint32_t s4, h4;
          uint2 lo;
          split4_f32(v[i], s4, lo, h4);
          *reinterpret_cast<uint32_t *>(sym + e) = s4;
          *reinterpret_cast<uint2 *>(out + g.off_res0 + 2 * (b * B + e)) = lo;
          *reinterpret_cast<uint32_t *>(out + g.off_res1 + b * B + e) = h4;
        } else {
          uint32_t s0, s1, r0, r1;
          if (DT == kBF16) {
            split4_bf16(v[i].x, v[i].y, s0, r0);
            split4_bf16(v[i].z, v[i].w, s1, r1);
          } else {
            split4_f16(v[i].x, v[i].y, s0, r0);
            split4_f16(v[i].z, v[i].w, s1, r1);
          }
          *reinterpret_cast<uint2 *>(sym + e) = make_uint2(s0, s1);
          *reinterpret_cast<uint2 *>(out + g.off_res0 + b * B + e) = make_uint2(r0, r1);
        }
      }
      }
      __syncwarp();

      // ---- a4: 32 interleaved rANS lanes, rounds R-1 .. 0
      uint32_t x = kL;
      uint32_t wp = 0;                         // words emitted so far (warp-uniform)
      constexpr uint32_t kCap = B / 2 - 64;    // words that fit before the raw threshold
#pragma unroll 4
      for (int j = C::kRounds - 1; j >= 0; --j) {
        const uint32_t s = sym[j * 32 + lane];
        const uint4 e = tab[s];
        const bool p = (x | 0x7FFFFu) >= e.y;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, p);
        if (p) {
          const uint32_t idx = wp + __popc(m & lt);
          if (idx < kCap) blk16[64 + idx] = (uint16_t)x;
          x >>= 16;
        }
        wp += __popc(m);
        const uint32_t q = __funnelshift_r(__umulhi(x, e.x), 0u, e.y);
        x = x + e.z + q * e.w;
      }
      K = wp;
      const uint32_t coded = (uint32_t)round16(128 + 2ull * K);
      if (coded >= B) {
        size = B;                               // stored raw (R13)
      } else {
        size = coded;
        blk32[lane] = x;
        const uint32_t pad_words = (coded - 128 - 2 * K) / 2;
        if ((uint32_t)lane < pad_words) blk16[64 + K + lane] = 0;
      }
    }
    if (lane == 0) {
      s_size[warp] = size;
      s_k[warp] = (size == (uint32_t)B) ? kRawBlock : K;
    }
    __syncthreads();

    // ---- a5: tile prefix by decoupled look-back (one warp)
    if (warp == 0) {
      unsigned long long agg = lane < kWarps ? s_size[lane] : 0u;
      agg = warp_sum_u64(agg);
      const unsigned long long excl = lookback(ws.tile_status, t, agg);
      if (lane == 0) s_prefix = excl;
    }
    __syncthreads();

    if (b < g.n_blocks) {
      unsigned long long off = s_prefix;
      for (int w = 0; w < warp; ++w) off += s_size[w];
      if (lane == 0) {
        reinterpret_cast<uint32_t *>(out + g.off_dir)[b] = s_k[warp];
        if (b % g.CB == 0) reinterpret_cast<unsigned long long *>(out + g.off_coff)[b / g.CB] = off;
      }
      const uint4 *srcv = reinterpret_cast<const uint4 *>(size == (uint32_t)B ? sym : blk);
      uint4 *dstv = reinterpret_cast<uint4 *>(out + g.off_pay + off);
      for (uint32_t i = lane; i < size / 16; i += 32) dstv[i] = srcv[i];
    }
    if (t == n_tiles - 1 && warp == kWarps - 1) {
      unsigned long long total = s_prefix;
      for (int w = 0; w < kWarps; ++w) total += s_size[w];
      finalize_stream<DT>(in, g, out, total, d_out_bytes);
    }
    __syncthreads();
  }
}

// ================================================================ k_decode
struct DecShared {
  static constexpr int kTab = 4096 * 4;          // decode table
  static constexpr int kOff = 1024 * 4;          // per-segment block offsets (relative to chunk)
  static constexpr int kWarpBuf = 2 * kMaxB;     // payload + symbols
  static constexpr int kBytes = kTab + kOff + kWarps * kWarpBuf;
};

__device__ __forceinline__ void set_err(CodecWs &ws, uint32_t code) { atomicCAS(ws.err, 0u, code); }

// Directory entry -> payload bytes of the block; flags entries no encoder emits.
__device__ __forceinline__ uint32_t dec_block_size(uint32_t d, uint32_t B, bool &bad) {
  if (d == kRawBlock) return B;
  if (d >= B / 2) {
    bad = true;
    return B;
  }
  const uint32_t sz = (uint32_t)round16(128 + 2ull * d);
  if (sz >= B) bad = true;
  return sz;
}

// a8: one warp decodes block b (payload at `off` within the payload section)
// and joins it with the residual plane into `out`.
template <int DT>
__device__ void decode_block(const uint8_t *__restrict__ in, const StreamGeom &g, unsigned long long payload,
                             uint32_t d, uint64_t b, unsigned long long off, const uint32_t *dtab, uint8_t *pay,
                             uint8_t *symb, uint8_t *__restrict__ out, CodecWs &ws) {
  const int lane = threadIdx.x & 31;
  const uint32_t B = g.B;
  bool bad = false;
  const uint32_t size = dec_block_size(d, B, bad);
  if (bad || off + size > payload) {
    if (lane == 0) set_err(ws, UZIP_ERR_CORRUPT_STREAM);
    return;
  }
  const bool raw = d == kRawBlock;
  const uint4 *srcv = reinterpret_cast<const uint4 *>(in + g.off_pay + off);
  uint4 *dstv = reinterpret_cast<uint4 *>(pay);
  for (uint32_t i = lane; i < size / 16; i += 32) dstv[i] = srcv[i];
  __syncwarp();
  const uint8_t *syms = pay;
  if (!raw) {
    const uint32_t *pay32 = reinterpret_cast<const uint32_t *>(pay);
    const uint16_t *pay16 = reinterpret_cast<const uint16_t *>(pay);
    const uint32_t lt = lanemask_lt();
    const uint32_t R = B / 32;
    uint32_t x = pay32[lane];
    int32_t p = (int32_t)d;
    for (uint32_t j = 0; j < R; ++j) {
      const uint32_t e = dtab[x & (kM - 1)];
      symb[j * 32 + lane] = (uint8_t)e;
      x = (e >> 20) * (x >> kProbBits) + ((e >> 8) & 0xFFFu);
      const bool need = x < kL;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
      const int32_t k = __popc(m);
      if (k > p) {
        bad = true;
        break;
      }
      if (need) x = (x << 16) | pay16[64 + p - k + __popc(m & lt)];
      p -= k;
    }
    if (bad || p != 0 || __any_sync(0xFFFFFFFFu, x != kL)) {
      if (lane == 0) set_err(ws, UZIP_ERR_CORRUPT_STREAM);
      __syncwarp();
      return;
    }
    syms = symb;
  }
  __syncwarp();
  // join with the residual plane, 128-bit stores
  if (DT == kF32) {
    for (uint32_t e = lane * 4; e < B; e += 128) {
      const uint32_t s4 = *reinterpret_cast<const uint32_t *>(syms + e);
      const uint2 lo = ldg_nc_v2(in + g.off_res0 + 2 * (b * B + e));
      const uint32_t h4 = ldg_nc_u32(in + g.off_res1 + b * B + e);
      *reinterpret_cast<uint4 *>(out + 4 * (b * B + e)) = join4_f32(s4, lo, h4);
    }
  } else {
    for (uint32_t e = lane * 8; e < B; e += 256) {
      const uint2 s8 = *reinterpret_cast<const uint2 *>(syms + e);
      const uint2 r8 = ldg_nc_v2(in + g.off_res0 + b * B + e);
      uint4 o;
      if (DT == kBF16) {
        join4_bf16(s8.x, r8.x, o.x, o.y);
        join4_bf16(s8.y, r8.y, o.z, o.w);
      } else {
        join4_f16(s8.x, r8.x, o.x, o.y);
        join4_f16(s8.y, r8.y, o.z, o.w);
      }
      *reinterpret_cast<uint4 *>(out + 2 * (b * B + e)) = o;
    }
  }
  __syncwarp();
}

template <int DT>
__global__ void __launch_bounds__(256, 2) k_decode(const uint8_t *__restrict__ in, uint64_t in_bytes,
                                                  uint8_t *__restrict__ out, uint64_t n, CodecWs ws,
                                                  int32_t *__restrict__ d_status) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t *dtab = reinterpret_cast<uint32_t *>(smem);
  uint32_t *soff = reinterpret_cast<uint32_t *>(smem + DecShared::kTab);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t *pay = smem + DecShared::kTab + DecShared::kOff + warp * DecShared::kWarpBuf;
  uint8_t *symb = pay + kMaxB;

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
    else if (!(B == 1024 || B == 2048 || B == 4096) || CB == 0 || payload > in_bytes)
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
      const uint64_t c = s0 / g.CB;
      const uint64_t c_first = c * g.CB;
      const uint64_t c_end = min(nb, c_first + g.CB);
      const uint64_t chunk_stop = min(cb1, c_end);
      __syncthreads();
      if (tid == 0) s_bad = 0;
      // ---- a7: decode table of chunk c: f:12 <<20 | (slot-cdf):12 <<8 | sym:8
      const uint16_t *ft = reinterpret_cast<const uint16_t *>(in + g.off_tab + 512 * c);
      const uint32_t f = ft[tid];
      uint32_t incl = f;
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t tt = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += tt;
      }
      if (lane == 31) s_red[warp] = incl;
      __syncthreads();
      uint32_t woff = 0, fsum = 0;
      for (int w = 0; w < kWarps; ++w) {
        if (w < warp) woff += s_red[w];
        fsum += s_red[w];
      }
      const uint32_t cdf = woff + incl - f;
      if (fsum != kM) {
        set_err(ws, UZIP_ERR_CORRUPT_STREAM);
        break;  // uniform: every thread saw the same sum
      }
      if (f == 0) s_bad = 1;
      // thread tid owns symbol tid; the 32 lanes of a warp fill the slots of the
      // warp's 32 symbols one symbol at a time
      for (int k = 0; k < 32; ++k) {
        const uint32_t fk = __shfl_sync(0xFFFFFFFFu, f, k);
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, cdf, k);
        const uint32_t sk = (uint32_t)(warp * 32 + k);
        for (uint32_t t = lane; t < fk; t += 32) dtab[ck + t] = (fk << 20) | (t << 8) | sk;
      }
      // ---- chunk bookkeeping: bytes before s0 inside the chunk; the CTA that
      // owns the chunk's first block also checks chunk_off[c] + sum == next.
      {
        const bool owner = c_first >= cb0;
        const uint64_t scan_end = owner ? c_end : s0;
        unsigned long long before = 0, chunk_total = 0;
        for (uint64_t bb = c_first + tid; bb < scan_end; bb += 256) {
          bool bad = false;
          const uint32_t sz = dec_block_size(dir[bb], B, bad);
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
      for (uint64_t seg = s0; seg < chunk_stop; seg += 1024) {
        const uint64_t seg_end = min(chunk_stop, seg + 1024);
        const unsigned long long run0 = s_base;
        unsigned long long run = run0;
        for (uint64_t bb0 = seg; bb0 < seg_end; bb0 += 256) {
          const uint64_t bb = bb0 + tid;
          uint32_t sz = 0;
          if (bb < seg_end) {
            bool bad = false;
            sz = dec_block_size(dir[bb], B, bad);
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
          decode_block<DT>(in, g, payload, dir[b], b, off, dtab, pay, symb, out, ws);
        }
        __syncthreads();
        if (tid == 0) s_base = run;
        __syncthreads();
      }
      s0 = chunk_stop;
    }
    // raw tail
    if (blockIdx.x == 0) {
      const uint64_t tail_bytes = (g.n - g.n_coded) * g.eb;
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
int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename K>
int occupancy(K kernel, int threads, size_t smem) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
  return occ > 0 ? occ : 1;
}

template <int DT, int B>
cudaError_t launch_encode_t(const void *in, const StreamGeom &g, void *out, uint64_t *d_out_bytes, void *ws_ptr,
                            cudaStream_t st, int max_ctas) {
  CodecWs ws = CodecWs::carve(ws_ptr, g.n_chunks);
  if (g.n_chunks > 0) {
    uint32_t max_parts = 1;
    for (uint64_t c = 0; c < g.n_chunks; c += (g.n_chunks > 1 ? g.n_chunks - 1 : 1)) {
      uint32_t p = (g.sample_len(c) + kHistSymsPerCta - 1) / kHistSymsPerCta;
      max_parts = p > max_parts ? p : max_parts;
    }
    dim3 grid(max_parts, (unsigned)g.n_chunks);
    k_table<DT><<<grid, 256, 0, st>>>((const uint8_t *)in, g, (uint8_t *)out, ws);
  }
  using C = EncCfg<DT, B>;
  auto kern = k_encode<DT, B>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  const uint64_t nt = g.n_tiles();
  int grid = sm_count() * occupancy(kern, 256, C::kSmem);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if ((uint64_t)grid > nt) grid = (int)(nt ? nt : 1);
  kern<<<grid, 256, C::kSmem, st>>>((const uint8_t *)in, g, (uint8_t *)out, ws, d_out_bytes);
  return cudaGetLastError();
}

template <int DT>
cudaError_t launch_encode_dt(const void *in, const StreamGeom &g, void *out, uint64_t *d_out_bytes, void *ws,
                             cudaStream_t st, int max_ctas) {
  switch (g.B) {
    case 1024: return launch_encode_t<DT, 1024>(in, g, out, d_out_bytes, ws, st, max_ctas);
    case 2048: return launch_encode_t<DT, 2048>(in, g, out, d_out_bytes, ws, st, max_ctas);
    default: return launch_encode_t<DT, 4096>(in, g, out, d_out_bytes, ws, st, max_ctas);
  }
}

template <int DT>
cudaError_t launch_decode_t(const void *in, uint64_t in_bytes, void *out, uint64_t n, void *ws_ptr,
                            int32_t *d_status, cudaStream_t st, int max_ctas, uint64_t est_blocks) {
  CodecWs ws = CodecWs::carve(ws_ptr, 0);
  auto kern = k_decode<DT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DecShared::kBytes);
    attr = true;
  }
  int grid = sm_count() * occupancy(kern, 256, DecShared::kBytes);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  const uint64_t want = (est_blocks + 3) / 4;
  if ((uint64_t)grid > want) grid = (int)(want ? want : 1);
  kern<<<grid, 256, DecShared::kBytes, st>>>((const uint8_t *)in, in_bytes, (uint8_t *)out, n, ws, d_status);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_compress(int dtype, const void *in, const StreamGeom &g, void *out, uint64_t *d_out_bytes,
                            void *ws, cudaStream_t st, int max_ctas) {
  switch (dtype) {
    case kBF16: return launch_encode_dt<kBF16>(in, g, out, d_out_bytes, ws, st, max_ctas);
    case kF16: return launch_encode_dt<kF16>(in, g, out, d_out_bytes, ws, st, max_ctas);
    default: return launch_encode_dt<kF32>(in, g, out, d_out_bytes, ws, st, max_ctas);
  }
}

cudaError_t launch_decompress(int dtype, const void *in, uint64_t in_bytes, void *out, uint64_t n, void *ws,
                              int32_t *d_status, cudaStream_t st, int max_ctas) {
  const uint64_t est_blocks = n / 1024;
  switch (dtype) {
    case kBF16: return launch_decode_t<kBF16>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    case kF16: return launch_decode_t<kF16>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
    default: return launch_decode_t<kF32>(in, in_bytes, out, n, ws, d_status, st, max_ctas, est_blocks);
  }
}

}  // namespace uzip
