// fused_impl.cuh -- the Uzip hot path for sm_100a (templates; instantiated per
// dtype and variant in fused_<dtype>_<enc|red>.cu so nvcc runs in parallel): table build and ONE persistent
// kernel per launch that encodes, transfers, decodes and reduces.
//
//   k_hist   a2     sampled per-chunk partial histograms ("the first 256 KB"
//                   of each chunk), several CTAs per chunk.
//   k_norm   a3     rule-N1 frequencies (R5) -> encode reciprocals and the
//                   serialized table; one launch pair covers every stream.
//   k_fused  E items  a1+a4+a5+a6: split (the residual leaves for every
//                   destination as soon as it is split: split-send),
//                   warp-per-block 32-lane rANS,
//                   decoupled look-back so each block is stored once at its
//                   final offset (Step 3 removed), stores straight
//                   into the destinations' staging, tile flag
//                   release (a12).
//            C items  plain copies (own allgather shard).
//            D items  a7+a8(+a9): acquire a tile flag, decode (table-driven),
//                   join; with several sources, decode each and fold in rank
//                   order in fp32 before one rounding (R11).
//
// Stream bytes equal the CPU oracle's (tests/test_gpu_codec.py,
// tests/test_gpu_comm.py); layout in DESIGN.md section 2.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>

#include "codec_dev.cuh"
#include "plan.h"
#include "uzip_internal.h"

// Tuning knobs (defaults measured best on B200; overridable for experiments with -D)
#ifndef UZIP_ENC_PIPE
#define UZIP_ENC_PIPE 0  // A/B: rounds per software-pipelined load group (0: UZIP_ENC_GROUP groups, loaded in place)
#endif
#ifndef UZIP_ENC_GROUP
#define UZIP_ENC_GROUP 8  // encoder rounds whose symbols/table entries are loaded ahead (r02b: 8 beats 4, 0.668 vs 0.676 ms)
#endif
#ifndef UZIP_RED_MINB
#define UZIP_RED_MINB 2   // resident CTAs per SM targeted by reduce launches (r02: 2 without spills beats 3 with)
#endif
#ifndef UZIP_ENC_TMA
#define UZIP_ENC_TMA 0    // A/B: stage each block's input into smem with a TMA bulk copy before the split
#endif
#ifndef UZIP_RING_WIDE
#define UZIP_RING_WIDE 24576  // ring bytes of f16 / fp8 encode launches (bf16 / fp32 and reduce: 16 KiB)
#endif
#ifndef UZIP_ENC_IMADCMP
#define UZIP_ENC_IMADCMP 1  // the encoder's renormalization test as IMAD + sign test (0.701 -> 0.676 ms)
#endif
#ifndef UZIP_ENC_MINB
#define UZIP_ENC_MINB 3   // resident CTAs per SM targeted by launches with encode items (measured)
#endif
#ifndef UZIP_DEC_ONLY_MINB
#define UZIP_DEC_ONLY_MINB 4  // ... and by decode-only launches (P2P / broadcast receivers)
#endif

namespace uzip {

// ================================================================ a2: sampled histograms
// Part `part` of chunk c's sample ("the first 256 KB") histogrammed by all 256 threads with
// per-warp shared-memory atomics into hist (8 x 256 counters, zeroed here); the part's partial
// histogram is stored to J.partial[c][part].  Used by the T items of k_fused and by k_hist.
constexpr int kHistThreads = 256;
constexpr int kHistWarps = kHistThreads / 32;

template <int DT>
__device__ __forceinline__ void sample_hist(const EncJob &J, uint64_t c, uint32_t part, uint32_t *hist) {
  const StreamGeom &g = J.g;
  const int tid = threadIdx.x, warp = warp_id();
  const uint32_t len = g.sample_len(c), parts = hist_parts(len, g.global);
  for (int i = tid; i < kHistWarps * 256; i += kHistThreads) hist[i] = 0;
  __syncthreads();
  constexpr uint32_t kPer = VecTraits<DT>::kSym;  // symbols per 16-byte vector
  constexpr int kUnroll = 8;
  const uint8_t *base = J.in + c * g.CB * g.B * group_bytes(DT);
  const uint32_t nvec = len / kPer;
  const uint32_t per = (nvec + parts - 1) / parts;
  const uint32_t v_lo = part * per, v_hi = min(nvec, v_lo + per);
  uint32_t *h = hist + 256 * warp;
  for (uint32_t v0 = v_lo; v0 < v_hi; v0 += kHistThreads * kUnroll) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t v = v0 + u * kHistThreads + tid;
      w[u] = v < v_hi ? ldg_nc_v4(base + (size_t)v * 16) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const bool ok = v0 + u * kHistThreads + tid < v_hi;
      uint32_t sw[4];
      vec_symbols<DT>(w[u], sw);
      // plain per-warp shared atomics: B200 resolves same-address lanes in the atomic unit
      // faster than a __match_any_sync warp aggregation (measured k_hist 37 -> 10 us per GiB)
#pragma unroll
      for (int k = 0; k < (int)kPer; ++k) {
        const uint32_t sy = (sw[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        if (ok) atomicAdd(&h[sy], 1u);
      }
    }
  }
  if (part == parts - 1)
    for (uint32_t i = nvec * kPer + tid; i < len; i += kHistThreads)  // sample not a vector multiple
      atomicAdd(&h[symbol_at<DT>(base, i)], 1u);
  __syncthreads();
  uint32_t sum = 0;
#pragma unroll
  for (int w = 0; w < kHistWarps; ++w) sum += hist[256 * w + tid];
  J.partial[(c * hist_cap(g.global) + part) * 256 + tid] = sum;
}

// Sum of `parts` partial rows (all 256 threads; returns the count of symbol tid).  Warp w takes rows
// w, w + 8, ..., each lane 8 columns as two 16-byte loads, 8 rows in flight; scr: 8 x 256 u32 of smem.
__device__ __forceinline__ uint32_t sum_rows(const uint32_t *rows, uint32_t parts, uint32_t *scr) {
  const int lane = threadIdx.x & 31, warp = warp_id();
  uint32_t a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint32_t r0 = warp; r0 < parts; r0 += 8 * kWarps) {
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t r = r0 + u * kWarps;
      const uint4 *q = reinterpret_cast<const uint4 *>(rows + (uint64_t)r * 256 + 8 * lane);
      v[2 * u] = r < parts ? ld_cg_v4(q) : make_uint4(0, 0, 0, 0);
      v[2 * u + 1] = r < parts ? ld_cg_v4(q + 1) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[0] += v[2 * u].x, a[1] += v[2 * u].y, a[2] += v[2 * u].z, a[3] += v[2 * u].w;
      a[4] += v[2 * u + 1].x, a[5] += v[2 * u + 1].y, a[6] += v[2 * u + 1].z, a[7] += v[2 * u + 1].w;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) scr[warp * 256 + 8 * lane + k] = a[k];
  __syncthreads();
  uint32_t sum = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) sum += scr[w * 256 + threadIdx.x];
  __syncthreads();
  return sum;
}

// A/B path (UZIP_TABLE_KERNELS=1): the same table build as two launches ahead of k_fused.
// k_hist grid (parts, chunks, streams); k_norm grid (chunks, streams) publishes flag = epoch + 1.
template <int DT>
__global__ void __launch_bounds__(kHistThreads) k_hist(const __grid_constant__ Plan P) {
  __shared__ uint32_t hist[kHistWarps * 256];
  const EncJob &J = P.e[blockIdx.z];
  if (J.raw) return;
  const uint32_t part = blockIdx.x, c = blockIdx.y;
  if (c >= J.g.n_chunks || part >= hist_parts(J.g.sample_len(c), J.g.global)) return;
  sample_hist<DT>(J, c, part, hist);
}

// a3, all 256 threads of a CTA: thread s holds cnt = count of symbol s in the chunk's sample; rule
// N1 (R5) -> the chunk's encode entries (enc, global), its 512-byte serialized table (tab16, global)
// and, if `tab` is not null, the entries in shared memory too.  red64/red32: 8 words of smem scratch.
__device__ __forceinline__ void norm_tables(uint32_t cnt, uint4 *enc, uint16_t *tab16, uint4 *tab,
                                            unsigned long long *red64, uint32_t *red32) {
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  // ---- rule N1 (R5): total and argmax (lowest symbol on ties): key = cnt<<8 | (255 - s)
  unsigned long long key = ((unsigned long long)cnt << 8) | (255u - tid);
  unsigned long long tot = cnt;
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
  for (int w = 0; w < 8; ++w) {
    best_key = red64[w] > best_key ? red64[w] : best_key;
    total += red32[w];
  }
  const uint32_t best = 255u - (uint32_t)(best_key & 0xFFu);
  uint32_t f;
  if (total == 0) f = kM / 256;
  else f = 1u + (uint32_t)(((unsigned long long)cnt * (kM - 256)) / total);
  __syncthreads();
  uint32_t fs = f;
  for (int o = 16; o; o >>= 1) fs += __shfl_xor_sync(0xFFFFFFFFu, fs, o);
  if (lane == 0) red32[warp] = fs;
  __syncthreads();
  uint32_t fsum = 0;
  for (int w = 0; w < 8; ++w) fsum += red32[w];
  if (total != 0 && tid == (int)best) f += kM - fsum;
  __syncthreads();
  uint32_t incl = f;  // exclusive prefix (cdf) over 256 symbols
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) red32[warp] = incl;
  __syncthreads();
  uint32_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += red32[w];
  const uint32_t cdf = woff + incl - f;
  const uint4 ent = make_enc_entry(f, cdf);
  enc[tid] = ent;
  tab16[tid] = (uint16_t)f;
  if (tab) tab[tid] = ent;
  // red32 / red64 free again; tab complete.  The caller's thread 0 then fences and releases the
  // chunk's flag: bar.sync + one gpu-scope fence cover every thread's stores (the grid-sync pattern)
  __syncthreads();
}

template <int DT>
__global__ void __launch_bounds__(256) k_norm(const __grid_constant__ Plan P) {
  __shared__ unsigned long long red64[8];
  __shared__ uint32_t red32[8];
  __shared__ uint32_t scr[kWarps * 256];
  const EncJob &J = P.e[blockIdx.y];
  if (J.raw) return;
  const StreamGeom &g = J.g;
  const int tid = threadIdx.x;
  const uint32_t c = blockIdx.x;
  if (c >= g.n_chunks) return;
  const uint32_t parts = hist_parts(g.sample_len(c), g.global), cap = hist_cap(g.global);
  const uint32_t sum = sum_rows(J.partial + (uint64_t)c * cap * 256, parts, scr);
  norm_tables(sum, J.enc + c * 256, J.tab16 + c * 256, nullptr, red64, red32);
  if (tid == 0) {
    __threadfence();
    st_release_gpu_u64(J.tflag + c, kCtlTag | ((*P.epoch & kEpochMask) + 1u));
  }
}

// ================================================================ shared pieces
// Look-back word: flag (2 bits: 1 aggregate, 2 inclusive prefix) | launch epoch (24 bits) | value
// (38 bits: stream offsets < 256 GiB).  A word whose epoch is not this launch's is "not ready", so
// the words never need resetting between launches (a 2^24-launch wrap could only alias a tile word
// left untouched for exactly that many launches of the same workspace).
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr int kEpochShift = 38;
constexpr unsigned long long kValMask = (1ull << kEpochShift) - 1;
__device__ __forceinline__ unsigned long long ep_bits(uint32_t ep) {
  return (unsigned long long)(ep & kEpochMask) << kEpochShift;
}

__device__ __forceinline__ void raise_err(const Plan &P, uint32_t code) { atomicCAS(P.err, 0u, code); }
// First error only: the code plus where it happened (site, expected, seen) for uzip_comm_error_detail.
__device__ __forceinline__ void raise_err_at(const Plan &P, uint32_t code, uint32_t site, uint32_t expect,
                                             unsigned long long seen, uint64_t where) {
  if (atomicCAS(P.err, 0u, code) == 0u) {
    P.err[1] = site;
    P.err[2] = expect;
    P.err[3] = (uint32_t)(seen >> 32);
    P.err[4] = (uint32_t)seen;
    P.err[5] = (uint32_t)where;
    P.err[6] = blockIdx.x;
    __threadfence_system();
  }
}

// Tile trace (Plan::trace): one event, thread-level.
__device__ __forceinline__ void trace_ev(const Plan &P, uint32_t kind, uint32_t job, uint64_t tile) {
  if (!P.trace) return;
  const uint32_t i = atomicAdd(P.trace_n, 1u);
  if (i < P.trace_cap) {
    P.trace[2ull * i] = ((unsigned long long)kind << 60) | ((unsigned long long)(job & 15u) << 56) |
                        (tile & ((1ull << 56) - 1));
    P.trace[2ull * i + 1] = globaltimer_ns();
  }
}

// Debug stress (UZIP_STRESS=seed): a pseudo-random pause of up to ~16 us at the protocol's hand-off
// points, so the loopback tests exercise late flags, early credits and reordered tiles.
__device__ __forceinline__ void stress_pause(const Plan &P, uint64_t salt) {
  if (!P.stress) return;
  uint64_t h = (salt + P.stress) * 0x9E3779B97F4A7C15ull + blockIdx.x * 0xBF58476D1CE4E5B9ull;
  h ^= h >> 31;
  if ((h & 3) == 0) __nanosleep((unsigned)((h >> 8) & 0x3FFF));
}

// Poll a tile flag until its epoch matches (thread-level; bounded by the
// plan's timeout, aborts when another CTA raised an error).
static __device__ bool wait_flag(const Plan &P, const unsigned long long *f, uint32_t epoch, unsigned long long &v) {
  unsigned long long t0 = 0;
  for (int spin = 0;; ++spin) {
    v = ld_acquire_sys_u64(f);
    if ((uint32_t)(v >> 32) == epoch) return true;
    if ((spin & 63) == 63) {
      if (ld_volatile_u32(P.err)) return false;
      const unsigned long long now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > P.timeout_ns) {
        raise_err_at(P, UZIP_ERR_TIMEOUT, 1, epoch, v, (uint64_t)(uintptr_t)f);
        return false;
      }
    }
    __nanosleep(32);
  }
}

// Credit: the destination consumed epoch-2 from this slot (a12).
static __device__ bool wait_credit(const Plan &P, const unsigned long long *cr, uint32_t epoch) {
  if (!cr || epoch <= 2) return true;
  unsigned long long t0 = 0;
  for (int spin = 0;; ++spin) {
    if (ld_acquire_sys_u64(cr) >= (unsigned long long)(epoch - 2)) return true;
    if ((spin & 63) == 63) {
      if (ld_volatile_u32(P.err)) return false;
      const unsigned long long now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > P.timeout_ns) {
        raise_err_at(P, UZIP_ERR_TIMEOUT, 2, epoch, ld_acquire_sys_u64(cr), (uint64_t)(uintptr_t)cr);
        return false;
      }
    }
    __nanosleep(64);
  }
}

// Poll a 64-bit flag until it equals `want` (gpu scope: a flag of this launch on this GPU).
static __device__ bool wait_u64(const Plan &P, const unsigned long long *f, unsigned long long want,
                                unsigned long long &seen) {
  unsigned long long t0 = 0;
  for (int spin = 0;; ++spin) {
    const unsigned long long v = ld_acquire_gpu_u64(f);
    if (v == want) return true;
    if ((spin & 63) == 63) {
      if (ld_volatile_u32(P.err)) return false;
      const unsigned long long now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > P.timeout_ns) {
        seen = v;
        raise_err_at(P, UZIP_ERR_TIMEOUT, 5, (uint32_t)want, v, (uint64_t)(uintptr_t)f);
        return false;
      }
    }
    __nanosleep(32);
  }
}

// Decoupled look-back over the tiles of one stream, in two halves so the
// aggregate can be published as soon as a tile is coded and the scan finished
// later.  publish: one thread.  finish: one full warp; returns the exclusive
// prefix of tile t, or ~0 on abort.
__device__ __forceinline__ void lookback_publish(unsigned long long *status, uint64_t t, unsigned long long agg,
                                                 uint32_t ep) {
  st_relaxed_u64(&status[t], (t == 0 ? kFlagInc : kFlagAgg) | ep_bits(ep) | agg);
}

static __device__ unsigned long long lookback_finish(const Plan &P, unsigned long long *status, uint64_t t,
                                              unsigned long long agg, uint32_t ep) {
  const int lane = threadIdx.x & 31;
  if (t == 0) return 0;
  unsigned long long excl = 0, t0 = 0;
  int64_t base = (int64_t)t - 1;
  const unsigned long long eb = ep_bits(ep), emask = (unsigned long long)kEpochMask << kEpochShift;
  for (int spin = 0;; ++spin) {
    const int64_t idx = base - lane;
    unsigned long long s = idx >= 0 ? ld_relaxed_u64(&status[idx]) : (kFlagInc | eb);
    uint32_t flag = (s & emask) == eb ? (uint32_t)(s >> 62) : 0u;  // another launch's word: not ready
    flag = flag == 3 ? 0u : flag;                                    // a control word (kCtlTag): not ready
    const uint32_t inc = __ballot_sync(0xFFFFFFFFu, flag == 2);
    const uint32_t notready = __ballot_sync(0xFFFFFFFFu, flag == 0);
    const int first_inc = inc ? __ffs(inc) - 1 : 31;
    const uint32_t needed = first_inc == 31 ? 0xFFFFFFFFu : ((2u << first_inc) - 1u);
    if (notready & needed) {
      if ((spin & 255) == 255) {
        bool stop = false;
        if (lane == 0) {
          const unsigned long long now = globaltimer_ns();
          if (ld_volatile_u32(P.err)) stop = true;
          else if (t0 == 0) t0 = now;
          else if (now - t0 > P.timeout_ns) {
            raise_err_at(P, UZIP_ERR_TIMEOUT, 3, (uint32_t)t, s, (uint64_t)(uintptr_t)status);
            stop = true;
          }
        }
        if (__shfl_sync(0xFFFFFFFFu, stop, 0)) return ~0ull;
      }
      __nanosleep(32);
      continue;
    }
    excl += warp_sum_u64(lane <= first_inc ? (s & kValMask) : 0ull);
    if (inc) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(&status[t], kFlagInc | eb | (excl + agg));
  return excl;
}

static __device__ unsigned long long lookback(const Plan &P, unsigned long long *status, uint64_t t,
                                       unsigned long long agg, uint32_t ep) {
  if ((threadIdx.x & 31) == 0) lookback_publish(status, t, agg, ep);
  return lookback_finish(P, status, t, agg, ep);
}

// ---------------------------------------------------------------- fp32 fold helpers (a9, R11)
template <int DT>
__device__ __forceinline__ float widen(uint32_t bits) {
  if (DT == kBF16) return __uint_as_float(bits << 16);
  if (DT == kF16) return __half2float(__ushort_as_half((unsigned short)bits));
  return __uint_as_float(bits);
}
template <int DT>
__device__ __forceinline__ uint32_t narrow(float v) {
  if (v != v) return DT == kF32 ? 0x7FFFFFFFu : 0x7FFFu;  // canonical NaN
  if (DT == kBF16) return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
  if (DT == kF16) return (uint32_t)__half_as_ushort(__float2half_rn(v));
  return __float_as_uint(v);
}
// One fold step of R (rank order): op 0 = fp32 sum without FMA contraction (R11); 1 / 2 = IEEE
// 754-2019 minimum / maximum (R25: NaN propagates, -0 < +0; canonicalised by narrow()).
__device__ __forceinline__ float fold(float acc, float x, bool first, uint32_t op) {
  if (first) return x;
  if (op == 0) return __fadd_rn(acc, x);
  if (acc != acc || x != x) return __int_as_float(0x7FFFFFFF);
  const bool sx = signbit(x), sa = signbit(acc);
  if (op == 1) return (x < acc || (x == acc && sx && !sa)) ? x : acc;
  return (x > acc || (x == acc && !sx && sa)) ? x : acc;
}

// Fold 16 bytes of elements into acc[0..kPer) (kPer = 8 for 2-byte types, 4 for fp32).
template <int DT>
__device__ __forceinline__ void fold_vec(float *acc, uint4 v, bool first, uint32_t op) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if (DT == kF32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = fold(acc[i], widen<DT>(w[i]), first, op);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] = fold(acc[2 * i], widen<DT>(w[i] & 0xFFFFu), first, op);
      acc[2 * i + 1] = fold(acc[2 * i + 1], widen<DT>(w[i] >> 16), first, op);
    }
  }
}
template <int DT>
__device__ __forceinline__ uint4 narrow_vec(const float *acc) {
  uint4 o;
  uint32_t *w = &o.x;
  if (DT == kF32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = narrow<DT>(acc[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = narrow<DT>(acc[2 * i]) | (narrow<DT>(acc[2 * i + 1]) << 16);
  }
  return o;
}

// ================================================================ k_fused
template <int DT, int B>
struct FusedCfg {
  static constexpr int kVec = VecTraits<DT>::kSym;          // symbols per 16-byte load
  static constexpr int kIters = B / (32 * kVec);            // loads per lane per block
#ifndef UZIP_SPLIT_BATCH
#define UZIP_SPLIT_BATCH 8
#endif
  static constexpr int kBatch = kIters < UZIP_SPLIT_BATCH ? kIters : UZIP_SPLIT_BATCH;  // 16-byte loads in flight per lane
  static constexpr int kRounds = B / 32;
  static constexpr int kEncTab = 4096;                      // 256 x uint4
  static constexpr int kWarpBuf = B + 256;                  // per warp: symbols/words (E) or payload + ring (D)
  static constexpr int kDecTab = 4096 * 4;
  static constexpr int kAcc = 4 * B;                        // fp32 accumulator per warp (reduce; in P.acc)
  // coded tile awaiting its offset: 16 KiB hold a bf16 / fp32 tile (8-bit exponents, ~1.5 KB per coded
  // block); f16 and fp8 symbols carry more bits (~2.3-2.8 KB per block on U[-1,1]), so their encode
  // launches park up to 24 KiB -- a tile larger than the ring finishes its look-back before it is stored
  static constexpr int ring(bool red) {
    return red ? 16384
               : B > 4096 ? 3 * B  // 8192 / 16384-symbol blocks: a coded bf16 tile is ~2.9 / 5.6 KB per block
               : (DT == kF16 || DT == kE4M3 || DT == kE5M2) ? UZIP_RING_WIDE : 16384;
  }
  static constexpr int kTmaStage = UZIP_ENC_TMA ? B * (int)group_bytes(DT) : 0;  // per warp (A/B only)
  static constexpr int smem(bool dec, bool red) {
    return kEncTab + kWarps * kWarpBuf + ring(red) + (dec ? kDecTab : 0) + kWarps * kTmaStage;
  }
};

struct FusedShared {
  uint32_t tk[2];
  uint32_t abort;
  uint32_t tile_cnt;
  unsigned long long tile_off;
  uint32_t size[kWarps], k[kWarps], ovf[kWarps];
  uint32_t psize[kWarps], pkdir[kWarps];  // the pending (coded, offset unknown) tile
  unsigned long long pagg, ptile_off;
  unsigned long long prefix;
  unsigned long long src_off[kMaxRanks];
  unsigned long long src_payload[kMaxRanks];
  uint32_t red[kWarps];
  unsigned long long red64[kWarps];
  uint32_t epoch;  // this launch's epoch (Plan::epoch)
  uint32_t is_last;
  // abort words of the other wait sites: each site has its own, so a warp still reading one site's
  // outcome never sees the next site's write (compute-sanitizer racecheck)
  uint32_t ab_credit, ab_table;
  unsigned long long tma_bar[kWarps];  // A/B (UZIP_ENC_TMA): one mbarrier per warp
  uint32_t tma_phase[kWarps];
};

// ---------------------------------------------------------------- E item
// Header (sizes before/after), zero pads and raw tail of a stream; one warp.
template <int DT>
static __device__ void finalize_stream(const EncJob &J, unsigned long long payload) {
  const int lane = threadIdx.x & 31;
  const StreamGeom &g = J.g;
  const uint64_t total = g.total(payload);
  if (lane == 0) {
    uint32_t h[16];
    for (int i = 0; i < 16; ++i) h[i] = 0;
    h[0] = 0x31425A55u;  // "UZB1"
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
    for (uint32_t d = 0; d < J.nd; ++d) {
      uint4 *o = reinterpret_cast<uint4 *>(J.dst[d]);
      for (int i = 0; i < 4; ++i) o[i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    }
    if (J.d_out_bytes) *J.d_out_bytes = total;
    if (J.wire_acc) atomicAdd(J.wire_acc, (unsigned long long)total * J.nd);
  }
  const uint64_t e1 = g.off_coff + 8 * g.n_chunks, e2 = g.off_dir + 4 * g.n_blocks;
  const uint64_t tail_bytes = g.tail_bytes();
  const uint8_t *tsrc = J.in + g.n_coded * g.eb;
  for (uint32_t d = 0; d < J.nd; ++d) {
    uint8_t *o = J.dst[d];
    for (uint64_t p = e1 + lane; p < g.off_dir; p += 32) o[p] = 0;
    for (uint64_t p = e2 + lane; p < g.off_pay; p += 32) o[p] = 0;
    uint8_t *tdst = o + g.off_tail(payload);
    for (uint64_t i = lane; i < tail_bytes; i += 32) tdst[i] = tsrc[i];
  }
}

// a1: split block b.  REV: symbol rows in coding order (row of round j at
// (R-1-j)*32, lanes in order within a row) for the encoder; otherwise element
// order (the stored-raw payload).  RES: also store the residual plane(s) to
// every destination (split-send: they leave before the exponents are coded).
template <int DT, int B, bool RES, bool REV, bool ND1, bool COH = false, bool SMEM = false>
__device__ __forceinline__ void split_block_t(const EncJob &J, const StreamGeom &g, uint64_t b, const uint8_t *src,
                                              uint8_t *buf) {
  using C = FusedCfg<DT, B>;
  const int lane = threadIdx.x & 31;
  // ND1: one destination (codec, P2P): the residual bases are computed once
  uint8_t *r0 = J.dst[0] + g.off_res0 + (DT == kF32 ? 2 : 1) * (b * B);
  uint8_t *r1 = J.dst[0] + g.off_res1 + b * B;
  // byte of the lane's first vector in buf; later vectors of the lane step by kVec*32 elements (one row
  // group), backwards in coding order (REV) -- an immediate offset in the store
  const uint32_t e0 = (uint32_t)lane * C::kVec;
  uint8_t *pos0 = buf + (REV ? (uint32_t)(B - 32) - (e0 & ~31u) + (e0 & 31u) : e0);
#pragma unroll
  for (int h = 0; h < C::kIters; h += C::kBatch) {
    uint4 v[C::kBatch];
#pragma unroll
    for (int i = 0; i < C::kBatch; ++i)
      v[i] = SMEM  ? *reinterpret_cast<const uint4 *>(src + (size_t)(lane + 32 * (h + i)) * 16)  // TMA-staged
             : COH ? ld_cg_v4(src + (size_t)(lane + 32 * (h + i)) * 16)   // written earlier in this launch
                   : ldg_nc_v4(src + (size_t)(lane + 32 * (h + i)) * 16);
#pragma unroll
    for (int i = 0; i < C::kBatch; ++i) {
      const uint32_t e = (uint32_t)(lane + 32 * (h + i)) * C::kVec;  // element within block
      uint8_t *sp = REV ? pos0 - 32 * C::kVec * (h + i) : pos0 + 32 * C::kVec * (h + i);
      if (DT == kF32) {
        uint32_t s4, h4;
        uint2 lo;
        split4_f32(v[i], s4, lo, h4);
        *reinterpret_cast<uint32_t *>(sp) = s4;
        if (RES) {
          if (ND1) {
            *reinterpret_cast<uint2 *>(r0 + 2 * e) = lo;
            *reinterpret_cast<uint32_t *>(r1 + e) = h4;
          } else {
            for (uint32_t d = 0; d < J.nd; ++d) {
              *reinterpret_cast<uint2 *>(J.dst[d] + g.off_res0 + 2 * (b * B + e)) = lo;
              *reinterpret_cast<uint32_t *>(J.dst[d] + g.off_res1 + b * B + e) = h4;
            }
          }
        }
      } else if (DT == kE5M2) {  // R24: the bytes are the symbols, no residual plane
        *reinterpret_cast<uint4 *>(sp) = v[i];
      } else {
        uint32_t s0, s1, q0, q1;
        if (DT == kBF16) {
          split4_bf16(v[i].x, v[i].y, s0, q0);
          split4_bf16(v[i].z, v[i].w, s1, q1);
        } else if (DT == kE4M3) {
          split4_e4m3(v[i].x, v[i].y, s0, q0);
          split4_e4m3(v[i].z, v[i].w, s1, q1);
        } else {
          split4_f16(v[i].x, v[i].y, s0, q0);
          split4_f16(v[i].z, v[i].w, s1, q1);
        }
        *reinterpret_cast<uint2 *>(sp) = make_uint2(s0, s1);
        if (RES) {
          if (ND1) {
            *reinterpret_cast<uint2 *>(r0 + e) = make_uint2(q0, q1);
          } else {
            for (uint32_t d = 0; d < J.nd; ++d)
              *reinterpret_cast<uint2 *>(J.dst[d] + g.off_res0 + b * B + e) = make_uint2(q0, q1);
          }
        }
      }
    }
  }
}

template <int DT, int B, bool RES, bool REV, bool COH = false, bool SMEM = false>
__device__ __forceinline__ void split_block(const EncJob &J, const StreamGeom &g, uint64_t b, const uint8_t *src,
                                            uint8_t *buf) {
  if (!RES || J.nd == 1) split_block_t<DT, B, RES, REV, true, COH, SMEM>(J, g, b, src, buf);
  else split_block_t<DT, B, RES, REV, false, COH, SMEM>(J, g, b, src, buf);
}

// A/B (UZIP_ENC_TMA): one TMA bulk copy (cp.async.bulk, mbarrier completion) moves the warp's whole
// input block into its smem stage; the split then reads shared memory instead of issuing LDG.128s.
__device__ __forceinline__ void tma_stage_block(const uint8_t *src, uint8_t *stage, uint32_t bytes,
                                                unsigned long long *bar, uint32_t *phase) {
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(bar), sdst = (uint32_t)__cvta_generic_to_shared(stage);
  if ((threadIdx.x & 31) == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sdst), "l"(src), "r"(bytes), "r"(sbar) : "memory");
  }
  const uint32_t ph = *phase;
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(sbar), "r"(ph) : "memory");
  __syncwarp();
  if ((threadIdx.x & 31) == 0) *phase = ph ^ 1u;
}

// a1 for one 16-byte vector of block b that is already in registers (the reduced output of the fused
// allreduce, a9): its symbols go to the encoder's row layout in buf (coding order, as split_block
// with REV), its residual bytes to every destination's residual plane(s).  e = first element.
template <int DT, int B>
__device__ __forceinline__ void split_vec(const EncJob &J, const StreamGeom &g, uint64_t b, uint32_t e, uint4 v,
                                          uint8_t *buf) {
  static_assert(DT == kBF16 || DT == kF16 || DT == kF32, "reduced dtypes (R22)");
  uint8_t *sp = buf + (uint32_t)(B - 32) - (e & ~31u) + (e & 31u);
  if (DT == kF32) {
    uint32_t s4, h4;
    uint2 lo;
    split4_f32(v, s4, lo, h4);
    *reinterpret_cast<uint32_t *>(sp) = s4;
    for (uint32_t d = 0; d < J.nd; ++d) {
      *reinterpret_cast<uint2 *>(J.dst[d] + g.off_res0 + 2 * (b * B + e)) = lo;
      *reinterpret_cast<uint32_t *>(J.dst[d] + g.off_res1 + b * B + e) = h4;
    }
  } else {
    uint32_t s0, s1, q0, q1;
    if (DT == kBF16) {
      split4_bf16(v.x, v.y, s0, q0);
      split4_bf16(v.z, v.w, s1, q1);
    } else {
      split4_f16(v.x, v.y, s0, q0);
      split4_f16(v.z, v.w, s1, q1);
    }
    *reinterpret_cast<uint2 *>(sp) = make_uint2(s0, s1);
    for (uint32_t d = 0; d < J.nd; ++d)
      *reinterpret_cast<uint2 *>(J.dst[d] + g.off_res0 + b * B + e) = make_uint2(q0, q1);
  }
}

// a4: 32 interleaved rANS lanes, rounds R-1 .. 0 (branch-free body); the
// symbols and table entries of 8 rounds are loaded ahead of their math.
// Words are compacted (ballot + popc) into emission order.  GLOBAL = false:
// words go to buf, behind the rows already read (limit 16 words per consumed
// row); a word that would overtake them sets `ovf` and is dropped.  GLOBAL =
// true (rare path): words go straight to every destination at payload offset
// `off` + 128.
template <int DT, int B, bool GLOBAL>
__device__ __forceinline__ void encode_block(const EncJob &J, const StreamGeom &g, unsigned long long off,
                                             uint8_t *buf, const uint4 *tab, uint32_t &x_out, uint32_t &K,
                                             bool &ovf) {
  using C = FusedCfg<DT, B>;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  uint16_t *buf16 = reinterpret_cast<uint16_t *>(buf);
  uint32_t x = kL, wp = 0;
  bool over = false;
  // Deferred word store (buf path): round u's word is stored during round u+1, so the store's
  // index (ballot -> popc) and its data register have a round of slack -- stored in place, the
  // store waited on the popc and the shift of x waited for the store to read x (ncu: the two
  // largest short_scoreboard stalls of the round loop).
  // Every lane stores every round: a lane without a word writes to its own spare slot past the
  // B-byte buffer (words B/2 + lane, inside the warp's B + 256 bytes), so the store needs no
  // predicate carried into the next round.
  const uint32_t spare = (uint32_t)B / 2 + (uint32_t)lane;
  uint32_t dw = 0, didx = spare;
  constexpr uint32_t kCap = B / 2 - 64;  // words that fit before the raw threshold
#if UZIP_ENC_PIPE
  if (!GLOBAL) {
    // software-pipelined groups of kH rounds: the next group's symbols and table entries are loaded
    // while this group codes (two register sets of kH entries), so the symbol -> entry load chain is
    // off the state chain except for the first group.  Words stay below the end of the coding group's
    // rows (lim), so the prefetched rows are never overwritten before they are read.
    constexpr int kH = UZIP_ENC_PIPE;
    constexpr int kNH = C::kRounds / kH;
    static_assert(kNH % 2 == 0, "pipelined encoder: an even number of groups");
    uint4 ea[kH], eb[kH];
    auto load = [&](uint4 *e, int h) {
#pragma unroll
      for (int u = 0; u < kH; ++u) e[u] = tab[buf[(kH * h + u) * 32 + lane]];
    };
    auto code = [&](const uint4 *ent, int h) {
      const uint32_t lim = min(kCap, (uint32_t)(16 * kH) * (h + 1));
#pragma unroll
      for (int u = 0; u < kH; ++u) {
        const uint4 e = ent[u];
        const uint32_t tt = x + e.w * (1u << 19);
        uint32_t m, nidx;
        buf16[didx] = (uint16_t)dw;
        dw = x;
        asm("{\n\t.reg .pred q;\n\t.reg .b32 r, c;\n\t"
            "setp.lt.s32 q, %3, 0;\n\t"
            "vote.sync.ballot.b32 %0, q, -1;\n\t"
            "and.b32 r, %0, %4;\n\t"
            "popc.b32 c, r;\n\t"
            "add.u32 r, %5, c;\n\t"
            "min.u32 r, r, %6;\n\t"
            "selp.b32 %1, r, %7, q;\n\t"
            "@q shr.b32 %2, %2, 16;\n\t}"
            : "=r"(m), "=r"(nidx), "+r"(x)
            : "r"(tt), "r"(lt), "r"(wp), "r"(lim - 1), "r"(spare));
        didx = nidx;
        wp += __popc(m);
        const uint32_t q = __funnelshift_r(__umulhi(x, e.x), 0u, e.y);
        x = x + e.z + q * e.w;
      }
      over |= wp > lim;
    };
    load(ea, 0);
#pragma unroll 1
    for (int h = 0; h < kNH; h += 2) {
      __syncwarp();  // every lane read rows h, h+1 before words may land in them
      load(eb, h + 1);
      code(ea, h);
      __syncwarp();
      if (h + 2 < kNH) load(ea, h + 2);
      code(eb, h + 1);
    }
    buf16[didx] = (uint16_t)dw;
    x_out = x;
    K = wp;
    ovf = over;
    return;
  }
#endif
  constexpr int kG = UZIP_ENC_GROUP;
#pragma unroll 1
  for (int G = 0; G < C::kRounds / kG; ++G) {
    uint4 ent[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) ent[u] = tab[buf[(kG * G + u) * 32 + lane]];
    __syncwarp();  // every lane read these rows before words may land in them
    const uint32_t lim = GLOBAL ? kCap : min(kCap, (uint32_t)(16 * kG) * (G + 1));
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const uint4 e = ent[u];
#if UZIP_ENC_IMADCMP
      if (!GLOBAL) {
        // x >= f << 19  <=>  x + (M - f) << 19 >= 2^31 (no overflow: both terms < 2^31): one IMAD on the
        // FMA pipe and a sign test instead of two ALU ops; the predicate drives the ballot, the word
        // slot select and a predicated shift in one PTX block (so it stays a predicate)
        const uint32_t tt = x + e.w * (1u << 19);
        uint32_t m, nidx;
        buf16[didx] = (uint16_t)dw;
        dw = x;
        asm("{\n\t.reg .pred q;\n\t.reg .b32 r, c;\n\t"
            "setp.lt.s32 q, %3, 0;\n\t"
            "vote.sync.ballot.b32 %0, q, -1;\n\t"
            "and.b32 r, %0, %4;\n\t"
            "popc.b32 c, r;\n\t"
            "add.u32 r, %5, c;\n\t"
            "min.u32 r, r, %6;\n\t"
            "selp.b32 %1, r, %7, q;\n\t"
            "@q shr.b32 %2, %2, 16;\n\t}"
            : "=r"(m), "=r"(nidx), "+r"(x)
            : "r"(tt), "r"(lt), "r"(wp), "r"(lim - 1), "r"(spare));
        didx = nidx;
        wp += __popc(m);
        const uint32_t q = UZIP_ENC_MULQ ? __umulhi(__umulhi(x, e.x), e.y) : __funnelshift_r(__umulhi(x, e.x), 0u, e.y);
        x = x + e.z + q * e.w;
        continue;
      }
#endif
      const bool p = UZIP_ENC_MULQ ? (int32_t)(x + e.w * (1u << 19)) < 0 : (x | 0x7FFFFu) >= e.y;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, p);
      const uint32_t idx = min(wp + __popc(m & lt), lim - 1);  // clamped words are never used
      if (GLOBAL) {
        if (p && idx + 1 < kCap)
          for (uint32_t d = 0; d < J.nd; ++d)
            *reinterpret_cast<uint16_t *>(J.dst[d] + g.off_pay + off + 128 + 2 * idx) = (uint16_t)x;
        x = p ? (x >> 16) : x;
      } else {
        buf16[didx] = (uint16_t)dw;
        dw = x, didx = p ? idx : spare;
        x = p ? (x >> 16) : x;  // (an inline-PTX predicated shift instead of the select: no change, 0.704 ms)
      }
      wp += __popc(m);
      const uint32_t q = UZIP_ENC_MULQ ? __umulhi(__umulhi(x, e.x), e.y) : __funnelshift_r(__umulhi(x, e.x), 0u, e.y);
      x = x + e.z + q * e.w;
    }
    over |= wp > lim;
  }
  if (!GLOBAL) buf16[didx] = (uint16_t)dw;
  x_out = x;
  K = wp;
  ovf = over;
}

// Exclusive prefix (roff) of the 8 per-warp block sizes of a tile at this warp, its own size and the
// tile's total: one shared load per lane and a 3-step shuffle scan instead of a loop over the warps.
__device__ __forceinline__ void tile_prefix(const uint32_t *sizes, int warp, uint32_t &roff, uint32_t &mine,
                                            uint32_t *total = nullptr) {
  const int lane = threadIdx.x & 31;
  const uint32_t v = lane < kWarps ? sizes[lane] : 0u;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  roff = __shfl_sync(0xFFFFFFFFu, incl - v, warp);
  mine = __shfl_sync(0xFFFFFFFFu, v, warp);
  if (total) *total = __shfl_sync(0xFFFFFFFFu, incl, kWarps - 1);
}

// A coded tile whose payload waits in the CTA's ring for its offset: the
// tile's aggregate is published as soon as it is coded, the look-back is
// finished one tile later (when every predecessor has long been coded), so
// warps never idle on stragglers.  Uniform across the CTA.
struct EncPending {
  int32_t job;  // -1: none
  uint64_t t;
};

template <int DT, int B>
static __device__ void resolve_pending(const Plan &P, FusedShared &S, const uint8_t *ring, EncPending &pd) {
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const int jidx = pd.job;
  const EncJob &J = P.e[jidx];
  const StreamGeom &g = J.g;
  const uint64_t t = pd.t;
  pd.job = -1;
  // warp 0 finishes the look-back, the other warps wait at the barrier (a CTA-wide walk, 256 words per
  // step, was measured slower: 0.746 vs 0.702 ms/GiB -- its per-step barriers cost every warp)
  if (warp == 0) {
    const unsigned long long excl = lookback_finish(P, J.tile_status, t, S.pagg, S.epoch);
    if (lane == 0) S.ptile_off = excl;
  }
  __syncthreads();
  const unsigned long long tile_off = S.ptile_off;
  if (tile_off != ~0ull) {
    const uint64_t b0 = t * kTileBlocks, b = b0 + warp;
    const uint64_t c = chunk_of(g, b0);
    uint32_t roff, size;
    tile_prefix(S.psize, warp, roff, size);
    if (b < g.n_blocks) {
      const unsigned long long off = tile_off + roff;
      for (uint32_t d = 0; d < J.nd; ++d) {
        if (lane == 0) {
          reinterpret_cast<uint32_t *>(J.dst[d] + g.off_dir)[b] = S.pkdir[warp];
          if ((uint32_t)b % g.CB == 0) reinterpret_cast<unsigned long long *>(J.dst[d] + g.off_coff)[chunk_of(g, b)] = off;
        }
        uint4 *o = reinterpret_cast<uint4 *>(J.dst[d] + g.off_pay + off);
        for (uint32_t i = lane; i < size / 16; i += 32) o[i] = reinterpret_cast<const uint4 *>(ring + roff)[i];
      }
      if (b == g.n_blocks - 1) finalize_stream<DT>(J, off + size);
    }
    if ((uint32_t)b0 % g.CB == 0 && warp == kWarps - 1) {  // the chunk's first tile carries its table
      const uint4 v = reinterpret_cast<const uint4 *>(J.tab16 + c * 256)[lane];
      for (uint32_t d = 0; d < J.nd; ++d) reinterpret_cast<uint4 *>(J.dst[d] + g.off_tab + 512ull * c)[lane] = v;
    }
    const bool flags = J.has_flags != 0;
    if (flags) {
      __syncwarp();
      if (lane == 0) {
        // every warp fences its own stores at system scope before counting in (a CTA-scope fence
        // + one system fence by the last warp was measured to lose tiles in the loopback bench)
        __threadfence_system();
        if (atomicAdd(&S.tile_cnt, 1u) == kWarps - 1) {
          S.tile_cnt = 0;
          const unsigned long long off16 = tile_off >> 4;
          for (uint32_t d = 0; d < J.nd; ++d)
            if (J.flag[d]) {
            stress_pause(P, t * 7 + d);
            st_release_sys_u64(J.flag[d] + t, ((unsigned long long)J.epoch[d] << 32) | off16);
          }
          trace_ev(P, kTrEFlag, (uint32_t)jidx, t);
        }
      }
    }
  }
  __syncthreads();  // the ring and the pending sizes are free again
}

// T item (a2 + a3 inside the fused kernel): part `part` of chunk c's sample is
// histogrammed into J.partial; the last part of the chunk to finish (epoch-tagged counter, so
// nothing is reset between launches) sums the partials, applies rule N1 and publishes the chunk's
// encode entries, serialized table and flag = epoch + 1.  E items of the chunk wait for the flag.
template <int DT, int B>
static __device__ void t_item(const Plan &P, const EncJob &J, uint64_t c, uint32_t part, uint8_t *smem,
                              FusedShared &S) {
  using C = FusedCfg<DT, B>;
  const int tid = threadIdx.x;
  uint32_t *hist = reinterpret_cast<uint32_t *>(smem + C::kEncTab);  // the warp buffers (free between items)
  sample_hist<DT>(J, c, part, hist);
  const uint32_t parts = hist_parts(J.g.sample_len(c), J.g.global), cap = hist_cap(J.g.global), ep = S.epoch;
  __syncthreads();
  if (tid == 0) {
    __threadfence();  // after the barrier: every thread's partial row is visible before it is counted
    const unsigned long long tag = kCtlTag | ((unsigned long long)ep << 32);
    unsigned long long old = ld_volatile_u64(J.tcount + c), want;  // tag | parts counted (L2, not L1)
    for (;;) {
      want = (old & ~0xFFFFFFFFull) == tag ? old + 1ull : (tag | 1ull);  // the first part of a launch restarts
      const unsigned long long seen = atomicCAS(J.tcount + c, old, want);
      if (seen == old) break;
      old = seen;
    }
    S.is_last = (uint32_t)want == parts ? 1u : 0u;
    __threadfence();
  }
  __syncthreads();
  if (!S.is_last) return;
#ifdef UZIP_SIMPLE_SUM
  uint32_t sum = 0;
  for (uint32_t p = 0; p < parts; ++p) sum += ld_cg_u32(J.partial + (c * cap + p) * 256 + tid);
#else
  const uint32_t sum = sum_rows(J.partial + c * cap * 256, parts, hist);
#endif
  norm_tables(sum, J.enc + c * 256, J.tab16 + c * 256, nullptr, S.red64, S.red);
  if (tid == 0) {
    __threadfence();
    st_release_gpu_u64(J.tflag + c, kCtlTag | (ep + 1u));
  }
}

// The destinations' slots of encode job jidx are free (a12): the first tile of the job in this CTA
// waits for their credits (or for k_credit, which waited already).  CTA-uniform; false = abort.
static __device__ bool credit_gate(const Plan &P, const EncJob &J, int jidx, uint32_t &credit_done, FusedShared &S) {
  if ((credit_done >> jidx) & 1u) return true;
  if (threadIdx.x == 0) {
    uint32_t ok = 1;
    if (P.credit_ready) ok = ld_volatile_u32(P.err) == 0;  // k_credit waited (or failed)
    else
      for (uint32_t d = 0; d < J.nd && ok; ++d) ok = wait_credit(P, J.credit[d], J.epoch[d]);
    S.ab_credit = ok ? 0u : 1u;
  }
  __syncthreads();
  if (S.ab_credit) return false;
  credit_done |= 1u << jidx;
  return true;
}

// a4-a6 for one tile whose blocks are split (symbols in each warp's buffer, residual stored): code
// every block (one warp each), park the coded tile or find its offset by look-back, store it to every
// destination, release the tile flags.  `src` is the tile's input, re-read for stored-raw blocks and
// the rare overflow path (COH: written earlier in this launch -- the fused allreduce's reduced shard).
template <int DT, int B, bool COH>
static __device__ void code_tile(const Plan &P, const EncJob &J, int jidx, uint64_t t, uint8_t *smem,
                                 FusedShared &S, uint8_t *ring, int ring_bytes, EncPending &pd, const uint8_t *in) {
  using C = FusedCfg<DT, B>;
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const bool flags = J.has_flags != 0;
  const StreamGeom &g = J.g;
  const uint4 *tab = reinterpret_cast<const uint4 *>(smem);
  uint8_t *buf = smem + C::kEncTab + warp * C::kWarpBuf;
  uint16_t *buf16 = reinterpret_cast<uint16_t *>(buf);
  const uint64_t b0 = t * kTileBlocks;
  const uint64_t c = g.n_blocks ? chunk_of(g, b0) : 0;
  const uint64_t b = b0 + warp;
  const uint8_t *src = in + b * (uint64_t)B * group_bytes(DT);
  uint32_t size = 0, kdir = 0, K = 0, x = kL;
  bool raw = false, ovf = false;
  if (b < g.n_blocks) {
    encode_block<DT, B, false>(J, g, 0, buf, tab, x, K, ovf);
    const uint32_t coded = (uint32_t)round16(128 + 2ull * K);
    raw = coded >= (uint32_t)B;  // stored raw (R13)
    size = raw ? (uint32_t)B : coded;
    kdir = raw ? kRawBlock : K;
    __syncwarp();
    if (raw) {
      split_block<DT, B, false, false, COH>(J, g, b, src, buf);  // payload = the symbols in element order
    } else if (!ovf && lane < 8) {
      buf16[K + lane] = 0;  // zero pad up to the 16-byte boundary (K + 8 <= kCap + 8 words fit)
    }
    __syncwarp();
  }
  if (lane == 0) {
    S.size[warp] = size;
    S.ovf[warp] = (ovf && !raw) ? 1u : 0u;
  }
  __syncthreads();
  if (pd.job >= 0) resolve_pending<DT, B>(P, S, ring, pd);  // the previous tile's offset is due now

  // ---- a5: tile prefix by decoupled look-back
  uint32_t sum, roff, mine;
  tile_prefix(S.size, warp, roff, mine, &sum);
  const uint32_t anyovf = __any_sync(0xFFFFFFFFu, (lane < kWarps) && S.ovf[lane & (kWarps - 1)]);
  if (g.n_blocks && !anyovf && sum <= (uint32_t)ring_bytes) {
    // park the coded tile in the ring, publish its aggregate, go on coding
    if (b < g.n_blocks) {
      uint8_t *r = ring + roff;
      if (raw) {
        for (uint32_t i = lane; i < size / 16; i += 32)
          reinterpret_cast<uint4 *>(r)[i] = reinterpret_cast<const uint4 *>(buf)[i];
      } else {
        reinterpret_cast<uint32_t *>(r)[lane] = x;
        for (uint32_t i = lane; i < (size - 128) / 16; i += 32)
          reinterpret_cast<uint4 *>(r + 128)[i] = reinterpret_cast<const uint4 *>(buf)[i];
      }
    }
    if (lane == 0) {
      S.psize[warp] = size;
      S.pkdir[warp] = kdir;
    }
    if (tid == 0) {
      S.pagg = sum;
      lookback_publish(J.tile_status, t, sum, S.epoch);
    }
    pd.job = jidx;
    pd.t = t;
    return;  // the item-end barrier publishes the ring contents to the resolving warps
  }
  if (warp == 0) {
    const unsigned long long excl = lookback(P, J.tile_status, t, sum, S.epoch);
    if (lane == 0) S.tile_off = excl;
  }
  __syncthreads();
  const unsigned long long tile_off = S.tile_off;
  if (tile_off == ~0ull) return;  // aborted (timeout / peer error)

  if (b < g.n_blocks) {
    const unsigned long long off = tile_off + roff;
    for (uint32_t d = 0; d < J.nd; ++d) {
      uint8_t *o = J.dst[d] + g.off_pay + off;
      if (lane == 0) {
        reinterpret_cast<uint32_t *>(J.dst[d] + g.off_dir)[b] = kdir;
        if ((uint32_t)b % g.CB == 0) reinterpret_cast<unsigned long long *>(J.dst[d] + g.off_coff)[chunk_of(g, b)] = off;
      }
      if (raw) {
        for (uint32_t i = lane; i < size / 16; i += 32)
          reinterpret_cast<uint4 *>(o)[i] = reinterpret_cast<const uint4 *>(buf)[i];
      } else {
        reinterpret_cast<uint32_t *>(o)[lane] = x;  // the block header: 32 final lane states
        if (!ovf)
          for (uint32_t i = lane; i < (size - 128) / 16; i += 32)
            reinterpret_cast<uint4 *>(o + 128)[i] = reinterpret_cast<const uint4 *>(buf)[i];
      }
    }
    if (ovf && !raw) {
      // rare: the words outran the consumed symbol rows -- code the block again,
      // now storing each word straight to its final place (offset known)
      __syncwarp();
      split_block<DT, B, false, true, COH>(J, g, b, src, buf);
      __syncwarp();
      uint32_t x2 = kL, K2 = 0;
      bool o2 = false;
      encode_block<DT, B, true>(J, g, off, buf, tab, x2, K2, o2);
      for (uint32_t d = 0; d < J.nd; ++d)
        for (uint32_t i = 2 * K + lane * 2; i < size - 128; i += 64)
          *reinterpret_cast<uint16_t *>(J.dst[d] + g.off_pay + off + 128 + i) = 0;
    }
    if (b == g.n_blocks - 1) finalize_stream<DT>(J, off + size);
  } else if (g.n_blocks == 0 && warp == 0) {  // no whole block: header + raw tail only
    finalize_stream<DT>(J, 0ull);
  }
  // the chunk's first tile carries its serialized table (the receiver waits for it)
  if (g.n_blocks && (uint32_t)b0 % g.CB == 0 && warp == kWarps - 1) {
    const uint4 v = reinterpret_cast<const uint4 *>(J.tab16 + c * 256)[lane];
    for (uint32_t d = 0; d < J.nd; ++d) reinterpret_cast<uint4 *>(J.dst[d] + g.off_tab + 512ull * c)[lane] = v;
  }
  if (flags) {  // the last warp of the tile to finish its stores releases the tile's flags (a12)
    __syncwarp();
    if (lane == 0) {
      __threadfence_system();
      if (atomicAdd(&S.tile_cnt, 1u) == kWarps - 1) {
        S.tile_cnt = 0;
        const unsigned long long off16 = tile_off >> 4;
        for (uint32_t d = 0; d < J.nd; ++d)
          if (J.flag[d]) {
            stress_pause(P, t * 7 + d);
            st_release_sys_u64(J.flag[d] + t, ((unsigned long long)J.epoch[d] << 32) | off16);
          }
        trace_ev(P, kTrEFlag, (uint32_t)jidx, t);
      }
    }
  }
}

// One encode tile: every warp codes one block; one warp finds the tile's
// offset by decoupled look-back over tiles; the last warp of the tile to
// finish its stores releases the tile's flags.
template <int DT, int B>
static __device__ void enc_item(const Plan &P, const EncJob &J, int jidx, uint64_t t, uint8_t *smem, FusedShared &S,
                         uint64_t &enc_key, uint32_t &credit_done, uint8_t *ring, int ring_bytes, EncPending &pd,
                         uint64_t next_it) {
  using C = FusedCfg<DT, B>;
  const int tid = threadIdx.x, warp = warp_id();
  (void)next_it;  // an L2 prefetch of the next tile by warp 0 was measured slower (r1: 0.784 vs 0.754 ms/GiB)
  if (!credit_gate(P, J, jidx, credit_done, S)) return;
  if (tid == 0) trace_ev(P, kTrEStart, (uint32_t)jidx, t);
  const bool flags = J.has_flags != 0;

  if (J.raw) {  // ---- below the threshold: raw 64 KiB tiles (a11)
    const uint64_t o0 = t * kRawTileBytes;
    const uint64_t len = min((uint64_t)kRawTileBytes, J.raw_bytes - o0);
    const uint64_t nv = len / 16;
    for (uint64_t i = tid; i < nv; i += 256) {
      const uint4 v = ldg_nc_v4(J.in + o0 + 16 * i);
      for (uint32_t d = 0; d < J.nd; ++d) *reinterpret_cast<uint4 *>(J.dst[d] + o0 + 16 * i) = v;
    }
    for (uint64_t i = nv * 16 + tid; i < len; i += 256) {
      const uint8_t v = J.in[o0 + i];
      for (uint32_t d = 0; d < J.nd; ++d) J.dst[d][o0 + i] = v;
    }
    __syncthreads();
    if (tid == 0 && flags) {
      __threadfence_system();
      for (uint32_t d = 0; d < J.nd; ++d)
        if (J.flag[d]) {
          stress_pause(P, t * 11 + d);
          st_release_sys_u64(J.flag[d] + t, (unsigned long long)J.epoch[d] << 32);
        }
      trace_ev(P, kTrEFlag, (uint32_t)jidx, t);
    }
    return;
  }

  const StreamGeom &g = J.g;
  uint4 *tab = reinterpret_cast<uint4 *>(smem);
  // One B-byte buffer per warp: symbol rows stored in coding order (round R-1
  // first); the coded words grow from byte 0 into the rows already consumed.
  uint8_t *buf = smem + C::kEncTab + warp * C::kWarpBuf;
  const uint64_t b0 = t * kTileBlocks;
  const uint64_t c = g.n_blocks ? chunk_of(g, b0) : 0;
  const uint64_t key = ((uint64_t)jidx << 48) | c;
  const uint64_t b = b0 + warp;
  if (b < g.n_blocks) {
    // ---- a1: split; the residual goes straight to every destination (split-send)
#if UZIP_ENC_TMA
    uint8_t *stage = smem + C::smem(true, false) - (kWarps - warp) * C::kTmaStage;
    tma_stage_block(J.in + b * (uint64_t)B * group_bytes(DT), stage, (uint32_t)C::kTmaStage, &S.tma_bar[warp],
                    &S.tma_phase[warp]);
    split_block<DT, B, true, true, false, true>(J, g, b, stage, buf);
#else
    split_block<DT, B, true, true>(J, g, b, J.in + b * (uint64_t)B * group_bytes(DT), buf);
#endif
    __syncwarp();
  }
  // the chunk's table after the split: a table still being built by its T items (small streams) is
  // waited for while the split's loads and residual stores are already done
  if (g.n_blocks && key != enc_key) {  // uniform; every warp left the previous tile's table behind
    if (!P.tables_ready) {
      if (tid == 0) {  // the chunk's table: published by its last T item (a smaller ticket)
        unsigned long long seen = 0;
        S.ab_table = wait_u64(P, J.tflag + c, kCtlTag | (S.epoch + 1u), seen) ? 0u : 1u;
      }
      __syncthreads();
      if (S.ab_table) return;
    }
    tab[tid] = J.enc[c * 256 + tid];  // after the acquire (gpu scope): plain loads see the T item's stores
    enc_key = key;
    __syncthreads();
  }
  code_tile<DT, B, false>(P, J, jidx, t, smem, S, ring, ring_bytes, pd, J.in);
}

// ---------------------------------------------------------------- C item
static __device__ void copy_item(const CopyJob &Cj, uint64_t t) {
  const uint64_t o0 = t * kRawTileBytes;
  const uint64_t len = min((uint64_t)kRawTileBytes, Cj.bytes - o0);
  const uint64_t nv = len / 16;
  for (uint64_t i = threadIdx.x; i < nv; i += 256)
    st_any16(Cj.dst + o0 + 16 * i, ldg_nc_v4(Cj.src + o0 + 16 * i));
  for (uint64_t i = nv * 16 + threadIdx.x; i < len; i += 256) Cj.dst[o0 + i] = Cj.src[o0 + i];
}

// Completion of one D item: the last tile of the job releases the sources' slots.
static __device__ void dec_done(const Plan &P, const DecJob &J, int jidx, uint64_t t) {
  if (threadIdx.x != 0) return;
  trace_ev(P, kTrDDone, (uint32_t)jidx, t);
  __threadfence();
  const uint32_t old = atomicAdd(J.done, 1u);
  if (old == (uint32_t)J.ntiles - 1) {
    __threadfence();
    *J.done = 0;
    for (uint32_t s = 0; s < J.nsrc; ++s)
      if ((int32_t)s != J.me && J.credit[s]) st_release_sys_u64(J.credit[s], (unsigned long long)J.epoch[s]);
  }
}

// Thread 0: acquire tile t of source s (and the chunk's first tile, which
// carries the table, when the table is not cached).  Sets S.abort on failure.
static __device__ void acquire_tile(const Plan &P, const DecJob &J, uint32_t s, uint64_t t, bool need_table,
                             FusedShared &S) {
  stress_pause(P, t * 131 + s);
  unsigned long long v = 0;
  bool ok = wait_flag(P, J.flag[s] + t, J.epoch[s], v);
  S.src_off[s] = (v & 0xFFFFFFFFull) << 4;
  if (ok && need_table && !J.raw && J.g.n_blocks) {
    const uint64_t first = (uint64_t)chunk_of(J.g, t * kTileBlocks) * J.g.CB / kTileBlocks;
    if (first != t) {
      unsigned long long v2;
      ok = wait_flag(P, J.flag[s] + first, J.epoch[s], v2);
    }
  }
  S.abort = ok ? 0u : 1u;
}

// Per-block payload offsets within a tile from the directory (all lanes of a warp).
__device__ __forceinline__ void tile_block(const uint8_t *stream, const StreamGeom &g, uint64_t b0, int warp,
                                           unsigned long long tile_off, uint32_t &K, unsigned long long &off,
                                           unsigned long long &tile_end, bool &bad) {
  const int lane = threadIdx.x & 31;
  const uint32_t *dir = reinterpret_cast<const uint32_t *>(stream + g.off_dir);
  uint32_t d = 0, sz = 0;
  bool bb = false;
  if (lane < kWarps && b0 + lane < g.n_blocks) {
    d = ld_cg_u32c(dir + b0 + lane);
    sz = block_size(d, g.B, bb);
  }
  bad = __any_sync(0xFFFFFFFFu, bb);
  uint32_t incl = sz;
  for (int o = 1; o < 8; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  K = __shfl_sync(0xFFFFFFFFu, d, warp);
  off = tile_off + __shfl_sync(0xFFFFFFFFu, incl - sz, warp);
  tile_end = tile_off + __shfl_sync(0xFFFFFFFFu, incl, kWarps - 1);
}

// Stage block payload into smem (warp).
__device__ __forceinline__ void stage_payload(const uint8_t *stream, const StreamGeom &g, unsigned long long off,
                                              uint32_t size, uint8_t *pay) {
  stage_block(stream + g.off_pay + off, size / 16, pay);
}

// Copy stream bytes [o, o+len) from the local staging to the same offset in
// every forward destination (all threads of the CTA).
__device__ __forceinline__ void fwd_range(const DecJob &J, const uint8_t *stream, uint64_t o, uint64_t len) {
  const uint64_t nv = len / 16;
  for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x) {
    const uint4 v = ld_cg_v4(stream + o + 16 * i);
    for (uint32_t d = 0; d < J.nfwd; ++d) *reinterpret_cast<uint4 *>(J.fdst[d] + o + 16 * i) = v;
  }
  for (uint64_t i = nv * 16 + threadIdx.x; i < len; i += blockDim.x) {
    const uint8_t v = stream[o + i];
    for (uint32_t d = 0; d < J.nfwd; ++d) J.fdst[d][o + i] = v;
  }
}

// Relay of one received tile (broadcast): the bytes the tile's flag covers --
// residual plane(s), directory entries, payload range, the chunk's table and
// offset on its first tile, header/pads/tail on the last -- are stored as
// received into the next hops' staging, then their flags are released with
// the same payload offset.  No decode, no re-encode.
template <int DT>
static __device__ void forward_tile(const Plan &P, const DecJob &J, uint64_t t, FusedShared &S, uint32_t &fwd_done,
                             int jidx) {
  const int tid = threadIdx.x;
  const StreamGeom &g = J.g;
  const uint8_t *stream = J.src[0];
  if (!((fwd_done >> jidx) & 1u)) {  // first forward of this job in this CTA: the hops' slots are free
    if (tid == 0) {
      uint32_t ok = 1;
      if (P.credit_ready) ok = ld_volatile_u32(P.err) == 0;
      else
        for (uint32_t d = 0; d < J.nfwd && ok; ++d) ok = wait_credit(P, J.fcredit[d], J.fepoch[d]);
      S.ab_credit = ok ? 0u : 1u;
    }
    __syncthreads();
    if (S.ab_credit) return;
    fwd_done |= 1u << jidx;
  }
  const unsigned long long tile_off = S.src_off[0];
  if (warp_id() == 0) {
    uint32_t K;
    unsigned long long off, tile_end;
    bool bad;
    tile_block(stream, g, t * kTileBlocks, 0, tile_off, K, off, tile_end, bad);
    if ((threadIdx.x & 31) == 0) S.ptile_off = bad ? tile_off : tile_end;
  }
  __syncthreads();
  const unsigned long long tile_end = S.ptile_off;
  const uint64_t b0 = t * kTileBlocks;
  const uint64_t nblk = g.n_blocks > b0 ? min((uint64_t)kTileBlocks, g.n_blocks - b0) : 0;
  if (nblk) {
    if (DT == kF32) {
      fwd_range(J, stream, g.off_res0 + 2 * b0 * g.B, 2 * nblk * g.B);
      fwd_range(J, stream, g.off_res1 + b0 * g.B, nblk * g.B);
    } else {
      fwd_range(J, stream, g.off_res0 + b0 * g.B, nblk * g.B);
    }
    fwd_range(J, stream, g.off_dir + 4 * b0, 4 * nblk);
    fwd_range(J, stream, g.off_pay + tile_off, tile_end - tile_off);
    if ((uint32_t)b0 % g.CB == 0) {
      const uint64_t c = chunk_of(g, b0);
      fwd_range(J, stream, g.off_tab + 512 * c, 512);
      fwd_range(J, stream, g.off_coff + 8 * c, 8);
    }
  }
  if (t == J.ntiles - 1) {  // header, section pads, raw tail
    fwd_range(J, stream, 0, kHeaderBytes);
    fwd_range(J, stream, g.off_coff + 8 * g.n_chunks, g.off_dir - (g.off_coff + 8 * g.n_chunks));
    fwd_range(J, stream, g.off_dir + 4 * g.n_blocks, g.off_pay - (g.off_dir + 4 * g.n_blocks));
    fwd_range(J, stream, g.off_tail(tile_end), g.tail_bytes());
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (uint32_t d = 0; d < J.nfwd; ++d)
      st_release_sys_u64(J.fflag[d] + t, ((unsigned long long)J.fepoch[d] << 32) | (tile_off >> 4));
  }
}

// ---------------------------------------------------------------- D item: decode (+ join)
template <int DT, int B, bool RED>
static __device__ void dec_item(const Plan &P, const DecJob &J, int jidx, uint64_t t, uint8_t *smem, FusedShared &S,
                         uint64_t &dec_key, uint32_t &fwd_done) {
  using C = FusedCfg<DT, B>;
  const int tid = threadIdx.x, warp = warp_id();
  const StreamGeom &g = J.g;
  const uint64_t b0 = t * kTileBlocks;
  const uint64_t c = g.n_blocks ? chunk_of(g, b0) : 0;
  const uint64_t key = (1ull << 63) | ((uint64_t)jidx << 48) | c;
  const bool need_table = key != dec_key;
  if (tid == 0) {
    acquire_tile(P, J, 0, t, need_table, S);
    trace_ev(P, kTrDAcq, (uint32_t)jidx, t);
  }
  __syncthreads();
  if (S.abort) return;
  const uint8_t *stream = J.src[0];
  if (J.raw) {
    const uint64_t o0 = t * kRawTileBytes;
    const uint64_t len = min((uint64_t)kRawTileBytes, J.raw_bytes - o0);
    const uint64_t nv = len / 16;
    for (uint64_t i = tid; i < nv; i += 256)
      st_any16(J.out + o0 + 16 * i, ld_cg_v4(stream + o0 + 16 * i));
    for (uint64_t i = nv * 16 + tid; i < len; i += 256) J.out[o0 + i] = stream[o0 + i];
    __syncthreads();
    dec_done(P, J, jidx, t);
    return;
  }
  if (J.nfwd) {  // relay first: the next hops receive the tile before it is decoded here
    forward_tile<DT>(P, J, t, S, fwd_done, jidx);
    if (S.abort) return;
  }
  uint32_t *dtab = reinterpret_cast<uint32_t *>(smem + C::kEncTab + kWarps * C::kWarpBuf + P.ring_bytes);
  if (g.n_blocks && need_table) {
    if (!build_dtab(reinterpret_cast<const uint16_t *>(stream + g.off_tab + 512 * c), dtab, S.red,
                    reinterpret_cast<uint32_t *>(smem + C::kEncTab))) {
      if (tid == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
      dec_key = ~0ull;
      return;
    }
    dec_key = key;
  }
  __syncthreads();
  uint8_t *pay = smem + C::kEncTab + warp * C::kWarpBuf;
  uint8_t *symb = pay + B;
  const uint64_t b = b0 + warp;
  uint32_t K;
  unsigned long long off, tile_end;
  bool bad;
  tile_block(stream, g, b0, warp, S.src_off[0], K, off, tile_end, bad);
  if (b < g.n_blocks && !bad) {
    const uint32_t size = K == kRawBlock ? (uint32_t)B : (uint32_t)round16(128 + 2ull * K);
    stage_payload(stream, g, off, size, pay);
    uint8_t *dst = J.out + b * (uint64_t)B * g.eb;
    if (K == kRawBlock) join_block<DT, B>(pay, stream, g, b, dst);
    else if (!decode_join_warp<DT, B>(pay, K, dtab, symb, stream, g, b, dst)) bad = true;
    __syncwarp();
  }
  if (bad && (threadIdx.x & 31) == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
  if (t == J.ntiles - 1) {  // raw tail
    const uint64_t tail_bytes = g.tail_bytes();
    const uint8_t *tsrc = stream + g.off_tail(tile_end);
    uint8_t *tdst = J.out + g.n_coded * g.eb;
    for (uint64_t i = tid; i < tail_bytes; i += 256) tdst[i] = tsrc[i];
  }
  __syncthreads();
  dec_done(P, J, jidx, t);
}

// Two consecutive tiles of a plain decode job at once (the D-item form of k_decode's pairing): every
// warp decodes block w of tile t and block w of tile t + 1 with their rANS chains interleaved
// (decode_join_warp2), both staged in the warp's buffer (two halves); blocks that are raw or larger
// than a half take the one-chain path.  The caller checked pair_tiles().
#ifndef UZIP_DEC_PAIR_TILES
#define UZIP_DEC_PAIR_TILES 1
#endif
template <int DT, int B, bool RED>
constexpr bool kDecPairOk = UZIP_DEC_PAIR_TILES && !RED && B == 4096 && (DT == kBF16 || DT == kF16 || DT == kE4M3);

__device__ __forceinline__ bool pair_tiles(const DecJob &J, uint64_t t) {
  const StreamGeom &g = J.g;
  return !J.raw && J.nfwd == 0 && J.nsrc == 1 && (t + 1) * kTileBlocks < g.n_blocks &&
         chunk_of(g, t * kTileBlocks) == chunk_of(g, (t + 1) * kTileBlocks);
}

template <int DT, int B>
static __device__ void dec_item2(const Plan &P, const DecJob &J, int jidx, uint64_t t, uint8_t *smem,
                                 FusedShared &S, uint64_t &dec_key) {
  using C = FusedCfg<DT, B>;
  constexpr uint32_t kHalf = C::kWarpBuf / 2, kStage2 = (kHalf - 256) & ~15u;
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const StreamGeom &g = J.g;
  const uint64_t b0 = t * kTileBlocks;
  const uint64_t c = chunk_of(g, b0);
  const uint64_t key = (1ull << 63) | ((uint64_t)jidx << 48) | c;
  const bool need_table = key != dec_key;
  if (tid == 0) {
    acquire_tile(P, J, 0, t, need_table, S);
    trace_ev(P, kTrDAcq, (uint32_t)jidx, t);
    if (!S.abort) {
      const unsigned long long o0 = S.src_off[0];
      acquire_tile(P, J, 0, t + 1, false, S);
      trace_ev(P, kTrDAcq, (uint32_t)jidx, t + 1);
      S.red64[0] = S.src_off[0];  // (scratch word: a new FusedShared field measurably raised k_fused's spills)
      S.src_off[0] = o0;
    }
  }
  __syncthreads();
  if (S.abort) return;
  const uint8_t *stream = J.src[0];
  uint32_t *dtab = reinterpret_cast<uint32_t *>(smem + C::kEncTab + kWarps * C::kWarpBuf + P.ring_bytes);
  if (need_table) {
    if (!build_dtab(reinterpret_cast<const uint16_t *>(stream + g.off_tab + 512 * c), dtab, S.red,
                    reinterpret_cast<uint32_t *>(smem + C::kEncTab))) {
      if (tid == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
      dec_key = ~0ull;
      return;
    }
    dec_key = key;
  }
  __syncthreads();
  uint8_t *buf = smem + C::kEncTab + warp * C::kWarpBuf;
  uint32_t KA, KB;
  unsigned long long offA, offB, endA, endB;
  bool badA, badB;
  tile_block(stream, g, b0, warp, S.src_off[0], KA, offA, endA, badA);
  tile_block(stream, g, b0 + kTileBlocks, warp, S.red64[0], KB, offB, endB, badB);
  (void)endA;
  const uint64_t bA = b0 + warp, bB = b0 + kTileBlocks + warp;
  const bool okA = bA < g.n_blocks && !badA, okB = bB < g.n_blocks && !badB;
  const uint32_t sA = KA == kRawBlock ? (uint32_t)B : (uint32_t)round16(128 + 2ull * KA);
  const uint32_t sB = KB == kRawBlock ? (uint32_t)B : (uint32_t)round16(128 + 2ull * KB);
  bool bad = badA || badB;
  if (okA && okB && KA != kRawBlock && KB != kRawBlock && sA <= kStage2 && sB <= kStage2) {
    uint8_t *payB = buf + kHalf;
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(buf), s1 = (uint32_t)__cvta_generic_to_shared(payB);
    const uint8_t *srcA = stream + g.off_pay + offA, *srcB = stream + g.off_pay + offB;
    for (uint32_t i = lane; i < sA / 16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + 16 * i), "l"(srcA + 16 * i) : "memory");
    for (uint32_t i = lane; i < sB / 16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s1 + 16 * i), "l"(srcB + 16 * i) : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    __syncwarp();
    bool gA, gB;
    decode_join_warp2<DT, B, false>(buf, KA, payB, KB, dtab, buf + kStage2, payB + kStage2, stream, g, bA, bB,
                                    J.out + bA * (uint64_t)B * g.eb, J.out + bB * (uint64_t)B * g.eb, gA, gB);
    bad = bad || !gA || !gB;
    __syncwarp();
  } else {
    for (int h = 0; h < 2; ++h) {
      const bool ok = h ? okB : okA;
      if (!ok) continue;
      const uint32_t K = h ? KB : KA, size = h ? sB : sA;
      const uint64_t b = h ? bB : bA;
      stage_payload(stream, g, h ? offB : offA, size, buf);
      uint8_t *dst = J.out + b * (uint64_t)B * g.eb;
      if (K == kRawBlock) join_block<DT, B>(buf, stream, g, b, dst);
      else if (!decode_join_warp<DT, B>(buf, K, dtab, buf + B, stream, g, b, dst)) bad = true;
      __syncwarp();
    }
  }
  if (bad && lane == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
  if (t + 1 == J.ntiles - 1) {  // raw tail
    const uint64_t tail_bytes = g.tail_bytes();
    const uint8_t *tsrc = stream + g.off_tail(endB);
    uint8_t *tdst = J.out + g.n_coded * g.eb;
    for (uint64_t i = tid; i < tail_bytes; i += 256) tdst[i] = tsrc[i];
  }
  __syncthreads();
  dec_done(P, J, jidx, t);
  dec_done(P, J, jidx, t + 1);
}

// The warp's fp32 accumulator lives in global memory (P.acc, B floats per
// (CTA, warp), L2-resident): every lane reads and writes only its own 8-element
// groups, the same ones for every source, so it is thread-private data moved
// with 128-bit accesses.  In smem it would take 128 KiB per CTA and hold the
// reduce kernel to one CTA per SM.
__device__ __forceinline__ void acc_load8(const float *p, float *v) {
  const float4 a = *reinterpret_cast<const float4 *>(p), b = *reinterpret_cast<const float4 *>(p + 4);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}
__device__ __forceinline__ void acc_store8(float *p, const float *v) {
  *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4 *>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

// Epilogue that folds a decoded source into the warp's fp32 accumulator (a9).
struct FoldEpi {
  float *acc;
  bool first;
  uint32_t op;
  template <int DT>
  __device__ __forceinline__ void apply(uint32_t e0, uint4 a, uint4 b) const {
    float v[8];
    if (!first) acc_load8(acc + e0, v);
    if (DT == kF32) {
      fold_vec<DT>(v, a, first, op);
      fold_vec<DT>(v + 4, b, first, op);
    } else {
      fold_vec<DT>(v, a, first, op);
    }
    acc_store8(acc + e0, v);
  }
};

// ---------------------------------------------------------------- D item: decode + reduce (a9)
template <int DT, int B>
static __device__ void red_item(const Plan &P, const DecJob &J, int jidx, uint64_t t, uint8_t *smem, FusedShared &S,
                         uint64_t &dec_key, uint64_t &enc_key, uint32_t &credit_done, uint8_t *ring, EncPending &pd) {
  using C = FusedCfg<DT, B>;
  const int tid = threadIdx.x, lane = tid & 31, warp = warp_id();
  const StreamGeom &g = J.g;
  const uint32_t eb = elem_bytes(DT);
  // fused allreduce (a9): this reduce job's tiles are also coded into the allgather stream e[ag_job]
  const bool ag = jidx == 0 && P.ag_job >= 0 && !J.raw;
  if (ag && !credit_gate(P, P.e[P.ag_job], P.ag_job, credit_done, S)) return;  // before the residual stores

  if (J.raw) {  // ---- below the threshold: fold raw tiles
    for (uint32_t s = 0; s < J.nsrc; ++s) {
      if ((int32_t)s == J.me) continue;
      if (tid == 0) acquire_tile(P, J, s, t, false, S);
      __syncthreads();
      if (S.abort) return;
    }
    const uint64_t o0 = t * kRawTileBytes;
    const uint64_t len = min((uint64_t)kRawTileBytes, J.raw_bytes - o0);
    const uint64_t nv = len / 16;
    for (uint64_t i = tid; i < nv; i += 256) {
      float acc[8];
      for (uint32_t s = 0; s < J.nsrc; ++s) {
        const uint8_t *p = J.src[s] + o0 + 16 * i;
        const uint4 v = ((int32_t)s == J.me) ? ldg_nc_v4(p) : ld_cg_v4(p);
        fold_vec<DT>(acc, v, s == 0, J.op);
      }
      *reinterpret_cast<uint4 *>(J.out + o0 + 16 * i) = narrow_vec<DT>(acc);
    }
    for (uint64_t i = nv * 16 / eb + tid; i < len / eb; i += 256) {  // scalar tail
      float acc = 0.f;
      for (uint32_t s = 0; s < J.nsrc; ++s) {
        const uint8_t *p = J.src[s] + o0 + i * eb;
        const uint32_t bits = DT == kF32 ? *reinterpret_cast<const uint32_t *>(p)
                                         : (uint32_t)*reinterpret_cast<const uint16_t *>(p);
        acc = fold(acc, widen<DT>(bits), s == 0, J.op);
      }
      const uint32_t r = narrow<DT>(acc);
      if (DT == kF32) *reinterpret_cast<uint32_t *>(J.out + o0 + i * eb) = r;
      else *reinterpret_cast<uint16_t *>(J.out + o0 + i * eb) = (uint16_t)r;
    }
    __syncthreads();
    dec_done(P, J, jidx, t);
    return;
  }

  const uint64_t b0 = t * kTileBlocks;
  const uint64_t c = g.n_blocks ? chunk_of(g, b0) : 0;
  const uint64_t b = b0 + warp;
  uint32_t *dtab = reinterpret_cast<uint32_t *>(smem + C::kEncTab + kWarps * C::kWarpBuf + C::ring(true));
  float *acc = P.acc + ((uint64_t)blockIdx.x * kWarps + warp) * B;
  uint8_t *pay = smem + C::kEncTab + warp * C::kWarpBuf;
  uint8_t *symb = pay + B;
  bool bad = false;

  for (uint32_t s = 0; s < J.nsrc; ++s) {
    const bool first = s == 0;
    if ((int32_t)s == J.me) {  // own shard: never compressed
      if (b < g.n_blocks) {
        const uint8_t *src = J.src[s] + b * (uint64_t)B * eb;
        // the same lane-to-element map as the decode epilogue (8 consecutive elements per lane
        // and group), so each accumulator element stays with one thread
        for (uint32_t e = lane * 8; e < (uint32_t)B; e += 256) {
          float a[8];
          if (!first) acc_load8(acc + e, a);
          fold_vec<DT>(a, ldg_nc_v4(src + e * eb), first, J.op);
          if (DT == kF32) fold_vec<DT>(a + 4, ldg_nc_v4(src + e * eb + 16), first, J.op);
          acc_store8(acc + e, a);
        }
      }
      __syncwarp();
      continue;
    }
    const uint64_t key = (2ull << 62) | ((uint64_t)jidx << 48) | ((uint64_t)s << 40) | c;
    const bool need_table = key != dec_key;
    if (tid == 0) acquire_tile(P, J, s, t, need_table, S);
    __syncthreads();
    if (S.abort) return;
    const uint8_t *stream = J.src[s];
    if (g.n_blocks && need_table) {
      if (!build_dtab(reinterpret_cast<const uint16_t *>(stream + g.off_tab + 512 * c), dtab, S.red,
                    reinterpret_cast<uint32_t *>(smem + C::kEncTab))) {
        if (tid == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
        dec_key = ~0ull;
        return;
      }
      dec_key = key;
    }
    __syncthreads();
    uint32_t K;
    unsigned long long off, tile_end;
    bool tb;
    tile_block(stream, g, b0, warp, S.src_off[s], K, off, tile_end, tb);
    bad |= tb;
    if (tid == 0) S.src_payload[s] = tile_end;
    if (b < g.n_blocks && !tb) {
      const uint32_t size = K == kRawBlock ? (uint32_t)B : (uint32_t)round16(128 + 2ull * K);
      stage_payload(stream, g, off, size, pay);
      FoldEpi epi{acc, first, J.op};
      if (K != kRawBlock) {
        if (!decode_join_warp_epi<DT, B>(pay, K, dtab, symb, stream, g, b, epi)) bad = true;
      } else {  // stored-raw block: symbols are the payload
        for (uint32_t e = lane * 8; e < (uint32_t)B; e += 256) {
          const uint2 s8 = *reinterpret_cast<const uint2 *>(pay + e);
          if (DT == kF32) {
            const uint4 lo = ld_cg_v4(stream + g.off_res0 + 2 * (b * B + e));
            const uint2 hi = ld_cg_v2(stream + g.off_res1 + b * B + e);
            epi.template apply<DT>(e, join4_f32(s8.x, make_uint2(lo.x, lo.y), hi.x),
                                   join4_f32(s8.y, make_uint2(lo.z, lo.w), hi.y));
          } else {
            const uint2 r8 = ld_cg_v2(stream + g.off_res0 + b * B + e);
            uint4 v;
            if (DT == kBF16) {
              join4_bf16(s8.x, r8.x, v.x, v.y);
              join4_bf16(s8.y, r8.y, v.z, v.w);
            } else {
              join4_f16(s8.x, r8.x, v.x, v.y);
              join4_f16(s8.y, r8.y, v.z, v.w);
            }
            epi.template apply<DT>(e, v, v);
          }
        }
      }
    }
    __syncwarp();
  }
  if (bad && lane == 0) raise_err(P, UZIP_ERR_CORRUPT_STREAM);
  if (b < g.n_blocks) {  // one rounding to the dtype, 128-bit stores
    uint8_t *dst = J.out + b * (uint64_t)B * eb;
    for (uint32_t e = lane * 8; e < (uint32_t)B; e += 256) {
      float a[8];
      acc_load8(acc + e, a);
      const uint4 v0 = narrow_vec<DT>(a);
      *reinterpret_cast<uint4 *>(dst + e * eb) = v0;
      uint4 v1 = v0;
      if (DT == kF32) *reinterpret_cast<uint4 *>(dst + e * eb + 16) = v1 = narrow_vec<DT>(a + 4);
      if constexpr (DT == kBF16 || DT == kF16 || DT == kF32) {
        if (ag) {  // a1 of the allgather phase on the reduced values, still in registers
          split_vec<DT, B>(P.e[P.ag_job], P.e[P.ag_job].g, b, e, v0, pay);
          if (DT == kF32) split_vec<DT, B>(P.e[P.ag_job], P.e[P.ag_job].g, b, e + 4, v1, pay);
        }
      }
    }
  }
  __syncthreads();
  if (t == J.ntiles - 1) {  // raw tails of every source, folded in rank order
    const uint64_t tail = g.n - g.n_coded;
    for (uint64_t i = tid; i < tail; i += 256) {
      float a = 0.f;
      for (uint32_t s = 0; s < J.nsrc; ++s) {
        const uint8_t *p = ((int32_t)s == J.me) ? J.src[s] + (g.n_coded + i) * eb
                                                : J.src[s] + g.off_tail(S.src_payload[s]) + i * eb;
        const uint32_t bits = DT == kF32 ? *reinterpret_cast<const uint32_t *>(p)
                                         : (uint32_t)*reinterpret_cast<const uint16_t *>(p);
        a = fold(a, widen<DT>(bits), s == 0, J.op);
      }
      const uint32_t r = narrow<DT>(a);
      if (DT == kF32) *reinterpret_cast<uint32_t *>(J.out + (g.n_coded + i) * eb) = r;
      else *reinterpret_cast<uint16_t *>(J.out + (g.n_coded + i) * eb) = (uint16_t)r;
    }
  }
  __syncthreads();
  if (ag) {
    const EncJob &A = P.e[P.ag_job];
    const StreamGeom &ga = A.g;
    const uint64_t ca = ga.n_blocks ? chunk_of(ga, b0) : 0;
    const uint64_t key = ((uint64_t)P.ag_job << 48) | ca;
    uint4 *tab = reinterpret_cast<uint4 *>(smem);
    unsigned long long *tabflag = A.tflag;  // per chunk: kCtlTag | (epoch + 1) = table published
    if (ga.n_blocks && (uint32_t)b0 % ga.CB == 0) {
      // the chunk's first tile is its sample (R26): histogram the symbols just split, rule N1, publish
      uint32_t *hist = dtab;  // 8 x 256 counters in the decode-table region
      dec_key = ~0ull;
      for (int i = tid; i < kWarps * 256; i += 256) hist[i] = 0;
      __syncthreads();
      if (b < ga.n_blocks) {
        uint32_t *h = hist + 256 * warp;
        for (uint32_t i = lane; i < (uint32_t)B / 4; i += 32) {
          const uint32_t w4 = reinterpret_cast<const uint32_t *>(pay)[i];
#pragma unroll
          for (int k = 0; k < 4; ++k) atomicAdd(&h[(w4 >> (8 * k)) & 0xFFu], 1u);
        }
      }
      __syncthreads();
      uint32_t cnt = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) cnt += hist[256 * w + tid];
      norm_tables(cnt, A.enc + ca * 256, A.tab16 + ca * 256, tab, S.red64, S.red);
      if (tid == 0) {
        __threadfence();
        st_release_gpu_u64(tabflag + ca, kCtlTag | (S.epoch + 1u));
      }
      enc_key = key;
    } else if (ga.n_blocks && key != enc_key) {
      if (tid == 0) {  // the chunk's first tile (a smaller ticket) publishes the table
        unsigned long long v = 0;
        S.ab_table = wait_u64(P, tabflag + ca, kCtlTag | (S.epoch + 1u), v) ? 0u : 1u;
      }
      __syncthreads();
      if (S.ab_table) return;
      tab[tid] = ld_cg_v4(A.enc + ca * 256 + tid);
      enc_key = key;
      __syncthreads();
    }
    code_tile<DT, B, true>(P, A, P.ag_job, t, smem, S, ring, P.ring_bytes, pd, A.in);
  }
  __syncthreads();
  dec_done(P, J, jidx, t);
}

// ---------------------------------------------------------------- the kernel
// MINB: resident CTAs per SM the register allocation targets.  Launches with
// encode items use UZIP_ENC_MINB (3: 85 registers, measured fastest for the
// encoder); decode-only launches use 4 (64 registers, like k_decode).
template <int DT, int B, bool RED, int MINB, bool DONLY = false>
__global__ void __launch_bounds__(256, MINB) k_fused(const __grid_constant__ Plan P) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ FusedShared S;
  const int tid = threadIdx.x;
  uint64_t enc_key = ~0ull, dec_key = ~0ull;
  uint32_t credit_done = 0, fwd_done = 0;
  using Cf = FusedCfg<DT, B>;
  uint8_t *ring = smem + Cf::kEncTab + kWarps * Cf::kWarpBuf;
  EncPending pd{-1, 0};
  const uint64_t nt = P.n_t_items, ne = P.n_e_items, nc = P.n_c_items, total = nt + ne + nc + P.n_d_items;
  if (UZIP_ENC_TMA && tid < kWarps) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&S.tma_bar[tid])));
    S.tma_phase[tid] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 0) {
    S.tile_cnt = 0;
    S.epoch = ld_volatile_u32(P.epoch) & kEpochMask;  // advanced only after every CTA has left
    S.tk[0] = atomicAdd(P.ticket, 1u);
  }
  __syncthreads();
  uint64_t it = uniform_u64(S.tk[0]);
  for (int par = 0; it < total; par ^= 1) {
    uint32_t nxt = 0;
    if (tid == 0) S.tk[par ^ 1] = nxt = atomicAdd(P.ticket, 1u);  // next ticket, read after the item's last barrier
    nxt = __shfl_sync(0xFFFFFFFFu, nxt, 0);  // warp 0 knows it now (L2 prefetch of that tile)
    // D items: job-major; a run of consecutive tiles per item (one decode-table build per source for
    // the run); after an abort every later tile of the run returns at once
    auto decode_items = [&](uint64_t k) {
      int j = 0;
      while (j + 1 < P.nd_jobs && k >= items_of(P.d[j])) k -= items_of(P.d[j++]);
      const DecJob &Jd = P.d[j];
      const uint64_t r = Jd.run > 1 ? Jd.run : 1, t1 = min(Jd.ntiles, (k + 1) * r);
      for (uint64_t t = k * r; t < t1; ++t) {
        if constexpr (DONLY && kDecPairOk<DT, B, RED>) {  // decode-only launches: their own register budget
          if (t + 1 < t1 && pair_tiles(Jd, t)) {  // two tiles of the run at once (two rANS chains per warp)
            dec_item2<DT, B>(P, Jd, j, t, smem, S, dec_key);
            ++t;
            continue;
          }
        }
        if constexpr (RED) {
          if (Jd.nsrc > 1) red_item<DT, B>(P, Jd, j, t, smem, S, dec_key, enc_key, credit_done, ring, pd);
          else dec_item<DT, B, RED>(P, Jd, j, t, smem, S, dec_key, fwd_done);
        } else {
          dec_item<DT, B, RED>(P, Jd, j, t, smem, S, dec_key, fwd_done);
        }
      }
    };
    if constexpr (DONLY) {
      // decode-only launch (P2P / broadcast receivers): no E/C item code in this instantiation, so
      // its register budget is the decoder's alone
      decode_items(it);
    } else if (it < nt) {  // T items: job-major, then chunk, then part (no pending tile exists yet)
      uint64_t k = it;
      int j = 0;
      while (j + 1 < P.ne && k >= t_items_of(P.e[j])) k -= t_items_of(P.e[j++]);
      uint64_t c;
      uint32_t part;
      t_item_at(P.e[j], k, c, part);
      t_item<DT, B>(P, P.e[j], c, part, smem, S);
    } else {
      it -= nt;
      int j = 0;
      uint64_t et = 0;
      if (it < ne) e_item_at(P, it, j, et);  // tile-major over the encode streams
      const bool coded_e = it < ne && !P.e[j].raw;
      if (pd.job >= 0 && !coded_e) resolve_pending<DT, B>(P, S, ring, pd);
      if (it < ne) {
        enc_item<DT, B>(P, P.e[j], j, et, smem, S, enc_key, credit_done, ring, P.ring_bytes, pd,
                        warp_id() == 0 ? (uint64_t)nxt : ~0ull);
      } else if (it < ne + nc) {
        copy_item(P.c, it - ne);
      } else {
        decode_items(it - ne - nc);
      }
    }
    __syncthreads();
    it = uniform_u64(S.tk[par ^ 1]);
  }
  if constexpr (!DONLY)
    if (pd.job >= 0) resolve_pending<DT, B>(P, S, ring, pd);
  if (tid == 0) {  // the last CTA out resets the ticket for the next launch
    __threadfence();
    if (atomicAdd(P.ticket + 1, 1u) == gridDim.x - 1) {
      P.ticket[0] = 0;
      P.ticket[1] = 0;
      *P.epoch = (S.epoch + 1u) & kEpochMask;  // every CTA read it at its start
      if (P.codec_call) {  // uzip_compress: the error word is private to this call
        if (ld_volatile_u32(P.err))
          for (int j = 0; j < P.ne; ++j)
            if (P.e[j].d_out_bytes) *P.e[j].d_out_bytes = 0;
        P.err[0] = 0;
      }
      __threadfence();
    }
  }
}

// ================================================================ launchers
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
inline int sm_count() {
  static int n[kMaxDevices] = {0};
  const int dev = current_device();
  if (n[dev] == 0) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

template <int DT>
cudaError_t launch_tables_t(const Plan &p, cudaStream_t st) {
  uint64_t max_chunks = 1;  // >= 1: the look-back words are reset even without chunks
  uint32_t max_parts = 1;
  for (int j = 0; j < p.ne; ++j) {
    const EncJob &J = p.e[j];
    if (J.raw) continue;
    max_chunks = J.g.n_chunks > max_chunks ? J.g.n_chunks : max_chunks;
    for (uint64_t c = 0; c < J.g.n_chunks; c += (J.g.n_chunks > 1 ? J.g.n_chunks - 1 : 1)) {
      const uint32_t parts = hist_parts(J.g.sample_len(c), J.g.global);
      max_parts = parts > max_parts ? parts : max_parts;
    }
  }
  k_hist<DT><<<dim3(max_parts, (unsigned)max_chunks, (unsigned)p.ne), kHistThreads, 0, st>>>(p);
  k_norm<DT><<<dim3((unsigned)max_chunks, (unsigned)p.ne), 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <int DT, int B, bool RED, int MINB, bool DONLY = false>
cudaError_t launch_fused_k(Plan p, cudaStream_t st, int max_ctas) {
  using C = FusedCfg<DT, B>;
  const bool dec = p.n_d_items > 0;
  // the ring parks coded tiles (encode launches only; none in the reduce variant)
  // (launches that also decode keep 16 KiB: their decode table follows the ring, 3 CTAs per SM)
  p.ring_bytes = (p.n_e_items > 0) ? (dec ? 16384 : C::ring(RED)) : 0;
  int smem = C::kEncTab + kWarps * C::kWarpBuf + p.ring_bytes + ((dec || RED) ? C::kDecTab : 0);
  if (UZIP_ENC_TMA && p.n_e_items > 0) smem = C::smem(true, RED);  // the stages sit at the end of the full layout
  auto kern = k_fused<DT, B, RED, MINB, DONLY>;
  static int attr_set[kMaxDevices] = {0};  // the attribute applies per device
  const int dev = current_device();
  if (attr_set[dev] < C::smem(true, RED)) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem(true, RED));
    if (e != cudaSuccess) return e;
    attr_set[dev] = C::smem(true, RED);
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  if (occ <= 0) occ = 1;
  const uint64_t items = p.n_t_items + p.n_e_items + p.n_c_items + p.n_d_items;
  int grid = sm_count() * occ;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  // Ranks sharing this GPU (loopback): a launch whose decode items spin on a
  // peer's flags may hold at most 1/share of the slots, so the peer's kernels
  // (the producers it waits for) always find an SM.
#ifndef UZIP_SHARE_ENC_CAP
#define UZIP_SHARE_ENC_CAP 0
#endif
  // Encode-only launches stay uncapped by default: capping them to 1/share did not let a receiver
  // launched after its sender start any earlier on the shared GPU (tile trace: 0 % of its tiles
  // decoded before the sender's last flag either way) and slowed the sender (loopback 1 GiB P2P 2.03-2.15
  // vs 1.98 ms).  A receiver launched first overlaps (98 % of its tiles decoded while the sender runs).
  if (p.share > 1 && (p.n_d_items > 0 || UZIP_SHARE_ENC_CAP) && grid > sm_count() * occ / (int)p.share)
    grid = sm_count() * occ / (int)p.share > 0 ? sm_count() * occ / (int)p.share : 1;
  if ((uint64_t)grid > items) grid = (int)(items ? items : 1);
  kern<<<grid, 256, smem, st>>>(p);
  return cudaGetLastError();
}

template <int DT, int B, bool RED>
cudaError_t launch_fused_t(const Plan &p, cudaStream_t st, int max_ctas) {
  if constexpr (RED) {
    return launch_fused_k<DT, B, RED, UZIP_RED_MINB>(p, st, max_ctas);
  } else {
    if (p.n_e_items > 0) return launch_fused_k<DT, B, RED, UZIP_ENC_MINB>(p, st, max_ctas);
    if (p.n_c_items == 0) return launch_fused_k<DT, B, RED, UZIP_DEC_ONLY_MINB, true>(p, st, max_ctas);
    return launch_fused_k<DT, B, RED, UZIP_DEC_ONLY_MINB>(p, st, max_ctas);
  }
}

// Load every kernel of this dtype/variant into the context now.  CUDA's lazy
// module loading synchronises the context when a kernel is first launched; a
// communicator whose peer kernels spin-wait inside the same context (loopback
// ranks) would then wait for a kernel that waits for it -- measured as a
// 5 s poll timeout in the loopback bench -- so communicators preload.
template <int DT, bool RED>
cudaError_t preload_t() {
  cudaFuncAttributes a;
  cudaError_t e = cudaSuccess;
  if constexpr (RED) {
    e = cudaFuncGetAttributes(&a, k_fused<DT, 1024, true, UZIP_RED_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 2048, true, UZIP_RED_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 4096, true, UZIP_RED_MINB>);
  } else {
    e = cudaFuncGetAttributes(&a, k_fused<DT, 1024, false, UZIP_ENC_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 2048, false, UZIP_ENC_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 4096, false, UZIP_ENC_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 1024, false, UZIP_DEC_ONLY_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 2048, false, UZIP_DEC_ONLY_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 4096, false, UZIP_DEC_ONLY_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 1024, false, UZIP_DEC_ONLY_MINB, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 2048, false, UZIP_DEC_ONLY_MINB, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 4096, false, UZIP_DEC_ONLY_MINB, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 8192, false, UZIP_ENC_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 8192, false, UZIP_DEC_ONLY_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 8192, false, UZIP_DEC_ONLY_MINB, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 16384, false, UZIP_ENC_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 16384, false, UZIP_DEC_ONLY_MINB>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_fused<DT, 16384, false, UZIP_DEC_ONLY_MINB, true>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_hist<DT>);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&a, k_norm<DT>);
  }
  return e;
}

template <int DT, bool RED>
cudaError_t launch_fused_b(const Plan &p, uint32_t B, cudaStream_t st, int max_ctas) {
  switch (B) {
    case 1024: return launch_fused_t<DT, 1024, RED>(p, st, max_ctas);
    case 2048: return launch_fused_t<DT, 2048, RED>(p, st, max_ctas);
    case 4096: return launch_fused_t<DT, 4096, RED>(p, st, max_ctas);
    default:
      // larger blocks (C2 block sweep): codec, P2P, allgather, all-to-all, broadcast; the reduce
      // kernel's accumulators hold kMaxB symbols per warp (the C ABI rejects larger B for reductions)
      if constexpr (RED) {
        return cudaErrorInvalidValue;
      } else {
        if (B == 8192) return launch_fused_t<DT, 8192, RED>(p, st, max_ctas);
        if (B == 16384) return launch_fused_t<DT, 16384, RED>(p, st, max_ctas);
        return cudaErrorInvalidValue;
      }
  }
}

}  // namespace uzip
