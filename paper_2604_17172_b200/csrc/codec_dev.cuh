// codec_dev.cuh -- device pieces of the decoder shared by k_decode (codec.cu)
// and the D items of k_fused (fused.cu): directory sizes, decode-table build
// (a7), 32-lane rANS decode (a8) and the join with the residual plane(s).
#pragma once

#include "uzip_device.cuh"

namespace uzip {

// Directory entry -> payload bytes of a block; flags entries no encoder emits.
__device__ __forceinline__ uint32_t block_size(uint32_t d, uint32_t B, bool &bad) {
  if (d == kRawBlock) return B;
  if (d >= B / 2) {
    bad = true;
    return B;
  }
  const uint32_t sz = (uint32_t)round16(128 + 2ull * d);
  if (sz >= B) bad = true;
  return sz;
}

// Decode table of one chunk: f:12 <<20 | (slot-cdf):12 <<8 | sym:8 (a7).
// All 256 threads; returns false (uniformly) if the table is invalid.  Every
// warp reads the 256 frequencies itself (8 per lane, one 16-byte load) and
// scans them, so the cdf needs no block-wide exchange; warp w owns slots
// [512w, 512w+512): it zeroes them, marks the first slot of each symbol that
// starts there, and each lane fills its 16 slots by a running max over the
// marks (balanced -- filling symbol by symbol left the warp owning the
// dominant exponents with ~128 serial stores).  One block barrier (for the
// per-symbol f/cdf scratch) instead of six; the caller's barrier publishes
// the table.  `scr`: 2 KiB of smem scratch (per-symbol f and cdf).
__device__ __forceinline__ bool build_dtab(const uint16_t *ft, uint32_t *dtab, uint32_t *s_red, uint32_t *scr) {
  (void)s_red;
  const int lane = threadIdx.x & 31, warp = warp_id();
  const uint4 q = ld_cg_v4(ft + 8 * lane);
  const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
  uint32_t f[8], c[8], loc = 0, zero = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    f[k] = (w4[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
    c[k] = loc;
    loc += f[k];
    zero |= f[k] == 0;
  }
  uint32_t incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t tt = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += tt;
  }
  const uint32_t fsum = __shfl_sync(0xFFFFFFFFu, incl, 31);
  if (fsum != kM || __any_sync(0xFFFFFFFFu, zero)) return false;  // same table in every warp: uniform
  const uint32_t base = incl - loc;
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k] += base;
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      scr[8 * lane + k] = f[k];
      scr[256 + 8 * lane + k] = c[k];
    }
  }
  const uint32_t w0 = 512u * (uint32_t)warp;  // this warp's slots [w0, w0 + 512)
  uint4 *d4 = reinterpret_cast<uint4 *>(dtab + w0 + 16 * lane);
#pragma unroll
  for (int i = 0; i < 4; ++i) d4[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  // marks; and the symbol covering slot w0 (the last one starting at or before it)
  uint32_t cover = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if ((c[k] >> 9) == (uint32_t)warp) dtab[c[k]] = 8u * lane + k;  // distinct first slots (f >= 1)
    if (c[k] <= w0) cover = 8u * lane + k;
  }
  for (int o = 16; o; o >>= 1) cover = max(cover, __shfl_xor_sync(0xFFFFFFFFu, cover, o));
  __syncwarp();
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 t = d4[i];
    v[4 * i] = t.x, v[4 * i + 1] = t.y, v[4 * i + 2] = t.z, v[4 * i + 3] = t.w;
  }
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = m = max(m, v[i]);
  uint32_t inc = m;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t tt = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc = max(inc, tt);
  }
  uint32_t pre = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  pre = max(lane == 0 ? 0u : pre, cover);
  __syncthreads();  // scr (warp 0) visible
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t sym = max(pre, v[4 * i + k]);
      const uint32_t slot = w0 + 16u * lane + 4 * i + k;
      e[k] = (scr[sym] << 20) | ((slot - scr[256 + sym]) << 8) | sym;
    }
    d4[i] = make_uint4(e[0], e[1], e[2], e[3]);
  }
  return true;  // the caller's barrier publishes dtab (and frees scr)
}

// Stage n16 16-byte words of a coded block into the warp's smem buffer with cp.async (L2 -> smem,
// .cg: never through L1, the bytes may have been written by a peer GPU): every lane's copies are
// in flight at once and hold no registers (a register-batched copy spilled the decoder).
#ifndef UZIP_DEC_NOCLAMP
#define UZIP_DEC_NOCLAMP 1  // k_decode's staged blocks: no clamp of the word index (1 GiB bf16 0.540 -> 0.524 ms)
#endif
#ifndef UZIP_DEC_PTR
#define UZIP_DEC_PTR 1  // k_decode pairs: word pointers as shared byte addresses updated by IMAD (0.524 -> 0.518 ms)
#endif
#ifndef UZIP_DEC_GE
#define UZIP_DEC_GE 1  // pairs: read address = s - 2*popc(m & lanemask_ge), both IMADs off the old s (no negation MOV)
#endif
#ifndef UZIP_DEC_PAIR_PF
#define UZIP_DEC_PAIR_PF 2  // pairs: residual prefetch distance in 8-round groups
#endif
#ifndef UZIP_DEC_PTRC
#define UZIP_DEC_PTRC 0  // A/B: the clamped pairs (k_fused receivers) use the pointer form too, clamped at word 0
#endif
#ifndef UZIP_DEC_RING16
#define UZIP_DEC_RING16 0  // A/B: pairs store both chains' symbols of a round with one 16-bit store
#endif
#ifndef UZIP_DEC_TADDR
#define UZIP_DEC_TADDR 0  // A/B: table address as LOP3 + IMAD
#endif
#ifndef UZIP_DEC_HI
#define UZIP_DEC_HI 0  // A/B: the state update's shifts as high multiplies (FMA pipe)
#endif
#ifndef UZIP_STAGE_ASYNC
#define UZIP_STAGE_ASYNC 1
#endif
__device__ __forceinline__ void stage_block(const uint8_t *src, uint32_t n16, uint8_t *pay) {
  const uint32_t lane = threadIdx.x & 31;
  if (UZIP_STAGE_ASYNC) {
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(pay);
    for (uint32_t i = lane; i < n16; i += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s0 + 16 * i), "l"(src + 16 * i) : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  } else {
    for (uint32_t i = lane; i < n16; i += 32) reinterpret_cast<uint4 *>(pay)[i] = ld_cg_v4(src + 16 * i);
  }
  __syncwarp();
}

// a8: one warp decodes the K-word block in `pay` (smem) into 8-bit symbols.
// Returns false if the block is corrupt (word overrun, end state != L).
template <int B>
__device__ __forceinline__ bool rans_decode_warp(const uint8_t *pay, uint32_t K, const uint32_t *dtab,
                                                 uint8_t *symb) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint32_t *pay32 = reinterpret_cast<const uint32_t *>(pay);
  const uint16_t *pay16 = reinterpret_cast<const uint16_t *>(pay) + 64;
  uint32_t x = pay32[lane];
  int32_t p = (int32_t)K;
#pragma unroll 8
  for (uint32_t j = 0; j < (uint32_t)(B / 32); ++j) {
    const uint32_t e = dtab[x & (kM - 1)];
    symb[j * 32 + lane] = (uint8_t)e;
    x = (e >> 20) * (x >> kProbBits) + ((e >> 8) & 0xFFFu);
    const bool need = x < kL;
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
    p -= __popc(m);
    // the k renormalizing lanes take the last k unread words in lane order;
    // a corrupt stream drives p negative: clamp the index, fail at the end
    const int32_t idx = max(p + __popc(m & lt), 0);
    const uint32_t w = pay16[idx];
    x = need ? ((x << 16) | w) : x;
  }
  return !(p != 0 || __any_sync(0xFFFFFFFFu, x != kL));
}

// Join 8-bit symbols (smem) with the residual plane(s) of block b; stores B
// elements of DT at dst (128-bit stores).
template <int DT, int B>
__device__ __forceinline__ void join_block(const uint8_t *syms, const uint8_t *stream, const StreamGeom &g,
                                           uint64_t b, uint8_t *dst) {
  const int lane = threadIdx.x & 31;
  if (DT == kF32) {
#pragma unroll 4
    for (uint32_t e = lane * 4; e < (uint32_t)B; e += 128) {
      const uint32_t s4 = *reinterpret_cast<const uint32_t *>(syms + e);
      const uint2 lo = ld_cg_v2(stream + g.off_res0 + 2 * (b * B + e));
      const uint32_t h4 = ld_cg_u32c(stream + g.off_res1 + b * B + e);
      st_any16(dst + 4 * e, join4_f32(s4, lo, h4));
    }
  } else if (DT == kE5M2) {  // the symbols are the bytes (R24)
#pragma unroll 4
    for (uint32_t e = lane * 16; e < (uint32_t)B; e += 512)
      st_any16(dst + e, *reinterpret_cast<const uint4 *>(syms + e));
  } else {
#pragma unroll 4
    for (uint32_t e = lane * 8; e < (uint32_t)B; e += 256) {
      const uint2 s8 = *reinterpret_cast<const uint2 *>(syms + e);
      const uint2 r8 = ld_cg_v2(stream + g.off_res0 + b * B + e);
      uint4 o;
      if (DT == kBF16) {
        join4_bf16(s8.x, r8.x, o.x, o.y);
        join4_bf16(s8.y, r8.y, o.z, o.w);
      } else if (DT == kE4M3) {
        join4_e4m3(s8.x, r8.x, o.x, o.y);
        join4_e4m3(s8.y, r8.y, o.z, o.w);
      } else {
        join4_f16(s8.x, r8.x, o.x, o.y);
        join4_f16(s8.y, r8.y, o.z, o.w);
      }
      st_any16(dst + 2 * e, o);
    }
  }
}

// a8 + join, streamed: one warp decodes a coded block 8 rounds at a time.
// The 8 rounds x 32 lanes of symbols land in a 256-byte ring (element order
// within the group), each lane then joins ITS 8 consecutive elements with the
// residual bytes it prefetched kPF groups earlier and stores 16 bytes (fp32:
// 32).  Per warp this needs the staged payload plus 256 bytes of smem, so more
// warps (rANS chains) fit on an SM.  Returns false on a corrupt block.
// Epilogue of the streamed decoder: receives the 8 joined elements of a lane
// (element offset e0 within the block; fp32 uses both vectors).
struct StoreEpi {
  uint8_t *dst;
  template <int DT>
  __device__ __forceinline__ void apply(uint32_t e0, uint4 a, uint4 b) const {
    if (DT == kF32) {
      st_any16(dst + 4 * e0, a);
      st_any16(dst + 4 * e0 + 16, b);
    } else if (DT == kE5M2) {
      st_any8(dst + e0, make_uint2(a.x, a.y));  // 8 symbols = 8 output bytes
    } else {
      st_any16(dst + 2 * e0, a);  // e0 counts groups: 2 bytes each (bf16, f16, e4m3 pair)
    }
  }
};

// NOCLAMP: `pay` is in k_decode's shared memory, where a corrupt stream's word index (at most B words
// below 0) still reads inside the CTA's window (the payload areas sit above the 17 KB table + offsets);
// in global memory (blocks decoded in place) or k_fused's layout the index is clamped at 0.
template <int DT, int B, class Epi, bool NOCLAMP = false>
__device__ __forceinline__ bool decode_join_warp_epi(const uint8_t *pay, uint32_t K, const uint32_t *dtab,
                                                     uint8_t *ring, const uint8_t *stream, const StreamGeom &g,
                                                     uint64_t b, const Epi &epi) {
  constexpr int kGroups = B / 256;
#ifndef UZIP_DEC_PF
#define UZIP_DEC_PF 4
#endif
  constexpr int kPF = UZIP_DEC_PF;  // residual prefetch distance in groups (divides kGroups)
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint32_t *pay32 = reinterpret_cast<const uint32_t *>(pay);
  const uint16_t *pay16 = reinterpret_cast<const uint16_t *>(pay) + 64;
  const uint8_t *res0 = stream + g.off_res0 + (DT == kF32 ? 2 : 1) * (b * B) + (DT == kF32 ? 16 : 8) * lane;
  const uint8_t *res1 = stream + g.off_res1 + b * B + 8 * lane;  // fp32 hi8 plane
  uint4 rlo[kPF];   // fp32: lo16 of 8 elements; bf16/f16/e4m3: .x/.y = 8 residual bytes; e5m2: none
  uint2 rhi[kPF];   // fp32: hi8 of 8 elements
#pragma unroll
  for (int i = 0; i < kPF; ++i) {
    if (DT == kF32) {
      rlo[i] = ld_cg_v4(res0 + 512 * i);
      rhi[i] = ld_cg_v2(res1 + 256 * i);
    } else if (DT != kE5M2) {
      const uint2 v = ld_cg_v2(res0 + 256 * i);
      rlo[i] = make_uint4(v.x, v.y, 0, 0);
    }
  }
  uint32_t x = pay32[lane];
  int32_t p = (int32_t)K;
#pragma unroll 1
  for (int g0 = 0; g0 < kGroups; g0 += kPF) {
#pragma unroll
    for (int q = 0; q < kPF; ++q) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t e = dtab[x & (kM - 1)];
        ring[u * 32 + lane] = (uint8_t)e;
        x = (e >> 20) * (x >> kProbBits) + ((e >> 8) & 0xFFFu);
        const bool need = x < kL;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, need);
        p -= __popc(m);
        // the k renormalizing lanes take the last k unread words in lane order;
        // a corrupt stream drives p negative: clamp the index (or not, NOCLAMP), fail at the end
        const int32_t idx = NOCLAMP ? p + __popc(m & lt) : max(p + __popc(m & lt), 0);
        const uint32_t w = pay16[idx];
        x = need ? ((x << 16) | w) : x;
      }
      __syncwarp();
      const uint2 s8 = *reinterpret_cast<const uint2 *>(ring + 8 * lane);
      const int gi = g0 + q;
      const uint32_t e0 = 256 * gi + 8 * lane;
      if (DT == kF32) {
        epi.template apply<DT>(e0, join4_f32(s8.x, make_uint2(rlo[q].x, rlo[q].y), rhi[q].x),
                               join4_f32(s8.y, make_uint2(rlo[q].z, rlo[q].w), rhi[q].y));
      } else if (DT == kE5M2) {
        const uint4 v = make_uint4(s8.x, s8.y, 0, 0);
        epi.template apply<DT>(e0, v, v);
      } else {
        uint4 v;
        if (DT == kBF16) {
          join4_bf16(s8.x, rlo[q].x, v.x, v.y);
          join4_bf16(s8.y, rlo[q].y, v.z, v.w);
        } else if (DT == kE4M3) {
          join4_e4m3(s8.x, rlo[q].x, v.x, v.y);
          join4_e4m3(s8.y, rlo[q].y, v.z, v.w);
        } else {
          join4_f16(s8.x, rlo[q].x, v.x, v.y);
          join4_f16(s8.y, rlo[q].y, v.z, v.w);
        }
        epi.template apply<DT>(e0, v, v);
      }
      if (gi + kPF < kGroups && DT != kE5M2) {
        if (DT == kF32) {
          rlo[q] = ld_cg_v4(res0 + 512 * (gi + kPF));
          rhi[q] = ld_cg_v2(res1 + 256 * (gi + kPF));
        } else {
          const uint2 v = ld_cg_v2(res0 + 256 * (gi + kPF));
          rlo[q] = make_uint4(v.x, v.y, 0, 0);
        }
      }
      __syncwarp();
    }
  }
  return !(p != 0 || __any_sync(0xFFFFFFFFu, x != kL));
}

// Two coded blocks per warp, their rANS chains interleaved round by round (a8): the decoder is bound by
// the latency of its table-lookup -> renormalization -> word-fetch chain, and a second independent
// chain in the same warp hides half of it.  One residual plane of one byte per symbol (bf16, f16,
// e4m3): pays / rings / residual prefetches per block; `ok` reports each block.
template <int DT, int B, bool NOCLAMP = (UZIP_DEC_NOCLAMP != 0)>
__device__ __forceinline__ void decode_join_warp2(const uint8_t *payA, uint32_t KA, const uint8_t *payB, uint32_t KB,
                                                  const uint32_t *dtab, uint8_t *ringA, uint8_t *ringB,
                                                  const uint8_t *stream, const StreamGeom &g, uint64_t bA,
                                                  uint64_t bB, uint8_t *dstA, uint8_t *dstB, bool &okA, bool &okB) {
  static_assert(DT == kBF16 || DT == kF16 || DT == kE4M3, "one residual byte per symbol");
  constexpr int kGroups = B / 256;
  constexpr int kPF = UZIP_DEC_PAIR_PF;  // residual prefetch distance in groups, per block (1 / 4: 0.542 / 0.553 vs 0.540 ms at 4 CTAs)
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint16_t *wA = reinterpret_cast<const uint16_t *>(payA) + 64;
  const uint16_t *wB = reinterpret_cast<const uint16_t *>(payB) + 64;
  const uint8_t *resA = stream + g.off_res0 + bA * B + 8 * lane;
  const uint8_t *resB = stream + g.off_res0 + bB * B + 8 * lane;
  uint2 rA[kPF], rB[kPF];
#pragma unroll
  for (int i = 0; i < kPF; ++i) {
    rA[i] = ld_cg_v2(resA + 256 * i);
    rB[i] = ld_cg_v2(resB + 256 * i);
  }
  uint32_t xA = reinterpret_cast<const uint32_t *>(payA)[lane], xB = reinterpret_cast<const uint32_t *>(payB)[lane];
  int32_t pA = (int32_t)KA, pB = (int32_t)KB;
#if UZIP_DEC_PTR
  const uint32_t sA0 = (uint32_t)__cvta_generic_to_shared(wA), sB0 = (uint32_t)__cvta_generic_to_shared(wB);
  uint32_t sA = sA0 + 2u * KA, sB = sB0 + 2u * KB;
  const uint32_t two = __shfl_sync(0xFFFFFFFFu, UZIP_DEC_GE ? 0xFFFFFFFEu : 2u, 0);  // +-2, opaque to ptxas: keeps the updates IMADs
#if UZIP_DEC_GE
  const uint32_t ge = ~lt;
#endif
#endif
#if UZIP_DEC_TADDR
  const uint32_t tbase = (uint32_t)__cvta_generic_to_shared(dtab);
  const uint32_t four = __shfl_sync(0xFFFFFFFFu, 4u, 0);  // opaque: the index scaling stays one IMAD
#endif
#if UZIP_DEC_HI
  // opaque 2^20 / 2^12 / -4096: x >> 12 = hi(x * 2^20), freq = e >> 20 = hi(e * 2^12); with e >> 8 = freq << 12 | bias,
  // x' = freq * (x >> 12) + bias = freq * ((x >> 12) - 4096) + (e >> 8)  (mod 2^32)
  const uint32_t k20 = __shfl_sync(0xFFFFFFFFu, 1u << 20, 0), k12 = __shfl_sync(0xFFFFFFFFu, 1u << 12, 0);
  const uint32_t m4096 = __shfl_sync(0xFFFFFFFFu, 0u - 4096u, 0);
#endif
#pragma unroll 1
  for (int g0 = 0; g0 < kGroups; g0 += kPF) {
#pragma unroll
    for (int q = 0; q < kPF; ++q) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#if UZIP_DEC_TADDR
        // table byte address = (x & 4095) * 4 + base as LOP3 + IMAD: two ops between x and the lookup
        // (ptxas emitted IMAD.SHL + LOP3 + IADD)
        uint32_t eA, eB;
        asm("{\n\t.reg .b32 i, a;\n\tand.b32 i, %1, 4095;\n\tmad.lo.u32 a, i, %2, %3;\n\tld.shared.u32 %0, [a];\n\t}"
            : "=r"(eA) : "r"(xA), "r"(four), "r"(tbase));
        asm("{\n\t.reg .b32 i, a;\n\tand.b32 i, %1, 4095;\n\tmad.lo.u32 a, i, %2, %3;\n\tld.shared.u32 %0, [a];\n\t}"
            : "=r"(eB) : "r"(xB), "r"(four), "r"(tbase));
#else
        const uint32_t eA = dtab[xA & (kM - 1)];
        const uint32_t eB = dtab[xB & (kM - 1)];
#endif
#if UZIP_DEC_RING16
        // both chains' symbols of this round in one 16-bit store (rounds 0-3 in ringA, 4-7 in ringB)
        *reinterpret_cast<uint16_t *>((u < 4 ? ringA : ringB) + ((u & 3) * 32 + lane) * 2) =
            (uint16_t)__byte_perm(eA, eB, 0x0040);
#else
        ringA[u * 32 + lane] = (uint8_t)eA;
        ringB[u * 32 + lane] = (uint8_t)eB;
#endif
#if UZIP_DEC_HI
        {
#if UZIP_DEC_HI == 1
          uint32_t hA, hB;
          asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(hA) : "r"(xA), "r"(k20), "r"(m4096));
          asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(hB) : "r"(xB), "r"(k20), "r"(m4096));
          xA = __umulhi(eA, k12) * hA + (eA >> 8);
          xB = __umulhi(eB, k12) * hB + (eB >> 8);
#elif UZIP_DEC_HI == 2
          xA = __umulhi(eA, k12) * __umulhi(xA, k20) + ((eA >> 8) & 0xFFFu);
          xB = __umulhi(eB, k12) * __umulhi(xB, k20) + ((eB >> 8) & 0xFFFu);
#else
          const uint32_t fA = __umulhi(eA, k12), fB = __umulhi(eB, k12);
          xA = fA * __umulhi(xA, k20) + (fA * m4096 + (eA >> 8));
          xB = fB * __umulhi(xB, k20) + (fB * m4096 + (eB >> 8));
#endif
        }
#else
        xA = (eA >> 20) * (xA >> kProbBits) + ((eA >> 8) & 0xFFFu);
        xB = (eB >> 20) * (xB >> kProbBits) + ((eB >> 8) & 0xFFFu);
#endif
        const bool nA = xA < kL, nB = xB < kL;
        const uint32_t mA = __ballot_sync(0xFFFFFFFFu, nA), mB = __ballot_sync(0xFFFFFFFFu, nB);
        uint32_t wa, wb;
#if UZIP_DEC_PTR
        if constexpr (NOCLAMP || UZIP_DEC_PTRC) {
          // shared-memory byte addresses of the read pointers, updated and offset by IMADs (FMA pipe)
          // instead of the index add + address IADD3 on the saturated ALU pipe
#if UZIP_DEC_GE
          // the k renormalizing lanes read the last k unread words: lane l's word sits popc(m & ge_l) words
          // below the old pointer (two = -2 here); both IMADs read the old pointer
          uint32_t aA = sA + two * __popc(mA & ge), aB = sB + two * __popc(mB & ge);
          if constexpr (!NOCLAMP) {  // k_fused's layout: a corrupt stream's reads stop at word 0
            aA = (uint32_t)max((int32_t)aA, (int32_t)sA0);
            aB = (uint32_t)max((int32_t)aB, (int32_t)sB0);
          }
          sA += two * __popc(mA);
          sB += two * __popc(mB);
#else
          sA -= two * __popc(mA);
          sB -= two * __popc(mB);
          uint32_t aA = sA + two * __popc(mA & lt), aB = sB + two * __popc(mB & lt);
          if constexpr (!NOCLAMP) {
            aA = (uint32_t)max((int32_t)aA, (int32_t)sA0);
            aB = (uint32_t)max((int32_t)aB, (int32_t)sB0);
          }
#endif
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(wa) : "r"(aA));
          asm volatile("ld.shared.u16 %0, [%1];" : "=r"(wb) : "r"(aB));
        } else
#endif
        {
        pA -= __popc(mA);
        pB -= __popc(mB);
        // NOCLAMP (k_decode): a corrupt stream drives p below 0 by at most B words, which stays inside
        // the CTA's shared memory (the payload areas sit above the 17 KB table + offsets); p != 0 at the
        // end reports it.  k_fused's layout clamps.
        const int32_t ia = pA + __popc(mA & lt), ib = pB + __popc(mB & lt);
        wa = wA[NOCLAMP ? ia : max(ia, 0)], wb = wB[NOCLAMP ? ib : max(ib, 0)];
        }
        xA = nA ? ((xA << 16) | wa) : xA;
        xB = nB ? ((xB << 16) | wb) : xB;
      }
      __syncwarp();
      const int gi = g0 + q;
      const uint32_t e0 = 256 * gi + 8 * lane;
#if UZIP_DEC_RING16
      // elements 8 lane .. 8 lane + 7 = round lane / 4, lanes 8 (lane % 4) ..: 16 bytes, A and B interleaved
      const uint4 v16 = *reinterpret_cast<const uint4 *>((lane < 16 ? ringA : ringB) + (lane & 15) * 16);
      const uint2 sA = make_uint2(__byte_perm(v16.x, v16.y, 0x6420), __byte_perm(v16.z, v16.w, 0x6420));
      const uint2 sB = make_uint2(__byte_perm(v16.x, v16.y, 0x7531), __byte_perm(v16.z, v16.w, 0x7531));
#else
      const uint2 sA = *reinterpret_cast<const uint2 *>(ringA + 8 * lane);
      const uint2 sB = *reinterpret_cast<const uint2 *>(ringB + 8 * lane);
#endif
      uint4 vA, vB;
      if (DT == kBF16) {
        join4_bf16(sA.x, rA[q].x, vA.x, vA.y);
        join4_bf16(sA.y, rA[q].y, vA.z, vA.w);
        join4_bf16(sB.x, rB[q].x, vB.x, vB.y);
        join4_bf16(sB.y, rB[q].y, vB.z, vB.w);
      } else if (DT == kE4M3) {
        join4_e4m3(sA.x, rA[q].x, vA.x, vA.y);
        join4_e4m3(sA.y, rA[q].y, vA.z, vA.w);
        join4_e4m3(sB.x, rB[q].x, vB.x, vB.y);
        join4_e4m3(sB.y, rB[q].y, vB.z, vB.w);
      } else {
        join4_f16(sA.x, rA[q].x, vA.x, vA.y);
        join4_f16(sA.y, rA[q].y, vA.z, vA.w);
        join4_f16(sB.x, rB[q].x, vB.x, vB.y);
        join4_f16(sB.y, rB[q].y, vB.z, vB.w);
      }
      st_any16(dstA + 2 * e0, vA);
      st_any16(dstB + 2 * e0, vB);
      if (gi + kPF < kGroups) {
        rA[q] = ld_cg_v2(resA + 256 * (gi + kPF));
        rB[q] = ld_cg_v2(resB + 256 * (gi + kPF));
      }
      __syncwarp();
    }
  }
#if UZIP_DEC_PTR
  if constexpr (NOCLAMP || UZIP_DEC_PTRC) {
    pA = (int32_t)(sA - sA0) / 2;
    pB = (int32_t)(sB - sB0) / 2;
  }
#endif
  okA = !(pA != 0 || __any_sync(0xFFFFFFFFu, xA != kL));
  okB = !(pB != 0 || __any_sync(0xFFFFFFFFu, xB != kL));
}

template <int DT, int B, bool NOCLAMP = false>
__device__ __forceinline__ bool decode_join_warp(const uint8_t *pay, uint32_t K, const uint32_t *dtab,
                                                 uint8_t *ring, const uint8_t *stream, const StreamGeom &g,
                                                 uint64_t b, uint8_t *dst) {
  StoreEpi epi{dst};
  return decode_join_warp_epi<DT, B, StoreEpi, NOCLAMP>(pay, K, dtab, ring, stream, g, b, epi);
}

}  // namespace uzip
