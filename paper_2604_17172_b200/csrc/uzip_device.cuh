// uzip_device.cuh -- device-side building blocks of the Uzip codec for sm_100a.
//
// This is the CUDA path's own restatement of the method (it shares nothing with
// oracle/): the float split of Step 1, the localized tables
// of P:357-370, warp-per-block rANS and the decode
// (P:391).  Stream layout: DESIGN.md section 2.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace uzip {

// ---------------------------------------------------------------- format constants
constexpr uint32_t kProbBits = 12;             // P (table precision)
constexpr uint32_t kM = 1u << kProbBits;        // 4096
constexpr uint32_t kLBits = 15;                 // states live in [2^15, 2^31)
constexpr uint32_t kL = 1u << kLBits;
constexpr uint32_t kLanes = 32;                 // interleaved states per block (one warp)
constexpr uint32_t kHeaderBytes = 64;
constexpr uint32_t kRawBlock = 0xFFFFFFFFu;
constexpr uint32_t kVersion = 1;
constexpr int kWarps = 8;                       // warps per CTA in the codec kernels
constexpr uint32_t kTileBlocks = kWarps;        // blocks per look-back tile
constexpr uint32_t kMaxB = 4096;                // largest block of the reduce kernels (fp32 accumulators)
constexpr uint32_t kMaxCodecB = 16384;          // largest block of the codec / P2P / allgather kernels
// block sizes the GPU kernels are instantiated for (C2 block sweep)
__host__ __device__ constexpr bool gpu_block_ok(uint32_t B) {
  return B == 1024 || B == 2048 || B == 4096 || B == 8192 || B == 16384;
}

enum Dtype : int { kBF16 = 0, kF16 = 1, kF32 = 2, kE4M3 = 3, kE5M2 = 4 };
constexpr int kNumDtypes = 5;

__host__ __device__ constexpr uint32_t elem_bytes(int dt) { return dt == kF32 ? 4u : (dt >= kE4M3 ? 1u : 2u); }
// A symbol group is the input that yields one symbol: one element, or a pair
// of e4m3 elements (R23).  Blocks, chunks and samples count groups.
__host__ __device__ constexpr uint32_t group_elems(int dt) { return dt == kE4M3 ? 2u : 1u; }
__host__ __device__ constexpr uint32_t group_bytes(int dt) { return elem_bytes(dt) * group_elems(dt); }
// residual plane bytes per group (f32 has two planes: lo16 + hi8)
__host__ __device__ constexpr uint32_t res_bytes(int dt) { return dt == kF32 ? 3u : (dt == kE5M2 ? 0u : 1u); }
__host__ __device__ constexpr uint64_t round16(uint64_t v) { return (v + 15u) & ~uint64_t(15); }

// Section offsets of a UZB1 stream, computed the same way
// on host and device from the header fields.
// n counts elements; n_blocks / n_coded count symbol groups; eb is the input
// bytes per group (= element bytes except e4m3 pairs).
struct StreamGeom {
  uint64_t n, n_blocks, n_coded, n_chunks;
  uint32_t B, CB, S, global, dtype, eb;
  uint32_t cb_log2;                       // log2(CB) if CB is a power of 2 (> 1), else 0
  uint64_t off_res0, off_res1, off_tab, off_coff, off_dir, off_pay;

  __host__ __device__ void init(int dt, uint64_t n_, uint32_t B_, uint32_t CB_, uint32_t S_, bool global_) {
    dtype = (uint32_t)dt;
    eb = group_bytes(dt);
    n = n_;
    B = B_;
    n_blocks = (n / group_elems(dt)) / B;
    n_coded = n_blocks * B;
    global = global_ ? 1u : 0u;
    if (global_) {
      CB = n_blocks ? (uint32_t)n_blocks : 1u;
      S = 0;
    } else {
      CB = CB_;
      S = S_;
    }
    n_chunks = (n_blocks + CB - 1) / CB;
    cb_log2 = 0;
    if (CB > 1 && (CB & (CB - 1)) == 0)
      while ((1u << cb_log2) < CB) ++cb_log2;
    off_res0 = kHeaderBytes;
    if (dt == kF32) {
      off_res1 = off_res0 + 2 * n_coded;
      off_tab = round16(off_res1 + n_coded);
    } else {
      off_res1 = off_res0;
      off_tab = round16(off_res0 + res_bytes(dt) * n_coded);
    }
    off_coff = off_tab + 512 * n_chunks;
    off_dir = round16(off_coff + 8 * n_chunks);
    off_pay = round16(off_dir + 4 * n_blocks);
  }
  __host__ __device__ uint64_t off_tail(uint64_t payload) const { return round16(off_pay + payload); }
  // raw tail: the elements after the last whole block
  __host__ __device__ uint64_t tail_bytes() const { return (n - n_coded * group_elems(dtype)) * elem_bytes(dtype); }
  __host__ __device__ uint64_t total(uint64_t payload) const { return off_tail(payload) + tail_bytes(); }
  __host__ __device__ uint64_t n_tiles() const { return (n_blocks + kTileBlocks - 1) / kTileBlocks; }
  __host__ __device__ uint32_t chunk_blocks_of(uint64_t c) const {
    uint64_t left = n_blocks - c * CB;
    return (uint32_t)(left < CB ? left : CB);
  }
  __host__ __device__ uint32_t sample_len(uint64_t c) const {
    uint64_t syms = (uint64_t)chunk_blocks_of(c) * B;
    return (uint32_t)((S == 0 || S > syms) ? syms : S);
  }
};

// Chunk of block b: 32-bit division (block indices fit 32 bits: the directory is u32), which
// compiles inline instead of the 64-bit division's runtime call.
__host__ __device__ __forceinline__ uint32_t chunk_of(const StreamGeom &g, uint64_t b) {
  return g.cb_log2 ? (uint32_t)b >> g.cb_log2 : (uint32_t)b / g.CB;  // default CB (1024 / 512) is a power of 2
}

// Decoder control words at the start of the caller's workspace (uzip_decompress): the first error
// and the CTA arrival counter, both reset by the last CTA (the encoder's workspace is EncWs, plan.h).
struct CodecWs {
  uint32_t *err;          // k_decode first error (self-resetting)
  uint32_t *dec_arrive;   // k_decode CTA arrivals (self-resetting)
  __host__ __device__ static CodecWs carve(void *base) {
    CodecWs w;
    uint8_t *p = (uint8_t *)base;
    w.err = (uint32_t *)(p + 4);
    w.dec_arrive = (uint32_t *)(p + 8);
    return w;
  }
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint4 ldg_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void *p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ldg_nc_u32(const void *p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ uint4 ld_cg_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_cg_v2(const void *p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_cg_u32c(const void *p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint16_t ld_cg_u16(const void *p) {
  uint16_t r;
  asm volatile("ld.global.cg.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}
// Cross-GPU flag protocol (a12): payload stores, then a system-scope release
// of the flag in the consumer's memory; the consumer polls with acquire.
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_gpu_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// NVLS multicast stores (f1): one store to a multicast address is replicated by the NVSwitch into
// every GPU bound to the multicast object (bit patterns travel unchanged: .f32 is only the width).
__device__ __forceinline__ void mc_store_v4(void *mc, uint4 v) {
  asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_store_v2(void *mc, uint2 v) {
  asm volatile("multimem.st.weak.global.v2.f32 [%0], {%1, %2};" ::"l"(mc), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void mc_store_b32(void *mc, uint32_t v) {
  asm volatile("multimem.st.weak.global.b32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
}
// Release of a tile flag to every bound GPU after the tile's multicast data stores.
__device__ __forceinline__ void mc_release_sys_u64(void *mc, unsigned long long v) {
  asm volatile("fence.proxy.alias;\n\tmultimem.st.release.sys.global.b64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// 16-byte store to an address that is only element-aligned (allgather slices
// of ragged counts); the alignment test is warp-uniform on every call site.
__device__ __forceinline__ void st_any16(uint8_t *p, uint4 v) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 15) == 0) {
    *reinterpret_cast<uint4 *>(p) = v;
  } else if ((a & 3) == 0) {
    uint32_t *q = reinterpret_cast<uint32_t *>(p);
    q[0] = v.x, q[1] = v.y, q[2] = v.z, q[3] = v.w;
  } else if ((a & 1) == 0) {
    uint16_t *q = reinterpret_cast<uint16_t *>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) q[2 * i] = (uint16_t)w[i], q[2 * i + 1] = (uint16_t)(w[i] >> 16);
  } else {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
  }
}
__device__ __forceinline__ void st_any8(uint8_t *p, uint2 v) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & 7) == 0) {
    *reinterpret_cast<uint2 *>(p) = v;
  } else {
    const uint32_t w[2] = {v.x, v.y};
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
  }
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
// Warp index as a value the compiler can prove warp-uniform (a broadcast), so
// warp-collective code under warp-indexed control flow compiles to plain
// VOTE/SHFL instead of WARPSYNC.COLLECTIVE sequences (measured in SASS).
__device__ __forceinline__ int warp_id() { return __shfl_sync(0xFFFFFFFFu, (int)(threadIdx.x >> 5), 0); }
__device__ __forceinline__ uint64_t uniform_u64(uint64_t v) {
  const uint32_t lo = __shfl_sync(0xFFFFFFFFu, (uint32_t)v, 0), hi = __shfl_sync(0xFFFFFFFFu, (uint32_t)(v >> 32), 0);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// (m & a) | (~m & b) as one LOP3
__device__ __forceinline__ uint32_t bitselect(uint32_t m, uint32_t a, uint32_t b) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(r) : "r"(m), "r"(a), "r"(b));
  return r;
}

// ---------------------------------------------------------------- a1 split / join
// Split of one 16-byte vector into symbols and residual (DESIGN.md
// section 2).  Byte-permute forms: 1.5 ALU ops per element.
// bf16 (s:15 e:14..7 m:6..0): symbol = e, residual = s<<7 | m.
__device__ __forceinline__ void split4_bf16(uint32_t w0, uint32_t w1, uint32_t &sym4, uint32_t &res4) {
  sym4 = __byte_perm(w0 >> 7, w1 >> 7, 0x6420);
  uint32_t lo = __byte_perm(w0, w1, 0x6420);
  uint32_t hi = __byte_perm(w0, w1, 0x7531);
  res4 = bitselect(0x80808080u, hi, lo);  // (hi & 0x80..) | (lo & 0x7F..) in one LOP3
}
// f16: symbol = high byte, residual = low byte (R3).
__device__ __forceinline__ void split4_f16(uint32_t w0, uint32_t w1, uint32_t &sym4, uint32_t &res4) {
  sym4 = __byte_perm(w0, w1, 0x7531);
  res4 = __byte_perm(w0, w1, 0x6420);
}
// f32 (s:31 e:30..23 m:22..0): symbol = e, lo16 = m[15:0], hi8 = s<<7 | m[22:16].
__device__ __forceinline__ void split4_f32(uint4 w, uint32_t &sym4, uint2 &lo, uint32_t &hi4) {
  uint32_t a = __byte_perm(w.x >> 23, w.y >> 23, 0x0040);
  uint32_t b = __byte_perm(w.z >> 23, w.w >> 23, 0x0040);
  sym4 = __byte_perm(a, b, 0x5410);
  lo.x = __byte_perm(w.x, w.y, 0x5410);
  lo.y = __byte_perm(w.z, w.w, 0x5410);
  uint32_t x01 = __byte_perm(w.x, w.y, 0x7362);
  uint32_t x23 = __byte_perm(w.z, w.w, 0x7362);
  uint32_t b2 = __byte_perm(x01, x23, 0x5410);
  uint32_t b3 = __byte_perm(x01, x23, 0x7632);
  hi4 = (b2 & 0x7F7F7F7Fu) | (b3 & 0x80808080u);
}

__device__ __forceinline__ void join4_bf16(uint32_t sym4, uint32_t res4, uint32_t &w0, uint32_t &w1) {
  uint32_t hb = (res4 & 0x80808080u) | ((sym4 >> 1) & 0x7F7F7F7Fu);
  uint32_t lb = ((sym4 << 7) & 0x80808080u) | (res4 & 0x7F7F7F7Fu);
  w0 = __byte_perm(lb, hb, 0x5140);
  w1 = __byte_perm(lb, hb, 0x7362);
}
__device__ __forceinline__ void join4_f16(uint32_t sym4, uint32_t res4, uint32_t &w0, uint32_t &w1) {
  w0 = __byte_perm(res4, sym4, 0x5140);
  w1 = __byte_perm(res4, sym4, 0x7362);
}
// e4m3 pairs (R23): 8 input bytes = 4 groups (a, b); symbol =
// exp_a<<4 | exp_b, residual = s_a<<7 | m_a<<4 | s_b<<3 | m_b.
__device__ __forceinline__ void split4_e4m3(uint32_t w0, uint32_t w1, uint32_t &sym4, uint32_t &res4) {
  const uint32_t A = __byte_perm(w0, w1, 0x6420), Bv = __byte_perm(w0, w1, 0x7531);  // a's, b's
  sym4 = ((A << 1) & 0xF0F0F0F0u) | ((Bv >> 3) & 0x0F0F0F0Fu);
  res4 = (A & 0x80808080u) | ((A << 4) & 0x70707070u) | ((Bv >> 4) & 0x08080808u) | (Bv & 0x07070707u);
}
__device__ __forceinline__ void join4_e4m3(uint32_t sym4, uint32_t res4, uint32_t &w0, uint32_t &w1) {
  const uint32_t A = (res4 & 0x80808080u) | ((sym4 >> 1) & 0x78787878u) | ((res4 >> 4) & 0x07070707u);
  const uint32_t Bv = ((res4 << 4) & 0x80808080u) | ((sym4 << 3) & 0x78787878u) | (res4 & 0x07070707u);
  w0 = __byte_perm(A, Bv, 0x5140);
  w1 = __byte_perm(A, Bv, 0x7362);
}
__device__ __forceinline__ uint4 join4_f32(uint32_t sym4, uint2 lo, uint32_t hi4) {
  uint32_t b2 = ((sym4 << 7) & 0x80808080u) | (hi4 & 0x7F7F7F7Fu);
  uint32_t b3 = (hi4 & 0x80808080u) | ((sym4 >> 1) & 0x7F7F7F7Fu);
  uint32_t h01 = __byte_perm(b2, b3, 0x5140);
  uint32_t h23 = __byte_perm(b2, b3, 0x7362);
  uint4 r;
  r.x = __byte_perm(lo.x, h01, 0x5410);
  r.y = __byte_perm(lo.x, h01, 0x7632);
  r.z = __byte_perm(lo.y, h23, 0x5410);
  r.w = __byte_perm(lo.y, h23, 0x7632);
  return r;
}

// Symbols per 16-byte input vector, and the symbols of one vector as
// little-endian symbol words (a1 for every dtype; residual planes are split
// by the encoder itself).
template <int DT>
struct VecTraits {
  static constexpr int kSym = DT == kF32 ? 4 : (DT == kE5M2 ? 16 : 8);
};
template <int DT>
__device__ __forceinline__ void vec_symbols(uint4 w, uint32_t sw[4]) {
  uint32_t r;
  if (DT == kBF16) {
    split4_bf16(w.x, w.y, sw[0], r);
    split4_bf16(w.z, w.w, sw[1], r);
  } else if (DT == kF16) {
    split4_f16(w.x, w.y, sw[0], r);
    split4_f16(w.z, w.w, sw[1], r);
  } else if (DT == kE4M3) {
    split4_e4m3(w.x, w.y, sw[0], r);
    split4_e4m3(w.z, w.w, sw[1], r);
  } else if (DT == kE5M2) {  // R24: every byte is a symbol
    sw[0] = w.x, sw[1] = w.y, sw[2] = w.z, sw[3] = w.w;
  } else {
    uint2 lo;
    split4_f32(w, sw[0], lo, r);
  }
}
// symbol i of a group-ordered input (scalar tail of a sample)
template <int DT>
__device__ __forceinline__ uint32_t symbol_at(const uint8_t *base, uint32_t i) {
  if (DT == kF32) return (reinterpret_cast<const uint32_t *>(base)[i] >> 23) & 0xFFu;
  if (DT == kBF16) return (reinterpret_cast<const uint16_t *>(base)[i] >> 7) & 0xFFu;
  if (DT == kF16) return reinterpret_cast<const uint16_t *>(base)[i] >> 8;
  if (DT == kE5M2) return base[i];
  return (((uint32_t)base[2 * i] << 1) & 0xF0u) | (((uint32_t)base[2 * i + 1] >> 3) & 0x0Fu);  // e4m3 pair
}

// ---------------------------------------------------------------- a3 encode table entry
// rANS encode needs floor(x/f) for x < f*2^19 < 2^31: a 32-bit reciprocal
// with shift s-1 (s = ceil(log2 f)) is exact below 2^31; f = 1 uses
// rcp = 2^32-1 (q = x-1) with the bias raised by M-1.  Entry:
//   x = rcp, y = f<<19 | shift (renorm threshold + funnel-shift amount),
//   z = bias, w = M - f.
#ifndef UZIP_ENC_MULQ
#define UZIP_ENC_MULQ 0  // A/B: measured slower (0.696 vs 0.679 ms: two IMAD.HI on the chain)
#endif
// Encode entry {rcp, y, z, M - f}: floor(x / f) = umulhi(umulhi(x, rcp), y) - d and
// x' = x + z + q' (M - f) with z = cdf + d (M - f) -- both high multiplies on the FMA pipe
// (UZIP_ENC_MULQ; y = 2^(32 - sh), or 2^32 - 1 for sh = 0, which undercounts by one).  The
// renormalization test x >= f << 19 reads M - f (x + (M - f) << 19 >= 2^31).  Without MULQ:
// y = f << 19 | sh, q = umulhi(x, rcp) >> sh (funnel shift, ALU pipe).
__host__ __device__ inline uint4 make_enc_entry(uint32_t f, uint32_t cdf) {
  uint4 e;
  uint32_t sh, d;  // post-shift of the 32-bit reciprocal; undercount of umulhi(x, rcp) against x / f
  if (f < 2) {
    e.x = 0xFFFFFFFFu;  // umulhi(x, 2^32 - 1) = x - 1
    sh = 0, d = 1;
  } else {
    uint32_t s = 0;
    while (f > (1u << s)) ++s;
    e.x = (uint32_t)(((1ull << (s + 31)) + f - 1) / f);
    sh = s - 1, d = 0;
  }
  if (UZIP_ENC_MULQ) {
    if (sh == 0) e.y = 0xFFFFFFFFu, d += 1;  // umulhi(t, 2^32 - 1) = t - 1 (t >= 1 here)
    else e.y = 1u << (32 - sh);
  } else {
    e.y = (f << 19) | sh;
  }
  e.w = kM - f;
  e.z = cdf + d * e.w;
  return e;
}

}  // namespace uzip
