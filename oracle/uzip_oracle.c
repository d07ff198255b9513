/*
 * uzip_oracle.c -- TEST INFRASTRUCTURE ONLY (see uzip_oracle.h).
 *
 * A plain, slow, obviously-correct single-threaded implementation of the
 * Uzip codec and collective fold, written from PAPER.md (arxiv 2604.17172)
 * with the readings of DESIGN.md.  No blocking, no fusion, no SIMD, no
 * reciprocal tricks: divisions are divisions, searches are searches.
 *
 * Paper passages followed (PAPER.md line numbers):
 *   Step 1 split + frequency table ............ P:147
 *   Step 2 independent block-wise ANS ......... P:161-165
 *   Step 3 coalescing into one buffer ......... P:168-170  (here: offsets)
 *   localized (per chunk) sampled tables ...... P:357-370
 *   warp-per-block (32 lanes) ................. P:421-424
 *   sizes before/after + dtype in metadata .... P:476-479
 *   chunk alignment, raw tail ................. P:458-465
 *   decompress before reduce, fixed fold ...... P:387-392
 */
#include "uzip_oracle.h"

#include <math.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* dtype facts (P:136 bf16 = 1 sign, 8 exponent, 7 fraction bits;      */
/* P:722 float16 = 5 exponent bits of 16, float32 = 8 exponent of 32). */
/* ------------------------------------------------------------------ */
size_t uzo_elem_bytes(int dtype) {
  switch (dtype) {
    case UZO_BF16: return 2;
    case UZO_F16: return 2;
    case UZO_F32: return 4;
    case UZO_E4M3: return 1;
    case UZO_E5M2: return 1;
    default: return 0;
  }
}

/* two e4m3 values form one 16-bit unit whose two 4-bit exponent
 * fields make one 8-bit symbol; every other dtype has one element per symbol. */
size_t uzo_group_elems(int dtype) { return dtype == UZO_E4M3 ? 2 : 1; }
size_t uzo_group_bytes(int dtype) { return uzo_elem_bytes(dtype) * uzo_group_elems(dtype); }
size_t uzo_res_bytes(int dtype) {
  switch (dtype) {
    case UZO_F32: return 3;
    case UZO_E5M2: return 0;
    default: return uzo_elem_bytes(dtype) ? 1 : 0;
  }
}

/* a1 split ("each value is decomposed into its exponent and
 * remaining bits"; bit maps SPEC S:29-31; R2, R3). */
void uzo_split_elem(int dtype, uint32_t bits, uint8_t *sym, uint32_t *res) {
  if (dtype == UZO_BF16) {
    uint32_t sign = (bits >> 15) & 1u;
    uint32_t expo = (bits >> 7) & 0xFFu;
    uint32_t frac = bits & 0x7Fu;
    *sym = (uint8_t)expo;
    *res = (sign << 7) | frac;
  } else if (dtype == UZO_F16) {
    /* R3: the symbol is the high byte (sign, 5 exponent bits, 2 fraction
     * MSBs), the residual the low byte. */
    *sym = (uint8_t)((bits >> 8) & 0xFFu);
    *res = bits & 0xFFu;
  } else if (dtype == UZO_E4M3) {
    /* e4m3 (s:7 e:6..3 m:2..0), pair (a, b): symbol = exp_a<<4 | exp_b,
     * residual = s_a<<7 | m_a<<4 | s_b<<3 | m_b */
    uint32_t a = bits & 0xFFu, b = (bits >> 8) & 0xFFu;
    uint32_t ea = (a >> 3) & 0xFu, eb = (b >> 3) & 0xFu;
    *sym = (uint8_t)((ea << 4) | eb);
    *res = ((a >> 7) << 7) | ((a & 7u) << 4) | ((b >> 7) << 3) | (b & 7u);
  } else if (dtype == UZO_E5M2) {
    /* SPEC S:33, S:94 (R24): the whole byte is the symbol, no residual */
    *sym = (uint8_t)(bits & 0xFFu);
    *res = 0;
  } else { /* UZO_F32 */
    uint32_t sign = (bits >> 31) & 1u;
    uint32_t expo = (bits >> 23) & 0xFFu;
    uint32_t frac = bits & 0x7FFFFFu;
    uint32_t lo16 = frac & 0xFFFFu;
    uint32_t hi8 = (sign << 7) | (frac >> 16);
    *sym = (uint8_t)expo;
    *res = lo16 | (hi8 << 16);
  }
}

uint32_t uzo_join_elem(int dtype, uint8_t sym, uint32_t res) {
  if (dtype == UZO_BF16) {
    uint32_t sign = (res >> 7) & 1u;
    uint32_t frac = res & 0x7Fu;
    return (sign << 15) | ((uint32_t)sym << 7) | frac;
  } else if (dtype == UZO_F16) {
    return ((uint32_t)sym << 8) | (res & 0xFFu);
  } else if (dtype == UZO_E4M3) {
    uint32_t ea = (uint32_t)sym >> 4, eb = (uint32_t)sym & 0xFu;
    uint32_t a = (((res >> 7) & 1u) << 7) | (ea << 3) | ((res >> 4) & 7u);
    uint32_t b = (((res >> 3) & 1u) << 7) | (eb << 3) | (res & 7u);
    return a | (b << 8);
  } else if (dtype == UZO_E5M2) {
    return sym;
  } else {
    uint32_t lo16 = res & 0xFFFFu;
    uint32_t hi8 = (res >> 16) & 0xFFu;
    uint32_t sign = hi8 >> 7;
    uint32_t frac = ((hi8 & 0x7Fu) << 16) | lo16;
    return (sign << 31) | ((uint32_t)sym << 23) | frac;
  }
}

/* n = number of symbol groups (elements for every dtype but e4m3: pairs). */
void uzo_split_array(int dtype, const void *in, size_t n, uint8_t *sym, uint32_t *res) {
  const uint8_t *b = (const uint8_t *)in;
  size_t w = uzo_group_bytes(dtype);
  for (size_t i = 0; i < n; ++i) {
    uint32_t bits = 0;
    for (size_t k = 0; k < w; ++k) bits |= (uint32_t)b[w * i + k] << (8 * k);
    uzo_split_elem(dtype, bits, &sym[i], &res[i]);
  }
}

void uzo_join_array(int dtype, const uint8_t *sym, const uint32_t *res, size_t n, void *out) {
  uint8_t *b = (uint8_t *)out;
  size_t w = uzo_group_bytes(dtype);
  for (size_t i = 0; i < n; ++i) {
    uint32_t v = uzo_join_elem(dtype, sym[i], res[i]);
    for (size_t k = 0; k < w; ++k) b[w * i + k] = (uint8_t)(v >> (8 * k));
  }
}

/* a2 histogram over the first `limit` symbols (limit==0: all)
 * "sampling a small portion of its assigned data range (e.g., the first
 * 256 KB)". */
void uzo_histogram(const uint8_t *sym, size_t n, size_t limit, uint32_t cnt[256]) {
  size_t m = n;
  if (limit != 0 && limit < n) m = limit;
  for (int s = 0; s < 256; ++s) cnt[s] = 0;
  for (size_t i = 0; i < m; ++i) cnt[sym[i]] += 1;
}

/* a3 rule N1 (R5): f[s] = 1 + floor(cnt[s]*(M-256)/T),
 * the remainder goes to the most frequent symbol (lowest on ties); an
 * all-zero histogram gives the uniform table M/256. */
void uzo_normalize(const uint32_t cnt[256], uint16_t freq[256]) {
  uint64_t total = 0;
  for (int s = 0; s < 256; ++s) total += cnt[s];
  if (total == 0) {
    for (int s = 0; s < 256; ++s) freq[s] = (uint16_t)(UZO_M / 256u);
    return;
  }
  uint32_t sum = 0;
  for (int s = 0; s < 256; ++s) {
    uint64_t scaled = ((uint64_t)cnt[s] * (uint64_t)(UZO_M - 256u)) / total;
    freq[s] = (uint16_t)(1u + (uint32_t)scaled);
    sum += freq[s];
  }
  int best = 0;
  for (int s = 1; s < 256; ++s)
    if (cnt[s] > cnt[best]) best = s;
  freq[best] = (uint16_t)(freq[best] + (UZO_M - sum));
}

static void cumulative(const uint16_t freq[256], uint32_t cdf[257]) {
  cdf[0] = 0;
  for (int s = 0; s < 256; ++s) cdf[s + 1] = cdf[s] + freq[s];
}

/* a4 rANS encode of one block, 32 interleaved lanes ("each
 * thread block ... applies ANS encoding locally"; P:422-424 one warp per
 * block).  Lane l codes symbols j*32+l; rounds run j = R-1 down to 0.
 * Before coding s the state is renormalized: while x >= f[s] << (31-P)
 * emit its low 16 bits (one word at most).  Then
 *   x = floor(x / f[s]) * M + (x mod f[s]) + cdf[s].
 * Words are appended in emission order (round R-1 first, lanes ascending
 * within a round).  R4 in DESIGN.md. */
uint32_t uzo_encode_block(const uint8_t *sym, uint32_t B, const uint16_t freq[256],
                          uint32_t states[32], uint16_t *words) {
  return uzo_encode_block_l(sym, B, freq, states, words, UZO_STATE_LBITS);
}

/* The same coder for a state interval [2^lbits, 2^(lbits+16)) (lbits 15 or 16).  lbits = 15 is the
 * stream format (R4); lbits = 16 is the interval of the survey's independent prototype, whose g1
 * micro-vector then pins this function's arithmetic byte for byte. */
uint32_t uzo_encode_block_l(const uint8_t *sym, uint32_t B, const uint16_t freq[256],
                            uint32_t states[32], uint16_t *words, uint32_t lbits) {
  uint32_t cdf[257];
  cumulative(freq, cdf);
  uint32_t x[32];
  for (uint32_t l = 0; l < UZO_LANES; ++l) x[l] = 1u << lbits;
  uint32_t K = 0;
  uint32_t R = B / UZO_LANES;
  for (uint32_t jj = R; jj > 0; --jj) {
    uint32_t j = jj - 1;
    for (uint32_t l = 0; l < UZO_LANES; ++l) {
      uint32_t s = sym[j * UZO_LANES + l];
      uint32_t f = freq[s];
      uint32_t x_max = f << (lbits + 16u - UZO_PROB_BITS);  /* (L >> P) << 16, times f */
      if (x[l] >= x_max) {
        words[K++] = (uint16_t)(x[l] & 0xFFFFu);
        x[l] >>= 16;
      }
      x[l] = (x[l] / f) * UZO_M + (x[l] % f) + cdf[s];
    }
  }
  for (uint32_t l = 0; l < UZO_LANES; ++l) states[l] = x[l];
  return K;
}

/* a8 decode of one block ("decompressed at the receiver").  Rounds
 * j = 0..R-1: slot = x mod M, s = the symbol whose [cdf, cdf+f) holds
 * slot, x = f*(x >> P) + slot - cdf.  Lanes whose state fell below L take
 * one word each; the k such lanes of a round read the last k unread words
 * of the stream, lanes ascending.  Corrupt unless exactly K words are
 * consumed and every lane ends at L (R4). */
int uzo_decode_block(const uint32_t states_in[32], const uint16_t *words, uint32_t K,
                     uint32_t B, const uint16_t freq[256], uint8_t *sym_out) {
  uint32_t cdf[257];
  cumulative(freq, cdf);
  if (cdf[256] != UZO_M) return UZO_ERR_CORRUPT_STREAM;
  uint8_t slot_sym[UZO_M];
  for (int s = 0; s < 256; ++s)
    for (uint32_t t = cdf[s]; t < cdf[s + 1]; ++t) slot_sym[t] = (uint8_t)s;
  uint32_t x[32];
  for (uint32_t l = 0; l < UZO_LANES; ++l) x[l] = states_in[l];
  uint32_t p = K;
  uint32_t R = B / UZO_LANES;
  for (uint32_t j = 0; j < R; ++j) {
    int need[32];
    uint32_t k = 0;
    for (uint32_t l = 0; l < UZO_LANES; ++l) {
      uint32_t slot = x[l] & (UZO_M - 1u);
      uint32_t s = slot_sym[slot];
      x[l] = (uint32_t)freq[s] * (x[l] >> UZO_PROB_BITS) + slot - cdf[s];
      sym_out[j * UZO_LANES + l] = (uint8_t)s;
      need[l] = x[l] < UZO_L;
      k += (uint32_t)need[l];
    }
    if (k > p) return UZO_ERR_CORRUPT_STREAM;
    uint32_t r = 0;
    for (uint32_t l = 0; l < UZO_LANES; ++l) {
      if (need[l]) {
        x[l] = (x[l] << 16) | words[p - k + r];
        ++r;
      }
    }
    p -= k;
  }
  if (p != 0) return UZO_ERR_CORRUPT_STREAM;
  for (uint32_t l = 0; l < UZO_LANES; ++l)
    if (x[l] != UZO_L) return UZO_ERR_CORRUPT_STREAM;
  return UZO_OK;
}

/* ------------------------------------------------------------------ */
/* UZB1 stream ("merged into a single        */
/* contiguous output buffer"; P:479 dtype and sizes before and after). */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t B, CB, S;
  int global;
  size_t n, n_blocks, n_coded, n_chunks;
  size_t off_res0, off_res1, off_tab, off_coff, off_dir, off_pay, off_tail, total;
  size_t payload_bytes;
} layout_t;

static size_t round16(size_t v) { return (v + 15u) & ~(size_t)15u; }

static void resolve_params(int dtype, const uzo_params *p, uint32_t *B, uint32_t *CB,
                           uint32_t *S, int *global) {
  size_t eb = uzo_group_bytes(dtype); /* input bytes per symbol */
  *B = (p && p->block_symbols) ? p->block_symbols : 4096u;
  *global = (p && p->global_table) ? 1 : 0;
  *CB = (p && p->chunk_blocks) ? p->chunk_blocks : (uint32_t)((8u << 20) / (*B * eb));
  if (*CB == 0) *CB = 1;
  *S = (p && p->sample_symbols) ? p->sample_symbols : (uint32_t)((256u << 10) / eb);
}

/* n counts ELEMENTS; blocks count symbol groups (n_coded groups are coded,
 * the remaining n - n_coded * group_elems elements form the raw tail). */
static void make_layout(int dtype, size_t n, uint32_t B, uint32_t CB, uint32_t S, int global,
                        size_t payload_bytes, layout_t *L) {
  size_t eb = uzo_elem_bytes(dtype);
  size_t ge = uzo_group_elems(dtype);
  L->B = B;
  L->n = n;
  L->n_blocks = (n / ge) / B;
  L->n_coded = L->n_blocks * B;
  L->global = global;
  if (global) {
    L->CB = L->n_blocks ? (uint32_t)L->n_blocks : 1u;
    L->S = 0;
  } else {
    L->CB = CB;
    L->S = S;
  }
  L->n_chunks = (L->n_blocks + L->CB - 1) / L->CB;
  L->off_res0 = UZO_HEADER_BYTES;
  if (dtype == UZO_F32) {
    L->off_res1 = L->off_res0 + 2 * L->n_coded;
    L->off_tab = round16(L->off_res1 + L->n_coded);
  } else {
    L->off_res1 = L->off_res0;
    L->off_tab = round16(L->off_res0 + uzo_res_bytes(dtype) * L->n_coded);
  }
  L->off_coff = L->off_tab + 512 * L->n_chunks;
  L->off_dir = round16(L->off_coff + 8 * L->n_chunks);
  L->off_pay = round16(L->off_dir + 4 * L->n_blocks);
  L->payload_bytes = payload_bytes;
  L->off_tail = round16(L->off_pay + payload_bytes);
  L->total = L->off_tail + (n - L->n_coded * ge) * eb;
}

static void put16(uint8_t *p, uint32_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put32(uint8_t *p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static void put64(uint8_t *p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint32_t get16(const uint8_t *p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8); }
static uint32_t get32(const uint8_t *p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= (uint32_t)p[i] << (8 * i);
  return v;
}
static uint64_t get64(const uint8_t *p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

static uint32_t load_elem(int dtype, const uint8_t *in, size_t i) {
  if (dtype == UZO_F32) return get32(in + 4 * i);
  if (dtype == UZO_E5M2) return in[i];
  return get16(in + 2 * i); /* bf16, f16, and an e4m3 pair */
}
static void store_elem(int dtype, uint8_t *out, size_t i, uint32_t v) {
  if (dtype == UZO_F32) put32(out + 4 * i, v);
  else if (dtype == UZO_E5M2) out[i] = (uint8_t)v;
  else put16(out + 2 * i, v);
}

/* Worst case: every block stored raw (O7 bound). */
size_t uzo_compress_bound(size_t n, int dtype, const uzo_params *p) {
  uint32_t B, CB, S;
  int global;
  if (uzo_elem_bytes(dtype) == 0) return 0;
  resolve_params(dtype, p, &B, &CB, &S, &global);
  layout_t L;
  make_layout(dtype, n, B, CB, S, global, ((n / uzo_group_elems(dtype)) / B) * (size_t)B, &L);
  return L.total;
}

#include <stdlib.h>

int uzo_compress(int dtype, const void *in_v, size_t n, const uzo_params *p, uint8_t *out,
                 size_t cap, size_t *out_bytes) {
  const uint8_t *in = (const uint8_t *)in_v;
  size_t eb = uzo_elem_bytes(dtype);
  if (eb == 0) return UZO_ERR_UNSUPPORTED_DTYPE;
  uint32_t B, CB, S;
  int global;
  resolve_params(dtype, p, &B, &CB, &S, &global);
  if (B < UZO_LANES || B % UZO_LANES != 0) return UZO_ERR_INVALID_ARG;

  layout_t L;
  make_layout(dtype, n, B, CB, S, global, 0, &L);

  /* Step 1: split every coded element into the symbol buffer (the
   * compressed part) and the residual buffer (the uncompressed part). */
  uint8_t *sym = (uint8_t *)malloc(L.n_coded ? L.n_coded : 1);
  uint32_t *res = (uint32_t *)malloc(sizeof(uint32_t) * (L.n_coded ? L.n_coded : 1));
  for (size_t i = 0; i < L.n_coded; ++i) uzo_split_elem(dtype, load_elem(dtype, in, i), &sym[i], &res[i]);

  /* Localized tables: one table per chunk from the chunk's sampled
   * prefix; global mode: one table over every symbol. */
  uint16_t *tables = (uint16_t *)malloc(512 * (L.n_chunks ? L.n_chunks : 1));
  for (size_t c = 0; c < L.n_chunks; ++c) {
    size_t first = c * L.CB * (size_t)B;
    size_t blocks = L.n_blocks - c * L.CB;
    if (blocks > L.CB) blocks = L.CB;
    uint32_t cnt[256];
    uzo_histogram(sym + first, blocks * B, L.S, cnt);
    uzo_normalize(cnt, tables + 256 * c);
  }

  /* Step 2: every block independently, variable-length. */
  uint32_t *dir = (uint32_t *)malloc(4 * (L.n_blocks ? L.n_blocks : 1));
  size_t *bsize = (size_t *)malloc(sizeof(size_t) * (L.n_blocks ? L.n_blocks : 1));
  uint32_t *bstates = (uint32_t *)malloc(4 * 32 * (L.n_blocks ? L.n_blocks : 1));
  uint16_t **bwords = (uint16_t **)malloc(sizeof(uint16_t *) * (L.n_blocks ? L.n_blocks : 1));
  size_t payload = 0;
  for (size_t b = 0; b < L.n_blocks; ++b) {
    size_t c = b / L.CB;
    bwords[b] = (uint16_t *)malloc(2 * (size_t)B);
    uint32_t K = uzo_encode_block(sym + b * B, B, tables + 256 * c, bstates + 32 * b, bwords[b]);
    size_t coded = round16(128 + 2 * (size_t)K);
    if (coded >= B) { /* R13: stored-raw escape, ties go raw */
      dir[b] = UZO_RAW_BLOCK;
      bsize[b] = B;
    } else {
      dir[b] = K;
      bsize[b] = coded;
    }
    payload += bsize[b];
  }
  make_layout(dtype, n, B, CB, S, global, payload, &L);
  int status = UZO_OK;
  if (L.total > cap) {
    status = UZO_ERR_CAPACITY;
    goto done;
  }
  memset(out, 0, L.total);

  /* header: dtype and sizes before/after compression */
  memcpy(out, "UZB1", 4);
  put16(out + 4, 1);
  out[6] = (uint8_t)dtype;
  out[7] = (uint8_t)(global ? 1 : 0);
  put64(out + 8, n);
  put32(out + 16, B);
  put32(out + 20, L.CB);
  put32(out + 24, L.S);
  out[28] = (uint8_t)UZO_PROB_BITS;
  out[29] = (uint8_t)UZO_LANES;
  out[30] = (uint8_t)UZO_STATE_LBITS;
  put32(out + 32, (uint32_t)L.n_blocks);
  put32(out + 36, (uint32_t)L.n_chunks);
  put64(out + 40, L.payload_bytes);
  put64(out + 48, L.total);

  /* residual plane(s), in element order (sent first) */
  for (size_t i = 0; i < L.n_coded; ++i) {
    if (dtype == UZO_F32) {
      put16(out + L.off_res0 + 2 * i, res[i] & 0xFFFFu);
      out[L.off_res1 + i] = (uint8_t)(res[i] >> 16);
    } else if (uzo_res_bytes(dtype) == 1) {
      out[L.off_res0 + i] = (uint8_t)res[i];
    }
  }
  for (size_t c = 0; c < L.n_chunks; ++c)
    for (int s = 0; s < 256; ++s) put16(out + L.off_tab + 512 * c + 2 * s, tables[256 * c + s]);
  /* Step 3 reduced to offsets: chunk_off = sizes of all blocks
   * of earlier chunks; block b sits after the blocks before it. */
  {
    size_t run = 0;
    for (size_t b = 0; b < L.n_blocks; ++b) {
      if (b % L.CB == 0) put64(out + L.off_coff + 8 * (b / L.CB), run);
      put32(out + L.off_dir + 4 * b, dir[b]);
      uint8_t *dst = out + L.off_pay + run;
      if (dir[b] == UZO_RAW_BLOCK) {
        memcpy(dst, sym + b * B, B);
      } else {
        for (int l = 0; l < 32; ++l) put32(dst + 4 * l, bstates[32 * b + l]);
        for (uint32_t w = 0; w < dir[b]; ++w) put16(dst + 128 + 2 * w, bwords[b][w]);
      }
      run += bsize[b];
    }
  }
  /* raw tail */
  memcpy(out + L.off_tail, in + L.n_coded * uzo_group_bytes(dtype), (n - L.n_coded * uzo_group_elems(dtype)) * eb);
  *out_bytes = L.total;

done:
  for (size_t b = 0; b < L.n_blocks; ++b) free(bwords[b]);
  free(bwords);
  free(bstates);
  free(bsize);
  free(dir);
  free(tables);
  free(res);
  free(sym);
  return status;
}

int uzo_decompress(const uint8_t *in, size_t in_bytes, void *out_v, size_t n, int dtype) {
  uint8_t *out = (uint8_t *)out_v;
  size_t eb = uzo_elem_bytes(dtype);
  if (eb == 0) return UZO_ERR_UNSUPPORTED_DTYPE;
  if (in_bytes < UZO_HEADER_BYTES) return UZO_ERR_CORRUPT_STREAM;
  if (memcmp(in, "UZB1", 4) != 0 || get16(in + 4) != 1) return UZO_ERR_CORRUPT_STREAM;
  if (in[6] != (uint8_t)dtype) return UZO_ERR_SIZE_MISMATCH;
  if (get64(in + 8) != (uint64_t)n) return UZO_ERR_SIZE_MISMATCH;
  uint32_t B = get32(in + 16), CB = get32(in + 20), S = get32(in + 24);
  int global = in[7] & 1;
  if ((in[7] & ~1u) != 0) return UZO_ERR_CORRUPT_STREAM;
  if (in[28] != UZO_PROB_BITS || in[29] != UZO_LANES || in[30] != UZO_STATE_LBITS)
    return UZO_ERR_CORRUPT_STREAM;
  if (B < UZO_LANES || B % UZO_LANES != 0 || B > (1u << 20) || CB == 0) return UZO_ERR_CORRUPT_STREAM;
  uint64_t payload = get64(in + 40);
  if (payload > in_bytes) return UZO_ERR_CORRUPT_STREAM;
  layout_t L;
  make_layout(dtype, n, B, CB, S, global, (size_t)payload, &L);
  if (global && L.CB != CB) return UZO_ERR_CORRUPT_STREAM;
  if (get32(in + 32) != L.n_blocks || get32(in + 36) != L.n_chunks) return UZO_ERR_CORRUPT_STREAM;
  if (get64(in + 48) != L.total || L.total > in_bytes) return UZO_ERR_CORRUPT_STREAM;

  uint8_t *sym = (uint8_t *)malloc(B);
  uint16_t *words = (uint16_t *)malloc(2 * (size_t)B);
  int status = UZO_OK;
  size_t run = 0;
  for (size_t c = 0; c < L.n_chunks && status == UZO_OK; ++c) {
    uint16_t freq[256];
    uint32_t sum = 0;
    for (int s = 0; s < 256; ++s) {
      freq[s] = (uint16_t)get16(in + L.off_tab + 512 * c + 2 * s);
      if (freq[s] == 0) status = UZO_ERR_CORRUPT_STREAM;
      sum += freq[s];
    }
    if (sum != UZO_M) status = UZO_ERR_CORRUPT_STREAM;
    if (get64(in + L.off_coff + 8 * c) != run) status = UZO_ERR_CORRUPT_STREAM;
    size_t b_end = (c + 1) * (size_t)L.CB;
    if (b_end > L.n_blocks) b_end = L.n_blocks;
    for (size_t b = c * (size_t)L.CB; b < b_end && status == UZO_OK; ++b) {
      uint32_t d = get32(in + L.off_dir + 4 * b);
      size_t size;
      if (d == UZO_RAW_BLOCK) {
        size = B;
      } else {
        size = round16(128 + 2 * (size_t)d);
        if (size >= B) { status = UZO_ERR_CORRUPT_STREAM; break; }
      }
      if (run + size > L.payload_bytes) { status = UZO_ERR_CORRUPT_STREAM; break; }
      const uint8_t *src = in + L.off_pay + run;
      if (d == UZO_RAW_BLOCK) {
        memcpy(sym, src, B);
      } else {
        uint32_t st[32];
        for (int l = 0; l < 32; ++l) st[l] = get32(src + 4 * l);
        for (uint32_t w = 0; w < d; ++w) words[w] = (uint16_t)get16(src + 128 + 2 * w);
        status = uzo_decode_block(st, words, d, B, freq, sym);
        if (status != UZO_OK) break;
      }
      for (uint32_t i = 0; i < B; ++i) {
        size_t e = b * (size_t)B + i;
        uint32_t r;
        if (dtype == UZO_F32)
          r = get16(in + L.off_res0 + 2 * e) | ((uint32_t)in[L.off_res1 + e] << 16);
        else if (uzo_res_bytes(dtype) == 1)
          r = in[L.off_res0 + e];
        else
          r = 0;
        store_elem(dtype, out, e, uzo_join_elem(dtype, sym[i], r));
      }
      run += size;
    }
  }
  if (status == UZO_OK && run != L.payload_bytes) status = UZO_ERR_CORRUPT_STREAM;
  if (status == UZO_OK)
    memcpy(out + L.n_coded * uzo_group_bytes(dtype), in + L.off_tail,
           (n - L.n_coded * uzo_group_elems(dtype)) * eb);
  free(words);
  free(sym);
  return status;
}

/* ------------------------------------------------------------------ */
/* a9 fold R (R11): widen to fp32, acc = x0,    */
/* acc = fl32(acc + xk) for k = 1..N-1 in rank order, round once (RNE), */
/* NaN -> canonical.                                                   */
/* ------------------------------------------------------------------ */
float uzo_widen_to_f32(int dtype, uint32_t bits) {
  float f;
  if (dtype == UZO_BF16) {
    uint32_t w = bits << 16;
    memcpy(&f, &w, 4);
  } else if (dtype == UZO_F16) {
    uint16_t h = (uint16_t)bits;
    _Float16 hf;
    memcpy(&hf, &h, 2);
    f = (float)hf; /* exact widening, IEEE 754 */
  } else {
    memcpy(&f, &bits, 4);
  }
  return f;
}

uint32_t uzo_round_from_f32(int dtype, float v) {
  if (isnan(v)) {
    if (dtype == UZO_F32) return 0x7FFFFFFFu;
    return 0x7FFFu;
  }
  uint32_t w;
  memcpy(&w, &v, 4);
  if (dtype == UZO_BF16) {
    /* round to nearest even on the 16 dropped bits */
    uint32_t lsb = (w >> 16) & 1u;
    return (w + 0x7FFFu + lsb) >> 16;
  } else if (dtype == UZO_F16) {
    _Float16 h = (_Float16)v; /* IEEE 754 conversion, round to nearest even */
    uint16_t hb;
    memcpy(&hb, &h, 2);
    return hb;
  }
  return w;
}

/* min / max fold ("sum, min, or max"; reading R25): IEEE 754-2019
 * minimum/maximum in rank order -- a NaN operand makes the result NaN
 * (canonical on output), -0 < +0, otherwise the smaller / larger value.
 * The result is one of the inputs, so the final rounding is exact. */
static float fold_min(float acc, float x) {
  if (isnan(acc) || isnan(x)) return NAN;
  if (x < acc) return x;
  if (x == acc && signbit(x) && !signbit(acc)) return x; /* -0 beats +0 */
  return acc;
}
static float fold_max(float acc, float x) {
  if (isnan(acc) || isnan(x)) return NAN;
  if (x > acc) return x;
  if (x == acc && !signbit(x) && signbit(acc)) return x; /* +0 beats -0 */
  return acc;
}

void uzo_reduce(int dtype, int op, const void *const *inputs, int nranks, size_t n, void *out_v) {
  if (op == UZO_OP_SUM) {
    uzo_reduce_sum(dtype, inputs, nranks, n, out_v);
    return;
  }
  uint8_t *out = (uint8_t *)out_v;
  for (size_t i = 0; i < n; ++i) {
    float acc = uzo_widen_to_f32(dtype, load_elem(dtype, (const uint8_t *)inputs[0], i));
    for (int k = 1; k < nranks; ++k) {
      float xk = uzo_widen_to_f32(dtype, load_elem(dtype, (const uint8_t *)inputs[k], i));
      acc = op == UZO_OP_MIN ? fold_min(acc, xk) : fold_max(acc, xk);
    }
    store_elem(dtype, out, i, uzo_round_from_f32(dtype, acc));
  }
}

void uzo_reduce_sum(int dtype, const void *const *inputs, int nranks, size_t n, void *out_v) {
  uint8_t *out = (uint8_t *)out_v;
  for (size_t i = 0; i < n; ++i) {
    volatile float acc = uzo_widen_to_f32(dtype, load_elem(dtype, (const uint8_t *)inputs[0], i));
    for (int k = 1; k < nranks; ++k) {
      float xk = uzo_widen_to_f32(dtype, load_elem(dtype, (const uint8_t *)inputs[k], i));
      acc = acc + xk;
    }
    store_elem(dtype, out, i, uzo_round_from_f32(dtype, acc));
  }
}
