/*
 * uzip_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the Uzip method
 * (arxiv 2604.17172, "PAPER.md" = /root/reference/PAPER.md).  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
 * may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path under paper_2604_17172_b200/csrc/.
 *
 * Every function cites the passage it follows.  Where the paper is silent
 * the reading taken is the one listed in DESIGN.md "Readings" (R1..R17,
 * numbered like SURVEY.md 8(c) Q1..Q17).
 *
 * Pins per function (tests/test_oracle_*.py, tests/test_golden.py):
 *   uzo_split_elem / uzo_join_elem      SPEC S:61-64 examples, exhaustive 2^16 bijections, numpy frexp
 *                                       fields; fp8 pairs / bytes (R23, R24) exhaustively
 *   uzo_histogram                       brute-force count (np.bincount)
 *   uzo_normalize                       S:132-134, invariants, the survey's g1/g4 tables
 *   uzo_encode_block / uzo_decode_block brute force over all 3^9 lane-0 sequences, information identity,
 *                                       byte-for-byte the survey's independent g1 prototype (K, sizes,
 *                                       final states, sha256), stored-raw tie blocks (O7)
 *   uzo_compress / uzo_decompress       round trips over dtypes x edge sizes, Shannon / N1-cost bounds
 *                                       from closed-form value distributions, the paper's printed ratios
 *                                       (Table 1), corrupt-stream errors
 *   uzo_reduce (sum / min / max)        numpy / torch fp32 folds, special-value tables, permutation
 *                                       invariance (R11, R25)
 *   wire streams (oracle/__init__.py)   decode to the plain definitions of the collectives (O13, R26)
 * The stream layout (UZB1) is this reproduction's definition: the paper prints no
 * format or worked stream, so bytes are compared GPU-vs-oracle, and the oracle against the pins above.
 */
#ifndef UZIP_ORACLE_H
#define UZIP_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes (same numbering as include/uzip.h, restated, not shared) */
enum { UZO_BF16 = 0, UZO_F16 = 1, UZO_F32 = 2, UZO_E4M3 = 3, UZO_E5M2 = 4 };

/* status codes (same numbering as include/uzip.h, restated, not shared) */
enum {
  UZO_OK = 0,
  UZO_ERR_INVALID_ARG = 1,
  UZO_ERR_UNSUPPORTED_DTYPE = 2,
  UZO_ERR_CAPACITY = 3,
  UZO_ERR_CORRUPT_STREAM = 4,
  UZO_ERR_SIZE_MISMATCH = 5
};

/* Format constants of the UZB1 stream. */
#define UZO_PROB_BITS 12u               /* P: table precision, M = 2^P      */
#define UZO_M (1u << UZO_PROB_BITS)     /* 4096                             */
#define UZO_STATE_LBITS 15u             /* L = 2^15, states in [L, 2^31)    */
#define UZO_L (1u << UZO_STATE_LBITS)
#define UZO_LANES 32u                   /* W: interleaved states per block  */
#define UZO_HEADER_BYTES 64u
#define UZO_RAW_BLOCK 0xFFFFFFFFu       /* directory sentinel: stored raw   */

typedef struct {
  uint32_t block_symbols;  /* B; multiple of 32; 0 -> default 4096            */
  uint32_t chunk_blocks;   /* CB; blocks per table chunk; 0 -> 8 MiB / (B*eb) */
  uint32_t sample_symbols; /* S_s; 0 -> 256 KiB / eb                          */
  uint32_t global_table;   /* 1 -> one table over every symbol (Step 1) */
} uzo_params;

size_t uzo_elem_bytes(int dtype);
/* A symbol group is the unit that yields one 8-bit symbol: one element for
 * bf16/f16/f32/e5m2, a pair of elements for e4m3 ("pack two FP8 values
 * into a single 16-bit unit").  group bytes = elem bytes * elems. */
size_t uzo_group_elems(int dtype);
size_t uzo_group_bytes(int dtype);
/* residual bytes per group: 1 (bf16, f16, e4m3), 3 (f32: lo16 + hi8 planes), 0 (e5m2) */
size_t uzo_res_bytes(int dtype);

/* a1 Split: one symbol group -> (symbol, residual).
 * bits holds the group's raw bits, little-endian (16 or 32 of them; for e4m3
 * the pair (a, b) = (bits & 0xFF, bits >> 8); for e5m2 the one byte).  For
 * f32 the residual is 24 bits: lo16 (bits 15..0) | hi8 << 16 where
 * hi8 = sign<<7 | bits 22..16.  For bf16/f16/e4m3 the residual is one byte,
 * for e5m2 it is empty (0). */
void uzo_split_elem(int dtype, uint32_t bits, uint8_t *sym, uint32_t *res);
uint32_t uzo_join_elem(int dtype, uint8_t sym, uint32_t res);
void uzo_split_array(int dtype, const void *in, size_t n, uint8_t *sym, uint32_t *res);
void uzo_join_array(int dtype, const uint8_t *sym, const uint32_t *res, size_t n, void *out);

/* a2 Histogram of the first `limit` symbols. */
void uzo_histogram(const uint8_t *sym, size_t n, size_t limit, uint32_t cnt[256]);

/* a3 Rule N1 normalization to sum M with floor 1 (R5, R6). */
void uzo_normalize(const uint32_t cnt[256], uint16_t freq[256]);

/* a4 32-lane interleaved rANS encode of one block of B symbols (P:161-165,
 * P:422-424).  words must hold B entries.  Returns the word count K. */
uint32_t uzo_encode_block(const uint8_t *sym, uint32_t B, const uint16_t freq[256],
                          uint32_t states[32], uint16_t *words);
uint32_t uzo_encode_block_l(const uint8_t *sym, uint32_t B, const uint16_t freq[256], uint32_t states[32],
                            uint16_t *words, uint32_t lbits);

/* a8 decode of one block; returns UZO_OK or UZO_ERR_CORRUPT_STREAM. */
int uzo_decode_block(const uint32_t states_in[32], const uint16_t *words, uint32_t K,
                     uint32_t B, const uint16_t freq[256], uint8_t *sym_out);

/* Whole stream (UZB1).  uzo_compress_bound is the capacity that always
 * suffices. */
size_t uzo_compress_bound(size_t n, int dtype, const uzo_params *p);
int uzo_compress(int dtype, const void *in, size_t n, const uzo_params *p,
                 uint8_t *out, size_t cap, size_t *out_bytes);
int uzo_decompress(const uint8_t *in, size_t in_bytes, void *out, size_t n, int dtype);

/* a9 fold R (R11): out[i] = rnd(((x0 + x1) + x2) + ...) in fp32, ranks in
 * order, NaN -> canonical NaN of the dtype. inputs[k] points at rank k's
 * n elements. */
void uzo_reduce_sum(int dtype, const void *const *inputs, int nranks, size_t n, void *out);

/* a9 with op (R25): UZO_OP_SUM is the fold above; UZO_OP_MIN / UZO_OP_MAX are IEEE 754-2019
 * minimum / maximum in rank order (NaN propagates, -0 < +0); same output rounding. */
enum { UZO_OP_SUM = 0, UZO_OP_MIN = 1, UZO_OP_MAX = 2 };
void uzo_reduce(int dtype, int op, const void *const *inputs, int nranks, size_t n, void *out);

/* fp32 -> dtype rounding used by the fold (exported for its pin test). */
uint32_t uzo_round_from_f32(int dtype, float v);
float uzo_widen_to_f32(int dtype, uint32_t bits);

#ifdef __cplusplus
}
#endif
#endif
