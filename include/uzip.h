/*
 * uzip.h -- C ABI of uzip-b200: lossless float compression fused into GPU
 * communication, after arxiv 2604.17172 ("Uzip"), B200 (sm_100a) only.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * Conventions for every call
 *  - Buffer pointers are DEVICE pointers (cudaMalloc / torch CUDA memory) on
 *    the calling thread's current device, 16-byte aligned (128-bit I/O).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Every data call is stream-ordered and asynchronous: it only
 *    validates arguments on the host and enqueues kernels; no host sync.
 *  - Synchronous errors are returned (bad pointer/alignment/dtype/size,
 *    capacity, communicator misuse).  Asynchronous errors found by a kernel
 *    (corrupt stream, size or dtype mismatch, poll timeout) are written to a
 *    device status word (`d_status` for uzip_decompress, the communicator's
 *    error word for collectives, read with uzip_comm_get_async_error).
 *  - count == 0 is valid and does nothing (returns UZIP_OK).
 *  - The caller owns all user buffers and must keep them alive until the
 *    stream work completes.  The library owns communicator staging memory.
 *
 * Stream format: UZB1, defined in DESIGN.md section 2 (header with dtype
 * and sizes before/after compression; residual plane first, P:300-311;
 * per-chunk tables; block directory; payload; raw tail,
 * P:458-465).
 */
#ifndef UZIP_H
#define UZIP_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define UZIP_API __attribute__((visibility("default")))
#else
#define UZIP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Element types the codec splits.  fp8: e4m3 pairs form one symbol (R23), e5m2
 * bytes are symbols (R24); fp8 is not reduced (reduce-scatter / allreduce, R22). */
typedef enum { UZIP_BF16 = 0, UZIP_F16 = 1, UZIP_F32 = 2, UZIP_E4M3 = 3, UZIP_E5M2 = 4 } uzip_dtype_t;

/* Reduction operators ("sum, min, or max"): the fold R in rank order -- sum in fp32 with
 * one rounding (R11); min / max = IEEE 754-2019 minimum / maximum, NaN propagates, -0 < +0 (R25). */
typedef enum { UZIP_SUM = 0, UZIP_MIN = 1, UZIP_MAX = 2 } uzip_op_t;

typedef enum {
  UZIP_OK = 0,
  UZIP_ERR_INVALID_ARG = 1,       /* null/misaligned pointer, bad rank/peer, bad params     */
  UZIP_ERR_UNSUPPORTED_DTYPE = 2, /* dtype outside uzip_dtype_t                             */
  UZIP_ERR_CAPACITY = 3,          /* out_capacity < uzip_compress_bound, ws too small       */
  UZIP_ERR_CORRUPT_STREAM = 4,    /* async: header, table, directory or block check failed  */
  UZIP_ERR_SIZE_MISMATCH = 5,     /* async: stream n/dtype differ from the call's           */
  UZIP_ERR_CUDA = 6,              /* a CUDA runtime call failed                              */
  UZIP_ERR_COMM = 7,              /* communicator setup / bootstrap failure; a call that    */
                                  /* needs co-scheduled co-resident ranks under serialised  */
                                  /* kernel execution (see uzip_comm_init_all)              */
  UZIP_ERR_TIMEOUT = 8,           /* async: a peer flag did not arrive in poll_timeout_ms   */
  UZIP_ERR_NOT_IMPLEMENTED = 9
} uzip_status_t;

/* Codec parameters; all-zero (or a NULL pointer) selects the defaults.
 *  block_symbols  B, symbols per independently coded block (Step 2);
 *                 GPU-supported: 1024, 2048, 4096 (default), 8192, 16384;
 *                 reduce-scatter / allreduce and uzip_compress_staged take
 *                 B <= 4096 (UZIP_ERR_INVALID_ARG otherwise).
 *  chunk_blocks   blocks sharing one localized frequency table;
 *                 default 8 MiB of input; must be a multiple of 8.
 *  sample_symbols leading symbols of each chunk that build its table
 *                 ("the first 256 KB"); default 256 KiB of input.
 *  global_table   1 = one table over every symbol (Step 1). */
typedef struct uzip_codec_params {
  uint32_t block_symbols;
  uint32_t chunk_blocks;
  uint32_t sample_symbols;
  uint32_t global_table;
} uzip_codec_params_t;

/* ---------------------------------------------------------------- codec */

/* Worst-case stream bytes for `count` elements: every block stored raw
 * (R13).  Returns 0 for an unsupported dtype. */
UZIP_API size_t uzip_compress_bound(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params);

/* Device workspace bytes needed by uzip_compress / uzip_decompress for
 * `count` elements.  The workspace must be zero-filled once before first use
 * (uzip_workspace_init); the kernels leave it reusable.  One workspace must
 * not be used by two calls in flight at the same time. */
UZIP_API size_t uzip_workspace_bytes(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params);
UZIP_API uzip_status_t uzip_workspace_init(void *ws, size_t ws_bytes, void *stream);

/* Compress `count` elements at `in` into one UZB1 stream at `out`
 * (Steps 1-3 of P:159-170 fused as in P:317-376: split + sampled per-chunk
 * tables + warp-per-block rANS + look-back compaction, no coalescing pass).
 * `out_capacity` must be >= uzip_compress_bound.  The stream's byte count is
 * written to the device word *d_out_bytes when the stream work completes
 * (0 = an internal kernel failure; a valid stream is at least 64 bytes).
 * Output bytes equal the CPU oracle's for the same input and params. */
UZIP_API uzip_status_t uzip_compress(const void *in, size_t count, uzip_dtype_t dtype, void *out,
                            size_t out_capacity, uint64_t *d_out_bytes, void *ws, size_t ws_bytes,
                            const uzip_codec_params_t *params, void *stream);

/* Decompress a UZB1 stream (at most `in_bytes` readable bytes at `in`) into
 * `count` elements of `dtype` at `out`.  Never reads or writes out of
 * bounds on corrupt input.  When the stream work
 * completes, *d_status holds UZIP_OK or the first error found
 * (UZIP_ERR_CORRUPT_STREAM / UZIP_ERR_SIZE_MISMATCH); on error the contents
 * of `out` are unspecified. */
UZIP_API uzip_status_t uzip_decompress(const void *in, size_t in_bytes, void *out, size_t count,
                              uzip_dtype_t dtype, int32_t *d_status, void *ws, size_t ws_bytes,
                              void *stream);

/* Ablation baseline: the paper's staged DietGPU-style compression, Steps 1-3 of
 * P:159-170 as separate global-memory passes -- split + one global table (Step 1), every block
 * coded into a temporary B-byte slot (Step 2), a prefix scan and a copy that merges the blocks
 * into one contiguous buffer (Step 3, "a third global memory write").  Same encoder and
 * format as uzip_compress with global_table = 1 (forced here), so the streams are identical.
 * bf16 / f16 / f32 only.  res_out (nullable, 16-byte aligned, stream bytes - 64 of room): the
 * residual plane(s) go there instead of into `out`, and split_done (nullable cudaEvent_t) is
 * recorded after Step 1, so the caller can move the plane into `out` with the copy engine while
 * Steps 2-3 run (copy-engine split-send).  The workspace (uzip_staged_workspace_bytes)
 * must be zero-filled once (uzip_workspace_init); calls leave it reusable. */
UZIP_API size_t uzip_staged_workspace_bytes(size_t count, uzip_dtype_t dtype, const uzip_codec_params_t *params);
UZIP_API uzip_status_t uzip_compress_staged(const void *in, size_t count, uzip_dtype_t dtype, void *out,
                                            size_t out_capacity, uint64_t *d_out_bytes, void *ws,
                                            size_t ws_bytes, const uzip_codec_params_t *params,
                                            void *res_out, void *split_done, void *stream);

/* NVLink SHARP multicast: *supported = CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED of
 * `device` (0 when the driver lacks multicast).  uzip_nvls_selftest creates a one-device multicast
 * object of >= `bytes`, binds device memory, stores a pattern through multimem.st and checks it
 * through the unicast mapping: UZIP_OK, UZIP_ERR_NOT_IMPLEMENTED (no multicast, or the node refuses to
 * create a multicast object), or an error. */
UZIP_API uzip_status_t uzip_nvls_supported(int device, int *supported);
UZIP_API uzip_status_t uzip_nvls_selftest(int device, size_t bytes);

/* ---------------------------------------------------------------- communicator */

typedef struct uzip_comm *uzip_comm_t;

/* Host bootstrap all-gather: every rank contributes `bytes_per_rank` bytes
 * from `send`; `recv` receives nranks*bytes_per_rank bytes in rank order.
 * Return 0 on success.  (The Python binding supplies torch.distributed.) */
typedef int (*uzip_allgather_fn)(const void *send, void *recv, size_t bytes_per_rank, void *ctx);

/* Communicator configuration; all-zero or NULL selects defaults.
 *  min_compress_bytes  compress only messages >= this (R10; default 1 MiB)
 *  staging_bytes       receive staging per peer = 2 slots, bounds the footprint (default 512 MiB)
 *  pipe_chunk_bytes    largest round (one UZB1 stream) in input bytes (P:249-252 large blocks;
 *                      default: as large as a slot allows; rounded down to a multiple of 16)
 *  max_ctas            CTAs of each fused kernel (0 = all SMs); loopback tests use small values
 *  poll_timeout_ms     peer-flag wait bound before UZIP_ERR_TIMEOUT (default 10000)
 *  codec               stream parameters used on the wire */
typedef struct uzip_config {
  uint64_t min_compress_bytes;
  uint64_t staging_bytes;
  uint64_t pipe_chunk_bytes;
  uint32_t max_ctas;
  uint32_t poll_timeout_ms;
  uzip_codec_params_t codec;
} uzip_config_t;

/* Multi-process init: one call per rank (one process per GPU), collective
 * over all ranks through `bootstrap`.  Staging and flag memory is allocated
 * here and mapped into peers with CUDA IPC ("directly write ...
 * into the communication buffer"; NVLink P:442). */
UZIP_API uzip_status_t uzip_comm_init(uzip_comm_t *comm, int nranks, int rank, int cuda_device,
                             uzip_allgather_fn bootstrap, void *ctx, const uzip_config_t *cfg);

/* Single-process init of `nranks` communicators (like ncclCommInitAll);
 * devices[r] may repeat (loopback: several ranks on one GPU).  Ranks that
 * share a GPU (here, or IPC ranks whose GPU UUIDs match) run their persistent
 * kernels side by side: a launch whose decode items spin on a peer holds at
 * most 1/k of the CTA slots for k co-resident ranks, and slot credits are
 * always awaited by a one-thread kernel, so every producer finds an SM.
 * Serialised execution (CUDA_LAUNCH_BLOCKING=1, a kernel profiler such as
 * ncu, or UZIP_SERIALIZED=1) runs one kernel at a time, so co-resident ranks
 * can only exchange data whose producer launch finishes before the consumer
 * launch starts: a send/recv of at most two staging slots.  Any other call
 * between co-resident ranks (a launch that both encodes for and decodes from
 * peers, a relay, or a round that waits for a slot credit) returns
 * UZIP_ERR_COMM at once instead of spinning until poll_timeout_ms. */
UZIP_API uzip_status_t uzip_comm_init_all(uzip_comm_t *comms, int nranks, const int *devices,
                                 const uzip_config_t *cfg);
UZIP_API uzip_status_t uzip_comm_destroy(uzip_comm_t comm);

/* Split-send P2P: the residual plane leaves for the peer as soon
 * as it is split, the entropy-coded exponents follow; the receiver decodes as
 * blocks land.  A send on rank a matches the next recv on `peer` with the
 * same count and dtype (FIFO per ordered pair, like NCCL).  As with NCCL,
 * calls of one communicator are issued in one order on one stream; a send and
 * a recv of the same rank placed on two streams to run concurrently may wait
 * on each other for SMs (the kernels are persistent and spin on their peer). */
UZIP_API uzip_status_t uzip_send(const void *buf, size_t count, uzip_dtype_t dtype, int peer, uzip_comm_t comm,
                        void *stream);
UZIP_API uzip_status_t uzip_recv(void *buf, size_t count, uzip_dtype_t dtype, int peer, uzip_comm_t comm,
                        void *stream);

/* Compress-on-send / decompress-on-receive collectives, one
 * direct exchange over NVSwitch (two for allreduce).
 *  allgather:      recvbuf[r*sendcount + i] = sendbuf_r[i]; one stream per rank sent to all peers
 *  reduce_scatter: recvbuf_r[i] = R(sendbuf_0[r*recvcount+i], ..., sendbuf_{N-1}[...]) with the
 *                  fixed-order fp32 fold R (R11); the own shard is never compressed
 *  allreduce:      two-shot = reduce_scatter + allgather of the reduced shards, any count: N shards of
 *                  ceil(count/N) elements rounded up to 16 bytes (the last ones shorter or empty);
 *                  compressed rounds run both phases in ONE launch, each reduced tile re-encoded from
 *                  registers into the allgather stream (a9; its chunk tables sampled from each
 *                  chunk's first tile, R26)
 *  (reduce_scatter needs recvcount * element bytes % 16 == 0: 16-byte aligned shards, R21)
 * In place: allreduce sendbuf == recvbuf; allgather sendbuf == recvbuf + rank*sendcount;
 * reduce_scatter recvbuf == sendbuf + rank*recvcount. */
UZIP_API uzip_status_t uzip_allgather(const void *sendbuf, void *recvbuf, size_t sendcount, uzip_dtype_t dtype,
                             uzip_comm_t comm, void *stream);
UZIP_API uzip_status_t uzip_reduce_scatter(const void *sendbuf, void *recvbuf, size_t recvcount,
                                  uzip_dtype_t dtype, uzip_op_t op, uzip_comm_t comm, void *stream);
UZIP_API uzip_status_t uzip_allreduce(const void *sendbuf, void *recvbuf, size_t count, uzip_dtype_t dtype,
                             uzip_op_t op, uzip_comm_t comm, void *stream);

/* All-to-all (MoE expert parallelism, KV scatter): sendbuf holds nranks chunks of `count`
 * elements, chunk j goes to rank j; recvbuf chunk i arrives from rank i.  Each non-own chunk is one
 * compressed stream (count*eb must be a multiple of 16); the own chunk is copied.  Out of place. */
UZIP_API uzip_status_t uzip_alltoall(const void *sendbuf, void *recvbuf, size_t count, uzip_dtype_t dtype,
                                     uzip_comm_t comm, void *stream);

/* Broadcast (RL weight sync, BASELINE configs[2]): after the call every rank's `buf`
 * holds the root's `count` elements.  Compressed messages (>= the threshold, >= 3 ranks) use a
 * compressed scatter + relay: the root encodes N-1 pieces once and sends piece k to receiver k
 * (root egress r*S instead of (N-1)*r*S); each receiver forwards the compressed bytes of its piece
 * to the other receivers without re-encoding, and decodes all pieces.  Otherwise the root's stream
 * (or raw bytes) is fanned out to every receiver. */
UZIP_API uzip_status_t uzip_broadcast(void *buf, size_t count, uzip_dtype_t dtype, int root, uzip_comm_t comm,
                                      void *stream);

/* First asynchronous error seen by the communicator's kernels (sync read). */
UZIP_API uzip_status_t uzip_comm_get_async_error(uzip_comm_t comm, uzip_status_t *err);

/* Byte accounting of the last call on this communicator (sync read).
 * raw_bytes: bytes this rank would have stored into peers uncompressed;
 * wire_bytes: bytes it actually stored (UZB1 streams: header, tables and
 * directory included, R17).  wire/raw is the call's compression ratio. */
typedef struct uzip_stats {
  uint64_t raw_bytes;
  uint64_t wire_bytes;
  uint32_t compressed;     /* 1 if the call took the compressed path */
  uint32_t reserved;
} uzip_stats_t;
UZIP_API uzip_status_t uzip_get_stats(uzip_comm_t comm, uzip_stats_t *out);

/* Debug: the async error word and where the first error happened (sync read into 16 words):
 * [0] status, [1] site (1 tile flag, 2 credit, 3 look-back), [2] expected epoch / tile,
 * [3..4] value seen (hi, lo), [5] low 32 bits of the polled address, [6] CTA index,
 * [7] rounds sent | received << 16 on the channel with the first other rank, [8..11] this rank's
 * credit words for peers 0 and 1 (slots 0, 1), [12..15] decode-job done counters 0..3. */
UZIP_API uzip_status_t uzip_comm_error_detail(uzip_comm_t comm, uint32_t *out16);

/* Debug/test: copy the first `bytes` of the staging slot (0 or 1) where
 * rank `src`'s rounds land on this rank into host memory (sync).  Round q of
 * the ordered pair (src, this rank) lands in slot q % 2 as one UZB1 stream
 * (the oracle's wire stream). */
/* Tile trace (overlap evidence without a timeline profiler): with UZIP_TRACE=1 in the
 * environment at communicator init, every fused launch appends events of two u64 -- kind:4 | job:4 |
 * tile:56, then %globaltimer ns -- kinds 1 = encode tile started, 2 = its flag released, 3 = decode tile
 * acquired, 4 = decode tile done.  Copies up to max_events of them to `host` (2 x u64 each), sets
 * *n_events and clears the buffer (synchronizes the device).  Off: *n_events = 0. */
UZIP_API uzip_status_t uzip_comm_trace(uzip_comm_t comm, unsigned long long *host, size_t max_events,
                                       size_t *n_events);
UZIP_API uzip_status_t uzip_comm_read_staging(uzip_comm_t comm, int src, int slot, void *host, size_t bytes);

UZIP_API const char *uzip_status_string(uzip_status_t s);

/* Library version string, e.g. "uzip-b200 0.1 sm_100a". */
UZIP_API const char *uzip_version(void);

#ifdef __cplusplus
}
#endif
#endif /* UZIP_H */
