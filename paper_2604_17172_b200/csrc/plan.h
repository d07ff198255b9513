// plan.h -- work description of one launch of the fused codec/communication
// kernel (fused.cu).  Shared by the host planners (api.cu, comm.cu) and the
// device code.
//
// A launch processes a ticket space [E items][C items][D items]:
//   E  encode one tile (8 blocks) of a UZB1 stream and store it into nd
//      destinations (local stream buffer for uzip_compress, or peers' staging
//      slots over NVLink for the collectives: "directly write the compressed
//      data into the communication buffer"), then release a tile
//      flag in each destination (a12).  Raw mode (below the threshold)
//      copies 64 KiB raw tiles instead.
//   C  plain copy tiles (the own shard of an allgather).
//   D  wait for a tile flag, decode the tile (a7-a8) and join into the output;
//      with nsrc > 1 it decodes the same tile from every source and folds them
//      in rank order in fp32 (a9, reading R11) -- decompress before reduce
//      (P:387-392).
#pragma once

#include "uzip_device.cuh"

namespace uzip {

constexpr int kMaxRanks = 8;
constexpr uint32_t kRawTileBytes = 64u << 10;

// Tiles (kTileBlocks blocks each) of a stream; a stream without whole blocks
// still has one tile (header + raw tail).
__host__ __device__ inline uint64_t tiles_of(const StreamGeom &g) {
  const uint64_t t = g.n_tiles();
  return t ? t : 1;
}

struct EncJob {
  const uint8_t *in;                        // local input of this stream
  StreamGeom g;                             // geometry (compressed mode)
  uint64_t raw_bytes;                       // raw mode: message bytes
  uint64_t ntiles;                          // >= 1
  uint32_t raw;                             // 1 = raw (uncoded) tiles
  uint32_t nd;                              // destinations
  uint8_t *dst[kMaxRanks];                  // stream base at each destination
  unsigned long long *flag[kMaxRanks];      // tile flags at each destination (null: no flags)
  const unsigned long long *credit[kMaxRanks];  // local word: last epoch the destination consumed from this slot
  uint32_t epoch[kMaxRanks];                // flag epoch per destination (round sequence + 1)
  uint4 *enc;                               // per-chunk encode entries (k_norm)
  uint16_t *tab16;                          // per-chunk serialized tables (k_norm)
  unsigned long long *tile_status;          // per-tile look-back words (zeroed by k_hist)
  uint32_t *partial;                        // k_hist partial histograms [chunk][kMaxHistParts][256]
  uint64_t *d_out_bytes;                    // codec: stream size (may be null)
  unsigned long long *wire_acc;             // comm: += stream bytes x nd (may be null)
};

struct DecJob {
  StreamGeom g;
  uint64_t raw_bytes;
  uint64_t ntiles;
  uint32_t raw;
  uint32_t nsrc;                            // 1: plain decode; > 1: decode + reduce over sources
  int32_t me;                               // reduce: index of the local (uncompressed) source, -1 none
  uint32_t op;                              // reduce: 0 sum, 1 min, 2 max (R11, R25)
  const uint8_t *src[kMaxRanks];            // stream base in local staging (me: local raw input)
  const unsigned long long *flag[kMaxRanks];  // local tile flags per source
  unsigned long long *credit[kMaxRanks];    // word at the source to release when the round is consumed
  uint32_t epoch[kMaxRanks];
  uint8_t *out;                             // output of this stream / shard
  uint32_t *done;                           // tiles finished (self-resetting counter in ws)
  uint32_t run;                             // consecutive tiles per D item (>= 1): one decode-table
                                            // build serves the run instead of one build per tile
  // relay (broadcast): every received tile is forwarded, as received, to nfwd peers before it is
  // decoded; the compressed bytes travel on without re-encoding (weight-sync broadcast)
  uint32_t nfwd;
  uint8_t *fdst[kMaxRanks];                 // stream base in each forward destination's staging
  unsigned long long *fflag[kMaxRanks];     // tile flags there
  const unsigned long long *fcredit[kMaxRanks];  // local credit words for those slots
  uint32_t fepoch[kMaxRanks];
};

// D items of a decode job (runs of `run` consecutive tiles).
__host__ __device__ inline uint64_t items_of(const DecJob &J) {
  return J.run > 1 ? (J.ntiles + J.run - 1) / J.run : J.ntiles;
}

struct CopyJob {
  const uint8_t *src;
  uint8_t *dst;
  uint64_t bytes;
  uint64_t ntiles;
};

struct Plan {
  int32_t ne, nd_jobs, has_copy, dtype;
  EncJob e[kMaxRanks];
  DecJob d[kMaxRanks];
  CopyJob c;
  uint64_t n_e_items, n_c_items, n_d_items;
  uint32_t *ticket;                         // self-resetting ticket + exit counter (2 words)
  uint32_t *err;                            // sticky async error word
  uint64_t timeout_ns;
  int32_t ring_bytes;                       // set by the launcher: smem ring for parked coded tiles
  uint32_t stress;                          // debug: != 0 injects pseudo-random delays (UZIP_STRESS)
  uint32_t credit_ready;                    // 1: k_credit already waited for every slot credit of this launch
  uint32_t share;                           // ranks whose kernels share this GPU (loopback / co-located processes)
  float *acc;                               // reduce: fp32 accumulators, B floats per (CTA, warp) (L2-resident)
  uint32_t codec_call;                      // 1: uzip_compress -- the last CTA out reports an internal
                                            // failure as *d_out_bytes = 0 and clears the error word
  // Fused allreduce (a9, R26): e[ag_job] (>= ne, so it has no E items of its own) is the allgather-phase
  // stream of this rank's reduced shard.  The reduce items of job d[0] round each reduced tile and
  // code it straight into that stream (one pass, no HBM round trip); the chunk's first tile samples
  // the table (tabflag[c] = e[ag_job].partial[c] publishes it to the other tiles of the chunk).
  int32_t ag_job;                           // -1: none
};

// Slot credits one launch needs (a12), waited for by k_credit -- one thread --
// before the fused kernel starts, so its CTAs never hold SM slots while the
// consumer that releases the credit still needs them (loopback, co-scheduled
// compute).
struct CreditWait {
  const unsigned long long *cr[2 * kMaxRanks];
  uint32_t epoch[2 * kMaxRanks];
  uint32_t n;
  uint32_t stress;
  uint32_t *err;
  uint64_t timeout_ns;
};

// k_hist splits a chunk's sample over up to kMaxHistParts CTAs of >= 16 Ki symbols.
constexpr uint32_t kMaxHistParts = 64;
__host__ __device__ inline uint32_t hist_parts(uint32_t sample_len) {
  const uint32_t p = (sample_len + 16383) / 16384;
  return p < 1 ? 1 : (p > kMaxHistParts ? kMaxHistParts : p);
}

// Workspace of one encode job: enc entries, serialized tables, look-back
// words, partial histograms (all written by k_hist/k_norm before use: no state
// survives a launch, so the layout may change from call to call).
struct EncWs {
  static uint64_t bytes(uint64_t n_chunks, uint64_t n_blocks) {
    return round16(4096 * n_chunks) + round16(512 * n_chunks) + round16(8 * (n_blocks + 1)) +
           round16(1024ull * kMaxHistParts * n_chunks);
  }
  static void carve(uint8_t *p, uint64_t n_chunks, uint64_t n_blocks, EncJob &j) {
    j.enc = reinterpret_cast<uint4 *>(p);
    p += round16(4096 * n_chunks);
    j.tab16 = reinterpret_cast<uint16_t *>(p);
    p += round16(512 * n_chunks);
    j.tile_status = reinterpret_cast<unsigned long long *>(p);
    p += round16(8 * (n_blocks + 1));
    j.partial = reinterpret_cast<uint32_t *>(p);
  }
};

static_assert(sizeof(Plan) <= 30000, "kernel parameter space");

cudaError_t launch_tables(int dtype, const Plan &p, cudaStream_t st);
cudaError_t preload_kernels();  // per device: defeat lazy loading for spin-waiting kernels
cudaError_t launch_fused(int dtype, const Plan &p, cudaStream_t st, int max_ctas);
cudaError_t launch_credit_wait(const CreditWait &w, cudaStream_t st);

}  // namespace uzip
