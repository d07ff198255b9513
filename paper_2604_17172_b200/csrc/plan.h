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
constexpr uint32_t kEpochMask = (1u << 24) - 1;  // launch epochs (Plan::epoch) are 24-bit
constexpr uint32_t kRawTileBytes = 64u << 10;

// Tiles (kTileBlocks blocks each) of a stream; a stream without whole blocks
// still has one tile (header + raw tail).
__host__ __device__ inline uint64_t tiles_of(const StreamGeom &g) {
  const uint64_t t = g.n_tiles();
  return t ? t : 1;
}

// Tables of an encode job are built inside the fused kernel by T items (a2 + a3): one per part of
// each chunk's sample; the last part of a chunk to finish applies rule N1 and publishes the chunk's
// table flag = epoch + 1 (table build fused into the single kernel).
struct EncJob {
  const uint8_t *in;                        // local input of this stream
  StreamGeom g;                             // geometry (compressed mode)
  uint64_t raw_bytes;                       // raw mode: message bytes
  uint64_t ntiles;                          // >= 1
  uint32_t raw;                             // 1 = raw (uncoded) tiles
  uint32_t nd;                              // destinations
  uint32_t has_flags;                       // some destination has tile flags (set by plan_flags)
  uint8_t *dst[kMaxRanks];                  // stream base at each destination
  unsigned long long *flag[kMaxRanks];      // tile flags at each destination (null: no flags)
  const unsigned long long *credit[kMaxRanks];  // local word: last epoch the destination consumed from this slot
  uint32_t epoch[kMaxRanks];                // flag epoch per destination (round sequence + 1)
  uint4 *enc;                               // per-chunk encode entries (k_norm)
  uint16_t *tab16;                          // per-chunk serialized tables (k_norm)
  unsigned long long *tile_status;          // per-tile look-back words (zeroed by k_hist)
  uint32_t *partial;                        // [chunk][hist_cap(global)][256] partial counts, a row per part
  unsigned long long *tflag;                // per chunk: table published = kCtlTag | (epoch + 1)
  unsigned long long *tcount;               // per chunk: kCtlTag | epoch << 32 | parts done (T items)
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
  uint64_t n_t_items, n_e_items, n_c_items, n_d_items;
  uint64_t e_tmin;                          // fewest tiles of any encode job (E items are tile-major)
  uint32_t *ticket;                         // self-resetting ticket + exit counter (2 words)
  uint32_t *epoch;                          // launch epoch of this workspace (24 bits): read by every CTA at
                                            // start, advanced by the last CTA out; tags the look-back words
                                            // and the per-chunk table flags, so nothing needs resetting
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
  uint32_t tables_ready;                    // 1: k_hist + k_norm built every encode table before this
                                            // launch (stream order), E items skip the table flag wait
  // optional tile trace (UZIP_TRACE=1, communicators only): events of 2 x u64 -- kind:4 | job:4 | tile:56,
  // %globaltimer ns -- appended through *trace_n (uzip_comm_trace); null when off
  unsigned long long *trace;
  uint32_t *trace_n;
  uint32_t trace_cap;
};

// Tile trace event kinds (overlap evidence: E items publish tiles while D items of the same round,
// on the peer, decode earlier ones).
enum TraceKind : uint32_t { kTrEStart = 1, kTrEFlag = 2, kTrDAcq = 3, kTrDDone = 4 };

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

// A chunk's sample is split over parts of >= 16 Ki symbols, at most hist_cap(global) of them (64 per
// chunk; the global-table mode samples the whole stream as one chunk: up to 512).
// Every part writes its own row of partial counts, so no state needs clearing between launches
// (a workspace may be reused for streams of other sizes, whose layout puts other data there).
__host__ __device__ inline uint32_t hist_cap(uint32_t global) { return global ? 512u : 64u; }
__host__ __device__ inline uint32_t hist_parts(uint32_t sample_len, uint32_t global) {
  const uint32_t p = (sample_len + 16383) / 16384, cap = hist_cap(global);
  return p < 1 ? 1 : (p > cap ? cap : p);
}
// Table flags and part counters are 64-bit words tagged with the top two bits set, a value no other
// workspace word ever holds (look-back words use flags 1 and 2 there; counts, tables and entries
// stay below 2^62), so a stale word of an earlier, differently laid-out call can never match.
constexpr unsigned long long kCtlTag = 3ull << 62;

// Workspace of one encode job: enc entries, serialized tables, look-back
// words, partial histograms (all written by k_hist/k_norm before use: no state
// survives a launch, so the layout may change from call to call).
struct EncWs {
  static uint64_t bytes(uint64_t n_chunks, uint64_t n_blocks, uint32_t global) {
    return round16(4096 * n_chunks) + round16(512 * n_chunks) + round16(8 * (n_blocks + 1)) +
           round16(1024ull * hist_cap(global) * n_chunks) + 2 * round16(8 * n_chunks);
  }
  static void carve(uint8_t *p, uint64_t n_chunks, uint64_t n_blocks, uint32_t global, EncJob &j) {
    j.enc = reinterpret_cast<uint4 *>(p);
    p += round16(4096 * n_chunks);
    j.tab16 = reinterpret_cast<uint16_t *>(p);
    p += round16(512 * n_chunks);
    j.tile_status = reinterpret_cast<unsigned long long *>(p);
    p += round16(8 * (n_blocks + 1));
    j.partial = reinterpret_cast<uint32_t *>(p);
    p += round16(1024ull * hist_cap(global) * n_chunks);
    j.tflag = reinterpret_cast<unsigned long long *>(p);
    p += round16(8 * n_chunks);
    j.tcount = reinterpret_cast<unsigned long long *>(p);
  }
};

// T items of an encode job: every chunk's sample split into hist_parts(sample, global) parts (all chunks but
// the last have the same sample length).
__host__ __device__ inline uint64_t t_items_of(const EncJob &J) {
  if (J.raw || J.g.n_blocks == 0) return 0;
  const uint64_t nc = J.g.n_chunks;
  return (nc - 1) * hist_parts(J.g.sample_len(0), J.g.global) + hist_parts(J.g.sample_len(nc - 1), J.g.global);
}
__host__ __device__ inline void t_item_at(const EncJob &J, uint64_t k, uint64_t &c, uint32_t &part) {
  const uint64_t nc = J.g.n_chunks, pf = hist_parts(J.g.sample_len(0), J.g.global);
  if (k < (nc - 1) * pf) {
    c = k / pf;
    part = (uint32_t)(k % pf);
  } else {
    c = nc - 1;
    part = (uint32_t)(k - (nc - 1) * pf);
  }
}

// E item `it` -> (job, tile).  Tile-major over the encode jobs (every destination receives tile t of
// its stream at about the same time); jobs may have different tile counts (uneven allreduce shards):
// below the smallest count the map is it % ne / it / ne, above it the jobs that still have tile t
// take turns in job order.
__host__ __device__ inline void e_item_at(const Plan &P, uint64_t it, int &job, uint64_t &tile) {
  const uint64_t ne = (uint64_t)P.ne;
  if (it < P.e_tmin * ne) {
    job = (int)(it % ne);
    tile = it / ne;
    return;
  }
  uint64_t r = it - P.e_tmin * ne;
  for (uint64_t t = P.e_tmin;; ++t) {
    for (int j = 0; j < P.ne; ++j)
      if (P.e[j].ntiles > t) {
        if (r == 0) {
          job = j;
          tile = t;
          return;
        }
        --r;
      }
  }
}

// Host: derive EncJob::has_flags of every encode job of a plan (call before the launch).
inline void plan_flags(Plan &p) {
  for (int j = 0; j < kMaxRanks; ++j) {
    p.e[j].has_flags = 0;
    for (uint32_t d = 0; d < p.e[j].nd; ++d) p.e[j].has_flags |= p.e[j].flag[d] != nullptr;
  }
  p.e_tmin = ~0ull;
  for (int j = 0; j < p.ne; ++j) p.e_tmin = p.e[j].ntiles < p.e_tmin ? p.e[j].ntiles : p.e_tmin;
  if (p.ne == 0) p.e_tmin = 0;
}

static_assert(sizeof(Plan) <= 30000, "kernel parameter space");

cudaError_t launch_tables(int dtype, const Plan &p, cudaStream_t st);
cudaError_t preload_kernels();  // per device: defeat lazy loading for spin-waiting kernels
cudaError_t launch_fused(int dtype, const Plan &p, cudaStream_t st, int max_ctas);
cudaError_t launch_credit_wait(const CreditWait &w, cudaStream_t st);

}  // namespace uzip
