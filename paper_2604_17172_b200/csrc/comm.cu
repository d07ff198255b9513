// comm.cu -- communicator and the compressed P2P / collective entry points.
//
// Host side only: it lays out the symmetric region every rank exports
// (staging slots, tile flags, credits), maps the peers' regions (CUDA IPC
// between processes, direct pointers in single-process mode), and turns each
// call into rounds of at most one staging slot, each round = k_hist + k_norm + one
// k_fused launch (fused.cu).  No host synchronization on the data path.
//
// Paper: split-send P2P, compress-on-send / decompress-
// (reduce)-on-receive collectives, two-shot allreduce,
// selective compression and threshold, bounded staging
// (P:487-490).  Readings R10-R12 in DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "plan.h"
#include "uzip_internal.h"

using namespace uzip;

namespace {

constexpr uint64_t kCtrlBytes = 256;
constexpr uint32_t kMagic = 0x555A4950u;  // "PIZU"

struct Layout {
  uint64_t slot_bytes, max_tiles;
  uint64_t off_credit, off_flags, off_stage, total;
  void init(int nranks, uint64_t slot) {
    slot_bytes = round16(slot);
    max_tiles = slot_bytes / 8192 + 2;
    off_credit = kCtrlBytes;
    off_flags = round16(off_credit + 8ull * kMaxRanks * 2);
    off_stage = (off_flags + 8ull * nranks * 2 * max_tiles + 4095) & ~4095ull;
    total = off_stage + (uint64_t)nranks * 2 * slot_bytes;
  }
  uint64_t credit(int dst, int slot) const { return off_credit + 8ull * (dst * 2 + slot); }
  uint64_t flags(int src, int slot) const { return off_flags + 8ull * ((uint64_t)(src * 2 + slot) * max_tiles); }
  uint64_t stage(int src, int slot) const { return off_stage + (uint64_t)(src * 2 + slot) * slot_bytes; }
};

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

struct uzip_comm {
  uint32_t magic;
  int nranks, rank, device;
  bool ipc;
  uzip_config_t cfg;
  Layout L;
  uint8_t *region;                 // own symmetric region
  uint8_t *peer[kMaxRanks];        // every rank's region as addressable from here
  uint32_t send_seq[kMaxRanks];    // rounds sent to / received from each peer (epoch = seq + 1)
  uint32_t recv_seq[kMaxRanks];
  uint8_t *ws;                     // local workspace: ticket, done counters, wire counter, encode jobs
  uint64_t ws_bytes, ws_job_bytes, max_chunks;
  cudaStream_t side;               // private stream for host reads (async error, stats)
  uzip_stats_t last;
  int nested;                      // inside uzip_allreduce: phases accumulate stats
  uint32_t call_rounds;            // fused launches issued by the current call
  uint32_t share;                  // ranks (incl. this one) whose kernels run on this same GPU
  float *acc;                      // reduce accumulators (allocated by the first reduce call)
  unsigned long long *trace;       // tile trace events (UZIP_TRACE=1), 2 x u64 each
  uint32_t *trace_n;
  uint32_t trace_cap;
};

namespace {

uint32_t *ws_ticket(uzip_comm *c) { return reinterpret_cast<uint32_t *>(c->ws); }
uint32_t *ws_done(uzip_comm *c, int j) { return reinterpret_cast<uint32_t *>(c->ws + 16) + j; }
unsigned long long *ws_wire(uzip_comm *c) { return reinterpret_cast<unsigned long long *>(c->ws + 64); }
uint8_t *ws_job(uzip_comm *c, int j) { return c->ws + 128 + (uint64_t)j * c->ws_job_bytes; }

uzip_config_t resolve_cfg(const uzip_config_t *in) {
  uzip_config_t c;
  memset(&c, 0, sizeof c);
  if (in) c = *in;
  auto env = [](const char *k, uint64_t dflt) -> uint64_t {
    const char *v = getenv(k);
    return v ? strtoull(v, nullptr, 0) : dflt;
  };
  if (!c.min_compress_bytes) c.min_compress_bytes = env("UZIP_MIN_COMPRESS_BYTES", 1ull << 20);
  if (c.min_compress_bytes == ~0ull) c.min_compress_bytes = ~0ull;  // never compress
  if (!c.staging_bytes) c.staging_bytes = env("UZIP_STAGING_BYTES", 512ull << 20);
  if (!c.pipe_chunk_bytes) c.pipe_chunk_bytes = env("UZIP_PIPE_CHUNK_BYTES", ~0ull);
  // rounds start at multiples of the pipe chunk: keep them 16-byte aligned for the 128-bit raw path
  c.pipe_chunk_bytes = std::max<uint64_t>(16, c.pipe_chunk_bytes & ~15ull);
  if (!c.max_ctas) c.max_ctas = (uint32_t)env("UZIP_MAX_CTAS", 0);
  if (!c.poll_timeout_ms) c.poll_timeout_ms = (uint32_t)env("UZIP_POLL_TIMEOUT_MS", 10000);
  return c;
}

// Allocate and zero the local region and workspace of a communicator.
uzip_status_t alloc_local(uzip_comm *c) {
  if (cudaSetDevice(c->device) != cudaSuccess) return UZIP_ERR_CUDA;
  if (c->cfg.staging_bytes < (2ull << 20)) return UZIP_ERR_INVALID_ARG;  // >= 2 slots of 1 MiB
  c->L.init(c->nranks, c->cfg.staging_bytes / 2);
  if (cudaMalloc(&c->region, c->L.total) != cudaSuccess) return UZIP_ERR_CUDA;
  if (cudaMemset(c->region, 0, c->L.off_stage) != cudaSuccess) return UZIP_ERR_CUDA;
  // workspace sized for the largest round any call can plan (one slot of elements)
  StreamGeom g;
  uzip_status_t st = resolve_geom(kBF16, c->L.slot_bytes / 2, &c->cfg.codec, &g);
  if (st != UZIP_OK) return st;
  c->max_chunks = g.n_chunks + 1;
  c->ws_job_bytes = EncWs::bytes(c->max_chunks, g.n_blocks + kTileBlocks, g.global);
  c->ws_bytes = 128 + (uint64_t)kMaxRanks * c->ws_job_bytes;
  if (cudaMalloc(&c->ws, c->ws_bytes) != cudaSuccess) return UZIP_ERR_CUDA;
  if (cudaMemset(c->ws, 0, c->ws_bytes) != cudaSuccess) return UZIP_ERR_CUDA;
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) return UZIP_ERR_CUDA;
  if (preload_kernels() != cudaSuccess) return UZIP_ERR_CUDA;
  if (getenv("UZIP_TRACE") && atoi(getenv("UZIP_TRACE")) != 0) {  // tile trace (overlap evidence)
    c->trace_cap = 1u << 20;
    if (cudaMalloc(&c->trace, 16ull * c->trace_cap + 16) != cudaSuccess) return UZIP_ERR_CUDA;
    c->trace_n = reinterpret_cast<uint32_t *>(c->trace + 2ull * c->trace_cap);
    if (cudaMemset(c->trace_n, 0, 16) != cudaSuccess) return UZIP_ERR_CUDA;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return UZIP_ERR_CUDA;
  return UZIP_OK;
}

uzip_comm *new_comm(int nranks, int rank, int device, const uzip_config_t *cfg) {
  uzip_comm *c = new uzip_comm;
  memset(c, 0, sizeof *c);
  c->magic = kMagic;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->cfg = resolve_cfg(cfg);
  return c;
}

void free_comm(uzip_comm *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->ipc)
    for (int p = 0; p < c->nranks; ++p)
      if (p != c->rank && c->peer[p]) cudaIpcCloseMemHandle(c->peer[p]);
  if (c->region) cudaFree(c->region);
  if (c->ws) cudaFree(c->ws);
  if (c->acc) cudaFree(c->acc);
  if (c->trace) cudaFree(c->trace);
  if (c->side) cudaStreamDestroy(c->side);
  c->magic = 0;
  delete c;
}

bool valid(uzip_comm *c) { return c && c->magic == kMagic; }

// ---------------------------------------------------------------- round planning
// Elements per round: the largest multiple of one table chunk (CB*B) whose
// worst-case stream fits a staging slot; raw rounds fill the slot.
uint64_t round_elems(uzip_comm *c, int dt, bool compressed, uint64_t count, StreamGeom *g_full) {
  const uint32_t eb = elem_bytes(dt);
  if (!compressed) return std::max<uint64_t>(1, std::min<uint64_t>(c->L.slot_bytes, c->cfg.pipe_chunk_bytes) / eb);
  StreamGeom g;
  resolve_geom(dt, count, &c->cfg.codec, &g);
  if (g_full) *g_full = g;
  const uint64_t cap = std::min<uint64_t>(c->L.slot_bytes, c->cfg.pipe_chunk_bytes) / eb;
  auto fits = [&](uint64_t elems) {
    StreamGeom t;
    resolve_geom(dt, elems, &c->cfg.codec, &t);
    return t.total(t.n_blocks * (uint64_t)t.B) <= c->L.slot_bytes && t.n_tiles() + 1 <= c->L.max_tiles &&
           t.n_chunks < c->max_chunks && EncWs::bytes(t.n_chunks, t.n_blocks, t.global) <= c->ws_job_bytes;
  };
  // whole table chunks when one fits a slot and the pipe chunk, else whole tiles (a round shorter
  // than a chunk has one chunk)
  const uint64_t ge = group_elems(dt);  // rounds split at symbol-group boundaries
  uint64_t unit = (g.global ? (uint64_t)g.B * kTileBlocks : (uint64_t)g.CB * g.B) * ge;
  if (unit > cap || !fits(unit)) unit = (uint64_t)g.B * kTileBlocks * ge;
  uint64_t lo = 1, hi = std::max<uint64_t>(1, cap / unit);
  while (lo < hi) {  // largest k <= cap / unit (at least 1) with k*unit fitting a slot and the workspace
    const uint64_t k = (lo + hi + 1) / 2;
    if (fits(k * unit)) lo = k;
    else hi = k - 1;
  }
  return lo * unit;
}

// Serialised kernel execution (CUDA_LAUNCH_BLOCKING=1, a kernel profiler, or the explicit knob):
// kernels of co-resident ranks can no longer run side by side (uzip.h, uzip_comm_init_all).
bool serialized_env() {
  static const int v = [] {
    const char *k = getenv("UZIP_SERIALIZED");
    if (k) return atoi(k) != 0 ? 1 : 0;
    const char *b = getenv("CUDA_LAUNCH_BLOCKING");
    if (b && atoi(b) != 0) return 1;
    const char *inj = getenv("CUDA_INJECTION64_PATH");  // ncu / nsys inject a library into the target
    if (inj && (strstr(inj, "nsight") || strstr(inj, "Nsight") || strstr(inj, "ncu"))) return 1;
    return 0;
  }();
  return v != 0;
}

bool compress_message(uzip_comm *c, uint64_t message_bytes) { return message_bytes >= c->cfg.min_compress_bytes; }

void base_plan(uzip_comm *c, Plan &p, int dt) {
  memset(&p, 0, sizeof p);
  p.ag_job = -1;
  p.dtype = dt;
  p.ticket = ws_ticket(c);
  p.epoch = reinterpret_cast<uint32_t *>(c->ws + 8);
  p.trace = c->trace;
  p.trace_n = c->trace_n;
  p.trace_cap = c->trace_cap;
  p.err = reinterpret_cast<uint32_t *>(c->region);
  p.acc = c->acc;
  p.timeout_ns = (uint64_t)c->cfg.poll_timeout_ms * 1000000ull;
  static const uint32_t stress = (uint32_t)strtoul(getenv("UZIP_STRESS") ? getenv("UZIP_STRESS") : "0", nullptr, 0);
  p.stress = stress;
  // debug knob: UZIP_SHARE_CAP=0 sizes launches as if the GPU were not shared (measurement of one
  // side alone only -- co-resident ranks that run concurrently need the cap)
  static const bool share_cap = !(getenv("UZIP_SHARE_CAP") && atoi(getenv("UZIP_SHARE_CAP")) == 0);
  p.share = (c->share && share_cap) ? c->share : 1;
}

// Encode job of `n` elements at `in` (round stream) into destinations dsts.
void enc_job(uzip_comm *c, Plan &p, int j, int dt, const uint8_t *in, uint64_t n, bool compressed,
             const std::vector<int> &dsts) {
  EncJob &J = p.e[j];
  memset(&J, 0, sizeof J);
  J.in = in;
  J.raw = compressed ? 0 : 1;
  J.raw_bytes = n * elem_bytes(dt);
  if (compressed) {
    resolve_geom(dt, n, &c->cfg.codec, &J.g);
    J.ntiles = tiles_of(J.g);
    EncWs::carve(ws_job(c, j), J.g.n_chunks, J.g.n_blocks, J.g.global, J);
  } else {
    J.ntiles = std::max<uint64_t>(1, (J.raw_bytes + kRawTileBytes - 1) / kRawTileBytes);
  }
  J.nd = (uint32_t)dsts.size();
  for (size_t i = 0; i < dsts.size(); ++i) {
    const int d = dsts[i];
    const uint32_t q = c->send_seq[d]++;
    const int slot = q & 1;
    J.dst[i] = c->peer[d] + c->L.stage(c->rank, slot);
    J.flag[i] = reinterpret_cast<unsigned long long *>(c->peer[d] + c->L.flags(c->rank, slot));
    J.credit[i] = reinterpret_cast<const unsigned long long *>(c->region + c->L.credit(d, slot));
    J.epoch[i] = q + 1;
  }
  J.wire_acc = ws_wire(c);
  p.ne = j + 1;
}

// Decode job: `srcs` in rank order; `me_idx` >= 0 marks the local raw input (reduce).
void dec_job(uzip_comm *c, Plan &p, int j, int dt, uint64_t n, bool compressed, const std::vector<int> &srcs,
             int me_idx, const uint8_t *own, uint8_t *out) {
  DecJob &J = p.d[j];
  memset(&J, 0, sizeof J);
  J.raw = compressed ? 0 : 1;
  J.raw_bytes = n * elem_bytes(dt);
  if (compressed) {
    resolve_geom(dt, n, &c->cfg.codec, &J.g);
    J.ntiles = tiles_of(J.g);
  } else {
    J.ntiles = std::max<uint64_t>(1, (J.raw_bytes + kRawTileBytes - 1) / kRawTileBytes);
  }
  J.nsrc = (uint32_t)srcs.size();
  J.me = me_idx;
  for (size_t i = 0; i < srcs.size(); ++i) {
    if ((int)i == me_idx) {
      J.src[i] = own;
      continue;
    }
    const int s = srcs[i];
    const uint32_t q = c->recv_seq[s]++;
    const int slot = q & 1;
    J.src[i] = c->region + c->L.stage(s, slot);
    J.flag[i] = reinterpret_cast<const unsigned long long *>(c->region + c->L.flags(s, slot));
    J.credit[i] = reinterpret_cast<unsigned long long *>(c->peer[s] + c->L.credit(c->rank, slot));
    J.epoch[i] = q + 1;
  }
  J.out = out;
  J.done = ws_done(c, j);
  // Plain decode jobs take their tiles in runs: a CTA's consecutive tickets are ~grid tiles apart,
  // i.e. in another 8 MiB chunk, so per-tile items rebuilt the 4096-slot decode table for every
  // tile.  Runs stay short next to the message so the receiver still follows the sender closely.
#ifndef UZIP_DEC_RUN_MAX
#define UZIP_DEC_RUN_MAX 8
#endif
  // Reduce jobs with one remote source (2 ranks) reuse that source's table across the run too; with
  // more sources the table changes with every source of a tile anyway, so they keep single tiles.
  J.run = 1;
  const int remote = (int)J.nsrc - (me_idx >= 0 ? 1 : 0);
  if (compressed && remote == 1) {
    J.run = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(UZIP_DEC_RUN_MAX, J.ntiles / 1024));
    // UZIP_DEC_RUN forces the run length (tests: paired-tile D items on small messages)
    static const int forced = getenv("UZIP_DEC_RUN") ? atoi(getenv("UZIP_DEC_RUN")) : 0;
    if (forced > 0) J.run = (uint32_t)forced;
  }
  p.nd_jobs = j + 1;
}

// Relay destinations of decode job j (broadcast): the received stream is also
// stored into `dsts`' staging for src = this rank (one round on each channel).
void fwd_setup(uzip_comm *c, Plan &p, int j, const std::vector<int> &dsts) {
  DecJob &J = p.d[j];
  J.nfwd = (uint32_t)dsts.size();
  for (size_t i = 0; i < dsts.size(); ++i) {
    const int d = dsts[i];
    const uint32_t q = c->send_seq[d]++;
    const int slot = q & 1;
    J.fdst[i] = c->peer[d] + c->L.stage(c->rank, slot);
    J.fflag[i] = reinterpret_cast<unsigned long long *>(c->peer[d] + c->L.flags(c->rank, slot));
    J.fcredit[i] = reinterpret_cast<const unsigned long long *>(c->region + c->L.credit(d, slot));
    J.fepoch[i] = q + 1;
  }
}

// A launch that can only finish while a co-resident peer's launch runs at the same time: it both
// encodes for and decodes from peers, relays, or reuses a slot whose credit a later consumer
// launch releases.
bool needs_coscheduling(const Plan &p) {
  bool remote_src = false, fwd = false, credit = false;
  for (int j = 0; j < p.nd_jobs; ++j) {
    remote_src |= p.d[j].nsrc > (p.d[j].me >= 0 ? 1u : 0u);
    fwd |= p.d[j].nfwd > 0;
    for (uint32_t d = 0; d < p.d[j].nfwd; ++d) credit |= p.d[j].fepoch[d] > 2;
  }
  for (int j = 0; j < p.ne + (p.ag_job >= 0 ? 1 : 0); ++j)
    for (uint32_t d = 0; d < p.e[j].nd; ++d) credit |= p.e[j].credit[d] && p.e[j].epoch[d] > 2;
  return (p.ne > 0 && remote_src) || fwd || credit;
}

uzip_status_t launch(uzip_comm *c, Plan &p, bool compressed, cudaStream_t st) {
  if (c->share > 1 && serialized_env() && needs_coscheduling(p)) return UZIP_ERR_COMM;  // fail fast, no hang
  plan_flags(p);
  static const bool dbg = getenv("UZIP_DEBUG_PLAN") != nullptr;
  if (dbg) {
    fprintf(stderr, "[rank %d] launch ne=%d nd=%d ag=%d:", c->rank, p.ne, p.nd_jobs, p.ag_job);
    for (int j = 0; j < p.ne + (p.ag_job >= 0 ? 1 : 0); ++j)
      fprintf(stderr, " E%d(raw%u n=%llu tiles=%llu ep=%u)", j, p.e[j].raw,
              (unsigned long long)(p.e[j].raw ? p.e[j].raw_bytes : p.e[j].g.n), (unsigned long long)p.e[j].ntiles,
              p.e[j].epoch[0]);
    for (int j = 0; j < p.nd_jobs; ++j)
      fprintf(stderr, " D%d(raw%u nsrc=%u me=%d tiles=%llu ep0=%u ep1=%u)", j, p.d[j].raw, p.d[j].nsrc, p.d[j].me,
              (unsigned long long)p.d[j].ntiles, p.d[j].epoch[0], p.d[j].epoch[1]);
    fprintf(stderr, "\n");
  }
  for (int j = 0; j < p.ne; ++j) p.n_e_items += p.e[j].ntiles;
  for (int j = 0; j < p.nd_jobs; ++j) p.n_d_items += items_of(p.d[j]);
  p.n_c_items = p.has_copy ? p.c.ntiles : 0;
  // the sampled tables: T items at the front of the fused kernel's ticket space (default), or the
  // k_hist + k_norm launches (A/B), which need no slot and overlap the credit wait
  if (compressed && p.ne > 0) {
    uint64_t chunks = 0;
    for (int j = 0; j < p.ne; ++j) chunks = std::max<uint64_t>(chunks, p.e[j].raw ? 0 : p.e[j].g.n_chunks);
    if (table_kernels(chunks, false)) {
      if (launch_tables(p.dtype, p, st) != cudaSuccess) return UZIP_ERR_CUDA;
      p.tables_ready = 1;
    } else {
      for (int j = 0; j < p.ne; ++j) p.n_t_items += t_items_of(p.e[j]);
    }
  }
  // From the third launch of a call on, a slot's credit comes from a consumer
  // launch of this same call: wait for it in k_credit (one thread) instead of
  // in every CTA of the fused kernel, which would hold SM slots the consumer
  // may need when both share a GPU (a12).  Ranks that share their GPU always
  // wait this way: a credit owed by an earlier call is just as likely to come
  // from a consumer kernel that is still queued behind the spinning producer
  // (measured: 8 back-to-back 30 MiB sends issued before their recvs timed out).
#ifndef UZIP_SHARED_CREDIT_KERNEL
#define UZIP_SHARED_CREDIT_KERNEL 1
#endif
  const bool first_rounds = c->call_rounds++ < 2;
  if (!first_rounds || (UZIP_SHARED_CREDIT_KERNEL && c->share > 1)) {
    CreditWait w;
    memset(&w, 0, sizeof w);
    for (int j = 0; j < p.ne + (p.ag_job >= 0 ? 1 : 0); ++j)  // + the fused allgather stream
      for (uint32_t d = 0; d < p.e[j].nd; ++d)
        if (p.e[j].credit[d] && p.e[j].epoch[d] > 2 && w.n < 2 * kMaxRanks) {
          w.cr[w.n] = p.e[j].credit[d];
          w.epoch[w.n++] = p.e[j].epoch[d];
        }
    for (int j = 0; j < p.nd_jobs; ++j)
      for (uint32_t d = 0; d < p.d[j].nfwd; ++d)
        if (p.d[j].fcredit[d] && p.d[j].fepoch[d] > 2 && w.n < 2 * kMaxRanks) {
          w.cr[w.n] = p.d[j].fcredit[d];
          w.epoch[w.n++] = p.d[j].fepoch[d];
        }
    if (w.n) {
      w.err = p.err;
      w.timeout_ns = p.timeout_ns;
      if (launch_credit_wait(w, st) != cudaSuccess) return UZIP_ERR_CUDA;
      p.credit_ready = 1;
    }
  }
  if (launch_fused(p.dtype, p, st, (int)c->cfg.max_ctas) != cudaSuccess) return UZIP_ERR_CUDA;
  return UZIP_OK;
}

std::vector<int> peers_from(uzip_comm *c) {  // rank+1, rank+2, ... (spreads first-hop load)
  std::vector<int> v;
  for (int i = 1; i < c->nranks; ++i) v.push_back((c->rank + i) % c->nranks);
  return v;
}

// Stats of a call: raw_bytes = bytes this rank would store into peers
// uncompressed; wire_bytes = bytes it actually stored (device counter for
// compressed streams).
uzip_status_t begin_call(uzip_comm *c, uint64_t egress_raw, bool compressed, cudaStream_t st) {
  if (cudaSetDevice(c->device) != cudaSuccess) return UZIP_ERR_CUDA;
  if (c->nested) {
    c->last.raw_bytes += egress_raw;
    return UZIP_OK;
  }
  c->call_rounds = 0;
  c->last.raw_bytes = egress_raw;
  c->last.compressed = compressed ? 1 : 0;
  c->last.wire_bytes = 0;
  if (cudaMemsetAsync(ws_wire(c), 0, 8, st) != cudaSuccess) return UZIP_ERR_CUDA;
  return UZIP_OK;
}

// fp32 accumulators of the reduce kernel: B (<= 4096) floats per warp of every
// CTA the largest grid can hold (4 per SM bounds the reduce kernel's occupancy).
uzip_status_t ensure_acc(uzip_comm *c) {
  if (c->acc) return UZIP_OK;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess) return UZIP_ERR_CUDA;
  const size_t bytes = (size_t)sms * 4 * kWarps * kMaxB * sizeof(float);
  return cudaMalloc(&c->acc, bytes) == cudaSuccess ? UZIP_OK : UZIP_ERR_CUDA;
}

uzip_status_t check_dtype(uzip_dtype_t dt) {
  return ((int)dt < 0 || (int)dt >= kNumDtypes) ? UZIP_ERR_UNSUPPORTED_DTYPE : UZIP_OK;
}
// reductions are defined for bf16/f16/f32 only (R22); the reduce kernel's fp32 accumulators hold
// blocks of at most kMaxB symbols (larger blocks: codec, P2P, allgather, all-to-all, broadcast only)
uzip_status_t check_reduce_dtype(uzip_comm_t c, uzip_dtype_t dt) {
  if ((int)dt < 0 || (int)dt > kF32) return UZIP_ERR_UNSUPPORTED_DTYPE;
  return c->cfg.codec.block_symbols > kMaxB ? UZIP_ERR_INVALID_ARG : UZIP_OK;
}

}  // namespace

// ================================================================ C ABI
extern "C" {

uzip_status_t uzip_comm_init(uzip_comm_t *comm, int nranks, int rank, int cuda_device, uzip_allgather_fn bootstrap,
                             void *ctx, const uzip_config_t *cfg) {
  NvtxRange nvtx_range("uzip_comm_init");
  if (!comm || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || !bootstrap)
    return UZIP_ERR_INVALID_ARG;
  *comm = nullptr;
  uzip_comm *c = new_comm(nranks, rank, cuda_device, cfg);
  c->ipc = true;
  uzip_status_t st = alloc_local(c);
  if (st != UZIP_OK) {
    free_comm(c);
    return st;
  }
  struct Card {
    cudaIpcMemHandle_t h;
    uint64_t total, slot, max_tiles;
    int32_t device, rank;
    unsigned char uuid[16];  // which physical GPU: co-located ranks share its SMs
  } mine, all[kMaxRanks];
  memset(&mine, 0, sizeof mine);
  if (cudaIpcGetMemHandle(&mine.h, c->region) != cudaSuccess) {
    free_comm(c);
    return UZIP_ERR_CUDA;
  }
  mine.total = c->L.total;
  mine.slot = c->L.slot_bytes;
  mine.max_tiles = c->L.max_tiles;
  mine.device = cuda_device;
  mine.rank = rank;
  {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cuda_device) == cudaSuccess) memcpy(mine.uuid, prop.uuid.bytes, 16);
  }
  if (bootstrap(&mine, all, sizeof(Card), ctx) != 0) {
    free_comm(c);
    return UZIP_ERR_COMM;
  }
  for (int p = 0; p < nranks; ++p) {
    if (all[p].rank != p || all[p].slot != mine.slot || all[p].total != mine.total) {
      free_comm(c);
      return UZIP_ERR_COMM;  // every rank must use the same configuration
    }
    if (memcmp(all[p].uuid, mine.uuid, 16) == 0) ++c->share;
    if (p == rank) {
      c->peer[p] = c->region;
      continue;
    }
    void *ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, all[p].h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      fprintf(stderr, "uzip_comm_init: rank %d cannot map rank %d: %s\n", rank, p, cudaGetErrorString(e));
      free_comm(c);
      return UZIP_ERR_COMM;
    }
    c->peer[p] = static_cast<uint8_t *>(ptr);
  }
  int dummy = 0, sink[kMaxRanks];
  if (bootstrap(&dummy, sink, sizeof(int), ctx) != 0) {  // everyone mapped everyone
    free_comm(c);
    return UZIP_ERR_COMM;
  }
  *comm = c;
  return UZIP_OK;
}

uzip_status_t uzip_comm_init_all(uzip_comm_t *comms, int nranks, const int *devices, const uzip_config_t *cfg) {
  NvtxRange nvtx_range("uzip_comm_init_all");
  if (!comms || !devices || nranks < 1 || nranks > kMaxRanks) return UZIP_ERR_INVALID_ARG;
  std::vector<uzip_comm *> cs(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    cs[r] = new_comm(nranks, r, devices[r], cfg);
    uzip_status_t st = alloc_local(cs[r]);
    if (st != UZIP_OK) {
      for (auto *c : cs) free_comm(c);
      return st;
    }
  }
  for (int r = 0; r < nranks; ++r) {
    cudaSetDevice(devices[r]);
    for (int p = 0; p < nranks; ++p) {
      cs[r]->peer[p] = cs[p]->region;
      if (devices[p] != devices[r]) {
        cudaError_t e = cudaDeviceEnablePeerAccess(devices[p], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          for (auto *c : cs) free_comm(c);
          return UZIP_ERR_CUDA;
        }
        cudaGetLastError();
      }
    }
  }
  for (int r = 0; r < nranks; ++r) {
    cs[r]->share = 0;
    for (int p = 0; p < nranks; ++p) cs[r]->share += devices[p] == devices[r];
    comms[r] = cs[r];
  }
  return UZIP_OK;
}

uzip_status_t uzip_comm_destroy(uzip_comm_t comm) {
  if (!valid(comm)) return UZIP_ERR_INVALID_ARG;
  cudaSetDevice(comm->device);
  cudaDeviceSynchronize();
  free_comm(comm);
  return UZIP_OK;
}

uzip_status_t uzip_send(const void *buf, size_t count, uzip_dtype_t dtype, int peer, uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_send");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_dtype(dtype)) return s;
  if (peer < 0 || peer >= c->nranks || peer == c->rank) return UZIP_ERR_INVALID_ARG;
  if (count == 0) return UZIP_OK;
  if (!buf || !aligned16(buf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const bool comp = compress_message(c, count * eb);
  cudaStream_t st = (cudaStream_t)stream;
  if (uzip_status_t s = begin_call(c, count * eb, comp, st)) return s;
  const uint64_t per = round_elems(c, dt, comp, count, nullptr);
  for (uint64_t o = 0; o < count; o += per) {
    const uint64_t n = std::min<uint64_t>(per, count - o);
    Plan p;
    base_plan(c, p, dt);
    enc_job(c, p, 0, dt, static_cast<const uint8_t *>(buf) + o * eb, n, comp, {peer});
    if (uzip_status_t s = launch(c, p, comp, st)) return s;
  }
  return UZIP_OK;
}

uzip_status_t uzip_recv(void *buf, size_t count, uzip_dtype_t dtype, int peer, uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_recv");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_dtype(dtype)) return s;
  if (peer < 0 || peer >= c->nranks || peer == c->rank) return UZIP_ERR_INVALID_ARG;
  if (count == 0) return UZIP_OK;
  if (!buf || !aligned16(buf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const bool comp = compress_message(c, count * eb);
  cudaStream_t st = (cudaStream_t)stream;
  if (uzip_status_t s = begin_call(c, 0, comp, st)) return s;
  const uint64_t per = round_elems(c, dt, comp, count, nullptr);
  for (uint64_t o = 0; o < count; o += per) {
    const uint64_t n = std::min<uint64_t>(per, count - o);
    Plan p;
    base_plan(c, p, dt);
    dec_job(c, p, 0, dt, n, comp, {peer}, -1, nullptr, static_cast<uint8_t *>(buf) + o * eb);
    if (uzip_status_t s = launch(c, p, comp, st)) return s;
  }
  return UZIP_OK;
}

uzip_status_t uzip_allgather(const void *sendbuf, void *recvbuf, size_t sendcount, uzip_dtype_t dtype,
                             uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_allgather");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_dtype(dtype)) return s;
  if (sendcount == 0) return UZIP_OK;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const int N = c->nranks, me = c->rank;
  const uint64_t msg = (uint64_t)N * sendcount * eb;  // R10: the user message (total output)
  const bool comp = N > 1 && compress_message(c, msg);
  cudaStream_t st = (cudaStream_t)stream;
  if (uzip_status_t s = begin_call(c, (uint64_t)(N - 1) * sendcount * eb, comp, st)) return s;
  const uint8_t *in = static_cast<const uint8_t *>(sendbuf);
  uint8_t *out = static_cast<uint8_t *>(recvbuf);
  const bool in_place = in == out + (uint64_t)me * sendcount * eb;
  const uint64_t per = round_elems(c, dt, comp, sendcount, nullptr);
  const std::vector<int> peers = peers_from(c);
  for (uint64_t o = 0; o < sendcount; o += per) {
    const uint64_t n = std::min<uint64_t>(per, sendcount - o);
    Plan p;
    base_plan(c, p, dt);
    if (N > 1) enc_job(c, p, 0, dt, in + o * eb, n, comp, peers);  // one stream, fanned out (a10)
    int j = 0;
    for (int s : peers) {
      dec_job(c, p, j, dt, n, comp, {s}, -1, nullptr, out + ((uint64_t)s * sendcount + o) * eb);
      ++j;
    }
    if (!in_place) {
      p.has_copy = 1;
      p.c.src = in + o * eb;
      p.c.dst = out + ((uint64_t)me * sendcount + o) * eb;
      p.c.bytes = n * eb;
      p.c.ntiles = (p.c.bytes + kRawTileBytes - 1) / kRawTileBytes;
    }
    if (uzip_status_t s = launch(c, p, comp, st)) return s;
  }
  return UZIP_OK;
}

uzip_status_t uzip_reduce_scatter(const void *sendbuf, void *recvbuf, size_t recvcount, uzip_dtype_t dtype,
                                  uzip_op_t op, uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_reduce_scatter");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_reduce_dtype(c, dtype)) return s;
  if ((int)op < 0 || (int)op > UZIP_MAX) return UZIP_ERR_INVALID_ARG;
  if (recvcount == 0) return UZIP_OK;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const int N = c->nranks, me = c->rank;
  if (N > 1 && (recvcount * eb) % 16 != 0) return UZIP_ERR_INVALID_ARG;  // shards stay 16-byte aligned (R21)
  const uint64_t msg = (uint64_t)N * recvcount * eb;  // R10: the user message (total input)
  const bool comp = compress_message(c, msg);
  cudaStream_t st = (cudaStream_t)stream;
  if (uzip_status_t s = begin_call(c, (uint64_t)(N - 1) * recvcount * eb, comp, st)) return s;
  if (uzip_status_t s = ensure_acc(c)) return s;
  const uint8_t *in = static_cast<const uint8_t *>(sendbuf);
  uint8_t *out = static_cast<uint8_t *>(recvbuf);
  const uint64_t per = round_elems(c, dt, comp, recvcount, nullptr);
  const std::vector<int> peers = peers_from(c);
  std::vector<int> all;
  for (int r = 0; r < N; ++r) all.push_back(r);
  for (uint64_t o = 0; o < recvcount; o += per) {
    const uint64_t n = std::min<uint64_t>(per, recvcount - o);
    Plan p;
    base_plan(c, p, dt);
    int j = 0;
    for (int d : peers) {  // shard d of my input -> its owner; my own shard is never compressed
      enc_job(c, p, j, dt, in + ((uint64_t)d * recvcount + o) * eb, n, comp, {d});
      ++j;
    }
    if (N == 1) {
      p.has_copy = in + o * eb != out + o * eb;
      p.c.src = in + o * eb;
      p.c.dst = out + o * eb;
      p.c.bytes = n * eb;
      p.c.ntiles = (p.c.bytes + kRawTileBytes - 1) / kRawTileBytes;
    } else {
      dec_job(c, p, 0, dt, n, comp, all, me, in + ((uint64_t)me * recvcount + o) * eb, out + o * eb);
      p.d[0].op = (uint32_t)op;
    }
    if (uzip_status_t s = launch(c, p, comp, st)) return s;
  }
  return UZIP_OK;
}

uzip_status_t uzip_allreduce(const void *sendbuf, void *recvbuf, size_t count, uzip_dtype_t dtype, uzip_op_t op,
                             uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_allreduce");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_reduce_dtype(c, dtype)) return s;
  if ((int)op < 0 || (int)op > UZIP_MAX) return UZIP_ERR_INVALID_ARG;
  if (count == 0) return UZIP_OK;
  const int N = c->nranks, me = c->rank, dt = (int)dtype;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return UZIP_ERR_INVALID_ARG;
  const uint32_t eb = elem_bytes(dt);
  // Two-shot over N shards of `shard` elements (the last ones shorter or empty when
  // count % N != 0): shards start on 16-byte boundaries, so any count works, as with NCCL (R21).
  const uint64_t align = 16 / eb;
  const uint64_t shard = ((count + N - 1) / N + align - 1) / align * align;
  auto len_of = [&](int j) -> uint64_t {
    const uint64_t lo = std::min<uint64_t>(count, (uint64_t)j * shard);
    return std::min<uint64_t>(shard, count - lo);
  };
  const bool comp = compress_message(c, count * eb);  // the user message decides both phases (R10)
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t *in = static_cast<const uint8_t *>(sendbuf);
  uint8_t *out = static_cast<uint8_t *>(recvbuf);
  if (N == 1) {
    if (uzip_status_t s2 = begin_call(c, 0, comp, st)) return s2;
    if (in != out && cudaMemcpyAsync(out, in, count * eb, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return UZIP_ERR_CUDA;
    return UZIP_OK;
  }
  static const bool fused_env = !(getenv("UZIP_AR_FUSED") && atoi(getenv("UZIP_AR_FUSED")) == 0);
  // One pass per round (a9, R26): one launch holds the reduce-scatter streams (E items), the reduce
  // items -- which round each reduced tile and code it straight into the allgather stream to the N-1
  // peers (no HBM round trip, no second table pass) -- and the decoders of the peers' allgather
  // streams, whose per-chunk tables are sampled from each chunk's first tile.  Below the threshold,
  // or with one global table (it needs every reduced symbol first), a round is two launches:
  // reduce-scatter, then allgather of the reduced shard (re-read from recvbuf).
  const bool fused = comp && fused_env && !c->cfg.codec.global_table;
  uint64_t egress = 0;
  for (int d = 0; d < N; ++d)
    if (d != me) egress += (len_of(d) + len_of(me)) * eb;
  if (uzip_status_t s2 = begin_call(c, egress, comp, st)) return s2;
  if (uzip_status_t s2 = ensure_acc(c)) return s2;
  const uint64_t per = round_elems(c, dt, comp, shard, nullptr);
  const std::vector<int> peers = peers_from(c);
  std::vector<int> all;
  for (int r = 0; r < N; ++r) all.push_back(r);
  auto part = [&](int j, uint64_t o) -> uint64_t { const uint64_t L = len_of(j); return L > o ? std::min(per, L - o) : 0; };
  for (uint64_t o = 0; o < shard; o += per) {
    const uint64_t nme = part(me, o);
    uint8_t *mine = out + ((uint64_t)me * shard + o) * eb;
    Plan p;
    base_plan(c, p, dt);
    int j = 0;
    for (int d : peers)  // shard d of my input -> its owner (reduce-scatter streams)
      if (const uint64_t n = part(d, o)) enc_job(c, p, j++, dt, in + ((uint64_t)d * shard + o) * eb, n, comp, {d});
    if (nme) {
      dec_job(c, p, 0, dt, nme, comp, all, me, in + ((uint64_t)me * shard + o) * eb, mine);
      p.d[0].op = (uint32_t)op;
    }
    if (fused && nme) {
      // single tiles per reduce item: the re-encoded tiles finish their look-back in tile order, so
      // runs of consecutive tiles per CTA would chain the CTAs (measured 4x slower at N = 2)
      p.d[0].run = 1;
      // the allgather stream of my reduced shard: e[ne], no E items of its own (p.ne unchanged)
      const int ne = p.ne;
      enc_job(c, p, ne, dt, mine, nme, true, peers);
      p.ne = ne;
      p.ag_job = ne;
      uzip_codec_params_t cp = c->cfg.codec;
      resolve_geom(dt, nme, &cp, &p.e[ne].g);
      cp.sample_symbols = kTileBlocks * p.e[ne].g.B;  // R26: the chunk's first tile is its sample
      resolve_geom(dt, nme, &cp, &p.e[ne].g);
    }
    if (fused) {
      int k = nme ? 1 : 0;
      for (int s : peers)  // the peers' reduced shards
        if (const uint64_t n = part(s, o)) dec_job(c, p, k++, dt, n, true, {s}, -1, nullptr, out + ((uint64_t)s * shard + o) * eb);
    }
    if (p.ne || p.nd_jobs)
      if (uzip_status_t s2 = launch(c, p, comp, st)) return s2;
    if (fused) continue;
    Plan q;  // allgather of the reduced shard (two-launch rounds)
    base_plan(c, q, dt);
    if (nme) enc_job(c, q, 0, dt, mine, nme, comp, peers);
    int k = 0;
    for (int s : peers)
      if (const uint64_t n = part(s, o)) dec_job(c, q, k++, dt, n, comp, {s}, -1, nullptr, out + ((uint64_t)s * shard + o) * eb);
    if (q.ne || q.nd_jobs)
      if (uzip_status_t s2 = launch(c, q, comp, st)) return s2;
  }
  return UZIP_OK;
}

uzip_status_t uzip_alltoall(const void *sendbuf, void *recvbuf, size_t count, uzip_dtype_t dtype, uzip_comm_t c,
                            void *stream) {
  NvtxRange nvtx_range("uzip_alltoall");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_dtype(dtype)) return s;
  if (count == 0) return UZIP_OK;
  if (!sendbuf || !recvbuf || !aligned16(sendbuf) || !aligned16(recvbuf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const int N = c->nranks, me = c->rank;
  if (N > 1 && (count * eb) % 16 != 0) return UZIP_ERR_INVALID_ARG;  // 16-byte aligned per-peer chunks
  {  // out of place only: E items read chunk d of sendbuf while D items write chunk s of recvbuf
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(sendbuf), b0 = reinterpret_cast<uintptr_t>(recvbuf);
    const uint64_t len = (uint64_t)N * count * eb;
    if (a0 < b0 + len && b0 < a0 + len) return UZIP_ERR_INVALID_ARG;
  }
  const uint64_t msg = (uint64_t)N * count * eb;                       // R10: the user message
  const bool comp = compress_message(c, msg);
  cudaStream_t st = (cudaStream_t)stream;
  if (uzip_status_t s = begin_call(c, (uint64_t)(N - 1) * count * eb, comp, st)) return s;
  const uint8_t *in = static_cast<const uint8_t *>(sendbuf);
  uint8_t *out = static_cast<uint8_t *>(recvbuf);
  const uint64_t per = round_elems(c, dt, comp, count, nullptr);
  const std::vector<int> peers = peers_from(c);
  for (uint64_t o = 0; o < count; o += per) {
    const uint64_t n = std::min<uint64_t>(per, count - o);
    Plan p;
    base_plan(c, p, dt);
    int j = 0;
    for (int d : peers) {  // chunk d of my input -> rank d, one stream each
      enc_job(c, p, j, dt, in + ((uint64_t)d * count + o) * eb, n, comp, {d});
      ++j;
    }
    j = 0;
    for (int s : peers) {
      dec_job(c, p, j, dt, n, comp, {s}, -1, nullptr, out + ((uint64_t)s * count + o) * eb);
      ++j;
    }
    const uint8_t *own = in + ((uint64_t)me * count + o) * eb;
    uint8_t *own_out = out + ((uint64_t)me * count + o) * eb;
    if (own != own_out) {
      p.has_copy = 1;
      p.c.src = own;
      p.c.dst = own_out;
      p.c.bytes = n * eb;
      p.c.ntiles = (p.c.bytes + kRawTileBytes - 1) / kRawTileBytes;
    }
    if (uzip_status_t s = launch(c, p, comp, st)) return s;
  }
  return UZIP_OK;
}

uzip_status_t uzip_broadcast(void *buf, size_t count, uzip_dtype_t dtype, int root, uzip_comm_t c, void *stream) {
  NvtxRange nvtx_range("uzip_broadcast");
  if (!valid(c)) return UZIP_ERR_INVALID_ARG;
  if (uzip_status_t s = check_dtype(dtype)) return s;
  if (root < 0 || root >= c->nranks) return UZIP_ERR_INVALID_ARG;
  if (count == 0 || c->nranks == 1) return UZIP_OK;
  if (!buf || !aligned16(buf)) return UZIP_ERR_INVALID_ARG;
  const int dt = (int)dtype;
  const uint32_t eb = elem_bytes(dt);
  const int N = c->nranks, me = c->rank;
  const uint64_t msg = count * eb;
  const bool comp = compress_message(c, msg);
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t *b = static_cast<uint8_t *>(buf);
  std::vector<int> rcv;  // receivers in rank order
  for (int r = 0; r < N; ++r)
    if (r != root) rcv.push_back(r);
  if (!comp || N == 2) {
    // fan-out: the root's one stream (or raw bytes) is stored to every receiver
    if (uzip_status_t s2 = begin_call(c, me == root ? (uint64_t)(N - 1) * msg : 0, comp, st)) return s2;
    const uint64_t per = round_elems(c, dt, comp, count, nullptr);
    for (uint64_t o = 0; o < count; o += per) {
      const uint64_t n = std::min<uint64_t>(per, count - o);
      Plan p;
      base_plan(c, p, dt);
      if (me == root) enc_job(c, p, 0, dt, b + o * eb, n, comp, rcv);
      else dec_job(c, p, 0, dt, n, comp, {root}, -1, nullptr, b + o * eb);
      if (uzip_status_t s2 = launch(c, p, comp, st)) return s2;
    }
    return UZIP_OK;
  }
  // compressed scatter + relay (SURVEY 8(e) weight sync): piece k goes root -> rcv[k] once, rcv[k]
  // forwards the compressed bytes to the other receivers; every receiver decodes every piece.
  const int R = N - 1;
  uint64_t P = (count + R - 1) / R;
  P = (P + 15) & ~15ull;  // pieces of 16 elements: 16-byte aligned for every dtype
  auto piece_len = [&](int k) -> uint64_t {
    const uint64_t lo = std::min<uint64_t>(count, (uint64_t)k * P), hi = std::min<uint64_t>(count, lo + P);
    return hi - lo;
  };
  int mine = -1;
  for (int k = 0; k < R; ++k)
    if (rcv[k] == me) mine = k;
  const uint64_t egress = me == root ? msg : (uint64_t)(R - 1) * piece_len(mine) * eb;
  if (uzip_status_t s2 = begin_call(c, egress, comp, st)) return s2;
  const uint64_t per = round_elems(c, dt, comp, P, nullptr);
  for (uint64_t o = 0; o < P; o += per) {
    Plan p;
    base_plan(c, p, dt);
    auto part = [&](int k) -> uint64_t { const uint64_t L = piece_len(k); return L > o ? std::min(per, L - o) : 0; };
    if (me == root) {
      int j = 0;
      for (int k = 0; k < R; ++k)
        if (const uint64_t n = part(k)) enc_job(c, p, j++, dt, b + ((uint64_t)k * P + o) * eb, n, comp, {rcv[k]});
    } else {
      int j = 0;
      if (const uint64_t n = part(mine)) {
        dec_job(c, p, j, dt, n, comp, {root}, -1, nullptr, b + ((uint64_t)mine * P + o) * eb);
        std::vector<int> hops;
        for (int k = 0; k < R; ++k)
          if (k != mine) hops.push_back(rcv[k]);
        fwd_setup(c, p, j, hops);
        ++j;
      }
      for (int k = 0; k < R; ++k)
        if (k != mine)
          if (const uint64_t n = part(k)) dec_job(c, p, j++, dt, n, comp, {rcv[k]}, -1, nullptr,
                                                  b + ((uint64_t)k * P + o) * eb);
    }
    if (uzip_status_t s2 = launch(c, p, comp, st)) return s2;
  }
  return UZIP_OK;
}

uzip_status_t uzip_comm_get_async_error(uzip_comm_t c, uzip_status_t *err) {
  if (!valid(c) || !err) return UZIP_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  uint32_t v = 0;
  if (cudaMemcpyAsync(&v, c->region, 4, cudaMemcpyDeviceToHost, c->side) != cudaSuccess) return UZIP_ERR_CUDA;
  if (cudaStreamSynchronize(c->side) != cudaSuccess) return UZIP_ERR_CUDA;
  *err = (uzip_status_t)v;
  return UZIP_OK;
}

uzip_status_t uzip_comm_error_detail(uzip_comm_t c, uint32_t *out16) {
  if (!valid(c) || !out16) return UZIP_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  unsigned long long cr[4] = {0, 0, 0, 0};
  bool ok = cudaMemcpyAsync(out16, c->region, 32, cudaMemcpyDeviceToHost, c->side) == cudaSuccess;
  for (int d = 0; d < 2 && d < c->nranks; ++d)  // credit words of peers 0,1 (slots 0,1)
    ok &= cudaMemcpyAsync(cr + 2 * d, c->region + c->L.credit(d, 0), 16, cudaMemcpyDeviceToHost, c->side) ==
          cudaSuccess;
  ok &= cudaMemcpyAsync(out16 + 12, c->ws + 16, 16, cudaMemcpyDeviceToHost, c->side) == cudaSuccess;
  ok &= cudaStreamSynchronize(c->side) == cudaSuccess;
  for (int i = 0; i < 4; ++i) out16[8 + i] = (uint32_t)cr[i];
  out16[7] = c->send_seq[c->rank ? 0 : 1] | (c->recv_seq[c->rank ? 0 : 1] << 16);
  return ok ? UZIP_OK : UZIP_ERR_CUDA;
}

uzip_status_t uzip_comm_read_staging(uzip_comm_t c, int src, int slot, void *host, size_t bytes) {
  if (!valid(c) || src < 0 || src >= c->nranks || src == c->rank || (slot & ~1) || !host) return UZIP_ERR_INVALID_ARG;
  if (bytes > c->L.slot_bytes) return UZIP_ERR_CAPACITY;
  cudaSetDevice(c->device);
  if (cudaMemcpyAsync(host, c->region + c->L.stage(src, slot), bytes, cudaMemcpyDeviceToHost, c->side) != cudaSuccess)
    return UZIP_ERR_CUDA;
  return cudaStreamSynchronize(c->side) == cudaSuccess ? UZIP_OK : UZIP_ERR_CUDA;
}

uzip_status_t uzip_comm_trace(uzip_comm_t c, unsigned long long *host, size_t max_events, size_t *n_events) {
  if (!valid(c) || !n_events) return UZIP_ERR_INVALID_ARG;
  *n_events = 0;
  if (!c->trace) return UZIP_OK;  // tracing off (UZIP_TRACE unset at init)
  cudaSetDevice(c->device);
  if (cudaDeviceSynchronize() != cudaSuccess) return UZIP_ERR_CUDA;
  uint32_t n = 0;
  if (cudaMemcpy(&n, c->trace_n, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return UZIP_ERR_CUDA;
  n = std::min<uint32_t>(n, c->trace_cap);
  const size_t k = std::min<size_t>(n, max_events);
  if (k && host && cudaMemcpy(host, c->trace, 16 * k, cudaMemcpyDeviceToHost) != cudaSuccess) return UZIP_ERR_CUDA;
  *n_events = k;
  return cudaMemset(c->trace_n, 0, 4) == cudaSuccess ? UZIP_OK : UZIP_ERR_CUDA;
}

uzip_status_t uzip_get_stats(uzip_comm_t c, uzip_stats_t *out) {
  if (!valid(c) || !out) return UZIP_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  unsigned long long w = 0;
  if (cudaMemcpyAsync(&w, ws_wire(c), 8, cudaMemcpyDeviceToHost, c->side) != cudaSuccess) return UZIP_ERR_CUDA;
  if (cudaStreamSynchronize(c->side) != cudaSuccess) return UZIP_ERR_CUDA;
  *out = c->last;
  out->wire_bytes = c->last.compressed ? w : c->last.raw_bytes;
  return UZIP_OK;
}

}  // extern "C"
