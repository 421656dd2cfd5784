// vx_handle.cuh — internals shared by the C-ABI translation units (vx_api.cu: handle
// lifecycle, data, host-buffer API, live batcher, comm; vx_stage.cu: the per-batch stage and
// the shard exchange).  Not part of the ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <map>

#include "../../include/vortex_b200.h"
#include "vx_internal.cuh"

// ---------------------------------------------------------------- NCCL (loaded lazily)
// NCCL is dlopen'ed on first use instead of linked: a host process (e.g. PyTorch) may
// already carry its own libnccl.so.2, and two copies under one soname break each other.
// Order: an already-loaded libnccl.so.2, $VX_NCCL_LIB, then the system library.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

NcclApi& nccl();

// thread-local error message (vx_last_error) + status
vx_status fail(vx_status s, const char* fmt, ...);

#define CU_TRY(expr)                                                                     \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(_e == cudaErrorMemoryAllocation ? VX_ERR_OOM : VX_ERR_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(_e), __FILE__, __LINE__);                    \
  } while (0)

#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      return fail(VX_ERR_NCCL, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(_r), __FILE__, \
                  __LINE__);                                                              \
  } while (0)

#define VX_TRY(expr)                 \
  do {                               \
    vx_status _s = (expr);           \
    if (_s != VX_OK) return _s;      \
  } while (0)

// 2-D row-major matrix [rows][cols] of `elem` bytes, box {box_cols, box_rows}, 128B swizzle.
vx_status make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem,
                       uint64_t rows, uint64_t cols, uint32_t box_cols, uint32_t box_rows,
                       uint64_t pitch = 0);  // row pitch in elements (0: cols)

// ---------------------------------------------------------------- handle

struct vx_index {
  vx_index_desc desc{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t row0 = 0, n_local = 0;
  float* docs = nullptr;
  uint16_t* tokens = nullptr;    // bf16 doc-token store [T][Nd][d] (default)
  float* tokens32 = nullptr;     // fp32 doc-token store (VX_FLAG_TOKENS_F32)
  CUtensorMap tmap_docs{};
  CUtensorMap tmap_tok{};
  uint16_t* docs16 = nullptr;    // bf16 shadow of the shard (coarse scan), may be null
  CUtensorMap tmap_docs16{};
  uint16_t* d_q16 = nullptr;     // [maxB][D] bf16 queries for the bf16 coarse scan
  int8_t* docs8 = nullptr;       // s8 shadow (one scale per shard, d_xnorm[5]), may be null
  CUtensorMap tmap_docs8{};
  // 64-row boxes of the same maps: the 128-document pair tiles (scan_tc2, QG = 2)
  CUtensorMap tmap_docs_h{}, tmap_docs16_h{}, tmap_docs8_h{};
  int8_t* d_q8 = nullptr;        // [maxB][D] s8 queries, per-row scales in d_qs8
  float* d_qs8 = nullptr;
  float xstats_host[8] = {};     // host copy of d_xnorm after every upload / synth
  int coarse = VX_COARSE_AUTO;
  int scan_tile = 0;             // documents per tensor-core tile (0 = auto)
  int kprime = 0;                // TC candidate set size k' (0 = auto; VX_OPT_KPRIME)
  int dbg_tc_bits = 0;           // timing-experiment knobs, read once from the environment at
  int dbg_tc_stages = 0;         //   create: VX_DEBUG_TC_NOSELECT (bit mask), VX_DEBUG_TC_STAGES,
  int dbg_seed_stride = 0;       //   VX_DEBUG_SEED_STRIDE (sample row stride, timing only)
  int dbg_seed_m = 0;            //   VX_DEBUG_SEED_M (sample rank of the scan seed, <= 32),
  int dbg_no_rep = 0;            //   VX_DEBUG_NO_REP (no small-batch query replication)
  int scan_seed = 1;             // seed the TC scan's admission thresholds (VX_OPT_SCAN_SEED)
  int i8_per_column = 0;         // s8 shadow column scales: 0 one per shard, 1 per column
  bool i8_demoted = false;       // AUTO left s8 after its certificate kept failing (vx_sync)
  uint64_t cert_seen_q = 0, cert_seen_l2 = 0, cert_seen_l3 = 0;  // demotion window origin
  int use_pairs = 2;             // CTA-pair scan for B > 128: 0 off, 1 on (256-query passes),
                                 // 2 on + 512-query passes for B > 256 (VX_OPT_SCAN_PAIRS)
  // options
  int scan_algo = VX_SCAN_AUTO;
  int maxsim_algo = VX_MAXSIM_AUTO;
  int grid = 0;
  // workspace
  float* d_q = nullptr;          // [maxB][D]
  float* d_qtok = nullptr;       // [maxB][maxNq][d]
  uint16_t* d_qtok16 = nullptr;  // bf16 copy for the shard exchange (half the broadcast bytes)
  uint64_t* d_part = nullptr;    // [maxB][grid][256]
  uint64_t* d_keys = nullptr;    // [maxB][maxK]
  int64_t* d_ids = nullptr;      // [maxB][maxK]
  float* d_ip = nullptr;         // [maxB][maxK]
  float* d_ms = nullptr;         // [maxB][maxK]
  int64_t* d_out_ids = nullptr;  // [maxB][maxK]
  float* d_out_ip = nullptr;
  float* d_out_ms = nullptr;
  void* d_send = nullptr;        // [maxB][maxK] x 8 B scratch (rank 0: the reduced MaxSim)
  void* d_recv = nullptr;        // [G][maxB][maxK] gathered keys (rank 0)
  float* d_lball = nullptr;      // [G][maxB][maxK] all-gathered coarse lower bounds (G > 1)
  float* d_tau = nullptr;        // [maxB] lower bound of the global exact k-th (G > 1)
  uint64_t* d_hkeys = nullptr;   // [maxB][maxK] exact keys of the re-rank head (G > 1)
  int32_t* d_hdr = nullptr;      // [4]
  uint64_t* d_ckeys = nullptr;   // [maxB][1024] merged coarse keys (TC path)
  unsigned* d_qctr = nullptr;     // [maxB] split re-rank: per-query CTA tickets (kept at 0)
  uint64_t* d_seedk = nullptr;   // [maxB][32] best sample keys per query (TC scan seeds)
  int* d_flags = nullptr;        // [maxB] certificate failures (TC path)
  unsigned int* d_xnorm = nullptr;  // [8] shard maxima (float bits, row_stats): |x|, |bf16 x|,
                                    // |x-bf16 x|, |sx x8|, |x-sx x8|; [5] sx; [6] scratch;
                                    // [7] sum of row norms (AUTO coarse heuristic)
  unsigned int* d_colmax = nullptr;  // [D] scratch: per-column |max| (s8 column scales)
  float* d_fq = nullptr;         // [maxB][D] queries gathered for the exact fallback
  int* d_fidx = nullptr;         // [maxB] flagged query indices
  int* d_fcount = nullptr;       // [2] flagged count of the last batch, running total
  unsigned* d_ctr = nullptr;     // ticket counter of the re-rank's fused compaction (0 at rest)
  vx::KTimer* d_ktimer = nullptr;  // [KT_N] device-side launch timers (vx_stats.kt_*)
  // pinned host staging
  void* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  int32_t* h_hdr = nullptr;
  int* h_flags = nullptr;
  // comm
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // stats
  vx_stats st{};
  cudaEvent_t ev[4] = {};        // eager-path timing events: scan begin/end, stage begin/end
  cudaEvent_t gev[4] = {};       // the same, recorded by captured graph nodes
  cudaEvent_t* tev = ev;         // events the code being issued records into
  cudaEvent_t* ev_start = ev;    // last batch: the array holding scan begin/end + stage begin
  cudaEvent_t* ev_end = ev;      //   ... and the one holding the stage end (read by vx_sync)
  cudaStream_t stream_last = nullptr;  // stream of the last batch's final part
  cudaEvent_t ev_done = nullptr;       // recorded there when it is not `stream` (vx_sync waits)
  bool done_pending = false;
  void* h_sync = nullptr;              // pinned: vx_sync's copies of the certificate counters
                                       // and the device timers (one async copy + one sync)
  cudaStream_t stream2 = nullptr;      // host API: query-token upload overlapping part 1
  cudaStream_t stream_cond = nullptr;  // captures the body of the certificate IF node
  cudaEvent_t tok_ev = nullptr;
  cudaEvent_t pev[10] = {};      // sharded rank 0 phases: start, bcast done, local done,
                                 //   gather done, end; then scan done, re-rank done,
                                 //   phase-2 bcast done, MaxSim done, reduce done ([5..9])
  bool phases_pending = false;
  bool timing_pending = false;
  bool scan_ev_valid = false;   // ev[0..1] hold this batch's scan span (eager runs only)
  bool stage_events = false;    // VX_OPT_STAGE_EVENTS
  bool graph_events = false;    // the graph being captured records its stage events
  // CUDA graphs per (op, B, k, nq)
  struct GraphEntry {
    cudaGraphExec_t exec;
    int launches;
    bool events;  // records the stage begin / end events (VX_OPT_STAGE_EVENTS at capture)
  };
  bool step_ev_valid = false;  // the last batch recorded its stage begin / end events
  bool use_graphs = false;
  std::map<uint64_t, GraphEntry> graphs;
  // Direct-I/O graphs (one GPU): the whole stage captured against the caller's own device
  // buffers, so a replay needs no copies in or out (each D2D copy around a replay is a
  // separate ~2-4 us operation — a fifth of a 100K-row small-batch step).  Keyed by shape AND
  // the buffer addresses; captured on the second sighting of an address tuple (a one-off
  // buffer never pays a capture), at most kIoGraphsPerShape tuples per shape.
  struct IoKey {
    uint64_t shape;
    uintptr_t p[5];
    bool operator<(const IoKey& o) const {
      if (shape != o.shape) return shape < o.shape;
      for (int i = 0; i < 5; ++i)
        if (p[i] != o.p[i]) return p[i] < o.p[i];
      return false;
    }
  };
  static constexpr int kIoGraphsPerShape = 4;
  std::map<IoKey, GraphEntry> io_graphs;
  std::map<IoKey, int> io_seen;
  std::map<uint64_t, int> io_per_shape;
};

// rows allocated past max_batch in the coarse query buffers (d_q16 / d_q8): the scan's query
// tensor maps span whole A tiles (<= 4 x 128 rows per pass)
constexpr int kQueryPadRows = 512;

static inline void count_launch(vx_index* h, int n = 1) { h->st.kernel_launches += n; }
static inline bool has_tokens(const vx_index* h) { return h->tokens || h->tokens32; }

// arm the device-side launch timers (start = max, everything else 0)
static inline vx_status ktimer_reset(vx_index* h) {
  vx::KTimer t[vx::KT_N] = {};
  for (auto& x : t) x.start = ~0ull;
  if (cudaMemcpy(h->d_ktimer, t, sizeof t, cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(VX_ERR_CUDA, "ktimer reset");
  return VX_OK;
}

// Captured stage graphs bake in every choice made at capture time (coarse format from the
// shard statistics, k', seed, tile, pairs, grid, scan / MaxSim algorithm), so any option
// change and any index upload / synth throws them away; the next batch of each shape
// re-captures.
static inline void drop_graphs(vx_index* h) {
  h->io_seen.clear();
  if (h->graphs.empty() && h->io_graphs.empty()) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
  for (auto& kv : h->io_graphs) cudaGraphExecDestroy(kv.second.exec);
  h->graphs.clear();
  h->io_graphs.clear();
  h->io_per_shape.clear();
}

// Timing events: inside a stream capture they must be EXTERNAL event nodes, or the graph only
// uses them for internal ordering and never records them for the host to read.
// Inside a capture (tev == gev) only with VX_OPT_STAGE_EVENTS: an external event node costs
// every replay ~2 us (100K-row B = 16 step: 92.8 -> 88.2 us without the two stage events).
static inline cudaError_t record_ev(vx_index* h, cudaEvent_t e, cudaStream_t st) {
  if (h->tev == h->gev && !h->stage_events) return cudaSuccess;
  if (h->tev == h->gev) h->graph_events = true;
  return cudaEventRecordWithFlags(e, st,
                                  h->tev == h->gev ? cudaEventRecordExternal : cudaEventRecordDefault);
}
// The scan's own begin / end events (tev[0], tev[1]): recorded on eager runs only.  Inside a
// captured stage an event node between the scan and the re-rank would cut the kernel-to-kernel
// edge the programmatic dependent launch of the re-rank needs; the scan kernels time
// themselves on the device anyway (vx_stats kt_*).
static inline cudaError_t record_scan_ev(vx_index* h, cudaEvent_t e, cudaStream_t st) {
  if (h->tev == h->gev) return cudaSuccess;
  h->scan_ev_valid = true;
  return cudaEventRecord(e, st);
}
// the same for events recorded without the tev indirection (sharded phase events)
static inline cudaError_t record_ext(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cudaEventRecordWithFlags(
      e, st, cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault);
}

static inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
static inline int kcap_of(int k) { return std::max(16, next_pow2(k)); }

// ---------------------------------------------------------------- pipeline pieces

static inline cudaStream_t pick_stream(vx_index* h, void* s) {
  return s ? reinterpret_cast<cudaStream_t>(s) : h->stream;
}

static inline vx_status check_batch(vx_index* h, int32_t B, int32_t k) {
  if (B < 1 || B > h->desc.max_batch)
    return fail(VX_ERR_INVALID, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (k < 1 || k > h->desc.max_k) return fail(VX_ERR_INVALID, "k %d outside [1, %d]", k, h->desc.max_k);
  return VX_OK;
}

// ---------------------------------------------------------------- the stage (vx_stage.cu)
int coarse_fmt(const vx_index* h);  // FMT_* the tensor-core pass uses (VX_OPT_COARSE resolved)
// AUTO leaves the s8 pass when its certificate keeps failing (fc: device counters)
void maybe_demote_i8(vx_index* h, const int* fc, uint64_t queries);
enum { OP_STOP = 0, OP_SEARCH = 1, OP_RESCORE = 2 };

vx_status run_maxsim(vx_index* h, const float* d_qtok, int B, int nq, const int64_t* d_cand, int C,
                     float* d_out, cudaStream_t st, int64_t id_lo = 0, int64_t id_hi = INT64_MAX,
                     const uint16_t* d_qtok16 = nullptr);
// part 1 / part 2 of the stage on any rank (the shard ranks call these from vx_shard_serve)
vx_status core_topk(vx_index* h, const float* d_q, int B, int k, cudaStream_t st);
vx_status core_rescore(vx_index* h, const float* d_qtok, int B, int nq, int k, int64_t* d_ids,
                       float* d_ip, float* d_ms, cudaStream_t st);
// rank-0 entry points: announce + part 1; part 2 of a search / of the fused stage
vx_status stage_begin(vx_index* h, int op, const float* d_q, int B, int nq, int k,
                      cudaStream_t st);
// one part of the stage (1: broadcast + top-k, 2: rescore) through its captured graph
vx_status run_part(vx_index* h, int part, int B, int nq, int k, cudaStream_t st);
vx_status stage_search_out(vx_index* h, int B, int k, int64_t* d_ids, float* d_ip,
                           cudaStream_t st);
vx_status stage_direct(vx_index* h, int op, const float* d_q, const float* d_qtok, int B, int nq,
                       int k, int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st,
                       bool* done);
vx_status stage_finish(vx_index* h, const float* d_qtok, int B, int nq, int k, int64_t* d_ids,
                       float* d_ip, float* d_ms, cudaStream_t st);
