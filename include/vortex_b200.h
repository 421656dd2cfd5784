/*
 * vortex_b200.h — C-ABI of the B200-native retrieval stage (exact inner-product
 * top-k over a sharded index + ColBERT/PreFLMR MaxSim re-scoring).
 *
 * This is the boundary a Vortex deployment binds instead of the simulated
 * search stage. The reference plugs operators in as
 *     using ComponentFn = std::function<std::vector<Payload>(const std::vector<Payload>&)>;
 *     Runtime::register_component(model_id, fn)            (proj/include/vortex/runtime.hpp:179, :202-211)
 * and today the search stage ("modelD", proj/assets/pipeline.json:7) is only a
 * profiled latency (proj/include/vortex/executor.hpp:172-182, profiles.csv:17-22).
 * The C++ adapter in include/vortex_b200_component.hpp wraps these entry points
 * into exactly that ComponentFn; see INTEGRATION.md for the reference-side
 * binding.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross this ABI.  Every call
 *    returns a vx_status; vx_last_error() returns a thread-local message.
 *  - Host-buffer entry points (vx_search, vx_maxsim, vx_search_rescore) own the
 *    H2D/D2H copies (through pinned staging) and return when results are on the
 *    host.  *_dev variants take device pointers and a cudaStream_t (as void*;
 *    NULL = the handle's own stream) and are asynchronous.
 *  - Output of a top-k: ids int64 [B][k] and scores float [B][k], ordered by
 *    score descending, then id ascending.  Missing entries (k > N) are id -1,
 *    score -INF.
 *  - Sharded mode (n_shards > 1): one handle per rank/GPU owns rows
 *    [floor(N*g/G), floor(N*(g+1)/G)).  Rank 0 is the operator: its search
 *    call broadcasts the batch to the other ranks over NCCL, every rank scans
 *    its shard and rescoring its local top-k, and the k x G candidates are
 *    gathered to rank 0 and merged.  Ranks != 0 sit in vx_shard_serve().
 *  - The library never falls back to the CPU.  If no usable sm_100 device is
 *    present, vx_index_create fails with VX_ERR_CUDA.
 */
#ifndef VORTEX_B200_H_
#define VORTEX_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_ABI_VERSION 1

typedef enum vx_status {
  VX_OK = 0,
  VX_ERR_INVALID = 1,     /* bad argument / shape (reference: errc::bad_config) */
  VX_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
  VX_ERR_OOM = 3,         /* device allocation failed (reference: errc::out_of_memory) */
  VX_ERR_NCCL = 4,        /* collective failure */
  VX_ERR_STATE = 5,       /* call not valid in this handle state (reference: errc::bad_transition) */
  VX_ERR_UNSUPPORTED = 6  /* shape outside the compiled kernel envelope */
} vx_status;

typedef struct vx_index vx_index;

/* Scan algorithm selection (vx_set_option VX_OPT_SCAN). */
enum { VX_SCAN_AUTO = 0, VX_SCAN_F32 = 1, VX_SCAN_TC = 2 };
/* Options. */
enum {
  VX_OPT_SCAN = 1,        /* one of VX_SCAN_* */
  VX_OPT_GRID = 2,        /* CTAs for the scan (0 = auto: one per SM) */
  VX_OPT_GRAPHS = 3,      /* 1 = replay pre-captured CUDA graphs per batch bucket */
  VX_OPT_MAXSIM = 4,      /* one of VX_MAXSIM_* */
  VX_OPT_COARSE = 5,      /* one of VX_COARSE_*: operand format of the tensor-core scan */
  VX_OPT_SCAN_TILE = 6,   /* documents per tensor-core scan tile: 0 (auto), 128 or 256 */
  VX_OPT_SCAN_PAIRS = 7   /* 2 (default): CTA-pair (cta_group::2) scan for B > 128, 512 queries
                             per pass (two query groups on 128-document tiles) when B > 256;
                             1: 256 queries per pass; 0: single-CTA kernels */,
  VX_OPT_KPRIME = 8       /* tensor-core candidate set k' re-ranked exactly: 0 (auto:
                             4 next_pow2(k) in [64, 256] for bf16/tf32, 8 next_pow2(k) in
                             [128, 1024] for s8) or a power of two in [16, 1024] */,
  VX_OPT_SCAN_SEED = 9    /* 1 (default): seed each query's tensor-core scan admission
                             threshold from a 1/64 row sample of the shard (shards of
                             >= 512K rows); 0: off.  Results are identical either way. */,
  VX_OPT_I8_SCALE = 10    /* s8 shadow scales: 0 (default) one per shard; 1 one per column
                             (folded into the query) — re-quantises the shard */,
  VX_OPT_STAGE_EVENTS = 11 /* 1: captured stages record their begin / end CUDA events
                             (vx_stats.last_step_ms on graph replays); 0 (default): only eager
                             runs do — each event node costs a replay ~2 us */
};
/* Coarse (candidate-selecting) tensor-core scan format.  Either way every reported score is
 * recomputed exactly in fp32 and certified.  BF16 reads a bf16 shadow
 * of the index (half the HBM bytes, 2x the tensor rate); TF32 reads the fp32 rows; I8 reads an
 * s8 shadow (one scale per shard, per-query scales; a quarter of the bytes, 2x the bf16 rate). */
enum { VX_COARSE_AUTO = 0, VX_COARSE_TF32 = 1, VX_COARSE_BF16 = 2, VX_COARSE_I8 = 3 };
/* vx_index_desc.flags */
enum {
  VX_FLAG_NO_BF16_SHADOW = 1, /* do not keep the bf16 copy of the index (saves N*D*2 B) */
  VX_FLAG_NO_I8_SHADOW = 2,   /* do not keep the s8 copy of the index (saves N*D B) */
  VX_FLAG_TOKENS_F32 = 4      /* fp32 doc-token store (SURVEY C2's fp32 variant: 4 B per
                                 element, MaxSim in exact in-order fp32 on the CUDA cores,
                                 query tokens unrounded); default bf16 */
};
/* MaxSim kernel selection (vx_set_option VX_OPT_MAXSIM).
 *  AUTO / TC: tensor-core kernel; for nq <= 64 the fp32 query tokens enter as bf16 hi + lo
 *             pairs (fp32-faithful: ~1e-6 relative to the fp64 MaxSim of the fp32 tokens),
 *             else rounded to bf16;
 *  TC_BF16Q:  tensor-core kernel, query tokens rounded to bf16 (~1e-3 relative);
 *  CC:        CUDA-core kernel, bf16-rounded query tokens, in-order fmaf chains
 *             (bit-identical to the oracle's VXO_F32 mode). */
enum { VX_MAXSIM_AUTO = 0, VX_MAXSIM_CC = 1, VX_MAXSIM_TC = 2, VX_MAXSIM_TC_BF16Q = 3 };

typedef struct vx_index_desc {
  int64_t n_docs;      /* global document count N (1 <= N < 2^32) */
  int32_t dim;         /* embedding dimension D (multiple of 32, <= 4096) */
  int32_t device;      /* CUDA device ordinal used by this handle */
  int32_t n_shards;    /* G: number of index shards (ranks); 1 = whole index */
  int32_t shard;       /* g: this handle's shard, 0 <= g < G */
  int32_t tok_per_doc; /* Nd: late-interaction tokens per document (0 = no token store) */
  int32_t tok_dim;     /* d: token dimension (multiple of 64 when Nd > 0) */
  int64_t tok_blocks;  /* T: token-store blocks; document id uses block (id mod T) */
  int32_t max_batch;   /* largest batch B accepted (workspace sizing) */
  int32_t max_k;       /* largest k accepted (<= 256) */
  int32_t max_qtok;    /* largest Nq accepted (<= 128) */
  int32_t flags;       /* VX_FLAG_* */
} vx_index_desc;

typedef struct vx_stats {
  uint64_t kernel_launches;   /* kernels this handle launched since creation / last reset */
  uint64_t batches;           /* search/maxsim batches served */
  uint64_t queries;           /* queries served */
  uint64_t graph_replays;     /* CUDA graph launches */
  uint64_t cert_fallbacks;    /* queries re-scanned exactly after both TC certificate levels
                                 failed */
  float last_scan_ms;         /* device time of the last scan kernel (CUDA events) */
  float last_step_ms;         /* device time of the last whole stage */
  double scan_ms_total;       /* sum of scan device times sampled by vx_sync */
  double step_ms_total;       /* sum of stage device times sampled by vx_sync */
  uint64_t timed_batches;     /* batches whose times were sampled (one per vx_sync) */
  float phase_ms[4];          /* sharded rank 0, last batch: broadcast, local stage,
                                 gather of the k x G keys + global merge, phase 2 (winner
                                 broadcast, owner MaxSim, max-reduce, order) */
  uint64_t cert_level2;       /* queries whose k'-candidate certificate failed and that went
                                 to the wide re-rank over the full per-CTA lists */
  uint64_t host_staged_bytes; /* host-buffer API: bytes memcpy'd through the handle's pinned
                                 staging (0 when every caller buffer was page-locked and DMA'd
                                 directly) */
  /* Device-side kernel timing (every launch, inside CUDA graphs, no host sync): [0] the
   * tensor-core scan passes, [1] the seeded sample pass, [2] the exact K1 scan, [3] MaxSim.
   * Duration = first CTA start -> last CTA end (%globaltimer); SM clock = CTA 0's clock64()
   * cycles over its %globaltimer span. */
  uint64_t kt_launches[4];
  double kt_ms[4];            /* summed durations */
  double kt_sm_mhz[4];        /* mean SM clock during those launches */
  float phase_detail_ms[6];   /* sharded rank 0, last batch, finer: local scan (sample + full
                                 passes), local re-rank incl. the tau all-gather, the rest of
                                 the local stage, phase-2 token + winner broadcast, owner
                                 MaxSim, max-reduce + order */
  uint64_t kt_rerank_launches; /* device-side timing of the exact re-rank launches (as kt_*) */
  double kt_rerank_ms;
  double kt_last_us[10];       /* [scan, sample, f32, maxsim, re-rank] x [start, end] of each
                                  kind's LAST launch, us after the earliest of those starts
                                  (both 0: no launch) — the gaps between a stage's kernels */
  uint64_t kt_origin_ns;       /* %globaltimer (ns) of that earliest start: the origin of
                                  kt_last_us, to place the kernels against other device stamps */
} vx_stats;

int32_t vx_abi_version(void);
const char* vx_last_error(void);

vx_status vx_index_create(const vx_index_desc* desc, vx_index** out);
vx_status vx_index_destroy(vx_index* h);
/* Rows owned by this handle: [*row0, *row0 + *n_local). */
vx_status vx_index_shard_range(const vx_index* h, int64_t* row0, int64_t* n_local);
vx_status vx_set_option(vx_index* h, int32_t option, int64_t value);
/* Effective value of an option; for VX_OPT_COARSE the format the tensor-core scan will use
 * (AUTO resolved: VX_COARSE_BF16, VX_COARSE_TF32 or VX_COARSE_I8). */
vx_status vx_get_option(const vx_index* h, int32_t option, int64_t* value);
vx_status vx_get_stats(const vx_index* h, vx_stats* out);
vx_status vx_reset_stats(vx_index* h);

/* Fill this shard's rows with the synthetic generator of vx_synth.h (seed). */
vx_status vx_index_synth(vx_index* h, uint64_t seed);
/* The same with a row distribution: 0 isotropic (= vx_index_synth), 1 anisotropic (power-law
 * per-dimension scales + outlier dimensions, vx_synth.h). */
vx_status vx_index_synth_dist(vx_index* h, uint64_t seed, int32_t dist);
/* Upload rows [row0, row0+n) (global ids, must lie inside this shard), fp32 row-major. */
vx_status vx_index_upload(vx_index* h, const float* rows, int64_t row0, int64_t n);
/* Copy rows [row0, row0+n) (global ids inside this shard) back to the host. */
vx_status vx_index_download(const vx_index* h, float* rows, int64_t row0, int64_t n);
/* Fill the token store with the generator (bf16 of the unit rows, seed). */
vx_status vx_tokens_synth(vx_index* h, uint64_t seed);
/* Upload token blocks [blk0, blk0+n): bf16 bits, [n][Nd][d]. */
vx_status vx_tokens_upload(vx_index* h, const uint16_t* tokens_bf16, int64_t blk0, int64_t n);
vx_status vx_tokens_download(const vx_index* h, uint16_t* tokens_bf16, int64_t blk0, int64_t n);
/* The same for an fp32 token store (VX_FLAG_TOKENS_F32). */
vx_status vx_tokens_upload_f32(vx_index* h, const float* tokens, int64_t blk0, int64_t n);
vx_status vx_tokens_download_f32(const vx_index* h, float* tokens, int64_t blk0, int64_t n);

/* Exact inner-product top-k of B queries (fp32 [B][D]).  Host buffers. */
vx_status vx_search(vx_index* h, const float* queries, int32_t B, int32_t k, int64_t* ids,
                    float* scores);
/* MaxSim of B queries' tokens (fp32 [B][Nq][d], rounded to bf16) against C
 * candidate ids per query ([B][C], -1 = skip -> -INF).  Host buffers. */
vx_status vx_maxsim(vx_index* h, const float* qtok, int32_t B, int32_t nq,
                    const int64_t* cand, int32_t C, float* out);
/* The fused stage: top-k by inner product, MaxSim of those k, results ordered
 * by MaxSim descending (ties: id ascending).  ip/maxsim are [B][k]. */
vx_status vx_search_rescore(vx_index* h, const float* queries, const float* qtok, int32_t B,
                            int32_t nq, int32_t k, int64_t* ids, float* ip, float* maxsim);

/* Row-gather variants: query i's vector at q_rows[i] (fp32 [D]) and its tokens at
 * tok_rows[i] (fp32 [nq][tok_dim]) — e.g. pointers straight into the runtime's query
 * payloads, so a batch is copied once, into the handle's pinned staging (the C++ operator
 * adapter uses these: SURVEY §8f "payload codec + pinned-host/H2D zero-copy"). */
vx_status vx_search_rows(vx_index* h, const float* const* q_rows, int32_t B, int32_t k,
                         int64_t* ids, float* scores);
vx_status vx_search_rescore_rows(vx_index* h, const float* const* q_rows,
                                 const float* const* tok_rows, int32_t B, int32_t nq, int32_t k,
                                 int64_t* ids, float* ip, float* maxsim);

/* Device-pointer variants (inputs already resident in HBM; asynchronous on stream). */
vx_status vx_search_dev(vx_index* h, const float* d_queries, int32_t B, int32_t k,
                        int64_t* d_ids, float* d_scores, void* stream);
vx_status vx_maxsim_dev(vx_index* h, const float* d_qtok, int32_t B, int32_t nq,
                        const int64_t* d_cand, int32_t C, float* d_out, void* stream);
vx_status vx_search_rescore_dev(vx_index* h, const float* d_queries, const float* d_qtok,
                                int32_t B, int32_t nq, int32_t k, int64_t* d_ids, float* d_ip,
                                float* d_maxsim, void* stream);
/* Wait for the handle's work; samples the last batch's scan/stage device times. */
vx_status vx_sync(vx_index* h);

/* Model-load step ("index preload", reference: exec::Executor::load_model,
 * proj/include/vortex/executor.hpp:129-149, and preload_one, elasticity.hpp:221-232):
 * with graphs enabled on a single-GPU handle, run and capture the stage graph of every
 * batch size 1..b_max for (op, k, nq) so that no batch the runtime dispatches later pays a
 * capture.  op: VX_PREPARE_SEARCH or VX_PREPARE_RESCORE.  Uses the handle's own
 * input buffers (filled with generator rows).  No-op (VX_OK) without graphs or with
 * nranks > 1. */
#define VX_PREPARE_SEARCH 1
#define VX_PREPARE_RESCORE 2
vx_status vx_prepare(vx_index* h, int32_t op, int32_t k, int32_t nq, int32_t b_max);

/* ---- Opportunistic, SLO-bounded batcher (reference: Runtime::maybe_dispatch,
 * proj/include/vortex/runtime.hpp:617-654: when the member is idle, dispatch the
 * min(|queue|, cap) oldest queries, never wait to fill).
 *
 * vx_batcher_simulate: replay on a virtual clock with a piecewise-linear latency profile
 * L(b) (knots, profile.hpp:90-109); no GPU.  arrivals_us sorted ascending.  Per query:
 * batch index, dispatch and completion time (us).  Completion = dispatch +
 * trunc(L(b)*1000) us, as SimExecutor::execute_batch (executor.hpp:172-182). */
vx_status vx_batcher_simulate(const uint64_t* arrivals_us, int64_t n, int32_t cap,
                              const int32_t* knot_batch, const double* knot_ms, int32_t n_knots,
                              int64_t* batch_of, uint64_t* dispatch_us, uint64_t* complete_us,
                              int64_t* n_batches);
/* Replica mode: `replicas` members of the stage, each batching as above, with the
 * reference's routing in front (Runtime::pick_member, runtime.hpp:522-536: power of two
 * choices on outstanding tags, ties to the lower index, draws from std::mt19937_64(seed) —
 * the runtime's seed is 7, runtime.hpp:188).  Per query: instance, dispatch and
 * completion time (us); n_batches counts batches over all instances. */
vx_status vx_batcher_simulate_replicas(const uint64_t* arrivals_us, int64_t n, int32_t replicas,
                                       int32_t cap, const int32_t* knot_batch,
                                       const double* knot_ms, int32_t n_knots, uint64_t seed,
                                       int32_t* instance_of, uint64_t* dispatch_us,
                                       uint64_t* complete_us, int64_t* n_batches);

/* Open-loop arrival trace (bench::arrival_times, bench.hpp:54-67): poisson != 0 draws
 * exponential gaps from std::mt19937_64(seed) exactly as the reference's sim::Rng does
 * (sim.hpp:95-98), else constant spacing; times in us, llround'ed. */
vx_status vx_arrival_times(double rate_qps, int64_t count, uint64_t seed, uint64_t start_us,
                           int32_t poisson, uint64_t* out);
/* vx_serve_trace: live mode — replays the arrival trace in wall-clock time through the
 * same batcher onto this handle's GPU stage (one batch in flight; each dispatched batch
 * is copied host->device, searched (and re-scored when qtok != NULL), and its results
 * copied back before the batch completes).  queries [n][D], qtok [n][nq][d] or NULL.
 * latency_us[i] = completion - planned arrival (bench.hpp:222).  ids [n][k] optional. */
vx_status vx_serve_trace(vx_index* h, const uint64_t* arrivals_us, int64_t n, int32_t cap,
                         const float* queries, const float* qtok, int32_t nq, int32_t k,
                         int64_t* ids, double* latency_us, int64_t* batch_of,
                         int64_t* n_batches);
/* Live replica mode: R whole-index handles (e.g. one per GPU) as the members of the stage,
 * each batching as above, queries routed at arrival by the reference's power of two choices
 * (Runtime::pick_member, runtime.hpp:522-536: outstanding = routed - completed, ties to the
 * lower index, draws from std::mt19937_64(seed)).  One host thread drives all members; the
 * queries queued behind a running batch are DMA'd into the member's second input buffer
 * while it computes.  Per query (all optional except latency_us): instance, dispatch and
 * completion time (us), the sequence numbers of its routing, dispatch and completion events
 * (one global counter: the queue every dispatch saw and the outstanding counts every routing
 * decision saw can be replayed), ids [n][k], latency, global batch index. */
vx_status vx_serve_trace_replicas(vx_index* const* handles, int32_t R, const uint64_t* arrivals_us,
                                  int64_t n, int32_t cap, const float* queries, const float* qtok,
                                  int32_t nq, int32_t k, uint64_t seed, int32_t* instance_of,
                                  uint64_t* dispatch_us, uint64_t* complete_us, uint64_t* admit_seq,
                                  uint64_t* dispatch_seq, uint64_t* complete_seq, int64_t* ids,
                                  double* latency_us, int64_t* batch_of, int64_t* n_batches);

/* Multi-GPU (one process per GPU).  Rank 0 creates the id, the host plumbing
 * (torch.distributed / MPI / a file) distributes the 128 bytes, every rank
 * calls vx_comm_init.  Ranks != 0 then call vx_shard_serve(), which returns
 * after rank 0 calls vx_shard_stop(). */
vx_status vx_comm_unique_id(uint8_t out_id[128]);
vx_status vx_comm_init(vx_index* h, const uint8_t id[128], int32_t nranks, int32_t rank);
vx_status vx_shard_serve(vx_index* h);
vx_status vx_shard_stop(vx_index* h);

#ifdef __cplusplus
}
#endif

#endif /* VORTEX_B200_H_ */
