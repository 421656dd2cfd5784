// vx_internal.cuh — shared declarations between the kernels and the C-ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vx_synth.h"

namespace vx {

// Device-side launch timing, kept per kernel kind (vx_ptx.cuh ktimer_begin / ktimer_end):
// every CTA folds its %globaltimer start / end into [start, end] with atomics, the last CTA to
// finish adds end - start to total_ns and re-arms the slot, so every launch — inside CUDA
// graphs, with no host synchronisation — is timed first-CTA-start to last-CTA-end.  CTA 0
// also accumulates clock64() cycles over its own %globaltimer span: the SM clock the kernel
// actually ran at.
struct KTimer {
  unsigned long long start, end, done, total_ns, launches, clk_cycles, clk_ns, last_start,
      last_end;  // the last launch's span (%globaltimer ns): the gaps between a stage's kernels
};
enum { KT_SCAN = 0, KT_SAMPLE = 1, KT_F32 = 2, KT_MAXSIM = 3, KT_RERANK = 4, KT_N = 5 };

// -------- exact fp32 scan (K1): scan_f32.cu
struct ScanF32Args {
  const float* q;      // [B][D] device, fp32
  int32_t B;           // queries in this launch (<= the config's BQ)
  int32_t D;           // dimension (multiple of 32)
  uint32_t n_local;    // rows in the shard
  int32_t kcap;        // per-CTA list length (power of 2, >= k, 16..256)
  int32_t cap;         // candidate buffer per query
  int32_t ns;          // pipeline stages
  uint64_t* part;      // [B][gridDim.x][kcap] keys (score desc, local id asc)
  const int* d_count;  // optional: queries actually present = min(B, *d_count - g0) (device)
  int32_t g0;
  KTimer* ktimer = nullptr;
};

// Returns the queries-per-launch bucket the f32 scan uses for a batch of B.
int scan_f32_bucket(int B);
// Dynamic smem bytes for (bucket, D, kcap); 0 if it does not fit.
size_t scan_f32_smem(int bucket, int D, int kcap, int* ns_out, int* cap_out);
cudaError_t launch_scan_f32(int bucket, const CUtensorMap* tmap, const ScanF32Args& a, int grid,
                            size_t smem, cudaStream_t st);
int scan_f32_tile_docs(int bucket);

// -------- tensor-core coarse scan (K2) + exact re-rank (K2b): scan_tc.cu
struct ScanTcArgs {
  uint32_t n_local;  // rows in the shard
  int32_t D;         // dimension (multiple of 32)
  int32_t B;         // queries in this launch (<= QT*128)
  int32_t ns;        // pipeline stages
  int32_t a_rows;    // TMA box rows of the query map (multiple of 8, <= 128)
  int32_t fmt;       // operand format: FMT_BF16 (kind::f16 on the bf16 shadow), FMT_TF32 (fp32
                     // rows read as TF32, kind::tf32) or FMT_I8 (s8 shadow, kind::i8, s32)
  int32_t dbg_no_select;  // timing experiments only (VX_DEBUG_TC_NOSELECT): skip the top-k
  uint64_t* part;    // [B][gridDim.x][KC] coarse keys
  // admission-threshold seeds (nullable): query q starts admitting at the coarse score of
  // key seed[q * seed_ld] (0 = no seed) instead of -inf — the m-th best coarse key of a
  // strided sample of the shard (vx_stage.cu local_topk_tc), so the lists skip the fill
  // phase; the re-rank's certificate bounds the documents the seed dropped
  const uint64_t* seed;
  int32_t seed_ld;
  int32_t kc;        // list length per CTA (pair) and query: 0 = kc_of(fmt), or kSampleKC
  KTimer* ktimer = nullptr;
  uint64_t* trace = nullptr;  // timing experiments only (VX_DEBUG_SCAN_TRACE): per CTA 8
                             // %globaltimer stamps (entry, setup done, first stage landed, last
                             // MMA issued, epilogue done, lists written)
  int32_t pdl = 0;   // launched as a programmatic dependent of the query conversion (single-CTA
                     // kernel): the prologue overlaps it; every thread waits before its roles
  int32_t rep = 1;   // single-CTA kernel, TD = 256, B <= 64: each query occupies rep = 128 /
                     // a_rows rows of the A tile, replica r selects over columns
                     // [r TD/rep, (r+1) TD/rep) — rep x the epilogue lanes on a small batch
};
// admission threshold a seed key stands for (-inf: none)
__device__ __forceinline__ float seed_thr(const uint64_t* seed, int ld, int q) {
  if (!seed) return -INFINITY;
  const uint64_t key = seed[(size_t)q * ld];
  return key ? vx_key_score(key) : -INFINITY;
}
// TF32 coarse-score error bound coefficient E = coef * ||q|| * max||x||: the tensor core
// truncates both operands to 10 mantissa bits (<= 2^-10 each).  The bf16 bound is computed
// from the actual rounding residuals (rerank_kernel in scan_tc.cu).
constexpr float kErrCoefTF32 = 0.001953125f;
cudaError_t launch_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st);
// s8 shadow of an n x D fp32 shard, x8[r][c] = rint(x[r][c] / s_c) with column scales s_c:
// one shard-wide value (default) or per_column s_c = max_r |x[r][c]| / 127 (0 for an all-zero
// column).  colmax_bits: D words of scratch; colscale: the D scales.
cudaError_t launch_to_i8_shadow(const float* in, int64_t n, int D, int8_t* out,
                                unsigned int* colmax_bits, float* colscale, int per_column,
                                cudaStream_t st);
// s8 copy of B query rows of D: q'[c] = q[c] s_c folds the document column scales into the
// query, then one scale per row sq = max|q'| / 127, q8 = rint(q' / sq); sq * (q8 . x8)
// approximates q . x (the certificate bounds the difference, scan_tc.cu cert_err_bound)
cudaError_t launch_rows_to_i8(const float* in, int B, int D, const float* colscale, int8_t* out,
                              float* scales, cudaStream_t st);
// xstats layout (d_xnorm, floats): [0] max|x|, [1] max|bf16 x|, [2] max|x - bf16 x|,
// [3] max|x8| (integer norm of the s8 row), [4] max|x - x^| (x^[c] = s_c x8[c]), [5] the s8
// coarse units' document factor (1: the column scales live in the query), [6] scratch,
// [7] sum of |x|; [8 .. 8+D) the column scales s_c
constexpr int kXstatColScale = 8;
// Coarse operand formats of the tensor-core scan (ScanTcArgs::fmt)
enum : int { FMT_BF16 = 1, FMT_TF32 = 2, FMT_I8 = 3 };
// Per-CTA (per-pair) candidate list length per query: 16, or 32 for the s8 coarse pass,
// whose candidate set k' is 4x larger (its error bound is ~4x the bf16 one).
__host__ __device__ constexpr int kc_of(int fmt) { return fmt == FMT_I8 ? 32 : 16; }
// list length of the seed's sample pass (vx_stage.cu): the seed is the m-th best of the
// union of the lists, and truncated lists only lower it (a valid, slightly looser seed)
constexpr int kSampleKC = 4;
// K3 merge: most keys per query staged in shared memory (96 KB; also the bound for fusing
// the merge into the re-rank)
constexpr int kMergeSmemKeys = 12288;
// s8 quantisation used by the shadow, the queries and the certificate's residuals
__device__ __forceinline__ int8_t vx_quant8(float v, float s) {
  const float r = rintf(v / s);
  return (int8_t)fminf(fmaxf(r, -127.0f), 127.0f);
}
constexpr int kTcListLen = 16;
size_t scan_tc_smem(int QT, int TD, int fmt, int* ns_out);
cudaError_t launch_scan_tc(int QT, int TD, const CUtensorMap* tq, const CUtensorMap* tx,
                           const ScanTcArgs& a, int grid, size_t smem, cudaStream_t st);
// CTA-pair variant for 128 < B <= 256 (scan_tc2.cu); grid must be even; lists per pair.
// H = 256-document halves per pair tile (1: 256-doc tiles, double-buffered; 2: 512-doc tiles)
size_t scan_tc2_smem(int H, int* ns_out);
cudaError_t launch_scan_tc2(int H, const CUtensorMap* tq, const CUtensorMap* tx,
                            const ScanTcArgs& a, int grid, size_t smem, cudaStream_t st);
// phase 0: the whole re-rank; sharded: phase 1 (head: exact keys of the k best coarse
// candidates -> hkeys, their scores -> lb) and phase 2 (tail, pruned by tau) around the
// exchange of lb (see scan_tc.cu)
// Fusions into the re-rank launch (all optional):
//  * merge: each CTA first merges its query's per-CTA lists (mlists + b * mld, mM keys) to
//    the coarse top-k' in cand (the K3 launch it replaces, vx_merge.cuh merge_topk_block);
//  * compact: the launch's last CTA (ticket counter ctr, zero on entry and reset on exit)
//    compacts the certificate failures of the WHOLE batch (flags_all[0, Ball)) for levels
//    2-3 and sets the captured stage's conditional handle (the cert_compact launch).
struct RerankFuse {
  int head = 0;  // sharded: head rows re-scored before the tau exchange (0: k).  G shards
                 // contribute G x head exact scores; tau = their k-th largest needs G head >= k
  const uint64_t* mlists = nullptr;
  int mM = 0;
  int filter = 1;  // the merge's sorted-list filter (VX_DEBUG_NO_MERGE_FILTER: A/B timing)
  int64_t mld = 0;
  unsigned* ctr = nullptr;
  const int* flags_all = nullptr;
  int Ball = 0;
  const float* qall = nullptr;
  int* fidx = nullptr;
  int* fcount = nullptr;
  float* fq = nullptr;
  unsigned long long cond = 0;
  int use_cond = 0;
  KTimer* ktimer = nullptr;
  // small batch, whole candidate set as the head (phase 0): S CTAs per query, CTA s re-scores
  // candidates [s k'/S, (s+1) k'/S) into ekeys[b][k'] (global); the query's last CTA to
  // finish (qctr[b] ticket, re-armed to 0) loads them and selects / certifies / writes.
  // The merge is then a launch of its own (every CTA reads the sorted candidates).
  int split = 1;
  uint64_t* ekeys = nullptr;
  unsigned* qctr = nullptr;
  uint64_t* trace = nullptr;  // timing experiments only (VX_DEBUG_RERANK_TRACE): per CTA 8
                              // %globaltimer stamps (entry, norms, dependency, merge, head,
                              // tail, sort, end)
};
cudaError_t launch_rerank(const float* docs, const float* q, int D, uint64_t* cand, int B,
                          int kp, const uint64_t* part, int grid, int ldlists, int kc, int k,
                          int64_t row0, const float* xstats, int fmt, const float* qscale,
                          uint64_t* out_keys, int64_t* out_ids, float* out_scores, int* flags,
                          cudaStream_t st, int phase = 0, const float* tau = nullptr,
                          uint64_t* hkeys = nullptr, float* lb = nullptr,
                          const uint64_t* seed = nullptr, int seed_ld = 0,
                          const RerankFuse& fuse = RerankFuse{});
// tau[B] = k-th largest of all[G][B][k] (G k <= 1024)
cudaError_t launch_shard_tau(const float* all, int G, int B, int k, float* tau, cudaStream_t st);
// second certificate level over the full per-CTA lists (compacted failing queries): two
// launches; wkeys = scratch of B x P_single x kc keys
cudaError_t launch_rerank_wide(const float* docs, const float* fq, int D, const int* fidx,
                               const int* fcount, const uint64_t* part_all, int B, int GS,
                               int P_pairs, int P_single, int kc, int k, int64_t row0,
                               const float* xstats, int fmt, const float* qscale,
                               uint64_t* wkeys, uint64_t* out_keys, int64_t* out_ids,
                               float* out_scores, int* flags, cudaStream_t st,
                               const uint64_t* seed = nullptr, int seed_ld = 0);
// per-shard maxima [max|x|, max|bf16(x)|, max|x - bf16(x)|] (floats as uint bits) and, when
// the s8 column scales are given, [3] max|x8| (integer norm), [4] max|x - s x8|
cudaError_t launch_row_stats(const float* docs, int64_t n, int D, unsigned int* out_bits,
                             cudaStream_t st, const float* colscale = nullptr);

// -------- top-k merge (K3): topk.cu
// For each query q: select the k largest keys among in[q][0..M), write them
// descending to out_keys[q][k] (re-keyed with id + id_base), ids (-1 for empty) and scores.
// ldin: keys between consecutive queries' candidate lists (0: M, i.e. contiguous)
// P, KC > 0: the input is P descending lists of KC keys per query (enables the sorted-list
// filter of vx_merge.cuh merge_topk_block)
cudaError_t launch_merge_topk(const uint64_t* in, int B, int M, int k, int64_t id_base,
                              uint64_t* out_keys, int64_t* out_ids, float* out_scores,
                              cudaStream_t st, const int* d_count = nullptr, int64_t ldin = 0,
                              int64_t ldout = 0, int P = 0, int KC = 0);
// Certificate failures (flags[B]) -> compacted list fidx/fcount and the flagged query rows
// gathered into fq; after the exact re-scan, scatter its [fcount][k] results back.
cudaError_t launch_cert_compact(const int* flags, int B, const float* q, int D, int* fidx,
                                int* fcount, float* fq, cudaStream_t st,
                                unsigned long long cond = 0, int use_cond = 0);
cudaError_t launch_cert_scatter(const int* fidx, const int* fcount, int B, int k,
                                const uint64_t* fkeys, const int64_t* fids, const float* fsc,
                                uint64_t* keys, int64_t* ids, float* scores, cudaStream_t st);
// Order k candidates per query by a float score descending (ties id asc) and
// permute the companion arrays: used to order by MaxSim after the IP top-k.
cudaError_t launch_order_by(const float* key_score, const int64_t* ids, const float* ip, int B,
                            int k, int64_t* out_ids, float* out_ip, float* out_ms,
                            cudaStream_t st, int planes = 1,
                            size_t plane_stride = 0);

// -------- synthetic fill: synth.cu
cudaError_t launch_synth_rows(float* out, uint64_t seed, int64_t row0, int64_t n, int D,
                              cudaStream_t st, uint32_t dist = 0);
cudaError_t launch_synth_tokens(uint16_t* out, uint64_t seed, int64_t blk0, int64_t nblk, int Nd,
                                int d, cudaStream_t st);

// -------- MaxSim (K4): maxsim.cu
struct MaxSimArgs {
  const float* qtok;     // [B][nq][d] fp32 (rounded to bf16 in-kernel)
  const uint16_t* qtok16 = nullptr;  // or already-rounded bf16 bits (shard exchange); with
                                     // split, two planes: hi at qtok16, lo at qtok16 + lo_off
  int64_t lo_off = 0;
  int split = 0;         // TC kernel: query tokens as bf16 hi + lo pairs (fp32-faithful)
  const int64_t* cand;   // [B][C] global doc ids, -1 = skip
  const uint16_t* table; // [T][Nd][d] bf16 bits
  const float* table32 = nullptr;  // or an fp32 store (VX_FLAG_TOKENS_F32): the CUDA-core
                                   // kernel then keeps the query tokens in fp32 too
  int64_t T;
  int32_t B, nq, C, Nd, d;
  float* out;            // [B][C]
  int64_t id_lo = 0, id_hi = INT64_MAX;  // ids outside [lo, hi) (another shard's) -> -INF, no loads
  float own_frac = 1.0f;  // expected fraction of candidates inside [lo, hi) (the launch sizes
                          // its candidate chunks by the OWNED work: 1 / G when sharded)
  KTimer* ktimer = nullptr;
};
cudaError_t launch_maxsim(const MaxSimArgs& a, cudaStream_t st);
// the fp32 token store (a.table32; nq <= 32, Nd <= 128, d % 4 == 0): register-tiled exact fp32
cudaError_t launch_maxsim_f32(const MaxSimArgs& a, cudaStream_t st);
// fp32 -> bf16 hi plane (out) + lo plane (out + n): hi = RNE(v), lo = RNE(v - hi)
cudaError_t launch_split_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st);
constexpr int kMaxSimSplitMaxNq = 64;  // hi/lo rows share the 128-row A tile
bool maxsim_tc_supported(int nq, int Nd, int d);
cudaError_t launch_maxsim_tc(const CUtensorMap* tt, const MaxSimArgs& a, cudaStream_t st);

}  // namespace vx
