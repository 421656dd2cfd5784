/*
 * vx_oracle.h — CPU oracle for the retrieval hot path.  TEST INFRASTRUCTURE ONLY:
 * imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg, as the checker and the timed CPU baseline.  The product
 * (paper_2511_02062_b200/) never links or calls it.
 *
 * What it restates (the reference has no retrieval arithmetic):
 *  - the stage semantics: a batch of query payloads in, per-query top-k ids and
 *    scores out, output i <-> input i  (proj/include/vortex/runtime.hpp:179,
 *    :656-672; stage D "Colbert search", pipeline.json:7);
 *  - exact flat inner-product top-k (BASELINE.json north_star; the paper's IVFPQ,
 *    PAPER.md:407, is approximate — exact flat is the deliberate spec);
 *  - ColBERT late interaction  score(q,d) = sum_i max_j <q_i, d_j>;
 *  - nearest-rank percentile (proj/include/vortex/bench.hpp:69-76).
 *
 * Arithmetic modes
 *  VXO_F64: products of the fp32 (or bf16) inputs accumulated in fp64 — the truth
 *           used for tie tolerances;
 *  VXO_F32: fp32 fused multiply-add chained over the dimension in index order
 *           (acc = fmaf(x[t], q[t], acc), t = 0..D-1), the order the GPU exact
 *           scan uses, so the two agree bit-for-bit.
 * Ordering everywhere: score descending, then id ascending.
 *
 * Parity status: the arithmetic is UNPINNED by the reference (it contains none);
 * this oracle is pinned against numpy fp64 golden vectors and hand-computed
 * known-answer tests (tests/golden/, tests/test_oracle.py).  The batcher /
 * operator boundary is pinned against the reference's own runtime compiled in
 * oracle/_ref (oracle/ref_driver.cpp).
 */
#ifndef VX_ORACLE_H_
#define VX_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VXO_F64 = 0, VXO_F32 = 1, VXO_F64_Q32 = 2 };
/* VXO_F64_Q32 (vxo_maxsim only): fp64 accumulation with the query tokens kept in fp32 — the
 * truth against the fp32 tokens a VXQ1 payload carries, so the bf16 rounding of the query
 * tokens on the GPU path shows up as error instead of being part of the reference. */

int vxo_threads(void);

/* Rows [row0, row0+n) of the synthetic matrix (vx_synth.h), fp32 [n][dim]. */
void vxo_synth_rows(uint64_t seed, int64_t row0, int64_t n, int32_t dim, float* out);
/* ... of distribution dist (0 isotropic, 1 anisotropic: vx_synth_mult). */
void vxo_synth_rows_dist(uint64_t seed, int64_t row0, int64_t n, int32_t dim, int32_t dist,
                         float* out);
/* Token blocks [blk0, blk0+nblk): bf16 bits [nblk][ntok][dim]; block b token j is
 * synthetic row b*ntok + j. */
void vxo_synth_tokens(uint64_t seed, int64_t blk0, int64_t nblk, int32_t ntok, int32_t dim,
                      uint16_t* out);

/* Token blocks blks[0..n) (any order, repeats allowed): bf16 bits [n][ntok][dim], block
 * blks[i] as in vxo_synth_tokens — the blocks a batch's candidates touch, without the whole
 * table. */
void vxo_synth_token_blocks(uint64_t seed, const int64_t* blks, int64_t n, int32_t ntok,
                            int32_t dim, uint16_t* out);

/* Single inner product in the given mode. */
double vxo_dot(const float* x, const float* q, int32_t dim, int32_t mode);

/* Exact flat IP top-k over X [n][dim] whose row r has id id_base + r.
 * ids [B][k] (-1 when k > n), scores [B][k] (as double; in VXO_F32 mode the
 * exact fp32 value).  threads <= 0 -> all cores.  Returns 0 on success. */
int vxo_flat_topk(const float* X, int64_t n, int32_t dim, int64_t id_base, const float* Q,
                  int32_t B, int32_t k, int32_t mode, int32_t threads, int64_t* ids,
                  double* scores);

/* MaxSim of query tokens qtok fp32 [B][nq][dim] (rounded to bf16 first, as the
 * GPU does, except in VXO_F64_Q32) against cand [B][C] ids; doc id uses token block (id mod T) of
 * `table` (bf16 [T][Nd][dim]).  cand -1 -> -INF.  out [B][C]. */
int vxo_maxsim(const float* qtok, int32_t B, int32_t nq, int32_t dim, const int64_t* cand,
               int32_t C, const uint16_t* table, int64_t T, int32_t Nd, int32_t mode,
               int32_t threads, double* out);
/* The same against an fp32 table [T][Nd][dim] (query tokens kept in fp32 in every mode). */
int vxo_maxsim_f32tab(const float* qtok, int32_t B, int32_t nq, int32_t dim, const int64_t* cand,
                      int32_t C, const float* table, int64_t T, int32_t Nd, int32_t mode,
                      int32_t threads, double* out);

/* The fused stage: IP top-k, MaxSim of those k, re-ordered by MaxSim desc (ties
 * id asc).  ids/ip/ms [B][k]. */
int vxo_search_rescore(const float* X, int64_t n, int32_t dim, const float* Q, const float* qtok,
                       int32_t B, int32_t nq, int32_t tdim, int32_t k, const uint16_t* table, int64_t T,
                       int32_t Nd, int32_t mode, int32_t threads, int64_t* ids, double* ip,
                       double* ms);

/* Nearest-rank percentile, bench.hpp:69-76 (v is sorted in place). */
double vxo_percentile(double* v, int64_t n, double p);

#ifdef __cplusplus
}
#endif

#endif /* VX_ORACLE_H_ */
