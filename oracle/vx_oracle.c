/*
 * vx_oracle.c — CPU restatement of the retrieval stage.  TEST INFRASTRUCTURE:
 * see vx_oracle.h for what it restates, the modes and the parity status.
 *
 * Build: oracle/Makefile  (gcc -O3 -march=x86-64-v4 -fopenmp, shared library).
 * The fp32 mode is also the timed CPU baseline (bench.py cpu_baseline /
 * --impl reference): queries are transposed so that one AVX-512 FMA advances 16
 * (query, doc) dot products by one dimension; each dot product is still an
 * in-order fmaf chain over the dimension, i.e. bit-identical to the GPU scan.
 */
#include "vx_oracle.h"

#include <immintrin.h>
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "../include/vx_synth.h"

int vxo_threads(void) { return omp_get_max_threads(); }

static int nthreads_of(int32_t threads) { return threads > 0 ? threads : omp_get_max_threads(); }

void vxo_synth_rows(uint64_t seed, int64_t row0, int64_t n, int32_t dim, float* out) {
  vxo_synth_rows_dist(seed, row0, n, dim, 0, out);
}

void vxo_synth_rows_dist(uint64_t seed, int64_t row0, int64_t n, int32_t dim, int32_t dist,
                         float* out) {
#pragma omp parallel
  {
    int32_t* v = (int32_t*)malloc(sizeof(int32_t) * (size_t)dim);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
      int64_t ss = 0;
      for (int32_t c = 0; c < dim; ++c) {
        v[c] = vx_synth_int_d(seed, (uint64_t)(row0 + r), (uint64_t)c, (uint32_t)dist);
        ss += (int64_t)v[c] * (int64_t)v[c];
      }
      float* o = out + r * (int64_t)dim;
      for (int32_t c = 0; c < dim; ++c) o[c] = vx_synth_finish(v[c], ss);
    }
    free(v);
  }
}

static void vxo_synth_tokens_one(uint64_t seed, int64_t blk, int32_t ntok, int32_t dim,
                                 uint16_t* out) {
  int32_t v[4096];
  for (int32_t j = 0; j < ntok; ++j) {
    uint64_t grow = (uint64_t)(blk * ntok + j);
    int64_t ss = 0;
    for (int32_t c = 0; c < dim; ++c) {
      v[c] = vx_synth_int(seed, grow, (uint64_t)c);
      ss += (int64_t)v[c] * (int64_t)v[c];
    }
    uint16_t* o = out + (int64_t)j * dim;
    for (int32_t c = 0; c < dim; ++c) o[c] = vx_f32_to_bf16_bits(vx_synth_finish(v[c], ss));
  }
}

void vxo_synth_tokens(uint64_t seed, int64_t blk0, int64_t nblk, int32_t ntok, int32_t dim,
                      uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < nblk; ++b)
    vxo_synth_tokens_one(seed, blk0 + b, ntok, dim, out + b * (int64_t)ntok * dim);
}

void vxo_synth_token_blocks(uint64_t seed, const int64_t* blks, int64_t n, int32_t ntok,
                            int32_t dim, uint16_t* out) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i)
    vxo_synth_tokens_one(seed, blks[i], ntok, dim, out + i * (int64_t)ntok * dim);
}

double vxo_dot(const float* x, const float* q, int32_t dim, int32_t mode) {
  if (mode == VXO_F32) {
    float acc = 0.0f;
    for (int32_t t = 0; t < dim; ++t) acc = fmaf(x[t], q[t], acc);
    return (double)acc;
  }
  double acc = 0.0;
  for (int32_t t = 0; t < dim; ++t) acc += (double)x[t] * (double)q[t];
  return acc;
}

/* ---- top-k lists: (score desc, id asc), kept sorted ---------------------- */

typedef struct {
  double s;
  int64_t id;
} vxo_ent;

static inline int better(double s, int64_t id, const vxo_ent* e) {
  return s > e->s || (s == e->s && id < e->id);
}

/* insert into list of current size *cnt (capacity k) */
static inline void topk_push(vxo_ent* L, int32_t* cnt, int32_t k, double s, int64_t id) {
  int32_t c = *cnt;
  if (c == k && !better(s, id, &L[k - 1])) return;
  int32_t pos = (c < k) ? c : k - 1;
  while (pos > 0 && better(s, id, &L[pos - 1])) {
    L[pos] = L[pos - 1];
    --pos;
  }
  L[pos].s = s;
  L[pos].id = id;
  if (c < k) *cnt = c + 1;
}

#define VXO_DB 8 /* docs per register block */

/* acc[r][b] = in-order fmaf chain over t of X[d0+r][t] * Qt[t][b], r < nb (<= VXO_DB),
 * b < Bp (multiple of 16).  AVX-512: 16 queries per register, up to 16 accumulators. */
static void block_f32(const float* X, int64_t d0, int32_t nb, int32_t dim, const float* Qt,
                      int32_t Bp, float* acc) {
  for (int32_t g0 = 0; g0 < Bp; g0 += 32) {
    int32_t mv = (Bp - g0 >= 32) ? 2 : 1;
    __m512 a[VXO_DB][2];
    for (int32_t r = 0; r < VXO_DB; ++r) a[r][0] = a[r][1] = _mm512_setzero_ps();
    const float* xr[VXO_DB];
    for (int32_t r = 0; r < VXO_DB; ++r) xr[r] = X + (d0 + (r < nb ? r : 0)) * (int64_t)dim;
    if (mv == 2) {
      for (int32_t t = 0; t < dim; ++t) {
        __m512 q0 = _mm512_loadu_ps(Qt + (int64_t)t * Bp + g0);
        __m512 q1 = _mm512_loadu_ps(Qt + (int64_t)t * Bp + g0 + 16);
        for (int32_t r = 0; r < VXO_DB; ++r) {
          __m512 xv = _mm512_set1_ps(xr[r][t]);
          a[r][0] = _mm512_fmadd_ps(xv, q0, a[r][0]);
          a[r][1] = _mm512_fmadd_ps(xv, q1, a[r][1]);
        }
      }
    } else {
      for (int32_t t = 0; t < dim; ++t) {
        __m512 q0 = _mm512_loadu_ps(Qt + (int64_t)t * Bp + g0);
        for (int32_t r = 0; r < VXO_DB; ++r)
          a[r][0] = _mm512_fmadd_ps(_mm512_set1_ps(xr[r][t]), q0, a[r][0]);
      }
    }
    for (int32_t r = 0; r < nb; ++r) {
      _mm512_storeu_ps(acc + r * Bp + g0, a[r][0]);
      if (mv == 2) _mm512_storeu_ps(acc + r * Bp + g0 + 16, a[r][1]);
    }
  }
}

int vxo_flat_topk(const float* X, int64_t n, int32_t dim, int64_t id_base, const float* Q,
                  int32_t B, int32_t k, int32_t mode, int32_t threads, int64_t* ids,
                  double* scores) {
  if (n < 0 || dim <= 0 || B <= 0 || k <= 0) return -1;
  int nt = nthreads_of(threads);
  int32_t Bp = (B + 15) & ~15;
  /* transposed, zero-padded queries */
  float* Qt = (float*)calloc((size_t)dim * Bp, sizeof(float));
  double* Qtd = (double*)calloc((size_t)dim * Bp, sizeof(double));
  for (int32_t b = 0; b < B; ++b)
    for (int32_t t = 0; t < dim; ++t) {
      Qt[(int64_t)t * Bp + b] = Q[(int64_t)b * dim + t];
      Qtd[(int64_t)t * Bp + b] = (double)Q[(int64_t)b * dim + t];
    }
  vxo_ent* lists = (vxo_ent*)malloc(sizeof(vxo_ent) * (size_t)nt * B * k);
  int32_t* counts = (int32_t*)calloc((size_t)nt * B, sizeof(int32_t));

#pragma omp parallel num_threads(nt)
  {
    int tid = omp_get_thread_num();
    vxo_ent* L = lists + (int64_t)tid * B * k;
    int32_t* C = counts + (int64_t)tid * B;
    float* accf = (float*)aligned_alloc(64, sizeof(float) * VXO_DB * Bp);
    double* accd = (double*)aligned_alloc(64, sizeof(double) * VXO_DB * Bp);
#pragma omp for schedule(static)
    for (int64_t d0 = 0; d0 < n; d0 += VXO_DB) {
      int32_t nb = (n - d0 < VXO_DB) ? (int32_t)(n - d0) : VXO_DB;
      if (mode == VXO_F32) {
        block_f32(X, d0, nb, dim, Qt, Bp, accf);
        for (int32_t r = 0; r < nb; ++r)
          for (int32_t b = 0; b < B; ++b)
            topk_push(L + (int64_t)b * k, &C[b], k, (double)accf[r * Bp + b], id_base + d0 + r);
      } else {
        memset(accd, 0, sizeof(double) * VXO_DB * Bp);
        for (int32_t t = 0; t < dim; ++t) {
          const double* qt = Qtd + (int64_t)t * Bp;
          for (int32_t r = 0; r < nb; ++r) {
            double xv = (double)X[(d0 + r) * (int64_t)dim + t];
            double* a = accd + r * Bp;
#pragma omp simd
            for (int32_t b = 0; b < Bp; ++b) a[b] += xv * qt[b];
          }
        }
        for (int32_t r = 0; r < nb; ++r)
          for (int32_t b = 0; b < B; ++b)
            topk_push(L + (int64_t)b * k, &C[b], k, accd[r * Bp + b], id_base + d0 + r);
      }
    }
    free(accf);
    free(accd);
  }
  /* merge per-thread lists */
  vxo_ent* fin = (vxo_ent*)malloc(sizeof(vxo_ent) * (size_t)k);
  for (int32_t b = 0; b < B; ++b) {
    int32_t fc = 0;
    for (int t = 0; t < nt; ++t) {
      vxo_ent* L = lists + ((int64_t)t * B + b) * k;
      int32_t c = counts[(int64_t)t * B + b];
      for (int32_t i = 0; i < c; ++i) topk_push(fin, &fc, k, L[i].s, L[i].id);
    }
    for (int32_t i = 0; i < k; ++i) {
      ids[(int64_t)b * k + i] = i < fc ? fin[i].id : -1;
      scores[(int64_t)b * k + i] = i < fc ? fin[i].s : -INFINITY;
    }
  }
  free(fin);
  free(lists);
  free(counts);
  free(Qt);
  free(Qtd);
  return 0;
}

/* ---- MaxSim ------------------------------------------------------------- */

static double maxsim_one(const float* qb /* bf16-rounded (VXO_F64_Q32: raw) fp32 [nq][dim] */, int32_t nq,
                         int32_t dim, const uint16_t* dt /* [Nd][dim] */, int32_t Nd,
                         int32_t mode) {
  if (mode == VXO_F32) {
    float total = 0.0f;
    for (int32_t i = 0; i < nq; ++i) {
      float best = -INFINITY;
      for (int32_t j = 0; j < Nd; ++j) {
        float acc = 0.0f;
        for (int32_t t = 0; t < dim; ++t)
          acc = fmaf(qb[(int64_t)i * dim + t], vx_bf16_bits_to_f32(dt[(int64_t)j * dim + t]), acc);
        if (acc > best) best = acc;
      }
      total += best;
    }
    return (double)total;
  }
  double total = 0.0;
  for (int32_t i = 0; i < nq; ++i) {
    double best = -INFINITY;
    for (int32_t j = 0; j < Nd; ++j) {
      double acc = 0.0;
      for (int32_t t = 0; t < dim; ++t)
        acc += (double)qb[(int64_t)i * dim + t] * (double)vx_bf16_bits_to_f32(dt[(int64_t)j * dim + t]);
      if (acc > best) best = acc;
    }
    total += best;
  }
  return total;
}

/* MaxSim against an fp32 doc-token table (the fp32 token store, VX_FLAG_TOKENS_F32): the
 * query tokens stay fp32 in every mode; VXO_F32 = one in-order fmaf chain per (query token,
 * doc token), max in order, the sum over query tokens in order (maxsim.cu maxsim_cc_kernel);
 * VXO_F64 / VXO_F64_Q32 = the same in fp64 (the truth). */
static double maxsim_one_f32(const float* q, int32_t nq, int32_t dim, const float* dt, int32_t Nd,
                             int32_t mode) {
  if (mode == VXO_F32) {
    float total = 0.0f;
    for (int32_t i = 0; i < nq; ++i) {
      float best = -INFINITY;
      for (int32_t j = 0; j < Nd; ++j) {
        float acc = 0.0f;
        for (int32_t t = 0; t < dim; ++t)
          acc = fmaf(q[(int64_t)i * dim + t], dt[(int64_t)j * dim + t], acc);
        if (acc > best) best = acc;
      }
      total += best;
    }
    return (double)total;
  }
  double total = 0.0;
  for (int32_t i = 0; i < nq; ++i) {
    double best = -INFINITY;
    for (int32_t j = 0; j < Nd; ++j) {
      double acc = 0.0;
      for (int32_t t = 0; t < dim; ++t)
        acc += (double)q[(int64_t)i * dim + t] * (double)dt[(int64_t)j * dim + t];
      if (acc > best) best = acc;
    }
    total += best;
  }
  return total;
}

int vxo_maxsim_f32tab(const float* qtok, int32_t B, int32_t nq, int32_t dim, const int64_t* cand,
                      int32_t C, const float* table, int64_t T, int32_t Nd, int32_t mode,
                      int32_t threads, double* out) {
  if (B <= 0 || nq <= 0 || dim <= 0 || C < 0 || T <= 0 || Nd <= 0) return -1;
  int nt = nthreads_of(threads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
  for (int64_t bc = 0; bc < (int64_t)B * C; ++bc) {
    int64_t b = bc / C;
    int64_t id = cand[bc];
    if (id < 0) {
      out[bc] = -INFINITY;
      continue;
    }
    out[bc] = maxsim_one_f32(qtok + b * nq * dim, nq, dim, table + (id % T) * (int64_t)Nd * dim, Nd,
                             mode);
  }
  return 0;
}

int vxo_maxsim(const float* qtok, int32_t B, int32_t nq, int32_t dim, const int64_t* cand,
               int32_t C, const uint16_t* table, int64_t T, int32_t Nd, int32_t mode,
               int32_t threads, double* out) {
  if (B <= 0 || nq <= 0 || dim <= 0 || C < 0 || T <= 0 || Nd <= 0) return -1;
  int nt = nthreads_of(threads);
  int64_t qn = (int64_t)B * nq * dim;
  float* qb = (float*)malloc(sizeof(float) * (size_t)qn);
  for (int64_t i = 0; i < qn; ++i)
    qb[i] = mode == VXO_F64_Q32 ? qtok[i] : vx_bf16_bits_to_f32(vx_f32_to_bf16_bits(qtok[i]));
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
  for (int64_t bc = 0; bc < (int64_t)B * C; ++bc) {
    int64_t b = bc / C;
    int64_t id = cand[bc];
    if (id < 0) {
      out[bc] = -INFINITY;
      continue;
    }
    const uint16_t* dt = table + (id % T) * (int64_t)Nd * dim;
    out[bc] = maxsim_one(qb + b * nq * dim, nq, dim, dt, Nd, mode);
  }
  free(qb);
  return 0;
}

int vxo_search_rescore(const float* X, int64_t n, int32_t dim, const float* Q, const float* qtok,
                       int32_t B, int32_t nq, int32_t tdim, int32_t k, const uint16_t* table, int64_t T,
                       int32_t Nd, int32_t mode, int32_t threads, int64_t* ids, double* ip,
                       double* ms) {
  int64_t* tid = (int64_t*)malloc(sizeof(int64_t) * (size_t)B * k);
  double* tsc = (double*)malloc(sizeof(double) * (size_t)B * k);
  double* tms = (double*)malloc(sizeof(double) * (size_t)B * k);
  int rc = vxo_flat_topk(X, n, dim, 0, Q, B, k, mode, threads, tid, tsc);
  if (rc == 0) rc = vxo_maxsim(qtok, B, nq, tdim, tid, k, table, T, Nd, mode, threads, tms);
  if (rc == 0) {
    vxo_ent* L = (vxo_ent*)malloc(sizeof(vxo_ent) * (size_t)k);
    for (int32_t b = 0; b < B; ++b) {
      int32_t c = 0;
      /* order by maxsim desc, id asc; carry ip alongside via index lookup */
      for (int32_t i = 0; i < k; ++i) {
        int64_t id = tid[(int64_t)b * k + i];
        if (id >= 0) topk_push(L, &c, k, tms[(int64_t)b * k + i], id);
      }
      for (int32_t i = 0; i < k; ++i) {
        int64_t o = (int64_t)b * k + i;
        if (i < c) {
          ids[o] = L[i].id;
          ms[o] = L[i].s;
          for (int32_t j = 0; j < k; ++j)
            if (tid[(int64_t)b * k + j] == L[i].id) ip[o] = tsc[(int64_t)b * k + j];
        } else {
          ids[o] = -1;
          ms[o] = -INFINITY;
          ip[o] = -INFINITY;
        }
      }
    }
    free(L);
  }
  free(tid);
  free(tsc);
  free(tms);
  return rc;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

double vxo_percentile(double* v, int64_t n, double p) {
  if (n <= 0) return NAN;
  qsort(v, (size_t)n, sizeof(double), cmp_double);
  int64_t rank = (int64_t)ceil(p / 100.0 * (double)n);
  if (rank < 1) rank = 1;
  if (rank > n) rank = n;
  return v[rank - 1];
}
