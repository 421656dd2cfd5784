// vx_merge.cuh — block-level device routines shared by the standalone kernels (topk.cu) and
// the fused re-rank (scan_tc.cu rerank_kernel): the merge of one query's candidate lists to
// its top-k (K3) and the compaction of the certificate failures of a batch.  Header-only so
// both translation units inline them (no relocatable device code).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "vx_internal.cuh"
#include "vx_sort.cuh"

namespace vx {

// timing experiments only (profiles/microbench/merge_bench.cu defines VX_MERGE_TRACE): clock64
// stamps of CTA 0's phases
#ifdef VX_MERGE_TRACE
__device__ unsigned long long g_merge_trace[32];
__device__ int g_merge_trace_n;
#define MERGE_STAMP()                                                             \
  do {                                                                            \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_merge_trace_n < 32)             \
      g_merge_trace[g_merge_trace_n++] = clock64();                               \
  } while (0)
#else
#define MERGE_STAMP() \
  do {                \
  } while (0)
#endif

constexpr int kMergeThreads = 256;
constexpr int kMaxK = 1024;  // merge: k' up to 1024 (the TC candidate set); order_by: k <= 256
constexpr int kMergeFilterKeys = 512;  // standalone merge: the sorted-list filter's buffer

// The merge of ONE query's lists L[0, M) to its best k keys, by the whole block (blockDim.x a
// multiple of 32, <= 1024; every thread calls it).  staged: nullable smem for the M keys
// (M <= kMergeSmemKeys, M even); sel: smem for next_pow2(max(k, 16)) keys.  Row `row` of the
// outputs (stride ldout).  Also the prologue of the fused re-rank (scan_tc.cu rerank_kernel).
//
// Sorted lists (P > 0: L = P lists of KC keys, each descending — the per-CTA lists of the scan,
// the shards' top-k lists): a filter first.  With S = the (j+1)-th key of every list and
// m (j+1) >= k, the m-th largest of S, T0, has at least m (j+1) >= k keys at or above it, so
// the k best keys are all >= T0; binary searches count each list's keys >= T0 and, when those
// (C) fit fbuf (fcap keys) and two keys per thread, ranking them gives the answer in order —
// no radix passes (each pass is a chain of barriers and atomics: 2 passes + collection + sort
// took ~17 K cycles for 2368 keys -> 64) and no sort (T0 and the C keys were two bitonic sorts:
// 5 K + 3.7 K of the filter's 13.6 K cycles; profiles/microbench/merge_bench.cu).  Otherwise
// (C too large, or T0 = 0: short lists) the radix select below runs as before.
// Inst: a separate instantiation per call site family (the fused re-rank keeps its own copy:
// one non-inlined body shared with a kernel of a larger register budget raised the re-rank
// from 80 to 116 registers)
template <int Inst = 0>
static __device__ __noinline__ void merge_topk_block(const uint64_t* __restrict__ L, int M, int k, int64_t id_base,
                                 uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_ids,
                                 float* __restrict__ out_scores, size_t row, int64_t ldout,
                                 uint64_t* staged, uint64_t* sel, int P = 0, int KC = 0,
                                 uint64_t* fbuf = nullptr, int fcap = 0) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix, s_mask;
  __shared__ int s_kk, s_done, s_above, s_eq;
  __shared__ int s_wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  MERGE_STAMP();
  if (staged && M <= kMergeSmemKeys && (M & 1) == 0) {  // stage (16-byte loads, all in flight)
    const uint4* src = reinterpret_cast<const uint4*>(L);
    uint4* dst = reinterpret_cast<uint4*>(staged);
    if ((reinterpret_cast<uintptr_t>(L) & 15) == 0) {
      for (int i = threadIdx.x; i < (M >> 1); i += blockDim.x) dst[i] = src[i];
    } else {
      for (int i = threadIdx.x; i < M; i += blockDim.x) staged[i] = L[i];
    }
    __syncthreads();
    L = staged;
  }
  MERGE_STAMP();
  if (P > 0 && KC > 0 && fbuf && P <= (int)blockDim.x && P <= fcap && k <= fcap &&
      (int64_t)P * KC == M) {
    const int j1 = (k + P - 1) / P;  // j + 1
    if (j1 <= KC) {
      const int m = (k + j1 - 1) / j1;  // <= P
      // t0 = the m-th largest of the lists' (j+1)-th keys, by rank (distinct documents:
      // distinct keys; 0 when fewer than m lists reach j + 1 keys)
      __shared__ uint64_t s_t0;
      if (threadIdx.x == 0) s_t0 = 0ull;
      for (int i = threadIdx.x; i < P; i += blockDim.x) fbuf[i] = L[(size_t)i * KC + (j1 - 1)];
      __syncthreads();
      MERGE_STAMP();
      if ((int)threadIdx.x < P) {
        const uint64_t v = fbuf[threadIdx.x];
        if (v != 0ull && rank_desc(fbuf, P, v) == m - 1) s_t0 = v;
      }
      __syncthreads();
      const uint64_t t0 = s_t0;
      MERGE_STAMP();
      if (t0 != 0ull) {
        // keys >= t0 in list p (descending: a prefix), by binary search; block prefix sum
        int c = 0;
        if ((int)threadIdx.x < P) {
          const uint64_t* lp = L + (size_t)threadIdx.x * KC;
          int lo = 0, hi = KC;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (lp[mid] >= t0) lo = mid + 1;
            else hi = mid;
          }
          c = lo;
        }
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) s_wsum[warp] = x;
        __syncthreads();
        MERGE_STAMP();
        int base = 0, C = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          const int v = s_wsum[w];
          if (w < warp) base += v;
          C += v;
        }
        // the C (>= k) survivors, all nonzero and distinct: ranked straight into the outputs
        if (C <= fcap && C <= 2 * (int)blockDim.x) {
          const int off = base + x - c;  // exclusive prefix of this list
          if (c) {
            const uint64_t* lp = L + (size_t)threadIdx.x * KC;
            for (int i = 0; i < c; ++i) fbuf[off + i] = lp[i];
          }
          __syncthreads();
          MERGE_STAMP();
          auto emit = [&](int r, uint64_t key) {
            const size_t o = row * ldout + r;
            if (key == 0ull) {
              if (out_keys) out_keys[o] = 0ull;
              if (out_ids) out_ids[o] = -1;
              if (out_scores) out_scores[o] = -INFINITY;
            } else {
              const int64_t gid = (int64_t)vx_key_id(key) + id_base;
              if (out_keys)
                out_keys[o] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (uint32_t)gid);
              if (out_ids) out_ids[o] = gid;
              if (out_scores) out_scores[o] = vx_key_score(key);
            }
          };
          rank_topk_block(fbuf, C, k, emit);
          for (int i = C + (int)threadIdx.x; i < k; i += blockDim.x) emit(i, 0ull);
          MERGE_STAMP();
          __syncthreads();
          MERGE_STAMP();
          return;
        }
      }
    }
  }

  // the digits every key shares need no pass: start at the first byte where the largest
  // and the smallest key differ (scores of one query's candidates share sign, exponent and
  // often leading mantissa bits — one or two of the ~3 passes).  Padding keys (0: a list
  // shorter than its slots, a pruned candidate) do not count for the smallest key — one of
  // them zeroed the shared prefix and cost every merge all eight passes (11-15 us of a
  // 16-query re-rank, VX_DEBUG_RERANK_TRACE); they never outrank a real key, and when fewer
  // than k real keys exist the selection below takes them all and pads with 0.
  uint64_t kmax = 0ull, kmin = ~0ull;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const uint64_t v = L[i];
    kmax = v > kmax ? v : kmax;
    kmin = (v != 0ull && v < kmin) ? v : kmin;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a = shfl_xor_u64(kmax, o), b = shfl_xor_u64(kmin, o);
    kmax = a > kmax ? a : kmax;
    kmin = b < kmin ? b : kmin;
  }
  __shared__ uint64_t s_mx[32], s_mn[32];
  if (lane == 0) {
    s_mx[warp] = kmax;
    s_mn[warp] = kmin;
  }
  __syncthreads();
  kmax = s_mx[0];
  kmin = s_mn[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    kmax = s_mx[w] > kmax ? s_mx[w] : kmax;
    kmin = s_mn[w] < kmin ? s_mn[w] : kmin;
  }
  MERGE_STAMP();
  if (kmax == 0ull) kmin = 0ull;  // no real key at all
  const int common_bytes = (kmax == kmin) ? 7 : (__clzll((long long)(kmax ^ kmin)) >> 3);
  uint64_t mask = common_bytes ? (~0ull << (64 - 8 * common_bytes)) : 0ull;
  uint64_t prefix = kmax & mask;
  int kk = k;
  for (int shift = 56 - 8 * common_bytes; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // histogram of the next digit over the keys still matching the prefix.  Top digits are
    // shared by most keys, so a warp whose live lanes all carry one digit adds once; mixed
    // warps add per lane (match.any aggregation was the kernel's critical path: its result
    // latency stalled every iteration — profiles/r02)
    // Four keys per thread per iteration: their chains are independent, so the warp keeps
    // four in flight (one key at a time left every iteration a ~300-cycle dependent chain).
    for (int i0 = 0; i0 < M; i0 += 4 * (int)blockDim.x) {
      uint64_t kx[4];
      bool lv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
        kx[u] = i < M ? L[i] : 0ull;
        lv[u] = i < M && (kx[u] & mask) == prefix;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned act = __ballot_sync(0xffffffffu, lv[u]);
        if (act == 0u) continue;
        const uint32_t dg = (uint32_t)(kx[u] >> shift) & 255u;
        const uint32_t d0 = __shfl_sync(0xffffffffu, dg, __ffs(act) - 1);
        const bool uni = __all_sync(0xffffffffu, !lv[u] || dg == d0);
        if (uni) {
          if (lane == 0) atomicAdd(&hist[d0], (uint32_t)__popc(act));
        } else if (lv[u]) {
          atomicAdd(&hist[dg], 1u);
        }
      }
    }
    __syncthreads();
    if (warp == 0) {
      // bins from the top: lane l owns digits 255-8l .. 248-8l; find the digit d holding
      // the kk-th key (descending) with a suffix scan over the lanes
      uint32_t c[8];
      uint32_t tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * lane - j];
        tot += c[j];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - tot;  // keys in higher digits than this lane's
      const bool mine = excl < (uint32_t)kk && incl >= (uint32_t)kk;
      const unsigned who = __ballot_sync(0xffffffffu, mine);
      if (who == 0) {
        // fewer than kk keys match at all: every one of them is selected; digit 0 (lane 31,
        // j = 7) becomes the "equal" bin, the other digits count as above it
        if (lane == 31) {
          s_prefix = prefix;
          s_mask = mask | (0xFFull << shift);
          s_kk = kk - (int)(incl - c[7]);
          s_done = 1;
        }
      } else if (lane == __ffs(who) - 1) {
        uint32_t above = excl;
        int d = 255 - 8 * lane;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (above + c[j] >= (uint32_t)kk) {
            d = 255 - 8 * lane - j;
            s_kk = kk - (int)above;
            s_done = (c[j] == (uint32_t)kk - above);
            break;
          }
          above += c[j];
        }
        s_prefix = prefix | ((uint64_t)d << shift);
        s_mask = mask | (0xFFull << shift);
      }
    }
    __syncthreads();
    prefix = s_prefix;
    mask = s_mask;
    kk = s_kk;
    MERGE_STAMP();
    if (s_done) break;
    __syncthreads();
  }
  int kp = 16;
  while (kp < k) kp <<= 1;
  for (int i = threadIdx.x; i < kp; i += blockDim.x) sel[i] = 0ull;
  if (threadIdx.x == 0) {
    s_above = 0;
    s_eq = 0;
  }
  __syncthreads();
  const int n_above = k - kk;
  for (int i0 = 0; i0 < M; i0 += 4 * (int)blockDim.x) {
    uint64_t kx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
      kx[u] = i < M ? L[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
      if (i >= M) continue;
      const uint64_t m = kx[u] & mask;
      if (m > prefix) {
        const int slot = atomicAdd(&s_above, 1);
        sel[slot] = kx[u];
      } else if (m == prefix) {
        const int slot = atomicAdd(&s_eq, 1);
        if (slot < kk) sel[n_above + slot] = kx[u];
      }
    }
  }
  __syncthreads();
  MERGE_STAMP();
  block_sort_desc(sel, kp);
  MERGE_STAMP();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    uint64_t key = sel[i];
    size_t o = row * ldout + i;
    if (key == 0ull) {
      if (out_keys) out_keys[o] = 0ull;
      if (out_ids) out_ids[o] = -1;
      if (out_scores) out_scores[o] = -INFINITY;
    } else {
      int64_t gid = (int64_t)vx_key_id(key) + id_base;
      if (out_keys)
        out_keys[o] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (uint32_t)gid);
      if (out_ids) out_ids[o] = gid;
      if (out_scores) out_scores[o] = vx_key_score(key);
    }
  }
  __syncthreads();  // sel / staged / the shared scalars are free again
  MERGE_STAMP();
}


// Compaction of the batch's certificate failures (flags[b] != 0, ascending b) into fidx /
// fcount and their fp32 queries into fq; sets the conditional handle of the captured stage.
// Whole block (blockDim.x a multiple of 32, <= 1024).
static __device__ __forceinline__ void cert_compact_block(const int* __restrict__ flags, int B,
                                                   const float* __restrict__ q, int D,
                                                   int* __restrict__ fidx, int* __restrict__ fcount,
                                                   float* __restrict__ fq,
                                                   cudaGraphConditionalHandle cond, int use_cond) {
  // stream compaction of the flagged queries (ascending order), blockDim.x flags per round:
  // warp ballots + a prefix over the 32 warp counts
  __shared__ int s_warp[32];
  __shared__ int s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += (int)blockDim.x) {
    const int b = b0 + (int)threadIdx.x;
    const bool f = b < B && flags[b] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      const int c = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = x - c;  // exclusive prefix
    }
    __syncthreads();
    const int base = s_base;
    if (f) fidx[base + s_warp[warp] + __popc(m & ((1u << lane) - 1u))] = b;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_base = base + s_warp[(blockDim.x >> 5) - 1] + __popc(m);
    __syncthreads();
  }
  const int n = s_base;
  if (threadIdx.x == 0) {
    fcount[0] = n;   // this batch
    fcount[1] += n;  // running total (vx_stats.cert_fallbacks)
    // captured stage: the rest of the certificate chain is the body of a conditional graph
    // node that runs only when some query failed (vx_stage.cu local_topk_tc)
    if (use_cond) cudaGraphSetConditional(cond, n > 0 ? 1u : 0u);
  }
  __threadfence_block();
  __syncthreads();
  for (int i = threadIdx.x; i < n * D; i += blockDim.x) {
    const int r = i / D;
    fq[i] = q[(size_t)fidx[r] * D + (i - r * D)];
  }
}


}  // namespace vx
