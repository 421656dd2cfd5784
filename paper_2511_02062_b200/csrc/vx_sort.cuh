// vx_sort.cuh — descending bitonic sort of u64 keys held in registers, for the small sorts of
// the stage (K3 merge output, the re-rank's k' exact keys, the MaxSim output order).
//
// A block-wide sort through shared memory pays one __syncthreads per stage: 55 stages for
// 1024 keys took ~20K cycles in the merge (profiles/microbench/merge_bench.cu).  Here element
// i = t * E + e lives in register e of thread t: strides < E are exchanged inside the thread,
// strides < 32 E between the lanes of a warp (shuffles, no barrier), and only the strides that
// cross warps go through shared memory — 6 barrier stages for 1024 keys on 256 threads.
#pragma once

#include <stdint.h>

namespace vx {

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

template <int E, int S>
__device__ __forceinline__ void in_thread_stage(uint64_t (&v)[E], int t, int size) {
  if constexpr (S < E) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if ((e & S) == 0) {
        const bool desc = (((t * E + e) & size) == 0);
        const uint64_t a = v[e], b = v[e + S];
        const bool sw = desc ? (a < b) : (a > b);
        v[e] = sw ? b : a;
        v[e + S] = sw ? a : b;
      }
    }
  }
}

// Sort N = nthreads * E keys (descending); v[e] is element t * E + e of thread t (t =
// threadIdx.x < nthreads; nthreads a power of two, a multiple of 32).  Every thread of the
// block calls it when the sort spans several warps (the barriers); threads >= nthreads only
// pass the barriers.  buf: N u64 of shared memory (cross-warp strides only).  Ends with the
// sorted keys back in v and nothing pending on buf.
template <int E>
__device__ __forceinline__ void reg_bitonic_desc(uint64_t (&v)[E], int nthreads, uint64_t* buf) {
  const int t = threadIdx.x;
  const int N = nthreads * E;
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < E) {
        // compile-time partner indices (a runtime e ^ stride would put v in local memory)
        if (stride == 1) in_thread_stage<E, 1>(v, t, size);
        else if (stride == 2) in_thread_stage<E, 2>(v, t, size);
        else if (stride == 4) in_thread_stage<E, 4>(v, t, size);
      } else if (stride < 32 * E) {
        const int pt = stride / E;  // partner lane distance
        const bool lower = (t & pt) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = shfl_xor_u64(v[e], pt);
          const bool desc = (((t * E + e) & size) == 0);
          const bool keep_max = lower == desc;
          v[e] = keep_max ? (v[e] > o ? v[e] : o) : (v[e] < o ? v[e] : o);
        }
      } else {
        if (t < nthreads) {
#pragma unroll
          for (int e = 0; e < E; ++e) buf[t * E + e] = v[e];
        }
        __syncthreads();
        if (t < nthreads) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = t * E + e, l = i ^ stride;
            const uint64_t o = buf[l];
            const bool desc = ((i & size) == 0);
            const bool keep_max = (i < l) == desc;
            v[e] = keep_max ? (v[e] > o ? v[e] : o) : (v[e] < o ? v[e] : o);
          }
        }
        __syncthreads();
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void sort_shared_e(uint64_t* keys, int n) {
  const int used = n / E;  // threads holding keys: min(n, blockDim.x), a multiple of 32
  uint64_t v[E];
  if ((int)threadIdx.x < used) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = keys[threadIdx.x * E + e];
  }
  __syncthreads();
  reg_bitonic_desc<E>(v, used, keys);
  if ((int)threadIdx.x < used) {
#pragma unroll
    for (int e = 0; e < E; ++e) keys[threadIdx.x * E + e] = v[e];
  }
  __syncthreads();
}

// Sort the n (power of two, 16 <= n <= 8 * blockDim.x) keys of the shared array keys[] in
// place, descending, with the whole block (blockDim.x a power of two >= 64; every thread
// must call it).  keys[] doubles as the exchange buffer: exactly n entries are touched.
__device__ __forceinline__ void block_sort_desc(uint64_t* keys, int n) {
  const int T = blockDim.x;
  if (n <= 64) {  // one warp, no barrier inside the sort
    if (threadIdx.x < 32) {
      uint64_t v[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = threadIdx.x * 2 + e;
        v[e] = i < n ? keys[i] : 0ull;
      }
      reg_bitonic_desc<2>(v, 32, nullptr);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = threadIdx.x * 2 + e;
        if (i < n) keys[i] = v[e];
      }
    }
    __syncthreads();
    return;
  }
  if (n <= T) sort_shared_e<1>(keys, n);
  else if (n <= 2 * T) sort_shared_e<2>(keys, n);
  else if (n <= 4 * T) sort_shared_e<4>(keys, n);
  else sort_shared_e<8>(keys, n);
}

// Rank of v among the n keys src[0, n) (shared memory): how many are strictly larger.  One
// broadcast load per key, no barrier — a bitonic sort of a few hundred keys is a chain of
// ~40 dependent shuffle/compare stages (5 K cycles for 256 keys, 3.7 K for ~150:
// profiles/microbench/merge_bench.cu), while ranking them all is ~n independent compares per
// thread.
__device__ __forceinline__ int rank_desc(const uint64_t* __restrict__ src, int n, uint64_t v) {
  int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  int j = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {  // 16-byte broadcast loads, 8 keys ahead
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
    for (; j + 8 <= n; j += 8) {
      const ulonglong2 a = s2[(j >> 1)], b = s2[(j >> 1) + 1], c = s2[(j >> 1) + 2],
                       d = s2[(j >> 1) + 3];
      r0 += (a.x > v) + (a.y > v);
      r1 += (b.x > v) + (b.y > v);
      r2 += (c.x > v) + (c.y > v);
      r3 += (d.x > v) + (d.y > v);
    }
  }
  for (; j + 4 <= n; j += 4) {
    r0 += src[j] > v;
    r1 += src[j + 1] > v;
    r2 += src[j + 2] > v;
    r3 += src[j + 3] > v;
  }
  for (; j < n; ++j) r0 += src[j] > v;
  return r0 + r1 + r2 + r3;
}

// Rank selection: src[0, n) holds n DISTINCT nonzero keys (shared memory, n <= 2 * blockDim.x);
// emit(r, key) is called for each of the min(n, k) largest with its descending position r.
// Whole block or any subset of it (no barrier inside: the caller orders src's writes before
// and emit's results after).
template <typename Emit>
__device__ __forceinline__ void rank_topk_block(const uint64_t* __restrict__ src, int n, int k,
                                                Emit&& emit) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t v = src[i];
    const int r = rank_desc(src, n, v);
    if (r < k) emit(r, v);
  }
}

}  // namespace vx
