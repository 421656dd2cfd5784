// vx_select.cuh — the per-query candidate selection shared by the tensor-core scan epilogues
// (scan_tc.cu, scan_tc2.cu).  One thread owns one query: it reads the query's accumulator row
// from TMEM 64 columns (= 64 documents) per tcgen05.ld and admits them (as one 64-column unit,
// or two 32-column halves where smem is short) into a register-resident descending list of
// KC order-preserving (score, id) keys.
//
// Fast path: the maxima of the unit's 8-column groups, compared on the raw accumulators
// (s32 for kind::i8: no conversions) against the query's admission threshold (the KC-th best
// key so far) — after the first tiles most units stop here.  Slow path: only the passing
// groups are compared, their passing positions are enumerated from a bit mask and inserted
// with an unrolled compare-exchange network; the raw words are parked in smem scratch (stride
// `ss` words between consecutive columns) so the enumeration can index them.  With 32 queries
// per warp the slow path is warp-divergent and taken by the warp whenever any lane passes,
// so its length, not its frequency per query, is what costs.
#pragma once

#include "vx_ptx.cuh"
#include "vx_synth.h"

#include <limits.h>

#include <type_traits>

namespace vx {

// Accumulator word -> an order-preserving comparable (s32 for kind::i8, fp32 otherwise).
template <int FMT>
struct AccOrd {
  using T = float;
  static VX_DEV T of(uint32_t w) { return __uint_as_float(w); }
  static VX_DEV T thr(float t) { return t; }
  static VX_DEV T mx(T a, T b) { return fmaxf(a, b); }
};
template <>
struct AccOrd<FMT_I8> {
  using T = int;
  static VX_DEV T of(uint32_t w) { return (int)w; }
  // thresholds are scores of admitted keys (exact integers) or -inf
  static VX_DEV T thr(float t) { return t == -INFINITY ? INT_MIN : (int)t; }
  static VX_DEV T mx(T a, T b) { return max(a, b); }
};

// Insert key (> L[KC-1]) into the descending list.  Every position is computed from the old
// list at once — new L[j] = key > L[j] ? (key > L[j-1] ? L[j-1] : key) : L[j] — instead of
// carrying the key through a compare-exchange chain: the same instruction count, but no
// dependency chain (one epilogue warp per SM sub-partition has nothing else to hide it).
template <int KC>
VX_DEV void list_insert(uint64_t (&L)[KC], uint64_t key) {
  bool c[KC];
#pragma unroll
  for (int j = 0; j < KC; ++j) c[j] = key > L[j];
#pragma unroll
  for (int j = KC - 1; j > 0; --j) L[j] = c[j] ? (c[j - 1] ? L[j - 1] : key) : L[j];
  L[0] = c[0] ? key : L[0];
}

// Fill of an EMPTY list (the thread's first unit, no seed): every column passes the -inf
// threshold, and inserting the 32 one by one (a 16-wide insert network each, no ILP between
// them) cost ~7 us at the end of a one-tile scan (VX_DEBUG_SCAN_TRACE, profiles/r02).  Instead
// sort the 32 keys with a register bitonic network (240 compare-exchanges, independent within
// a stage) and keep the best KC.  Same list as the inserts: keys are unique (distinct ids).
template <int FMT, int KC>
VX_DEV void fill_sorted32(const uint32_t* r, uint32_t doc0, uint32_t n_local, uint64_t (&L)[KC]) {
  uint64_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i)
    v[i] = doc0 + i < n_local ? vx_make_key(acc_score<FMT>(r[i]), doc0 + i) : 0ull;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool desc = (i & k) == 0;
          const uint64_t a = v[i], b = v[l];
          const bool sw = desc ? (a < b) : (a > b);
          v[i] = sw ? b : a;
          v[l] = sw ? a : b;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KC; ++j) L[j] = j < 32 ? v[j] : 0ull;
}

// Admit W (32 or 64) consecutive accumulator columns (documents doc0 ..) of this thread's
// query.  scratch: W words per thread, stride ss.
template <int FMT, int KC, int W>
VX_DEV void admit(const uint32_t* r, uint32_t doc0, uint32_t n_local, uint32_t* scratch, int ss,
                  uint64_t (&L)[KC], float& thr) {
  using O = AccOrd<FMT>;
  using T = typename O::T;
  using M = typename std::conditional<W == 64, unsigned long long, uint32_t>::type;
  constexpr int NG = W / 8;
  // maxima of the 8-column groups (independent trees), then of all W
  T gm[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    T m0 = O::mx(O::of(r[8 * g + 0]), O::of(r[8 * g + 1]));
    T m1 = O::mx(O::of(r[8 * g + 2]), O::of(r[8 * g + 3]));
    T m2 = O::mx(O::of(r[8 * g + 4]), O::of(r[8 * g + 5]));
    T m3 = O::mx(O::of(r[8 * g + 6]), O::of(r[8 * g + 7]));
    gm[g] = O::mx(O::mx(m0, m1), O::mx(m2, m3));
  }
  T m = gm[0];
#pragma unroll
  for (int g = 1; g < NG; ++g) m = O::mx(m, gm[g]);
  const T t = O::thr(thr);
  if (m < t) return;
  if constexpr (W == 32 && KC <= 32) {
    if (L[0] == 0ull && thr == -INFINITY) {  // empty, unseeded list: bulk fill
      fill_sorted32<FMT, KC>(r, doc0, n_local, L);
      if (L[KC - 1] != 0ull) thr = vx_key_score(L[KC - 1]);
      return;
    }
  }
  // only the passing groups are compared and parked (warp-divergent: the warp takes this
  // path when any of its 32 queries passes, so it has to stay short)
  M mask = 0;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    if (gm[g] < t) continue;
    uint32_t gmask = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      gmask |= (O::of(r[8 * g + e]) >= t ? 1u : 0u) << e;
      scratch[(8 * g + e) * ss] = r[8 * g + e];
    }
    mask |= (M)gmask << (8 * g);
  }
  bool ins = false;
  while (mask) {
    const int i = (W == 64 ? __ffsll((long long)mask) : __ffs((int)mask)) - 1;
    mask &= mask - 1;
    const uint32_t doc = doc0 + i;
    if (doc >= n_local) break;  // positions are increasing: the rest are padding
    const uint64_t key = vx_make_key(acc_score<FMT>(scratch[i * ss]), doc);
    if (key <= L[KC - 1]) continue;
    list_insert<KC>(L, key);
    ins = true;
  }
  // a list that is not full keeps its threshold (-inf, or the query's seed)
  if (ins && L[KC - 1] != 0ull) thr = vx_key_score(L[KC - 1]);
}

}  // namespace vx
