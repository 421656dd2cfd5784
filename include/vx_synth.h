/*
 * vx_synth.h — counter-based synthetic data generator shared bit-for-bit by
 * the CUDA product (device fill of the index / token store) and the CPU oracle.
 *
 * Why a shared generator: the index at the BASELINE configs is 0.3–31 GB, so
 * the GPU fills it in place instead of uploading it, and the oracle must see the
 * identical fp32 bits to make a bit-exact top-k id comparison meaningful.
 *
 * Definition (all integer arithmetic until one fp64 divide per element, so the
 * result is identical on any IEEE-754 host or device):
 *   h(seed,row,col) = splitmix64(splitmix64(seed*PHI + row) ^ (col*C2))
 *   v(seed,row,col) = sum of the four 16-bit limbs of h  - 131070      (Irwin–Hall n=4,
 *                     symmetric, integer in [-131070, 131070], ~N(0, 37837^2))
 *   x(row,col)      = (float)( (double)v / sqrt((double) sum_c v(row,c)^2) )
 * i.e. every row is an L2-normalised direction (the sum of squares is exact in
 * int64: 1024 * 131070^2 < 2^45).  Tokens are the same rows rounded to bf16 with
 * round-to-nearest-even done on the integer bit pattern.
 *
 * Seeds used by the benches/tests: docs 42, queries 43,
 * query tokens 44, doc tokens 45.
 *
 * Distributions (dist): 0 = the isotropic rows above; 1 = ANISOTROPIC — before the
 * normalisation v(row,col) is multiplied by the integer m(col) = (1 + 32 / (1 + col/4)) x
 * (4 if col % 97 == 13 else 1): power-law per-dimension scale (the leading dimensions carry up
 * to 33x the spread of the tail) plus sparse outlier dimensions (x4), the shape of real text
 * embeddings that defeats one quantisation scale per shard.  Still exact integer arithmetic
 * (|v m| < 2^25, sum of squares < 2^61).
 */
#ifndef VX_SYNTH_H_
#define VX_SYNTH_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define VX_HD __host__ __device__ __forceinline__
#else
#define VX_HD static inline
#endif

VX_HD uint64_t vx_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Integer pre-normalisation value of element (row, col). */
VX_HD int32_t vx_synth_int(uint64_t seed, uint64_t row, uint64_t col) {
  uint64_t h = vx_splitmix64(seed * 0x9E3779B97F4A7C15ull + row);
  h = vx_splitmix64(h ^ (col * 0xD1B54A32D192ED03ull));
  int32_t s = (int32_t)(h & 0xFFFFu) + (int32_t)((h >> 16) & 0xFFFFu) +
              (int32_t)((h >> 32) & 0xFFFFu) + (int32_t)(h >> 48);
  return s - 131070;
}

/* Integer column multiplier of distribution dist (see the header comment). */
VX_HD int32_t vx_synth_mult(uint32_t dist, uint64_t col) {
  if (dist == 0) return 1;
  const int32_t m = 1 + (int32_t)(32u / (1u + (uint32_t)(col / 4u)));
  return (col % 97u == 13u) ? 4 * m : m;
}

VX_HD int32_t vx_synth_int_d(uint64_t seed, uint64_t row, uint64_t col, uint32_t dist) {
  return vx_synth_int(seed, row, col) * vx_synth_mult(dist, col);
}

/* Final fp32 element given the row's exact integer sum of squares. */
VX_HD float vx_synth_finish(int32_t v, int64_t sumsq) {
  if (sumsq == 0) return 0.0f;
  double nrm = sqrt((double)sumsq);
  return (float)((double)v / nrm);
}

/* fp32 -> bf16 bits, round-to-nearest-even on the bit pattern (no NaN inputs). */
VX_HD uint16_t vx_f32_to_bf16_bits(float f) {
  union { float f; uint32_t u; } c;
  c.f = f;
  uint32_t u = c.u;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

VX_HD float vx_bf16_bits_to_f32(uint16_t b) {
  union { float f; uint32_t u; } c;
  c.u = ((uint32_t)b) << 16;
  return c.f;
}

/* Score -> order-preserving uint32 (larger float => larger key). */
VX_HD uint32_t vx_order_f32(float f) {
  union { float f; uint32_t u; } c;
  c.f = f;
  return (c.u & 0x80000000u) ? ~c.u : (c.u | 0x80000000u);
}

VX_HD float vx_unorder_f32(uint32_t k) {
  union { float f; uint32_t u; } c;
  c.u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return c.f;
}

/* Top-k sort key: score descending, then id ascending, as ONE descending u64.
 * ids are 32-bit (an index shard or a whole index < 2^32 documents). */
VX_HD uint64_t vx_make_key(float score, uint32_t id) {
  return ((uint64_t)vx_order_f32(score) << 32) | (uint64_t)(0xFFFFFFFFu - id);
}
VX_HD float vx_key_score(uint64_t key) { return vx_unorder_f32((uint32_t)(key >> 32)); }
VX_HD uint32_t vx_key_id(uint64_t key) { return 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu); }

#endif /* VX_SYNTH_H_ */
