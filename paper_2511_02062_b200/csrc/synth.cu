// synth.cu — in-place fill of the index shard and the token store with the
// counter-based generator of include/vx_synth.h (bit-identical to the oracle:
// integer limbs, exact int64 sum of squares, one IEEE fp64 sqrt + divide).
// One warp per row; the row's sum of squares is an order-independent int64
// warp reduction, so the result does not depend on the launch shape.
#include <cuda_runtime.h>

#include "vx_internal.cuh"

namespace vx {

template <typename OutT, bool kBf16>
__global__ void synth_rows_kernel(OutT* __restrict__ out, uint64_t seed, int64_t row0,
                                  int64_t n, int D, uint32_t dist = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * wpb) {
    int64_t ss = 0;
    for (int c = lane; c < D; c += 32) {
      int64_t v = vx_synth_int_d(seed, (uint64_t)(row0 + r), (uint64_t)c, dist);
      ss += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    OutT* o = out + r * (int64_t)D;
    for (int c = lane; c < D; c += 32) {
      float x = vx_synth_finish(vx_synth_int_d(seed, (uint64_t)(row0 + r), (uint64_t)c, dist), ss);
      if constexpr (kBf16)
        o[c] = vx_f32_to_bf16_bits(x);
      else
        o[c] = x;
    }
  }
}

static int fill_grid(int64_t rows) {
  int64_t blocks = (rows + 7) / 8;
  if (blocks > 148 * 64) blocks = 148 * 64;
  return (int)(blocks < 1 ? 1 : blocks);
}

cudaError_t launch_synth_rows(float* out, uint64_t seed, int64_t row0, int64_t n, int D,
                              cudaStream_t st, uint32_t dist) {
  synth_rows_kernel<float, false><<<fill_grid(n), 256, 0, st>>>(out, seed, row0, n, D, dist);
  return cudaGetLastError();
}

// fp32 -> bf16 (RNE on the bit pattern, vx_synth.h): the coarse-scan shadow of the index
// and the per-batch query copy.  8 elements per thread (two 16-byte loads, one 16-byte store).
__global__ void to_bf16_kernel(const float4* __restrict__ in, uint4* __restrict__ out, int64_t n8) {
  // the scan behind a query conversion is its programmatic dependent (ScanTcArgs::pdl): let it
  // launch now — it waits for this grid's completion before reading anything
  asm volatile("griddepcontrol.launch_dependents;" :::);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = in[2 * i], b = in[2 * i + 1];
    uint4 o;
    o.x = vx_f32_to_bf16_bits(a.x) | ((uint32_t)vx_f32_to_bf16_bits(a.y) << 16);
    o.y = vx_f32_to_bf16_bits(a.z) | ((uint32_t)vx_f32_to_bf16_bits(a.w) << 16);
    o.z = vx_f32_to_bf16_bits(b.x) | ((uint32_t)vx_f32_to_bf16_bits(b.y) << 16);
    o.w = vx_f32_to_bf16_bits(b.z) | ((uint32_t)vx_f32_to_bf16_bits(b.w) << 16);
    out[i] = o;
  }
}

cudaError_t launch_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;  // callers pass rows of D (multiple of 32)
  const int64_t n8 = n / 8;
  int64_t blocks = (n8 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  to_bf16_kernel<<<(int)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in),
                                              reinterpret_cast<uint4*>(out), n8);
  return cudaGetLastError();
}

// fp32 -> (hi, lo) bf16 planes for the fp32-faithful MaxSim operand (maxsim_tc.cu): the
// residual v - hi is exact in fp32, its RNE lo leaves |v - hi - lo| <= 2^-17 |v|.
__global__ void split_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ hi,
                                  uint16_t* __restrict__ lo, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = in[i];
    const uint16_t h = vx_f32_to_bf16_bits(v);
    hi[i] = h;
    lo[i] = vx_f32_to_bf16_bits(v - vx_bf16_bits_to_f32(h));
  }
}

cudaError_t launch_split_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  split_bf16_kernel<<<(int)blocks, 256, 0, st>>>(in, out, out + n, n);
  return cudaGetLastError();
}

// ---- s8 coarse operands.  The index shadow uses ONE scale per shard, sx = max|x| / 127, so
// for a fixed query every document's s32 dot product is in the same units and the scan can
// select on the raw integer; queries use one scale per row, sq = max|q| / 127.  Rounding:
// v8 = clamp(rint(v / s), -127, 127); the certificate bounds the residual v - s * v8.
// Per-column maxima: a block walks rows (coalesced: threads own columns), keeps its columns'
// running |max| in registers (D <= 1024 = 4 per thread) and folds them with one atomicMax
// per column at the end (float bits of non-negative values order like the floats).
__global__ void col_absmax_kernel(const float* __restrict__ in, int64_t n, int D,
                                  unsigned int* __restrict__ colmax_bits) {
  float m[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const float* x = in + r * D;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = threadIdx.x + j * blockDim.x;
      if (c < D) m[j] = fmaxf(m[j], fabsf(x[c]));
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = threadIdx.x + j * blockDim.x;
    if (c < D) atomicMax(&colmax_bits[c], __float_as_uint(m[j]));
  }
}

// per_column: s_c = max|x_c| / 127; else one scale for the shard, s = max_c max|x_c| / 127
// (the default: with queries drawn like the documents, folding per-column scales into the
// query widens its quantisation error more than it narrows the documents' — DESIGN.md §4)
__global__ void col_scale_kernel(const unsigned int* __restrict__ colmax_bits, int D,
                                 float* __restrict__ colscale, int per_column) {
  __shared__ unsigned int s_max;
  if (threadIdx.x == 0) s_max = 0u;
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) atomicMax(&s_max, colmax_bits[c]);
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    const float mx = __uint_as_float(per_column ? colmax_bits[c] : s_max);
    colscale[c] = mx > 0.0f ? mx / 127.0f : 0.0f;
  }
}

__global__ void to_i8_cols_kernel(const float4* __restrict__ in, int64_t n4, int D4,
                                  const float4* __restrict__ colscale, char4* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    const float4 s = colscale[i % D4];
    out[i] = make_char4(s.x > 0.0f ? vx_quant8(v.x, s.x) : 0, s.y > 0.0f ? vx_quant8(v.y, s.y) : 0,
                        s.z > 0.0f ? vx_quant8(v.z, s.z) : 0, s.w > 0.0f ? vx_quant8(v.w, s.w) : 0);
  }
}

cudaError_t launch_to_i8_shadow(const float* in, int64_t n, int D, int8_t* out,
                                unsigned int* colmax_bits, float* colscale, int per_column,
                                cudaStream_t st) {
  if (D % 4 || D > 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(colmax_bits, 0, (size_t)D * 4, st);
  if (e != cudaSuccess) return e;
  int64_t rb = n < 148 * 8 ? n : 148 * 8;
  col_absmax_kernel<<<(int)(rb < 1 ? 1 : rb), 256, 0, st>>>(in, n, D, colmax_bits);
  col_scale_kernel<<<1, 1024, 0, st>>>(colmax_bits, D, colscale, per_column);
  const int64_t n4 = n * D / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  to_i8_cols_kernel<<<(int)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(in), n4, D / 4,
                                                 reinterpret_cast<const float4*>(colscale),
                                                 reinterpret_cast<char4*>(out));
  return cudaGetLastError();
}

// per-row scales (queries), document column scales folded in: one block per row
__global__ void rows_to_i8_kernel(const float* __restrict__ in, int D,
                                  const float* __restrict__ colscale, int8_t* __restrict__ out,
                                  float* __restrict__ scales) {
  asm volatile("griddepcontrol.launch_dependents;" :::);  // as to_bf16_kernel
  __shared__ float s_m[32];
  const float* x = in + (size_t)blockIdx.x * D;
  float m = 0.0f;
  for (int t = threadIdx.x; t < D; t += blockDim.x) m = fmaxf(m, fabsf(x[t] * colscale[t]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? s_m[threadIdx.x] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) s_m[0] = v > 0.0f ? v / 127.0f : 1.0f;
  }
  __syncthreads();
  const float sc = s_m[0];
  if (threadIdx.x == 0) scales[blockIdx.x] = sc;
  for (int t = threadIdx.x; t < D; t += blockDim.x)
    out[(size_t)blockIdx.x * D + t] = vx_quant8(x[t] * colscale[t], sc);
}

cudaError_t launch_rows_to_i8(const float* in, int B, int D, const float* colscale, int8_t* out,
                              float* scales, cudaStream_t st) {
  rows_to_i8_kernel<<<B, 256, 0, st>>>(in, D, colscale, out, scales);
  return cudaGetLastError();
}

cudaError_t launch_synth_tokens(uint16_t* out, uint64_t seed, int64_t blk0, int64_t nblk, int Nd,
                                int d, cudaStream_t st) {
  int64_t rows = nblk * Nd;
  synth_rows_kernel<uint16_t, true><<<fill_grid(rows), 256, 0, st>>>(out, seed, blk0 * Nd, rows,
                                                                     d);
  return cudaGetLastError();
}

}  // namespace vx
