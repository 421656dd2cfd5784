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
                                  int64_t n, int D) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t r = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * wpb) {
    int64_t ss = 0;
    for (int c = lane; c < D; c += 32) {
      int64_t v = vx_synth_int(seed, (uint64_t)(row0 + r), (uint64_t)c);
      ss += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    OutT* o = out + r * (int64_t)D;
    for (int c = lane; c < D; c += 32) {
      float x = vx_synth_finish(vx_synth_int(seed, (uint64_t)(row0 + r), (uint64_t)c), ss);
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
                              cudaStream_t st) {
  synth_rows_kernel<float, false><<<fill_grid(n), 256, 0, st>>>(out, seed, row0, n, D);
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
