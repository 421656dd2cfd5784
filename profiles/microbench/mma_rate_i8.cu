// mma_rate_i8.cu — tcgen05.mma throughput, kind::f16 (bf16 x bf16 -> f32, K=16 per MMA) vs
// kind::i8 (s8 x s8 -> s32, K=32 per MMA), M=128 (cta_group::1) x N=256, SS operands.  One
// warp per CTA walks the loop (warp-uniform state) and an elected lane issues 4 MMAs per
// iteration on resident smem; one commit at the end.  Prints cycles per MMA and the SM clock.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../../paper_2511_02062_b200/csrc mma_rate_i8.cu -o mma_rate_i8
#include <cstdio>
#include <vector>

#include "vx_ptx.cuh"

using namespace vx;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
               "r"(idesc), "r"(acc) : "memory");
}
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <bool I8>
__global__ void __launch_bounds__(128, 1) kern(int iters, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    reinterpret_cast<uint32_t*>(smem)[i] = I8 ? (h & 0x7f7f7f7fu) : (0x3c003c00u | (h & 0x03ff03ffu));
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  const int warp = warp_idx_uniform();
  if (warp == 0) tmem_alloc(slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  uint64_t c0 = clock64(), t0 = gtimer();
  if (warp == 0) {
    constexpr uint32_t idesc = I8 ? idesc_i8(128, 256) : make_idesc(1u, 128u, 256u);
    const uint64_t a0 = umma_desc_sw128(smem_u32(smem)), b0 = umma_desc_sw128(smem_u32(smem + 16384));
    for (int it = 0; it < iters; ++it) {
      __syncwarp();
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (I8) mma_i8(tmem, a0 + 2 * j, b0 + 2 * j, idesc, j != 0);
          else mma_f16_ss(tmem, a0 + 2 * j, b0 + 2 * j, idesc, j != 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(bar);
    __syncwarp();
  }
  if (threadIdx.x == 0) mbar_wait(bar, 0);
  uint64_t c1 = clock64(), t1 = gtimer();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = c1 - c0;
    out[blockIdx.x * 2 + 1] = t1 - t0;
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

template <bool I8>
static void run(int iters) {
  const int smem = 16384 + 32768 + 64 + 1024, grid = 148;
  cudaFuncSetAttribute(kern<I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, grid * 16);
  for (int rep = 0; rep < 3; ++rep) {
    kern<I8><<<grid, 128, smem>>>(iters, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return; }
    std::vector<unsigned long long> h(grid * 2);
    cudaMemcpy(h.data(), d, grid * 16, cudaMemcpyDeviceToHost);
    double cyc = 0, ns = 0;
    for (int i = 0; i < grid; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
    cyc /= grid; ns /= grid;
    const double mma = 4.0 * iters, k = I8 ? 32 : 16;
    const double ops = 2.0 * 128 * 256 * k * mma * grid;
    printf("%s: %.1f cyc/MMA (M=128 N=256 K=%d) at %.0f MHz -> %.0f T(FL)OP/s\n", I8 ? "kind::i8 " : "kind::f16",
           cyc / mma, (int)k, cyc / ns * 1e3, ops / (ns * 1e-9) / 1e12);
  }
  cudaFree(d);
}

int main() {
  run<false>(100000);
  run<true>(100000);
  run<false>(100000);
  run<true>(100000);
  return 0;
}
