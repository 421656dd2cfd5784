// mma_rate.cu — tcgen05.mma issue-rate microbenchmark (bf16, SS operands, fp32 accumulate).
// One CTA per SM (or one CTA pair per TPC); one elected thread issues `iters` MMAs back to
// back on resident smem operands, one commit at the end.  Reports SM cycles (clock64),
// wall ns (%globaltimer) -> the effective SM clock and MAC/clk/SM the tensor core sustains.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../../paper_2511_02062_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vx_ptx.cuh"

using namespace vx;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// mode 0: cta_group::1 M=128 N=NN; mode 1: cta_group::2 M=256 N=NN (cluster of 2)
template <int MODE>
__global__ void __launch_bounds__(192, 1) mma_kernel(int iters, int nn, int nacc, int nld, int cpc, int ns,
                                                     unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;                 // 128 rows x 128 B
  uint8_t* sB = smem + 16384;         // up to 256 rows x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint64_t* full = bar + 1;     // [8]
  uint64_t* empty = full + 8;   // [8]
  uint64_t* dummy = empty + 8;  // [1]
  uint32_t* slot = reinterpret_cast<uint32_t*>(dummy + 1);
  // fill operands with pseudo-random bf16 (finite, |v| < 2)
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    const uint32_t lo = 0x3c00u | (h & 0x3ffu) | ((h >> 10) & 0x8000u);
    const uint32_t hi = 0x3c00u | ((h >> 16) & 0x3ffu) | ((h << 5) & 0x8000u);
    reinterpret_cast<uint32_t*>(smem)[i] = lo | (hi << 16);
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 8; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(dummy, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (MODE == 1) tmem_alloc_pair(slot, 512); else tmem_alloc(slot, 512);
  }
  tc_fence_before();
  if (MODE == 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const bool issuer = MODE == 1 ? (cluster_ctarank() == 0 && threadIdx.x == 128) : threadIdx.x == 128;
  uint64_t c0 = clock64(), t0 = gtimer();
  if (issuer) {
    const uint32_t idesc = make_idesc(1u, MODE == 1 ? 256u : 128u, (uint32_t)nn);
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    int s = 0;
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const int j = it & 3;
      if (ns > 0 && j == 0) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
      }
      const uint32_t d = tmem + (uint32_t)((it >> 2) % nacc) * (uint32_t)nn;
      if (MODE == 1)
        mma_pair(0, d, umma_desc_sw128(a + j * 32), umma_desc_sw128(b + j * 32), idesc, j != 0);
      else
        mma_f16_ss(d, umma_desc_sw128(a + j * 32), umma_desc_sw128(b + j * 32), idesc, j != 0);
      if (j == 3) {
        if (ns > 0) {
          if (MODE == 1) mma_commit_pair(&empty[s], 0x3); else mma_commit(&empty[s]);
          if (++s == ns) { s = 0; ph ^= 1; }
        }
        for (int c = ns > 0 ? 1 : 0; c < cpc; ++c) {
          if (MODE == 1) mma_commit_pair(dummy, 0x3); else mma_commit(dummy);
        }
      }
    }
    if (MODE == 1) mma_commit_pair(bar, 0x3); else mma_commit(bar);
  }
  if (threadIdx.x == 160 && ns > 0 && (MODE == 0 || cluster_ctarank() == 0)) {
    // producer emulation: wait for the stage to drain, re-arm it (no bytes)
    int s = 0;
    uint32_t ph = 0;
    for (int c = 0; c < iters / 4; ++c) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], 0);
      if (++s == ns) { s = 0; ph ^= 1; }
    }
  }
  if (warp < 4 && nld > 0) {
    // concurrent TMEM readers (an epilogue draining the other accumulator buffer)
    uint32_t acc = 0;
    const uint32_t col = tmem + 256u + ((uint32_t)(warp * 32) << 16);
    for (int i = 0; i < nld; ++i) {
      uint32_t r[32];
      tmem_ld32(col + (uint32_t)(i & 7) * 32u, r);
      tmem_ld_wait();
      acc += r[0] ^ r[31];
    }
    if (acc == 0x12345678u) out[0] = 0;
  }
  if (threadIdx.x == 128) mbar_wait(bar, 0);
  uint64_t c1 = clock64(), t1 = gtimer();
  tc_fence_before();
  if (MODE == 1) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 128) {
    out[blockIdx.x * 2] = c1 - c0;
    out[blockIdx.x * 2 + 1] = t1 - t0;
  }
  if (warp == 0) {
    tc_fence_after();
    if (MODE == 1) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
static void run(int nn, int nacc, int iters, int grid, int nld = 0, int cpc = 0, int ns = 0) {
  auto k = mma_kernel<MODE>;
  const int smem = 16384 + 32768 + 256 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, grid * 16);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MODE == 1 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k, iters, nn, nacc, nld, cpc, ns, d);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    if (err != cudaSuccess || e2 != cudaSuccess) {
      printf("error %s / %s\n", cudaGetErrorString(err), cudaGetErrorString(e2));
      exit(1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(grid * 2);
    cudaMemcpy(h.data(), d, grid * 16, cudaMemcpyDeviceToHost);
    double cyc = 0, tns = 0;
    for (int i = 0; i < grid; ++i) {
      cyc += h[2 * i];
      tns += h[2 * i + 1];
    }
    cyc /= grid;
    tns /= grid;
    const double M = MODE == 1 ? 256 : 128;
    const double macs_per_sm = M * nn * 16.0 * iters / (MODE == 1 ? 2 : 1);
    const double sms = grid;
    printf("mode=%d N=%d nacc=%d nld=%d cpc=%d ns=%d iters=%d grid=%d: %.0f cyc %.0f ns -> %.0f MHz, %.1f cyc/mma, "
           "%.0f MAC/clk/SM, %.0f TFLOP/s (event %.3f ms)\n",
           MODE, nn, nacc, nld, cpc, ns, iters, grid, cyc, tns, cyc / tns * 1e3, cyc / iters,
           macs_per_sm / cyc, 2.0 * macs_per_sm * sms / (tns * 1e-9) / 1e12, ms);
  }
  cudaFree(d);
}

int main() {
  const int it = 200000;
  // cpc = commits per 4-MMA chunk; ns = emulated producer ring depth (0 = none)
  run<1>(256, 1, it, 148);
  run<1>(256, 1, it, 148, 0, 1, 0);
  run<1>(256, 1, it, 148, 0, 2, 0);
  run<1>(256, 1, it, 148, 0, 1, 4);
  run<1>(256, 1, it, 148, 0, 2, 4);
  run<1>(256, 1, it, 148, 0, 1, 8);
  run<0>(256, 1, it, 148, 0, 2, 4);
  return 0;
}
