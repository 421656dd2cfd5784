// gather_bench.cu — the HBM ceiling of the exact re-rank's access pattern: random whole rows
// of a 10M x 768 fp32 matrix (3 KB each), B = 1024 queries x R rows, no arithmetic.
//   ring  : per-thread private rings of S slots x CH bytes filled by cp.async.bulk (the
//           re-rank's ring mode), warp-uniform waits
//   ldg   : warp per row, coalesced 16-byte loads, U rows in flight per warp (registers)
//   seq   : the same bytes read contiguously (the streaming ceiling)
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../../paper_2511_02062_b200/csrc gather_bench.cu -o gather_bench
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "vx_ptx.cuh"

using namespace vx;

constexpr int D = 768;

__global__ void ring_kernel(const float* __restrict__ X, const uint32_t* __restrict__ rows,
                            int nrows, int T, int S, int CH, float* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[4 * 256];
  const int t = threadIdx.x;
  if (t < T)
    for (int i = 0; i < S; ++i) mbar_init(&bars[i * T + t], 1);
  fence_barrier_init();
  __syncthreads();
  if (t >= T) return;
  const int nch = D * 4 / CH;
  // this CTA's rows: [r0, r1); thread t takes rows r0 + t, r0 + t + T, ...
  const int per = (nrows + gridDim.x - 1) / gridDim.x;
  const int r0 = blockIdx.x * per, r1 = min(nrows, r0 + per);
  const int my_rows = r1 - r0 > t ? (r1 - r0 - t + T - 1) / T : 0;
  const int n_items = my_rows * nch;
  const int n_warp = __shfl_sync(0xffffffffu, n_items, 0);
  auto issue = [&](int n) {
    const int r = n / nch, c = n - r * nch;
    const uint32_t row = rows[r0 + t + r * T];
    const int sl = n % S;
    mbar_expect_tx(&bars[sl * T + t], (uint32_t)CH);
    bulk_load(sm + ((size_t)sl * T + t) * (CH + 16), reinterpret_cast<const uint8_t*>(X + (size_t)row * D) + (size_t)c * CH,
              (uint32_t)CH, &bars[sl * T + t]);
  };
  for (int n = 0; n < S - 1 && n < n_items; ++n) issue(n);
  float acc = 0.f;
  for (int n = 0; n < n_warp; ++n) {
    const bool mine = n < n_items;
    if (n + S - 1 < n_items) issue(n + S - 1);
    const int sl = n % S;
    while (!__all_sync(0xffffffffu, !mine || mbar_try_wait(&bars[sl * T + t], (uint32_t)((n / S) & 1)))) {
    }
    if (mine) acc += reinterpret_cast<const float*>(sm + ((size_t)sl * T + t) * (CH + 16))[0];
  }
  if (acc == 12345.f) *sink = acc;
}

// the re-rank's staging (scan_tc.cu rescore): one CTA per query, R threads each stage their
// row's DC-float chunk per item through NB buffers (one mbarrier per buffer, R arrivals), items
// streamed NB - 1 ahead across rounds; `rows_per_q` rows per query; no arithmetic
__global__ void stream_kernel(const float* __restrict__ X, const uint32_t* __restrict__ rows,
                              int rows_per_q, int R, int DC, int NB, float* sink) {
  extern __shared__ __align__(128) float buf[];
  __shared__ __align__(8) uint64_t bars[4];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bars[i], (uint32_t)R);
    fence_barrier_init();
  }
  __syncthreads();
  const uint32_t* myrows = rows + (size_t)blockIdx.x * rows_per_q;
  const int nch = D / DC, RS = DC + 4;
  const int nitems = ((rows_per_q + R - 1) / R) * nch;
  auto issue = [&](int i) {
    if (t < R) {
      const int r = i / nch, c = i - r * nch;
      const int idx = r * R + t;
      const uint32_t bytes = idx < rows_per_q ? (uint32_t)DC * 4u : 0u;
      mbar_expect_tx(&bars[i % NB], bytes);
      if (bytes) bulk_load(buf + ((size_t)(i % NB) * R + t) * RS, X + (size_t)myrows[idx] * D + (size_t)c * DC, bytes, &bars[i % NB]);
    }
  };
  for (int i = 0; i < NB - 1 && i < nitems; ++i) issue(i);
  float acc = 0.f;
  for (int i = 0; i < nitems; ++i) {
    if (i + NB - 1 < nitems) issue(i + NB - 1);
    mbar_wait(&bars[i % NB], (uint32_t)((i / NB) & 1));
    if (t < R) acc += buf[((size_t)(i % NB) * R + t) * RS];
    __syncthreads();
  }
  if (acc == 12345.f) *sink = acc;
}

template <int U>
__global__ void ldg_kernel(const float* __restrict__ X, const uint32_t* __restrict__ rows, int nrows,
                           float* sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int r = gw * U; r < nrows; r += nw * U) {
    float4 v[U][6];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rr = r + u < nrows ? r + u : r;
      const float4* p = reinterpret_cast<const float4*>(X + (size_t)rows[rr] * D);
#pragma unroll
      for (int j = 0; j < 6; ++j) v[u][j] = __ldg(p + lane + 32 * j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 6; ++j) acc += v[u][j].x + v[u][j].w;
  }
  if (acc == 12345.f) *sink = acc;
}

__global__ void seq_kernel(const float4* __restrict__ X, size_t n4, float* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(X + i);
    acc += v.x + v.w;
  }
  if (acc == 12345.f) *sink = acc;
}

int main(int argc, char** argv) {
  const size_t N = 10000000;
  const int B = 1024, R = argc > 1 ? atoi(argv[1]) : 720;
  const int nrows = B * R;
  float* X;
  if (cudaMalloc(&X, N * D * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(X, 0, N * D * 4);
  std::vector<uint32_t> h(nrows);
  std::mt19937 rng(1);
  for (auto& r : h) r = rng() % N;
  uint32_t* rows;
  float* sink;
  cudaMalloc(&rows, nrows * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(rows, h.data(), nrows * 4, cudaMemcpyHostToDevice);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)nrows * D * 4;
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  auto timeit = [&](auto&& fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int i = 0; i < 5; ++i) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(z);
      cudaEventSynchronize(z);
      float ms;
      cudaEventElapsedTime(&ms, a, z);
      best = ms < best ? ms : best;
    }
    return best;
  };
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    struct SC { int R, DC, NB; };
    const SC scs[] = {{64, 192, 2}, {64, 128, 3}, {64, 96, 3}, {32, 384, 2}, {64, 384, 2},
                      {32, 768, 2}, {16, 768, 2}, {128, 96, 2}, {64, 192, 3}, {128, 192, 2},
                      {32, 192, 3}, {64, 64, 4}};
    for (const SC& c : scs) {
      const size_t smem = (size_t)c.NB * c.R * (c.DC + 4) * 4;
      const float ms = timeit([&] {
        stream_kernel<<<B, 256, smem>>>(X, rows, R, c.R, c.DC, c.NB, sink);
      });
      printf("stream R=%3d DC=%3d NB=%d smem=%6zu (%d CTA/SM): %.3f ms %.2f TB/s (%s)\n", c.R, c.DC,
             c.NB, smem, (int)((227 * 1024) / (smem + 1024)), ms, bytes / ms / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  struct RC { int T, S, CH, ctas_per_sm; };
  const RC rcs[] = {{64, 2, 768, 2},  {64, 3, 768, 2},  {64, 4, 512, 2},  {32, 2, 3072, 1},
                    {32, 3, 1536, 1}, {64, 3, 1024, 1}, {128, 3, 512, 1}, {64, 2, 1536, 1},
                    {96, 2, 1024, 1}, {48, 3, 1536, 1}, {64, 3, 768, 1},  {128, 2, 768, 1}};
  for (const RC& c : rcs) {
    const size_t smem = (size_t)c.S * c.T * (c.CH + 16);
    if (smem > 200 * 1024 || (c.ctas_per_sm == 2 && smem > 100 * 1024)) {
      printf("ring T=%d S=%d CH=%d: smem %zu too big\n", c.T, c.S, c.CH, smem);
      continue;
    }
    const int grid = nsm * c.ctas_per_sm;
    const float ms = timeit([&] {
      ring_kernel<<<grid, 256, smem>>>(X, rows, nrows, c.T, c.S, c.CH, sink);
    });
    printf("ring T=%3d S=%d CH=%4d ctas/SM=%d smem=%6zu: %.3f ms %.2f TB/s (%s)\n", c.T, c.S, c.CH,
           c.ctas_per_sm, smem, ms, bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int blocks : {nsm * 4, nsm * 8}) {
    float ms = timeit([&] { ldg_kernel<2><<<blocks, 256>>>(X, rows, nrows, sink); });
    printf("ldg U=2 blocks=%d: %.3f ms %.2f TB/s\n", blocks, ms, bytes / ms / 1e9);
    ms = timeit([&] { ldg_kernel<4><<<blocks, 256>>>(X, rows, nrows, sink); });
    printf("ldg U=4 blocks=%d: %.3f ms %.2f TB/s\n", blocks, ms, bytes / ms / 1e9);
  }
  {
    const float ms = timeit([&] { seq_kernel<<<nsm * 8, 256>>>(reinterpret_cast<const float4*>(X), (size_t)(bytes / 16), sink); });
    printf("seq: %.3f ms %.2f TB/s\n", ms, bytes / ms / 1e9);
  }
  return 0;
}
