// merge_bench.cu — times K3 (merge_topk_kernel, topk.cu) alone with CUDA events: B queries x
// M = P*KC sorted-per-list coarse keys -> top k', the shapes of the small-batch stage.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../../paper_2511_02062_b200/csrc merge_bench.cu -o merge_bench
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2511_02062_b200/csrc/topk.cu"

__global__ void empty_kernel() {}

int main() {
  struct Case { int B, P, KC, k; };
  const Case cases[] = {{16, 148, 16, 64}, {16, 148, 32, 1024}, {1024, 74, 32, 1024}, {16, 148, 16, 10}};
  for (const Case& c : cases) {
    const int M = c.P * c.KC;
    std::vector<uint64_t> h((size_t)c.B * M);
    std::mt19937_64 rng(1);
    std::normal_distribution<float> nd(0.f, 0.036f);
    for (int b = 0; b < c.B; ++b)
      for (int p = 0; p < c.P; ++p) {
        std::vector<uint64_t> l(c.KC);
        for (int j = 0; j < c.KC; ++j) {
          float s = std::fabs(nd(rng)) + 0.1f;
          l[j] = vx_make_key(s, (uint32_t)(rng() % 100000));
        }
        std::sort(l.rbegin(), l.rend());
        for (int j = 0; j < c.KC; ++j) h[((size_t)b * c.P + p) * c.KC + j] = l[j];
      }
    uint64_t *din, *dout;
    cudaMalloc(&din, h.size() * 8);
    cudaMalloc(&dout, (size_t)c.B * c.k * 8);
    cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, z;
    cudaEventCreate(&a);
    cudaEventCreate(&z);
    for (int w = 0; w < 3; ++w) vx::launch_merge_topk(din, c.B, M, c.k, 0, dout, nullptr, nullptr, 0);
    const int it = 50;
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < it; ++i) vx::launch_merge_topk(din, c.B, M, c.k, 0, dout, nullptr, nullptr, st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(z, st);
    cudaEventSynchronize(z);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, z);
    printf("merge B=%d M=%d (P=%d x KC=%d) -> k'=%d: %.2f us/launch (%s)\n", c.B, M, c.P, c.KC, c.k,
           ms * 1e3 / it, cudaGetErrorString(cudaGetLastError()));
    cudaFree(din);
    cudaFree(dout);
  }
  {  // calibration: an empty kernel per graph node
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 50; ++i) empty_kernel<<<16, 256, 0, st>>>();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaEvent_t a, z;
    cudaEventCreate(&a);
    cudaEventCreate(&z);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(z, st);
    cudaEventSynchronize(z);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, z);
    printf("empty kernel in a graph: %.2f us/node\n", ms * 1e3 / 50);
  }
  return 0;
}
