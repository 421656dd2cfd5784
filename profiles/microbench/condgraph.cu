// condgraph.cu — the cost of a graph's tail: a conditional IF node (body skipped) after the
// last kernel, vs. plain kernel nodes.  %globaltimer stamps: s0 (a kernel before the graph on
// the same stream), the graph's own kernels, s1 (a kernel after it).
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 condgraph.cu -o condgraph
#include <algorithm>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void stamp(unsigned long long* out) { *out = gt(); }
// a 148-CTA kernel that stamps at its end (last CTA) and optionally sets the condition
__global__ void work(unsigned long long* out, cudaGraphConditionalHandle h, int set) {
  __shared__ int s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    if (set) cudaGraphSetConditional(h, 0u);
    *out = gt();
  }
}
__global__ void body(int* p) { if (threadIdx.x == 0) p[blockIdx.x] = 1; }

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  unsigned long long* ts;
  int* dp;
  cudaMalloc(&ts, 64 * 8);
  cudaMalloc(&dp, 1 << 20);
  const char* names[] = {"work", "work -> work", "work -> IF(set 0 in kernel){6 kernels}",
                         "work -> IF(default 0){6 kernels}", "work -> IF(set 0){1 kernel}"};
  for (int variant = 0; variant < 5; ++variant) {
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h = 0;
    if (variant >= 2)
      cudaGraphConditionalHandleCreate(&h, g, variant == 3 ? 0u : 1u,
                                       variant == 3 ? cudaGraphCondAssignDefault : 0u);
    cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
    work<<<148, 128, 0, st>>>(ts + 1, h, variant == 2 || variant == 4);
    if (variant == 1) work<<<148, 128, 0, st>>>(ts + 1, h, 0);
    cudaGraph_t body_g = nullptr;
    if (variant >= 2) {
      cudaGraphNode_t node;
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps;
      size_t nd;
      cudaGraph_t cg;
      cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd);
      cudaGraphAddNode(&node, cg, deps, nd, &cp);
      cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies);
      body_g = cp.conditional.phGraph_out[0];
      cudaStream_t bs;
      cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking);
      cudaStreamBeginCaptureToGraph(bs, body_g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
      for (int i = 0; i < (variant == 4 ? 1 : 6); ++i) body<<<16, 128, 0, bs>>>(dp);
      cudaGraph_t tmp;
      cudaStreamEndCapture(bs, &tmp);
    }
    cudaGraph_t gout;
    cudaError_t e = cudaStreamEndCapture(st, &gout);
    cudaGraphExec_t ge;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    if (e != cudaSuccess) {
      printf("%s: %s\n", names[variant], cudaGetErrorString(e));
      cudaGetLastError();
      continue;
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<double> pre, post, ev;
    for (int r = 0; r < 30; ++r) {
      cudaEventRecord(a, st);
      stamp<<<1, 1, 0, st>>>(ts + 0);
      cudaGraphLaunch(ge, st);
      stamp<<<1, 1, 0, st>>>(ts + 2);
      cudaEventRecord(b, st);
      cudaStreamSynchronize(st);
      unsigned long long t[3];
      cudaMemcpy(t, ts, sizeof t, cudaMemcpyDeviceToHost);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 5) {
        pre.push_back((t[1] - t[0]) * 1e-3);
        post.push_back((t[2] - t[1]) * 1e-3);
        ev.push_back(ms * 1e3);
      }
    }
    auto med = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    printf("%-44s stamp -> last kernel end %.2f us | last kernel end -> next stamp %.2f us | event->event %.2f us (%s)\n",
           names[variant], med(pre), med(post), med(ev), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
