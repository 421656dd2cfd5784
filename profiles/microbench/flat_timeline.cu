// flat_timeline.cu — where the configs[0] step (100K x 768, B = 16, top-10, one captured
// graph per batch) spends the time between its kernels: %globaltimer stamps from one-thread
// kernels on the caller's stream right before and after vx_search_dev, against the library's
// own device-side kernel timers (vx_stats.kt_last_us, origin kt_origin_ns).  L2 flushed before
// every step, as bench.py does.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include \
//          flat_timeline.cu -L../../paper_2511_02062_b200 -lvortex_b200 \
//          -Xlinker -rpath,'$ORIGIN/../../paper_2511_02062_b200' -o flat_timeline
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#include "vortex_b200.h"

__global__ void stamp_kernel(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
__global__ void flush_kernel(int4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_int4((int)i, 0, 0, 0);
}

#define CK(x)                                                              \
  do {                                                                     \
    if ((x) != 0) {                                                        \
      fprintf(stderr, "%s failed: %s\n", #x, vx_last_error());             \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 16, k = 10, D = 768, reps = 20;
  const int64_t N = argc > 2 ? atoll(argv[2]) : 100000;
  vx_index_desc d = {};
  d.n_docs = N;
  d.dim = D;
  d.n_shards = 1;
  d.max_batch = 64;
  d.max_k = 100;
  vx_index* h = nullptr;
  CK(vx_index_create(&d, &h));
  CK(vx_index_synth(h, 42));
  CK(vx_set_option(h, VX_OPT_GRAPHS, 1));
  std::vector<float> q((size_t)B * D);
  std::mt19937 rng(43);
  std::normal_distribution<float> nd(0.f, 1.f);
  for (auto& v : q) v = nd(rng);
  float *dq, *dsc;
  int64_t* dids;
  unsigned long long* ts;
  int4* fl;
  const size_t nfl = (256u << 20) / 16;
  cudaMalloc(&dq, q.size() * 4);
  cudaMalloc(&dsc, (size_t)B * k * 4);
  cudaMalloc(&dids, (size_t)B * k * 8);
  cudaMalloc(&ts, 64 * 8);
  cudaMalloc(&fl, nfl * 16);
  cudaMemcpy(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t ea, eb;
  cudaEventCreate(&ea);
  cudaEventCreate(&eb);
  for (int w = 0; w < 5; ++w) CK(vx_search_dev(h, dq, B, k, dids, dsc, st));
  CK(vx_sync(h));
  std::vector<double> pre, scan, gap, rr, post, tot, ev, bare;
  for (int r = 0; r < reps; ++r) {
    flush_kernel<<<1184, 256, 0, st>>>(fl, nfl);
    stamp_kernel<<<1, 1, 0, st>>>(ts + 2);  // two adjacent stamps: the bare kernel-to-kernel gap
    stamp_kernel<<<1, 1, 0, st>>>(ts + 3);
    cudaEventRecord(ea, st);
    stamp_kernel<<<1, 1, 0, st>>>(ts + 0);
    CK(vx_search_dev(h, dq, B, k, dids, dsc, st));
    stamp_kernel<<<1, 1, 0, st>>>(ts + 1);
    cudaEventRecord(eb, st);
    cudaStreamSynchronize(st);
    CK(vx_sync(h));
    vx_stats s;
    CK(vx_get_stats(h, &s));
    unsigned long long t[4];
    cudaMemcpy(t, ts, sizeof t, cudaMemcpyDeviceToHost);
    float ms = 0;
    cudaEventElapsedTime(&ms, ea, eb);
    const double o = (double)s.kt_origin_ns;
    const double s0 = o + s.kt_last_us[0] * 1e3, s1 = o + s.kt_last_us[1] * 1e3;
    const double r0 = o + s.kt_last_us[8] * 1e3, r1 = o + s.kt_last_us[9] * 1e3;
    pre.push_back((s0 - (double)t[0]) * 1e-3);
    scan.push_back((s1 - s0) * 1e-3);
    gap.push_back((r0 - s1) * 1e-3);
    rr.push_back((r1 - r0) * 1e-3);
    post.push_back(((double)t[1] - r1) * 1e-3);
    tot.push_back((double)(t[1] - t[0]) * 1e-3);
    bare.push_back((double)(t[3] - t[2]) * 1e-3);
    ev.push_back(ms * 1e3);
  }
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  printf("B=%d N=%lld (median of %d, us): stamp->scan start %.2f | scan %.2f | scan end->rerank start %.2f | "
         "rerank %.2f | rerank end->stamp %.2f | stamp->stamp %.2f | event->event %.2f | bare stamp gap %.2f\n",
         B, (long long)N, reps, med(pre), med(scan), med(gap), med(rr), med(post), med(tot), med(ev), med(bare));
  vx_index_destroy(h);
  return 0;
}
