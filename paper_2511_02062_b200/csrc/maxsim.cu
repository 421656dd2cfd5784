// maxsim.cu — K4: ColBERT/PreFLMR late-interaction re-scoring
//   score(q, d) = sum_{i<Nq} max_{j<Nd} <q_i, d_j>
// for B queries x C candidates, doc tokens bf16 in HBM (token block = id mod T),
// query tokens rounded to bf16, fp32 accumulation.
//
// This file holds the CUDA-core kernel (in-order fp32 FMA chains, bit-identical to
// the oracle's VXO_F32 MaxSim); the tcgen05 tensor-core kernel is maxsim_tc.cu.
#include <cuda_runtime.h>
#include <math.h>

#include "vx_internal.cuh"

namespace vx {

constexpr int kMsThreads = 128;

// One CTA per (candidate, query).  Thread j owns doc token j (Nd <= 128... looped
// for larger Nd); query tokens are broadcast from smem.
__global__ void __launch_bounds__(kMsThreads)
    maxsim_cc_kernel(const MaxSimArgs a) {
  extern __shared__ float sm[];
  const int b = blockIdx.y, c = blockIdx.x;
  const int nq = a.nq, d = a.d, Nd = a.Nd;
  const int DS = d + 1;                   // padded doc-token row (conflict-free)
  float* q_s = sm;                        // [nq][d]
  float* d_s = q_s + nq * d;              // [Nd][d+1]
  float* best = d_s + Nd * DS;            // [nq]
  float* wm = best + nq;                  // [warps][nq] per-warp running max
  const int64_t id = a.cand[(size_t)b * a.C + c];
  if (id < 0 || id < a.id_lo || id >= a.id_hi) {  // no candidate / another shard's
    if (threadIdx.x == 0) a.out[(size_t)b * a.C + c] = -INFINITY;
    return;
  }
  const float* qt = a.qtok ? a.qtok + (size_t)b * nq * d : nullptr;
  const uint16_t* qt16 = a.qtok16 ? a.qtok16 + (size_t)b * nq * d : nullptr;
  for (int i = threadIdx.x; i < nq * d; i += blockDim.x)
    q_s[i] = vx_bf16_bits_to_f32(qt16 ? qt16[i] : vx_f32_to_bf16_bits(qt[i]));
  const uint16_t* dt = a.table + (size_t)(id % a.T) * Nd * d;
  for (int i = threadIdx.x; i < Nd * d; i += blockDim.x) {
    int j = i / d, t = i - j * d;
    d_s[j * DS + t] = vx_bf16_bits_to_f32(dt[i]);
  }
  for (int i = threadIdx.x; i < (int)(blockDim.x >> 5) * nq; i += blockDim.x) wm[i] = -INFINITY;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j0 = 0; j0 < Nd; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    for (int i = 0; i < nq; ++i) {
      float acc = -INFINITY;
      if (j < Nd) {
        acc = 0.0f;
        const float* dr = d_s + j * DS;
        const float* qr = q_s + i * d;
        for (int t = 0; t < d; ++t) acc = fmaf(qr[t], dr[t], acc);
      }
      // max over the doc tokens of this warp; each warp owns its row of wm
      for (int o = 16; o > 0; o >>= 1) acc = fmaxf(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (lane == 0) wm[warp * nq + i] = fmaxf(wm[warp * nq + i], acc);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    float m = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wm[w * nq + i]);
    best[i] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float total = 0.0f;
    for (int i = 0; i < nq; ++i) total += best[i];
    a.out[(size_t)b * a.C + c] = total;
  }
}

cudaError_t launch_maxsim(const MaxSimArgs& a, cudaStream_t st) {
  if (a.B <= 0 || a.C <= 0) return cudaSuccess;
  size_t smem = sizeof(float) * ((size_t)a.nq * a.d + (size_t)a.Nd * (a.d + 1) + (size_t)a.nq * (1 + kMsThreads / 32));
  cudaError_t e = cudaFuncSetAttribute(maxsim_cc_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.C, a.B);
  maxsim_cc_kernel<<<grid, kMsThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vx
