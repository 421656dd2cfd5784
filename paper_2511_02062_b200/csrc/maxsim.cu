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
#include "vx_ptx.cuh"

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
  uint64_t kt_c0 = 0, kt_g0 = 0;
  ktimer_begin(a.ktimer, kt_c0, kt_g0);
  const int64_t id = a.cand[(size_t)b * a.C + c];
  if (id < 0 || id < a.id_lo || id >= a.id_hi) {  // no candidate / another shard's
    if (threadIdx.x == 0) a.out[(size_t)b * a.C + c] = -INFINITY;
    ktimer_end(a.ktimer, kt_c0, kt_g0);
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
    // four query tokens at a time: four independent in-order chains per thread (each dot
    // product is still the oracle's single chain over t)
    for (int i0 = 0; i0 < nq; i0 += 4) {
      float acc[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      if (j < Nd) {
        const float* dr = d_s + j * DS;
        const float* qr = q_s + i0 * d;
        const int ni = nq - i0 < 4 ? nq - i0 : 4;
        float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
        if (ni == 4) {
          for (int t = 0; t < d; ++t) {
            const float x = dr[t];
            a0 = fmaf(qr[t], x, a0);
            a1 = fmaf(qr[d + t], x, a1);
            a2 = fmaf(qr[2 * d + t], x, a2);
            a3 = fmaf(qr[3 * d + t], x, a3);
          }
        } else {
          for (int t = 0; t < d; ++t) {
            const float x = dr[t];
            a0 = fmaf(qr[t], x, a0);
            if (ni > 1) a1 = fmaf(qr[d + t], x, a1);
            if (ni > 2) a2 = fmaf(qr[2 * d + t], x, a2);
          }
        }
        acc[0] = a0;
        acc[1] = ni > 1 ? a1 : -INFINITY;
        acc[2] = ni > 2 ? a2 : -INFINITY;
        acc[3] = ni > 3 ? a3 : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u >= nq) break;
        float m = acc[u];
        // max over the doc tokens of this warp; each warp owns its row of wm
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wm[warp * nq + i0 + u] = fmaxf(wm[warp * nq + i0 + u], m);
      }
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
  ktimer_end(a.ktimer, kt_c0, kt_g0);
}

// The fp32 token store (VX_FLAG_TOKENS_F32): exact fp32 MaxSim with a register tile.  One CTA
// per (candidate, query), 128 threads: thread = 4 query tokens (ig = tid / 16, tokens 4 ig + v)
// x 8 doc tokens (jg = tid % 16, tokens jg + 16 u: consecutive lanes read consecutive rows,
// conflict-free with the 4-float row padding), 32 accumulators, each an in-order fmaf chain over
// t (float4 steps of the shared rows) — bit-identical to the oracle's VXO_F32 over the fp32
// table; 8 independent chains per query token hide the FMA latency and each LDS.128 feeds 8
// (doc) or 4 (query) FMAs.  The max over doc tokens is a 16-lane shuffle max, the sum over
// query tokens runs in order on one thread.
constexpr int kMsF32Threads = 128;
__global__ void __launch_bounds__(kMsF32Threads)
    maxsim_f32_kernel(const MaxSimArgs a) {
  extern __shared__ __align__(16) float smf[];
  const int b = blockIdx.y, c = blockIdx.x;
  const int nq = a.nq, d = a.d, Nd = a.Nd;
  const int RS = d + 4;                    // padded row (16-byte aligned)
  float* q_s = smf;                        // [32][RS] (rows >= nq zero)
  float* d_s = q_s + 32 * RS;              // [128][RS] (rows >= Nd zero)
  float* best = d_s + 128 * RS;            // [32]
  uint64_t kt_c0 = 0, kt_g0 = 0;
  ktimer_begin(a.ktimer, kt_c0, kt_g0);
  const int64_t id = a.cand[(size_t)b * a.C + c];
  if (id < 0 || id < a.id_lo || id >= a.id_hi) {
    if (threadIdx.x == 0) a.out[(size_t)b * a.C + c] = -INFINITY;
    ktimer_end(a.ktimer, kt_c0, kt_g0);
    return;
  }
  const float4* qt = reinterpret_cast<const float4*>(a.qtok + (size_t)b * nq * d);
  const float4* dt = reinterpret_cast<const float4*>(a.table32 + (size_t)(id % a.T) * Nd * d);
  const int d4 = d >> 2;
  // staging: eight 16-byte loads in flight per thread before their stores (a load-store loop
  // waited one global latency per 16 bytes: 40 round trips for a 64 KB block)
  auto stage = [&](const float4* __restrict__ src, float* dst, int rows, int valid) {
    const int n = rows * d4;
    for (int i0 = 0; i0 < n; i0 += 8 * (int)blockDim.x) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
        const int r = i / d4;
        v[u] = (i < n && r < valid) ? src[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * (int)blockDim.x + (int)threadIdx.x;
        if (i < n) {
          const int r = i / d4, t4 = i - r * d4;
          *reinterpret_cast<float4*>(dst + r * RS + 4 * t4) = v[u];
        }
      }
    }
  };
  stage(qt, q_s, 32, nq);
  stage(dt, d_s, 128, Nd);
  __syncthreads();
  const int ig = threadIdx.x >> 4, jg = threadIdx.x & 15;
  float acc[4][8];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[v][u] = 0.0f;
  for (int t = 0; t < d; t += 4) {
    float4 qv[4], dv[8];
#pragma unroll
    for (int v = 0; v < 4; ++v) qv[v] = *reinterpret_cast<const float4*>(q_s + (4 * ig + v) * RS + t);
#pragma unroll
    for (int u = 0; u < 8; ++u) dv[u] = *reinterpret_cast<const float4*>(d_s + (jg + 16 * u) * RS + t);
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[v][u] = fmaf(qv[v].x, dv[u].x, acc[v][u]);
        acc[v][u] = fmaf(qv[v].y, dv[u].y, acc[v][u]);
        acc[v][u] = fmaf(qv[v].z, dv[u].z, acc[v][u]);
        acc[v][u] = fmaf(qv[v].w, dv[u].w, acc[v][u]);
      }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    float m = -INFINITY;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (jg + 16 * u < Nd) m = fmaxf(m, acc[v][u]);
    // the 16 lanes of this query-token group (lane bits 0-3)
    for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (jg == 0) best[4 * ig + v] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float total = 0.0f;
    for (int i = 0; i < nq; ++i) total += best[i];
    a.out[(size_t)b * a.C + c] = total;
  }
  ktimer_end(a.ktimer, kt_c0, kt_g0);
}

cudaError_t launch_maxsim_f32(const MaxSimArgs& a, cudaStream_t st) {
  if (a.B <= 0 || a.C <= 0) return cudaSuccess;
  if (a.nq > 32 || a.Nd > 128 || (a.d & 3) || !a.table32 || !a.qtok) return cudaErrorInvalidValue;
  const size_t smem = sizeof(float) * ((size_t)(32 + 128) * (a.d + 4) + 32);
  cudaError_t e = cudaFuncSetAttribute(maxsim_f32_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.C, a.B);
  maxsim_f32_kernel<<<grid, kMsF32Threads, smem, st>>>(a);
  return cudaGetLastError();
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
