// topk.cu — K3: merge of per-CTA (or per-shard) candidate key lists into the
// final per-query top-k, and the MaxSim re-ordering of the stage output.
//
// One CTA per query.  MSB-first radix select over the u64 keys (8-bit digits,
// histogram in smem) narrows to the bin holding the k-th key — usually 2-3 passes
// over the M = P*kcap candidates, staged once into smem (M <= kMergeSmemKeys: every pass
// re-reading them from L2 made each pass a chain of dependent ~0.5 us loads — 14-18 us per
// merge at B = 16, where a few CTAs run alone) — then one collection
// pass gathers exactly k keys and a block bitonic sort orders them
// (score desc, id asc; the key encodes both, vx_synth.h vx_make_key).
// Padding keys (0) rank below every real key and come out as id -1 / -INF.
#include <cuda_runtime.h>
#include <math.h>

#include "vx_internal.cuh"
#include "vx_ptx.cuh"
#include "vx_sort.cuh"
#include "vx_merge.cuh"

namespace vx {

__device__ __forceinline__ void block_bitonic_desc(uint64_t* buf, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc = (lo & size) == 0;
        uint64_t a = buf[lo], b = buf[hi];
        if ((a < b) == desc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kMergeThreads)
    merge_topk_kernel(const uint64_t* __restrict__ in, int M, int64_t ldin, int k, int64_t id_base,
                      uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_ids,
                      float* __restrict__ out_scores, const int* __restrict__ d_count,
                      int64_t ldout, int P, int KC) {
  if (d_count && (int)blockIdx.x >= *d_count) return;  // device-sized batch (cert fallback)
  // dynamic smem: [M] staged keys, then [kMergeFilterKeys] for the sorted-list filter
  extern __shared__ uint64_t staged[];
  __shared__ uint64_t sel[kMaxK];
  const bool st = M <= kMergeSmemKeys && (M & 1) == 0;
  merge_topk_block(in + (size_t)blockIdx.x * ldin, M, k, id_base, out_keys, out_ids, out_scores,
                   blockIdx.x, ldout, st ? staged : nullptr, sel, st ? P : 0, KC,
                   st ? staged + M : nullptr, kMergeFilterKeys);
}

cudaError_t launch_merge_topk(const uint64_t* in, int B, int M, int k, int64_t id_base,
                              uint64_t* out_keys, int64_t* out_ids, float* out_scores,
                              cudaStream_t st, const int* d_count, int64_t ldin,
                              int64_t ldout, int P, int KC) {
  if (k < 1 || k > kMaxK || M < k) return cudaErrorInvalidValue;
  const size_t smem =
      (M <= kMergeSmemKeys && (M & 1) == 0) ? (size_t)(M + kMergeFilterKeys) * 8 : 0;
  static bool attr[64] = {};  // once per device: the largest staging size
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(merge_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (kMergeSmemKeys + kMergeFilterKeys) * 8);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev] = true;
  }
  merge_topk_kernel<<<B, kMergeThreads, smem, st>>>(in, M, ldin > 0 ? ldin : M, k, id_base,
                                                 out_keys, out_ids, out_scores, d_count,
                                                 ldout > 0 ? ldout : k, P, KC);
  return cudaGetLastError();
}

// Stage output order: MaxSim descending, then id ascending.  k <= 256, one CTA per query.
// planes > 1 (sharded phase 2): ms holds `planes` [B][k] arrays (one per shard, -inf where the
// shard does not own the winner) and each score is their max — the max-reduce fused in.
__global__ void __launch_bounds__(256)
    order_by_kernel(const float* __restrict__ ms, const int64_t* __restrict__ ids,
                    const float* __restrict__ ip, int k, int64_t* __restrict__ out_ids,
                    float* __restrict__ out_ip, float* __restrict__ out_ms, int planes,
                    size_t plane_stride) {
  __shared__ uint64_t buf[256];
  __shared__ float s_ip[256], s_ms[256];
  __shared__ int64_t s_id[256];
  int kp = 16;
  while (kp < k) kp <<= 1;
  const size_t base = (size_t)blockIdx.x * k;
  for (int i = threadIdx.x; i < kp; i += blockDim.x) {
    uint64_t key = 0ull;
    if (i < k) {
      int64_t id = ids[base + i];
      float m = ms[base + i];
      for (int g = 1; g < planes; ++g) m = fmaxf(m, ms[(size_t)g * plane_stride + base + i]);
      s_ip[i] = ip[base + i];
      s_ms[i] = m;
      s_id[i] = id;
      // position i is carried in the low bits; ties on MaxSim resolve by id
      // because the IP top-k list is id-unique and we rank (ms desc, id asc).
      if (id >= 0) {
        uint32_t ord = vx_order_f32(m);
        key = ((uint64_t)ord << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)id);
      }
    }
    buf[i] = key;
  }
  __syncthreads();
  block_sort_desc(buf, kp);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    uint64_t key = buf[i];
    if (key == 0ull) {
      out_ids[base + i] = -1;
      out_ip[base + i] = -INFINITY;
      out_ms[base + i] = -INFINITY;
      continue;
    }
    uint32_t id32 = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
    // find the source slot (k <= 256: linear scan of smem)
    int src = 0;
    for (int j = 0; j < k; ++j)
      if (s_id[j] >= 0 && (uint32_t)s_id[j] == id32) {
        src = j;
        break;
      }
    out_ids[base + i] = s_id[src];
    out_ip[base + i] = s_ip[src];
    out_ms[base + i] = s_ms[src];
  }
}

cudaError_t launch_order_by(const float* key_score, const int64_t* ids, const float* ip, int B,
                            int k, int64_t* out_ids, float* out_ip, float* out_ms,
                            cudaStream_t st, int planes, size_t plane_stride) {
  if (k < 1 || k > 256 || planes < 1) return cudaErrorInvalidValue;
  order_by_kernel<<<B, 256, 0, st>>>(key_score, ids, ip, k, out_ids, out_ip, out_ms, planes,
                                     plane_stride);
  return cudaGetLastError();
}

}  // namespace vx

namespace vx {

// ---- device-side handling of tensor-core certificate failures (no host round trip, so the
// whole stage can live in one CUDA graph)

__global__ void cert_scatter_kernel(const int* __restrict__ fidx, const int* __restrict__ fcount,
                                    int k, const uint64_t* __restrict__ fkeys,
                                    const int64_t* __restrict__ fids, const float* __restrict__ fsc,
                                    uint64_t* __restrict__ keys, int64_t* __restrict__ ids,
                                    float* __restrict__ scores) {
  const int i = blockIdx.x;
  if (i >= *fcount) return;
  const size_t dst = (size_t)fidx[i] * k, src = (size_t)i * k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    keys[dst + j] = fkeys[src + j];
    ids[dst + j] = fids[src + j];
    scores[dst + j] = fsc[src + j];
  }
}

__global__ void __launch_bounds__(1024)
    cert_compact_kernel(const int* __restrict__ flags, int B, const float* __restrict__ q, int D,
                        int* __restrict__ fidx, int* __restrict__ fcount, float* __restrict__ fq,
                        cudaGraphConditionalHandle cond, int use_cond) {
  cert_compact_block(flags, B, q, D, fidx, fcount, fq, cond, use_cond);
}

cudaError_t launch_cert_compact(const int* flags, int B, const float* q, int D, int* fidx,
                                int* fcount, float* fq, cudaStream_t st, unsigned long long cond,
                                int use_cond) {
  cert_compact_kernel<<<1, 1024, 0, st>>>(flags, B, q, D, fidx, fcount, fq,
                                          (cudaGraphConditionalHandle)cond, use_cond);
  return cudaGetLastError();
}

cudaError_t launch_cert_scatter(const int* fidx, const int* fcount, int B, int k,
                                const uint64_t* fkeys, const int64_t* fids, const float* fsc,
                                uint64_t* keys, int64_t* ids, float* scores, cudaStream_t st) {
  cert_scatter_kernel<<<B, 128, 0, st>>>(fidx, fcount, k, fkeys, fids, fsc, keys, ids, scores);
  return cudaGetLastError();
}

}  // namespace vx
