// maxsim_tc.cu — K4: fused tensor-core MaxSim (tcgen05 kind::f16, bf16 in / fp32 accumulate)
//   score(q, d) = sum_{i<Nq} max_{j<Nd} <q_i, d_j>          (ColBERT late interaction)
//
// One CTA per (query, chunk of its candidates); 2 CTAs per SM.
//   A = the query's tokens, bf16, M = 128 rows (rows >= Nq are zero), resident in smem for
//       the whole chunk (written once by the CTA, SWIZZLE_128B, K-major);
//   B = one candidate's doc-token block [Nd rows][d] bf16, TMA-streamed from the token store
//       (block = id mod T), NS-stage ring;
//   D = TMEM accumulator [query token (lane)][doc token (column)], double-buffered.
// Epilogue (4 warps): thread = query token; tcgen05.ld its Nd scores, row max in registers,
// warp-sum over query tokens, cross-warp sum in smem -> one fp32 score per candidate.  The
// token x token matrix never leaves the SM.
//
// fp32-faithful query tokens (a.split, nq <= 64): the fp32 tokens the payload carries are
// split into bf16 hi = RNE(q) and lo = RNE(q - hi) (|q - hi - lo| <= 2^-17 |q|; every
// bf16 x bf16 product is exact in fp32).  The A tile has 128 rows and nq <= 64 of them would
// be padding, so the lo rows take the padding: lane quadrant w holds tokens 16w..16w+15, hi
// in its lanes 0-15 and lo in lanes 16-31.  The epilogue adds lane l + 16's accumulator to
// lane l's (one shuffle per column) before the row max, so <hi + lo, d_j> costs no extra MMA
// and no HBM bytes.  Measured vs the fp64 MaxSim of the fp32 tokens: ~1e-6 relative, where
// rounding the query tokens to bf16 alone leaves ~1e-3 (tests/test_gpu_headline.py).
#include <cuda_runtime.h>
#include <math.h>

#include "vx_internal.cuh"
#include "vx_ptx.cuh"

namespace vx {

constexpr int kMsStages = 2;
constexpr int kMsThreads = 6 * 32;  // producer, MMA, 4 epilogue warps

template <int ND, int DK>
struct MsCfg {
  static constexpr int kATile = 128 * 128;                 // one K-block of A: 128 rows x 128 B
  static constexpr int kABytes = DK * kATile;
  static constexpr int kStageBytes = DK * ND * 128;        // one candidate block
  static constexpr int kTmemCols = 2 * ND;                 // double-buffered accumulator
  static constexpr size_t kSmem = (size_t)kABytes + (size_t)kMsStages * kStageBytes +
                                  (2 * kMsStages + 4) * 8 + 2 * 4 * 4 + 16 + 1024;
};

template <int ND, int DK>
__global__ void __launch_bounds__(kMsThreads, 2)
    maxsim_tc_kernel(const __grid_constant__ CUtensorMap tt, const MaxSimArgs a, int chunk,
                     int cpq) {
  using C = MsCfg<ND, DK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (size_t)kMsStages * C::kStageBytes);
  uint64_t* empty = full + kMsStages;
  uint64_t* tfull = empty + kMsStages;
  uint64_t* tempty = tfull + 2;
  float* partial = reinterpret_cast<float*>(tempty + 2);  // [2 bufs][4 quads]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(partial + 8);

  const int warp = warp_idx_uniform(), lane = threadIdx.x & 31;
  const int b = blockIdx.x / cpq;
  const int c0 = (blockIdx.x % cpq) * chunk;
  const int c1 = min(a.C, c0 + chunk);
  const int nq = a.nq;
  const int64_t* cand = a.cand + (size_t)b * a.C;
  uint64_t kt_c0 = 0, kt_g0 = 0;
  ktimer_begin(a.ktimer, kt_c0, kt_g0);
  // candidates another shard owns (or none, id < 0) are skipped by every role: no loads,
  // no MMA, the epilogue writes -INF; the ring advances only over owned candidates
  auto owned = [&](int c) {
    const int64_t id = cand[c];
    return id >= 0 && id >= a.id_lo && id < a.id_hi;
  };

  // A tile: query tokens -> bf16 (RNE), SWIZZLE_128B K-major; rows without a token are zero.
  // Split: row r = 32 w + l holds token 16 w + (l & 15), its hi part for l < 16, lo for l >= 16.
  {
    const float* qt = a.qtok ? a.qtok + (size_t)b * nq * a.d : nullptr;
    const uint16_t* qt16 = a.qtok16 ? a.qtok16 + (size_t)b * nq * a.d : nullptr;
    const int chunks16 = DK * 128 * 8;  // 16-byte chunks in the A tile
    for (int i = threadIdx.x; i < chunks16; i += blockDim.x) {
      const int kb = i / (128 * 8), rem = i % (128 * 8), r = rem >> 3, ch = rem & 7;
      const int tok = a.split ? ((r >> 5) << 4) + (r & 15) : r;
      const int part = a.split ? (r >> 4) & 1 : 0;  // 0: hi (or plain RNE), 1: lo
      uint32_t w[4] = {0, 0, 0, 0};
      if (tok < nq && qt16) {
        const uint16_t* src16 = qt16 + (part ? a.lo_off : 0);
        const uint4 v = *reinterpret_cast<const uint4*>(src16 + (size_t)tok * a.d + kb * 64 + ch * 8);
        w[0] = v.x;
        w[1] = v.y;
        w[2] = v.z;
        w[3] = v.w;
      } else if (tok < nq) {
        const float* src = qt + (size_t)tok * a.d + kb * 64 + ch * 8;
        auto conv = [&](float v) -> uint32_t {
          const uint16_t h = vx_f32_to_bf16_bits(v);
          return part ? vx_f32_to_bf16_bits(v - vx_bf16_bits_to_f32(h)) : h;
        };
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = conv(src[2 * e]) | (conv(src[2 * e + 1]) << 16);
      }
      uint4* dst = reinterpret_cast<uint4*>(sA + kb * C::kATile + r * 128 + ((ch ^ (r & 7)) << 4));
      *dst = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tt);
    for (int s = 0; s < kMsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  fence_proxy_async();  // generic-proxy smem writes (A tile) -> visible to the tensor core
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (int c = c0; c < c1; ++c) {
        if (!owned(c)) continue;
        const int64_t blk = cand[c] % a.T;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], C::kStageBytes);
#pragma unroll
        for (int kb = 0; kb < DK; ++kb)
          tma_load_2d(sB + (size_t)s * C::kStageBytes + kb * ND * 128, &tt, &full[s], kb * 64,
                      (int32_t)(blk * a.Nd), pol);
        if (++s == kMsStages) {
          s = 0;
          ph ^= 1;
        }
      }
      // producer tail: every async commit-arrive on our barriers has landed before exit
      for (int i = 0; i < kMsStages; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        if (++s == kMsStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // whole warp walks the pipeline, one elected lane issues (uniform-datapath descriptors)
    constexpr uint32_t idesc = make_idesc(1u /*BF16*/, 128u, (uint32_t)ND);
    const uint64_t da = umma_desc_sw128(smem_u32(sA));
    const uint64_t db0 = umma_desc_sw128(smem_u32(sB));
    int s = 0, buf = 0;
    uint32_t ph = 0, bph = 0;
    for (int c = c0; c < c1; ++c) {
      if (!owned(c)) continue;
      mbar_wait(&tempty[buf], bph ^ 1);
      mbar_wait(&full[s], ph);
      tc_fence_after();
      __syncwarp();
      if (elect_one()) {
        const uint64_t db = db0 + (uint64_t)(s * (C::kStageBytes >> 4));
#pragma unroll
        for (int kb = 0; kb < DK; ++kb)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            mma_f16_ss(tmem_base + (uint32_t)(buf * ND),
                       da + (uint64_t)(kb * (C::kATile >> 4) + 2 * j),
                       db + (uint64_t)(kb * (ND * 128 >> 4) + 2 * j), idesc,
                       (kb | j) != 0 ? 1u : 0u);
        mma_commit(&empty[s]);
        mma_commit(&tfull[buf]);
      }
      __syncwarp();
      if (++s == kMsStages) {
        s = 0;
        ph ^= 1;
      }
      if (++buf == 2) {
        buf = 0;
        bph ^= 1;
      }
    }
  } else {
    const int quad = warp & 3;
    const bool split = a.split != 0;
    const int tok0 = split ? quad * 16 : quad * 32;  // first token of this lane quadrant
    const bool active = tok0 < nq;  // warp-uniform: does this lane quadrant hold tokens?
    int buf = 0;
    uint32_t bph = 0;
    for (int c = c0; c < c1; ++c) {
      if (!owned(c)) {
        if (warp == 2 && lane == 0) a.out[(size_t)b * a.C + c] = -INFINITY;
        continue;
      }
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
      float mx = -INFINITY;
      if (active) {
        const uint32_t col = tmem_base + (uint32_t)(buf * ND) + ((uint32_t)(quad * 32) << 16);
#pragma unroll
        for (int cc = 0; cc < ND / 32; ++cc) {
          uint32_t r[32];
          tmem_ld32(col + cc * 32, r);
          tmem_ld_wait();
          if (split) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float v = __uint_as_float(r[i]);
              mx = fmaxf(mx, v + __shfl_down_sync(0xffffffffu, v, 16));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(r[i]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      const bool mine = split ? (lane < 16 && tok0 + lane < nq) : (tok0 + lane < nq);
      float v = (active && mine) ? mx : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) partial[buf * 4 + quad] = v;
      named_bar_sync(1, 128);
      if (warp == 2 && lane == 0) {
        const float total = partial[buf * 4 + 0] + partial[buf * 4 + 1] + partial[buf * 4 + 2] +
                            partial[buf * 4 + 3];
        a.out[(size_t)b * a.C + c] = total;
      }
      if (++buf == 2) {
        buf = 0;
        bph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  ktimer_end(a.ktimer, kt_c0, kt_g0);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

template <int ND, int DK>
static cudaError_t launch_ms(const CUtensorMap* tt, const MaxSimArgs& a, cudaStream_t st) {
  using C = MsCfg<ND, DK>;
  auto kfn = maxsim_tc_kernel<ND, DK>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
  if (e != cudaSuccess) return e;
  // CTAs: 2 per SM.  Fewer queries than CTA slots: split each query's candidates into
  // slots / B chunks so the grid is ONE full wave (B = 64, C = 100: 4 x 25 -> 256 CTAs; a
  // ceil(B*C / slots) chunk gave 320 CTAs = 1.08 waves and a 40 % tail).  Otherwise chunks
  // of ~B*C / slots candidates (2..64, at least 2 for the pipeline).
  // Sharded (own_frac = 1/G): chunks are sized by the candidates this shard OWNS, so a CTA
  // still streams ~the same number of blocks and the grid shrinks G-fold (each CTA pays its
  // A-tile build, barrier and TMEM setup once: 2048 CTAs for ~16 owned candidates each at
  // G = 4 spent that setup on 1/4 of the work).
  const int slots = 2 * 148;
  const float of = a.own_frac > 0.f && a.own_frac < 1.f ? a.own_frac : 1.f;
  int chunk;
  if (a.B < slots) {
    const int cpq0 = slots / a.B;
    chunk = (a.C + cpq0 - 1) / cpq0;
  } else {
    const long pairs = (long)((double)a.B * a.C * of + 0.5);
    chunk = (int)((pairs + slots - 1) / slots);
    chunk = chunk > 64 ? 64 : chunk;
    chunk = (int)(chunk / of);  // positions per CTA for `chunk` owned candidates
  }
  chunk = chunk < 2 ? 2 : chunk;
  chunk = chunk > a.C ? a.C : chunk;
  const int cpq = (a.C + chunk - 1) / chunk;
  kfn<<<a.B * cpq, kMsThreads, C::kSmem, st>>>(*tt, a, chunk, cpq);
  return cudaGetLastError();
}

bool maxsim_tc_supported(int nq, int Nd, int d) {  // split additionally needs nq <= 64
  return nq >= 1 && nq <= 128 && (Nd == 64 || Nd == 128 || Nd == 256) && (d == 64 || d == 128);
}

cudaError_t launch_maxsim_tc(const CUtensorMap* tt, const MaxSimArgs& a, cudaStream_t st) {
  if (a.B <= 0 || a.C <= 0) return cudaSuccess;
  if (a.split && a.nq > kMaxSimSplitMaxNq) return cudaErrorInvalidValue;
  if (a.d == 128) {
    if (a.Nd == 128) return launch_ms<128, 2>(tt, a, st);
    if (a.Nd == 64) return launch_ms<64, 2>(tt, a, st);
    if (a.Nd == 256) return launch_ms<256, 2>(tt, a, st);
  } else if (a.d == 64) {
    if (a.Nd == 128) return launch_ms<128, 1>(tt, a, st);
    if (a.Nd == 64) return launch_ms<64, 1>(tt, a, st);
    if (a.Nd == 256) return launch_ms<256, 1>(tt, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace vx
