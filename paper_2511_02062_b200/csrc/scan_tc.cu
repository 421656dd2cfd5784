// scan_tc.cu — K2: tensor-core (tcgen05, kind::tf32) coarse scan of an index shard with a
// fused per-CTA top-16 per query, followed by K2b: exact fp32 re-ranking of the merged
// coarse top-k' with a correctness certificate.
//
// Why: the exact fp32 CUDA-core scan (scan_f32.cu) is shared-memory-bandwidth bound at
// B >= 16 (ncu, profiles/r01); the tensor pipe does the B x N x D contraction ~30x faster,
// so the scan stays HBM-bound up to B ~ 256.  TF32 products are not exact, so the tensor
// pass only SELECTS candidates; every reported score is recomputed exactly (in-order fmaf
// chain, bit-identical to the oracle) and a certificate proves that no document outside
// the candidate set can enter the exact top-k (else the query is re-scanned exactly).
//
// K2 layout (one CTA per SM, persistent over 128-document tiles):
//   A = queries   [QT x 128 rows][32 fp32 per K-chunk]  (TMA, SWIZZLE_128B, L2 evict_last)
//   B = documents [128 rows][32 fp32 per K-chunk]        (TMA, SWIZZLE_128B, L2 evict_first)
//   D = scores in TMEM: lane = query, column = document (fp32), NBUF accumulator buffers
//   warp 0: TMA producer; warp 1: TMEM allocator + single-thread MMA issuer;
//   warps 2..: epilogue — thread = one query: tcgen05.ld its 128 scores of the tile and
//   keep its 16 best (score desc, id asc) in registers (branch-free insertion).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "vx_internal.cuh"
#include "vx_merge.cuh"
#include "vx_ptx.cuh"
#include "vx_select.cuh"
#include "vx_sort.cuh"

namespace vx {

constexpr int kTcStageUnit = 16384;   // one 128-row x 128-byte operand tile
constexpr int kRerankMaxBufs = 4;      // re-rank: chunk buffers in the staging stream
constexpr int kRerankMergeSel = 1024;   // fused merge: selection buffer (k' <= 1024)
constexpr int kRerankMergeFilter = 1024;  // fused merge: sorted-list filter buffer

// QT: 128-query tiles per launch (A operands); TD: documents per tile (MMA N, 128 or 256).
// A bigger TD re-streams the query tiles from L2 half as often per document byte.
template <int QT, int TD>
struct TcCfg {
  static constexpr int EG = QT == 1 ? 1 : 2;                       // epilogue warp groups
  static constexpr int kThreads = (2 + 4 * EG) * 32;
  static constexpr int NBUF = (2 * QT * TD <= 512) ? 2 : 1;         // accumulator buffers
  static constexpr int kTmemCols = NBUF * QT * TD;                  // 256 or 512
  static constexpr int kStageBytes = QT * kTcStageUnit + TD * 128;
  static constexpr int QPT = QT / EG;                               // query tiles per epilogue thread
};

template <int QT, int TD, int FMT, int KC>
__global__ void __launch_bounds__(TcCfg<QT, TD>::kThreads, 1)
    scan_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tx,
                   const ScanTcArgs a) {
  using C = TcCfg<QT, TD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int ns = a.ns;
  // epilogue scratch: the 32 scores of a passing chunk per thread, [32][QT*128] floats
  uint64_t* lists = reinterpret_cast<uint64_t*>(smem + (size_t)ns * C::kStageBytes);
  uint64_t* full = lists + (size_t)QT * 128 * 16;
  uint64_t* empty = full + ns;
  uint64_t* tfull = empty + ns;
  uint64_t* tempty = tfull + C::NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + C::NBUF);

  const int warp = warp_idx_uniform(), lane = threadIdx.x & 31;
  // K-chunk = one 128-byte swizzle atom: 32 fp32 (kind::tf32), 64 bf16 (kind::f16), 128 s8
  constexpr int cw = FMT == FMT_TF32 ? 32 : (FMT == FMT_I8 ? 128 : 64);
  const int nch = a.D / cw;
  const uint32_t n_local = a.n_local;
  const int ntiles = (int)((n_local + TD - 1) / TD);
  uint64_t kt_c0 = 0, kt_g0 = 0;
  if (!a.pdl) ktimer_begin(a.ktimer, kt_c0, kt_g0);
  uint64_t* trc = a.trace ? a.trace + (size_t)blockIdx.x * 16 : nullptr;
  if (trc && threadIdx.x == 0) trc[0] = gtimer_ns();

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tx);
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * C::EG);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // launched early behind the query conversion (ScanTcArgs::pdl): launch, barrier setup and
  // the TMEM allocation overlapped it; nothing below runs before its queries are visible.
  // The device timer then starts here (the kernel's own time, not its wait).
  if (a.pdl) {
    pdl_wait();
    ktimer_begin(a.ktimer, kt_c0, kt_g0);
  }
  if (trc && threadIdx.x == 0) trc[1] = gtimer_ns();
  // the re-rank behind this pass may be scheduled now (it waits for our completion before
  // reading the lists; its prologue — smem carve-out, query norms — overlaps our tail)
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_first();
      const uint64_t pol_q = policy_evict_last();
      const uint32_t bytes = (uint32_t)(QT * a.rep * a.a_rows * 128 + TD * 128);
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], bytes);
          uint8_t* st = smem + (size_t)s * C::kStageBytes;
#pragma unroll
          for (int qt = 0; qt < QT; ++qt)
            tma_load_2d(st + qt * kTcStageUnit, &tq, &full[s], c * cw, qt * 128, pol_q);
          // replicated small batch (QT = 1): the same a_rows query rows again at row offsets
          // r a_rows (the SW128 swizzle is address-based, so every copy is laid out alike)
          for (int r = 1; r < a.rep; ++r)
            tma_load_2d(st + r * a.a_rows * 128, &tq, &full[s], c * cw, 0, pol_q);
#pragma unroll
          for (int h = 0; h < TD; h += 128)  // the document map's box is 128 rows
            tma_load_2d(st + QT * kTcStageUnit + h * 128, &tx, &full[s], c * cw, tile * TD + h,
                        pol_x);
          if (++s == ns) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      // Producer tail: wait until the MMA's commits have released every stage, so no async
      // mbarrier arrive can land in this CTA's smem after it exits (it would corrupt the
      // next kernel resident on the SM).
      for (int i = 0; i < ns; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        if (++s == ns) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected
    // lane issues; loop state warp-uniform -> uniform-datapath descriptors, see scan_tc2.cu)
    constexpr uint32_t idesc = make_idesc_fmt(FMT, 128u, (uint32_t)TD);
    const uint64_t d0 = umma_desc_sw128(smem_u32(smem));
    int s = 0;
    uint32_t ph = 0;
    int buf = 0;
    uint32_t bph = 0;
    bool first = true;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      mbar_wait(&tempty[buf], bph ^ 1);
      tc_fence_after();
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (trc && first && lane == 0) trc[2] = gtimer_ns();
        first = false;
        __syncwarp();
        if (elect_one()) {
          const uint64_t ds = d0 + (uint64_t)(s * (C::kStageBytes >> 4));  // start addr >> 4
#pragma unroll
          for (int qt = 0; qt < QT; ++qt) {
            const uint32_t d = tmem_base + (uint32_t)((buf * QT + qt) * TD);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              mma_ss<FMT>(d, ds + (uint64_t)(qt * (kTcStageUnit >> 4) + 2 * j),
                           ds + (uint64_t)(QT * (kTcStageUnit >> 4) + 2 * j), idesc,
                           (c | j) != 0 ? 1u : 0u);
          }
          mma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == ns) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) mma_commit(&tfull[buf]);
      __syncwarp();
      if (++buf == C::NBUF) {
        buf = 0;
        bph ^= 1;
      }
    }
    if (trc && lane == 0) trc[3] = gtimer_ns();
  } else {
    // ------------------------------------------------ epilogue: thread = query
    const int e = warp - 2;
    const int g = e >> 2;                 // epilogue group
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int m = quad * 32 + lane;       // query row within a 128-query tile
    // Selection (vx_select.cuh): 64 columns per TMEM load, a max filter per 32-column half
    // against the query's admission threshold, rare insertions via smem scratch.
    constexpr int NEPI = 4 * C::EG * 32;
    uint32_t* scratch = reinterpret_cast<uint32_t*>(lists) + (e * 32 + lane);  // [32][NEPI]
    uint64_t L[C::QPT][KC];
#pragma unroll
    for (int t = 0; t < C::QPT; ++t)
#pragma unroll
      for (int j = 0; j < KC; ++j) L[t][j] = 0ull;
    // replicated small batch (rep > 1, QT = 1, TD = 256): row m holds query m % a_rows, its
    // replica m / a_rows selects over columns [replica TD/rep, +TD/rep).  a_rows >= 32: one
    // replica per warp; a_rows = 16: two per warp (lane halves), one 64-column load.
    const int rep = QT == 1 && TD == 256 ? a.rep : 1;
    const int qrow = rep > 1 ? m % a.a_rows : m;
    const int repl = rep > 1 ? m / a.a_rows : 0;
    float thr[C::QPT];
#pragma unroll
    for (int t = 0; t < C::QPT; ++t) {
      const int q = (g + t * C::EG) * 128 + qrow;
      thr[t] = q < a.B ? seed_thr(a.seed, a.seed_ld, q) : -INFINITY;
    }
    int buf = 0;
    uint32_t bph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
      if (trc && warp == 2 && lane == 0) trc[7] = gtimer_ns();  // last tile's accumulator ready
      if (rep > 1) {
        const int q = qrow;
        const uint32_t colq = tmem_base + (uint32_t)(buf * TD) + ((uint32_t)(quad * 32) << 16);
        if (a.a_rows == 16) {
          // warp = replicas 2 quad, 2 quad + 1 (32 columns each): one 64-column load
          uint32_t r[64];
          tmem_ld64(colq + quad * 64, r);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
          const int half = lane >> 4;
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = half ? r[32 + i] : r[i];
          if (q < a.B && !(a.dbg_no_select & 1))
            admit<FMT, KC, 32>(v, (uint32_t)tile * TD + quad * 64 + half * 32, n_local, scratch,
                               NEPI, L[0], thr[0]);
        } else {
          const int cr = TD / rep;  // 64 (rep 4) or 128 (rep 2) columns per replica
#pragma unroll 1
          for (int cc = 0; cc < cr / 64; ++cc) {
            uint32_t r[64];
            tmem_ld64(colq + repl * cr + cc * 64, r);
            tmem_ld_wait();
            if (cc == cr / 64 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[buf]);
            }
            if (q >= a.B || (a.dbg_no_select & 1)) continue;
            const uint32_t doc0 = (uint32_t)tile * TD + repl * cr + cc * 64;
            admit<FMT, KC, 32>(r, doc0, n_local, scratch, NEPI, L[0], thr[0]);
            admit<FMT, KC, 32>(r + 32, doc0 + 32, n_local, scratch, NEPI, L[0], thr[0]);
          }
        }
      } else {
#pragma unroll
      for (int t = 0; t < C::QPT; ++t) {
        const int qt = g + t * C::EG;
        const int q = qt * 128 + m;
        const uint32_t col = tmem_base + (uint32_t)((buf * QT + qt) * TD) +
                             ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
        for (int cc = 0; cc < TD / 64; ++cc) {
          uint32_t r[64];
          tmem_ld64(col + cc * 64, r);
          tmem_ld_wait();
          if (t == C::QPT - 1 && cc == TD / 64 - 1) {
            // last chunk of the buffer in registers: release it before the selection
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
          }
          if (q >= a.B || (a.dbg_no_select & 1)) continue;
          const uint32_t doc0 = (uint32_t)tile * TD + cc * 64;
          admit<FMT, KC, 32>(r, doc0, n_local, scratch, NEPI, L[t], thr[t]);
          admit<FMT, KC, 32>(r + 32, doc0 + 32, n_local, scratch, NEPI, L[t], thr[t]);
        }
      }
      }
      if (++buf == C::NBUF) {
        buf = 0;
        bph ^= 1;
      }
    }
    if (trc && warp == 2 && lane == 0) trc[4] = gtimer_ns();
    if (trc && warp >= 3 && lane == 0) trc[10 + warp] = gtimer_ns();  // [13..15]
    if (rep > 1) {
      // merge each query's rep replica lists into ONE per-CTA list: its KC-th key is >= every
      // replica's KC-th key, so "every document of this CTA outside the list has key <= the
      // list's last key" still holds (certificate 1).  Buffer: the operand ring, idle now
      // (the last tile's MMAs completed before its tfull arrive).
      // rows padded to KC + 1 keys (the 16 merging lanes read distinct banks); the heads of the
      // rep lists stay in registers and only the consumed list's next key is loaded per step
      // (the per-step reload of all rep heads, bank-conflicted, took ~7 us at the end of a
      // one-tile scan — VX_DEBUG_SCAN_TRACE)
      constexpr int MS = KC + 1;
      uint64_t* mb = reinterpret_cast<uint64_t*>(smem);  // [128][KC + 1]
#pragma unroll
      for (int j = 0; j < KC; ++j) mb[m * MS + j] = L[0][j];
      mb[m * MS + KC] = 0ull;  // sentinel past each list's end
      if (trc && threadIdx.x == 128) trc[8] = gtimer_ns();
      named_bar_sync(1, 128);
      if (trc && threadIdx.x == 128) trc[9] = gtimer_ns();
      if (m < a.a_rows && m < a.B) {
        int pos[8];
        uint64_t head[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          pos[r] = 0;
          head[r] = r < rep ? mb[(r * a.a_rows + m) * MS] : 0ull;
        }
        uint64_t* out = a.part + ((size_t)m * gridDim.x + blockIdx.x) * KC;
        // branch-free: the winner's list index selects one refill load (lanes picking different
        // lists diverged into up to 8 serial load paths per step — ~4 us of a one-tile pass)
#pragma unroll 1
        for (int j = 0; j < KC; ++j) {
          uint64_t best = head[0];
          int br = 0;
#pragma unroll
          for (int r = 1; r < 8; ++r) {
            const bool gt = head[r] > best;
            best = gt ? head[r] : best;
            br = gt ? r : br;
          }
          out[j] = best;
          int np = 0;
#pragma unroll
          for (int r = 0; r < 8; ++r) np = r == br ? pos[r] + 1 : np;
          np = min(np, KC);
          const uint64_t nk = mb[(br * a.a_rows + m) * MS + np];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            pos[r] = r == br ? np : pos[r];
            head[r] = r == br ? nk : head[r];
          }
        }
        if (trc && threadIdx.x == 128) trc[10] = gtimer_ns();
      }
    } else {
#pragma unroll
    for (int t = 0; t < C::QPT; ++t) {
      const int qt = g + t * C::EG;
      const int q = qt * 128 + m;
      if (q < a.B) {
        uint64_t* out = a.part + ((size_t)q * gridDim.x + blockIdx.x) * KC;
#pragma unroll
        for (int j = 0; j < KC; ++j) out[j] = L[t][j];
      }
    }
    }
  }
  if (trc && threadIdx.x == 128) trc[11] = gtimer_ns();
  tc_fence_before();
  if (trc && threadIdx.x == 128) trc[12] = gtimer_ns();
  __syncthreads();
  if (trc && threadIdx.x == 0) trc[5] = gtimer_ns();
  if (trc && threadIdx.x == 64) trc[6] = gtimer_ns();
  ktimer_end(a.ktimer, kt_c0, kt_g0);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// Certificate-2 error bound E for one query (see rerank_kernel): qn = |q|, qh = |q^| and
// qr = |q - q^| for the coarse operand q^ of the query (bf16(q), or sq * q8), each already
// inflated for fp32 rounding; xstats = shard maxima [|x|, |bf16 x|, |x - bf16 x|, |sx x8|,
// |x - sx x8|, sx].
__device__ __forceinline__ float cert_err_bound(int fmt, int D, float qn, float qh, float qr,
                                                const float* __restrict__ xstats) {
  float e;
  if (fmt == FMT_TF32) e = kErrCoefTF32 * qn * xstats[0];
  // s8 (column scales s_c folded into the query, q' = q s): with x^ = s x8 and the query's
  // coarse operand q~ = sq q8 / s, q.x - sq (q8.x8) = q.(x - x^) + (q' - sq q8).x8 exactly, so
  // |err| <= |q| max|x - x^| + |q' - sq q8| max|x8|  (qr = |q' - sq q8|, xstats[3] = max|x8|)
  else if (fmt == FMT_I8) e = qn * xstats[4] + qr * xstats[3];
  else e = qh * xstats[2] + qr * xstats[1] + qr * xstats[2];
  const float xmax = fmt == FMT_I8 ? xstats[0] : fmaxf(xstats[0], xstats[1]);
  // fp32 accumulation slack: the exact in-order chain and the tensor core's fp32 sum each
  // err <= ~D 2^-24 |q||x| (2x margin for the tensor core's accumulation rounding): 2^-12
  // covers D <= 1008; longer rows scale it
  const float slack = fmaxf(0.000244140625f, (float)(4 * D + 64) * 5.9604645e-8f);
  return e * 1.001f + slack * fmaxf(qn, qh) * xmax + 1e-30f;
}

// The query's coarse operand q^ (bf16 RNE, or sq * rint(q / sq) for s8 — the same rounding
// as the scan's operands) as squared-norm partial sums: |q|^2, |q^|^2, |q - q^|^2.  The
// whole block reduces into red[0..2] (smem, 3 x 32 floats); also copies q into qs.
__device__ __forceinline__ void query_norms(const float* __restrict__ q, int D, int fmt, float sq,
                                            float* __restrict__ qs, float* red,
                                            const float* __restrict__ xstats) {
  float ss = 0.0f, sh = 0.0f, sr = 0.0f;
  const float* colscale = xstats + kXstatColScale;
  for (int t = threadIdx.x; t < D; t += blockDim.x) {
    const float v = q[t];
    // s8: the residual of q' = q s (the scan's own q8 rounding, rows_to_i8_kernel)
    const float vq = fmt == FMT_I8 ? v * colscale[t] : v;
    const float vh = fmt == FMT_I8 ? sq * (float)vx_quant8(vq, sq)
                                   : vx_bf16_bits_to_f32(vx_f32_to_bf16_bits(v));
    if (qs) qs[t] = v;
    ss = fmaf(v, v, ss);
    sh = fmaf(vh, vh, sh);
    sr = fmaf(vq - vh, vq - vh, sr);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = ss;
    red[32 + (threadIdx.x >> 5)] = sh;
    red[64 + (threadIdx.x >> 5)] = sr;
  }
}
// after a __syncthreads: the three norms (inflated for the fp32 sums: s x8 rounds to fp32, so
// the s8 residual gets 1e-3 of margin, bf16 residuals are exact, Sterbenz)
__device__ __forceinline__ void query_norms_final(const float* red, int fmt, float* qn, float* qh,
                                                  float* qr) {
  float a = 0.0f, b = 0.0f, c = 0.0f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    a += red[w];
    b += red[32 + w];
    c += red[64 + w];
  }
  *qn = sqrtf(a) * 1.0001f;
  *qh = sqrtf(b) * 1.0001f;
  *qr = sqrtf(c) * (fmt == FMT_I8 ? 1.001f : 1.0001f);
}

// ------------------------------------------------------------------- K2b: exact re-rank
// One CTA per query.  cand: the merged coarse top-k' keys (score desc); part: the per-CTA
// lists of K2 (certificate 1); docs/queries fp32.  Writes the exact top-k and flags[b] = 1
// when the certificate fails (the caller re-scans that query with the exact kernel).
//
// Candidate pruning (|exact - cscale c| <= E for every document): the k best coarse
// candidates are re-scored first ("head"); their minimum exact score L is <= the exact k-th,
// so any later candidate with cscale c_j + E < L cannot enter the top-k, and — candidates
// being sorted by coarse key — only the prefix down to cscale c >= L - E is fetched
// ("tail"; 10M x 768 s8, k' = 1024: ~600 of the 1024 rows, where the a-priori bound
// cscale c_k - 2E keeps all of them).  Sharded, tau[b] (the k-th largest of every shard's
// head scores, shard_tau_kernel) <= the GLOBAL exact k-th replaces L when larger, so each
// shard fetches only what can reach the global top-k.
//   phase 0: head + tail in one launch (one shard);
//   phase 1: head only — exact head keys to hkeys[b][k], their scores to lb[b][k];
//   phase 2: tail, from hkeys and tau.
// two CTAs per SM (the staging stream is sized for it): at most 128 registers.  (Three per
// SM — launch bounds 256 x 3 fit in 80 registers without spills — with the staging cut to
// 72 KB per CTA was slower at every split: 0.70-0.86 vs 0.62 ms per 1024-query launch,
// profiles/r02/rerank/three_per_sm.txt.)
__global__ void __launch_bounds__(256, 2)
    rerank_kernel(const float* __restrict__ docs, const float* __restrict__ qv, int D,
                  uint64_t* __restrict__ cand, int kp, const uint64_t* __restrict__ part,
                  int grid, int ldlists, int kc, int k, int64_t row0,
                  const float* __restrict__ xstats, int fmt, const float* __restrict__ qscale,
                  uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_ids,
                  float* __restrict__ out_scores, int* __restrict__ flags, int rows_per_round,
                  int dchunk, int phase, const float* __restrict__ tau, uint64_t* __restrict__ hkeys,
                  float* __restrict__ lb, const uint64_t* __restrict__ seed, int seed_ld,
                  int head_all, int nbuf, const RerankFuse fz) {
  uint64_t* trc = fz.trace ? fz.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (trc && threadIdx.x == 0) trc[0] = gtimer_ns();
  uint64_t kt_c0 = 0, kt_g0 = 0;
  ktimer_begin(fz.ktimer, kt_c0, kt_g0);
  extern __shared__ __align__(16) float rsm[];
  float* qs = rsm;                                             // [D]
  uint64_t* keys = reinterpret_cast<uint64_t*>(rsm + ((D + 3) & ~3));  // [kp]
  float* rowbuf = reinterpret_cast<float*>(keys + kp);         // [2][R][DC+4] row chunks
  __shared__ float s_red[96];
  __shared__ float s_min[8];
  __shared__ int s_fail;
  __shared__ __align__(8) uint64_t s_bar[kRerankMaxBufs];
  const int S = fz.split;  // CTAs per query (RerankFuse::split)
  const int b = blockIdx.x / S, sidx = blockIdx.x - b * S;
  const float* q = qv + (size_t)b * D;
  // coarse keys are in the coarse pass's units: the s8 pass scores sq * sx * (s32 dot)
  const float sq = fmt == FMT_I8 ? qscale[b] : 1.0f;
  const float cscale = fmt == FMT_I8 ? sq * xstats[5] : 1.0f;
  query_norms(q, D, fmt, sq, qs, s_red, xstats);  // the certificate's error bound, below
  // everything below reads the scan's output (lists, candidates, seeds, scales of the query
  // conversion): with programmatic dependent launch this CTA may have started early
  if (trc && threadIdx.x == 0) trc[1] = gtimer_ns();
  pdl_wait();
  if (trc && threadIdx.x == 0) trc[2] = gtimer_ns();
  if (threadIdx.x == 0) {
    s_fail = 0;
    for (int i = 0; i < (nbuf & 15); ++i) mbar_init(&s_bar[i], (uint32_t)rows_per_round);
  }
  if (threadIdx.x == 0) fence_barrier_init();
  __syncthreads();
  float qn, qh, qr;
  query_norms_final(s_red, fmt, &qn, &qh, &qr);
  const float E = cert_err_bound(fmt, D, qn, qh, qr, xstats);
  if (fz.mlists) {  // fused K3: this query's lists -> its coarse top-k' (staged in rowbuf)
    uint64_t* staged = reinterpret_cast<uint64_t*>(rowbuf);
    uint64_t* msel = staged + ((fz.mM + 1) & ~1);
    // the sorted-list filter pays off when its survivors fit one register sort (k' <= 512;
    // at k' = 1024 they never do and the filter's own sort would be wasted)
    const bool filt = fz.filter && kp <= kRerankMergeFilter / 2;
    merge_topk_block(fz.mlists + (size_t)b * fz.mld, fz.mM, kp, 0, cand + (size_t)b * kp, nullptr,
                     nullptr, 0, kp, staged, msel, filt ? grid : 0, kc, msel + kRerankMergeSel,
                     kRerankMergeFilter);
  }
  if (trc && threadIdx.x == 0) trc[3] = gtimer_ns();
  const uint64_t* cb = cand + (size_t)b * kp;
  const uint64_t tprime = cb[kp - 1];  // coarse k'-th key (0: fewer than k' candidates)
  // head rows; head_all (small batch, latency-bound: the pruning saves bytes nobody waits
  // for, and a second gather round costs its full latency) re-scores all k' in one round
  const int kh0 = fz.head > 0 && fz.head < k ? fz.head : k;
  const int kh = head_all ? kp : (kh0 < kp ? kh0 : kp);
  // The candidate rows are random 3 KB gathers from HBM (DRAM-page unfriendly); per-thread
  // loads left too few bytes in flight (measured 85 us at B=128).  Instead each round stages
  // R rows into smem with one TMA bulk copy per row (R x 3 KB in flight per SM), then R
  // threads run the in-order fmaf chains from smem (row stride D+4 floats: the LDS.128 of
  // 8 consecutive lanes hit distinct banks).
  // Rows are staged in DC-float chunks through NB buffers (one mbarrier each, R arrivals):
  // the chunks of all rounds form ONE stream (item i = round i / nch, chunk i % nch), NB - 1
  // items ahead of the chains, across round boundaries — the next round's first chunk is in
  // flight while this round's last one is scored (a double buffer that restarted at every
  // round exposed one full gather latency per 64 rows: ~0.73 of the copy peak).  The
  // accumulators carry across a row's chunks, so the fmaf order is the oracle's.
  // (Per-thread rings and cp.async variants were measured slower: lanes waiting on their own
  // slots diverge, and LDGSTS keeps too few bytes in flight — profiles/r02/README.md.)
  const int R = rows_per_round, DC = dchunk, RS = DC + 4, nch = D / DC, NB = nbuf & 15,
            PF = nbuf >> 4;
  int chunk_no = 0;  // items issued so far (both calls); item i uses buffer / barrier i % NB
  auto rescore = [&](int j0, int j1) {  // exact keys of candidates [j0, j1) into keys[]
    const int t = threadIdx.x;
    const int nitems = ((j1 - j0 + R - 1) / R) * nch;
    const int base = chunk_no;
    auto row_key = [&](int r) -> uint64_t {
      const int idx = j0 + r * R + t;
      return (t < R && idx < j1) ? cb[idx] : 0ull;
    };
    auto issue = [&](int i) {  // item i of this call -> buffer (base + i) % NB
      if (t < R) {
        const int r = i / nch, c = i - r * nch, no = base + i;
        const uint64_t ck = row_key(r);
        const uint32_t bytes = ck ? (uint32_t)DC * 4u : 0u;
        uint64_t* bar = &s_bar[no % NB];
        mbar_expect_tx(bar, bytes);  // every staging thread arrives once (count R)
        if (ck)
          bulk_load(rowbuf + ((size_t)(no % NB) * R + t) * RS,
                    docs + (size_t)vx_key_id(ck) * D + (size_t)c * DC, bytes, bar);
      }
    };
    // L2 prefetch PF items beyond the staging window: the bulk copies then find their lines in
    // L2 (the CTA keeps only NB - 1 chunks in flight in smem — 2 of 8 warps stream, and with a
    // full HBM latency per item the chain warps sat at the barrier half the time, ncu)
    auto prefetch = [&](int i) {
      if (t < R && i < nitems) {
        const int r = i / nch, c = i - r * nch;
        const uint64_t pk = row_key(r);
        if (pk) {
          const float* src = docs + (size_t)vx_key_id(pk) * D + (size_t)c * DC;
          for (int o = 0; o < DC; o += 32) prefetch_l2(src + o);
        }
      }
    };
    for (int i = 0; i < NB - 1 && i < nitems; ++i) issue(i);
    for (int i = NB - 1; i < NB - 1 + PF; ++i) prefetch(i);
    float acc = 0.0f;
    uint64_t ck = 0ull;
    for (int i = 0; i < nitems; ++i) {
      // the buffer item i - 1 used: released by the __syncthreads that closed item i - 1
      if (i + NB - 1 < nitems) issue(i + NB - 1);
      if (PF) prefetch(i + NB - 1 + PF);
      const int r = i / nch, c = i - r * nch, no = base + i;
      if (c == 0) {
        ck = row_key(r);
        acc = 0.0f;
      }
      mbar_wait(&s_bar[no % NB], (uint32_t)((no / NB) & 1));
      if (ck) {
        const float4* x = reinterpret_cast<const float4*>(rowbuf + ((size_t)(no % NB) * R + t) * RS);
        const float4* q4 = reinterpret_cast<const float4*>(qs + (size_t)c * DC);
        for (int u0 = 0; u0 < (DC >> 2); u0 += 8) {  // 8 float4s loaded ahead of 32 fmafs
          float4 xv[8], qv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            xv[u] = x[u0 + u];
            qv[u] = q4[u0 + u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            acc = fmaf(xv[u].x, qv[u].x, acc);
            acc = fmaf(xv[u].y, qv[u].y, acc);
            acc = fmaf(xv[u].z, qv[u].z, acc);
            acc = fmaf(xv[u].w, qv[u].w, acc);
          }
        }
      }
      if (c == nch - 1) {
        const int idx = j0 + r * R + t;
        if (t < R && idx < j1) keys[idx] = ck ? vx_make_key(acc, vx_key_id(ck)) : 0ull;
      }
      __syncthreads();  // this buffer is refilled NB - 1 items later
    }
    chunk_no = base + nitems;
    __syncthreads();  // keys[] complete
  };
  if (phase == 2) {
    for (int i = threadIdx.x; i < kh; i += blockDim.x) keys[i] = hkeys[(size_t)b * k + i];
    __syncthreads();
  } else if (S > 1) {
    // split head: this CTA's slice to ekeys; the query's last CTA continues with all of them
    const int j0 = (int)((int64_t)kh * sidx / S), j1 = (int)((int64_t)kh * (sidx + 1) / S);
    rescore(j0, j1);
    uint64_t* ek = fz.ekeys + (size_t)b * kp;
    for (int i = j0 + threadIdx.x; i < j1; i += blockDim.x) ek[i] = keys[i];
    __shared__ int s_lastq;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();  // this slice before the ticket
      s_lastq = atomicAdd(fz.qctr + b, 1u) == (unsigned)(S - 1);
    }
    __syncthreads();
    if (!s_lastq) {
      ktimer_end(fz.ktimer, kt_c0, kt_g0);
      return;
    }
    __threadfence();  // every slice (each fenced before its ticket)
    for (int i = threadIdx.x; i < kh; i += blockDim.x) keys[i] = ek[i];
    if (threadIdx.x == 0) fz.qctr[b] = 0u;  // re-armed for the next launch (graph replays)
    __syncthreads();
  } else {
    rescore(0, kh);
  }
  if (phase == 1) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const uint64_t key = i < kh ? keys[i] : 0ull;
      hkeys[(size_t)b * k + i] = key;
      lb[(size_t)b * k + i] = key ? vx_key_score(key) : -INFINITY;
    }
    return;
  }
  if (trc && threadIdx.x == 0) trc[4] = gtimer_ns();
  // L = the head's minimum exact score (a bound on the exact k-th once k heads exist); also
  // its smallest key, for the final selection
  // (over the first k candidates only — the k best coarse ones, cand is descending — so that
  // with the whole candidate set as the head (small batch) the selection below still sees
  // ~k + a few survivors, not all k')
  const int kl = kh < k ? kh : k;
  float m = INFINITY;
  uint64_t mk = ~0ull;
  for (int i = threadIdx.x; i < kl; i += blockDim.x) {
    m = fminf(m, keys[i] ? vx_key_score(keys[i]) : -INFINITY);
    mk = keys[i] < mk ? keys[i] : mk;
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const uint64_t y = shfl_xor_u64(mk, o);
    mk = y < mk ? y : mk;
  }
  __shared__ uint64_t s_mk[8];
  if ((threadIdx.x & 31) == 0) {
    s_min[threadIdx.x >> 5] = m;
    s_mk[threadIdx.x >> 5] = mk;
  }
  __syncthreads();
  float L = s_min[0];
  mk = s_mk[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    L = fminf(L, s_min[w]);
    mk = s_mk[w] < mk ? s_mk[w] : mk;
  }
  if (kh < k) L = -INFINITY;
  // the final top-k are all >= the smallest head key when the head holds k real keys (k keys
  // are >= it); otherwise every real key stays in the running
  const uint64_t sel_floor = (kl >= k && mk != 0ull) ? mk : 1ull;
  const float tb = tau ? tau[b] : -INFINITY;
  const float lim = fmaxf(L, tb) - E;
  int kpe = kp;  // candidates re-ranked: the prefix with cscale c >= lim
  if (lim > -INFINITY) {
    int lo = kh, hi = kp;  // first index whose candidate falls below lim (cb is descending)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const uint64_t c = cb[mid];
      if (c != 0ull && vx_key_score(c) * cscale >= lim) lo = mid + 1;
      else hi = mid;
    }
    kpe = lo;
  }
  for (int i = kpe + threadIdx.x; i < kp; i += blockDim.x) keys[i] = 0ull;
  rescore(kh, kpe);
  if (trc && threadIdx.x == 0) trc[5] = gtimer_ns();
  // certificate 1: no CTA that truncated its list (KC kept) had its last key inside the
  // top-k' (sharded: a truncated list whose dropped keys are all bounded below tau is harmless)
  for (int t = threadIdx.x; t < grid; t += blockDim.x) {
    const uint64_t last = part[((size_t)b * ldlists + t) * kc + (kc - 1)];
    if (last != 0ull && (tprime == 0ull || last >= tprime) &&
        !(vx_key_score(last) * cscale + E < tb))
      s_fail = 1;
  }
  __syncthreads();
  // the exact top-k: the keys >= sel_floor (the k head keys and the few tail keys that beat
  // the head's worst: ~k + a few) compacted and ranked into keys[0, k) — a bitonic sort of all
  // k' keys took 8.8 us per CTA at k' = 1024 (VX_DEBUG_RERANK_TRACE); the sort remains the
  // fallback when more than 2 x 256 survive.  (A radix top-k instead, as a second call site of
  // the merge, took the kernel from 80 to 173 registers: one CTA per SM.)
  {
    __shared__ int s_cnt;
    uint64_t* surv = reinterpret_cast<uint64_t*>(rowbuf);  // the staging is drained
    constexpr int kSurvCap = 512;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < kp; i += blockDim.x) {
      const uint64_t key = keys[i];
      if (key >= sel_floor) {
        const int slot = atomicAdd(&s_cnt, 1);
        if (slot < kSurvCap) surv[slot] = key;
      }
    }
    __syncthreads();
    const int C = s_cnt;
    if (C <= kSurvCap && C <= 2 * (int)blockDim.x) {
      rank_topk_block(surv, C, k, [&](int r, uint64_t key) { keys[r] = key; });
      for (int i = C + (int)threadIdx.x; i < k; i += blockDim.x) keys[i] = 0ull;
      __syncthreads();
    } else {
      block_sort_desc(keys, kp);
    }
  }
  if (trc && threadIdx.x == 0) trc[6] = gtimer_ns();
  // seeded scan (ScanTcArgs::seed): the lists also dropped every document whose coarse score
  // is below the seed, so a document outside the candidates has coarse score
  // <= max(s(T'), seed)
  const float sd = seed_thr(seed, seed_ld, b);
  if (threadIdx.x == 0 && (tprime != 0ull || sd > -INFINITY)) {
    // certificate 2: every document outside the candidates has coarse score <= s(T'), so
    // its exact score <= s(T') + E; the exact k-th must beat that bound strictly.
    //   bf16 coarse: with q16 = bf16(q), rq = q - q16 (x16, rx likewise, per shard maxima
    //   from row_stats_kernel), q.x - q16.x16 = q16.rx + rq.x16 + rq.rx, so by Cauchy-Schwarz
    //   |q.x - q16.x16| <= |q16| max|rx| + |rq| max|x16| + |rq| max|rx|: a rigorous bound
    //   from the actual rounding residuals (the worst case 2u|q||x| = 2^-7 |q||x| is ~2x
    //   looser).  TF32 coarse: per-operand truncation <= 2^-10 -> 2^-9 |q| max|x|.
    //   Both: + max(2^-12, (4D+64) 2^-24) |q| max|x| for the fp32 accumulation of the tensor
    //   core and of the exact in-order chain (each <= D 2^-24 relative; cert_err_bound).
    // Sharded: a document outside the candidates is also out of the GLOBAL top-k when its
    // bound is below tau (the shard then reports fewer than k keys, padded with 0).
    const float bound = fmaxf(tprime ? vx_key_score(tprime) : -INFINITY, sd) * cscale + E;
    const uint64_t ek = keys[k - 1];
    if (!(bound < tb) && (ek == 0ull || !(vx_key_score(ek) > bound))) s_fail = 1;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const uint64_t key = keys[i];
    const size_t o = (size_t)b * k + i;
    if (key == 0ull) {
      out_keys[o] = 0ull;
      out_ids[o] = -1;
      out_scores[o] = -INFINITY;
    } else {
      const int64_t gid = (int64_t)vx_key_id(key) + row0;
      out_keys[o] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (uint32_t)gid);
      out_ids[o] = gid;
      out_scores[o] = vx_key_score(key);
    }
  }
  if (threadIdx.x == 0) flags[b] = s_fail;
  if (trc && threadIdx.x == 0) trc[7] = gtimer_ns();
  __syncthreads();
  ktimer_end(fz.ktimer, kt_c0, kt_g0);
  if (fz.ctr) {  // fused compaction: the last CTA of the launch takes the whole batch
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      __threadfence();  // this CTA's flag before its ticket
      s_last = atomicAdd(fz.ctr, 1u) == gridDim.x / S - 1;  // one finishing CTA per query
    }
    __syncthreads();
    if (s_last) {
      __threadfence();  // every other CTA's flag (they fenced before their tickets)
      cert_compact_block(fz.flags_all, fz.Ball, fz.qall, D, fz.fidx, fz.fcount, fz.fq,
                         (cudaGraphConditionalHandle)fz.cond, fz.use_cond);
      if (threadIdx.x == 0) *fz.ctr = 0u;  // re-armed for the next launch (graph replays)
    }
  }
}

// ------------------------------------------------------------------- K2c: wide re-rank
// Second certificate level for the (rare) queries whose k'-candidate certificate failed:
// the per-CTA (per-pair) lists hold more than the k' candidates.  With T'' = the largest
// KC-th key among FULL lists (the deepest truncation point), every document whose coarse key
// is >= T'' is in some list (a document outside its list has key < that list's last key <=
// T''), so re-ranking all list entries >= T'' exactly (up to P x KC rows) and checking
// exact k-th > coarse(T'') + E certifies the query without touching the index again.  T''
// sits ~5-7x deeper than the k'-th candidate, so the gap almost always clears E; queries
// that still fail go on to the exact re-scan.
// Two launches: wide_score_kernel spreads each failing query's rows over S CTAs (one row per
// thread, the in-order fmaf chain of the exact oracle — a row cannot be split across lanes
// without changing the rounding, so rows in flight are what hides the gather latency; one
// CTA per query took ~0.5 ms for 2 queries of a 10M x 768 batch), wide_select_kernel sorts
// and certifies.  Both walk the compacted failing queries i = blockIdx / S, += gridDim / S.

// T'' and the query's list block; every query's lists start at a stride of P_single lists
// (K2 / K2-pairs share it)
__device__ __forceinline__ void wide_lists(const uint64_t* part_all, int b, int B, int GS,
                                           int P_pairs, int P_single, int kc,
                                           const uint64_t** lists, int* P) {
  const int g0 = (b / GS) * GS, Bg = min(GS, B - g0);
  *P = (P_pairs > 0 && Bg > 128) ? P_pairs : P_single;
  *lists = part_all + (size_t)b * P_single * kc;
}
__device__ __forceinline__ uint64_t wide_t2(const uint64_t* lists, int P, int kc,
                                            unsigned long long* s_t2) {
  if (threadIdx.x == 0) *s_t2 = 0ull;
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const uint64_t last = lists[(size_t)p * kc + (kc - 1)];
    if (last) atomicMax(s_t2, (unsigned long long)last);
  }
  __syncthreads();
  return *s_t2;
}

__global__ void __launch_bounds__(256)
    wide_score_kernel(const float* __restrict__ docs, const float* __restrict__ fq, int D,
                      const int* __restrict__ fidx, const int* __restrict__ fcount,
                      const uint64_t* __restrict__ part_all, int B, int GS, int P_pairs,
                      int P_single, int kc, int S, uint64_t* __restrict__ wkeys) {
  extern __shared__ __align__(16) float qs[];  // [D]
  __shared__ unsigned long long s_t2;
  const int n = *fcount, W = gridDim.x / S, s = blockIdx.x % S;
  const int Mmax = P_single * kc;
  for (int i = blockIdx.x / S; i < n; i += W) {
    const int b = fidx[i];
    const uint64_t* lists;
    int P;
    wide_lists(part_all, b, B, GS, P_pairs, P_single, kc, &lists, &P);
    const uint64_t t2 = wide_t2(lists, P, kc, &s_t2);
    for (int t = threadIdx.x; t < D; t += blockDim.x) qs[t] = fq[(size_t)i * D + t];
    __syncthreads();
    const int M = P * kc, chunk = (M + S - 1) / S;
    const int j1 = min(M, (s + 1) * chunk);
    for (int j = s * chunk + threadIdx.x; j < j1; j += blockDim.x) {
      const uint64_t ck = lists[j];
      uint64_t key = 0ull;
      if (ck != 0ull && ck >= t2) {
        const float4* x = reinterpret_cast<const float4*>(docs + (size_t)vx_key_id(ck) * D);
        float acc = 0.0f;
        const int nv = D >> 2;
        // 24 loads in flight, then the in-order chain (8 left every row a chain of 24
        // dependent gathers: 28-49 us for the 2-3 queries of a 10M-row batch)
        for (int c0 = 0; c0 < nv; c0 += 24) {
          float4 v[24];
#pragma unroll
          for (int u = 0; u < 24; ++u)
            if (c0 + u < nv) v[u] = __ldg(x + c0 + u);
#pragma unroll
          for (int u = 0; u < 24; ++u)
            if (c0 + u < nv) {
              const int c = c0 + u;
              acc = fmaf(v[u].x, qs[4 * c + 0], acc);
              acc = fmaf(v[u].y, qs[4 * c + 1], acc);
              acc = fmaf(v[u].z, qs[4 * c + 2], acc);
              acc = fmaf(v[u].w, qs[4 * c + 3], acc);
            }
        }
        key = vx_make_key(acc, vx_key_id(ck));
      }
      wkeys[(size_t)i * Mmax + j] = key;
    }
    __syncthreads();  // qs / s_t2 are reused by the next query
  }
}

__global__ void __launch_bounds__(256)
    wide_select_kernel(const float* __restrict__ fq, int D, const int* __restrict__ fidx,
                       const int* __restrict__ fcount, const uint64_t* __restrict__ part_all,
                       int B, int GS, int P_pairs, int P_single, int kc, int k, int64_t row0,
                       const float* __restrict__ xstats, int fmt,
                       const float* __restrict__ qscale, const uint64_t* __restrict__ wkeys,
                       uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_ids,
                       float* __restrict__ out_scores, int* __restrict__ flags,
                       const uint64_t* __restrict__ seed, int seed_ld) {
  extern __shared__ __align__(16) uint64_t keys[];  // [Mmax (even)] staged keys + [kp2] top-k
  __shared__ float s_red[96];
  __shared__ unsigned long long s_t2;
  __shared__ int s_fail;
  const int n = *fcount;
  const int Mmax = P_single * kc;
  uint64_t* sel = keys + ((Mmax + 1) & ~1);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = fidx[i];
    const uint64_t* lists;
    int P;
    wide_lists(part_all, b, B, GS, P_pairs, P_single, kc, &lists, &P);
    const uint64_t t2 = wide_t2(lists, P, kc, &s_t2);
    const int M = P * kc;
    const float sq = fmt == FMT_I8 ? qscale[b] : 1.0f;
    const float cscale = fmt == FMT_I8 ? sq * xstats[5] : 1.0f;
    query_norms(fq + (size_t)i * D, D, fmt, sq, nullptr, s_red, xstats);
    // the k best exact keys, descending, into sel[0, k) (K3's radix select over the staged
    // keys: a shared-memory bitonic sort of all next_pow2(M) keys took 52 us per launch at
    // 10M x 768, profiles/r02/ncu_final/launches_bench.csv)
    merge_topk_block<1>(wkeys + (size_t)i * Mmax, M, k, 0, sel, nullptr, nullptr, 0, k,
                     (M & 1) == 0 && M <= kMergeSmemKeys ? keys : nullptr, sel);
    if (threadIdx.x == 0) {
      int fail = 0;
      // documents outside every list: coarse <= max(s(T''), seed) (seeded scan)
      const float cb = fmaxf(t2 ? vx_key_score(t2) : -INFINITY, seed_thr(seed, seed_ld, b));
      if (cb > -INFINITY) {
        float qn, qh, qr;
        query_norms_final(s_red, fmt, &qn, &qh, &qr);
        const float E = cert_err_bound(fmt, D, qn, qh, qr, xstats);
        const uint64_t ek = sel[k - 1];
        fail = (ek == 0ull || !(vx_key_score(ek) > cb * cscale + E)) ? 1 : 0;
      }
      s_fail = fail;
      flags[b] = fail;
    }
    __syncthreads();
    if (!s_fail) {  // else the exact re-scan writes this query
      for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const uint64_t key = sel[j];
        const size_t o = (size_t)b * k + j;
        if (key == 0ull) {
          out_keys[o] = 0ull;
          out_ids[o] = -1;
          out_scores[o] = -INFINITY;
        } else {
          const int64_t gid = (int64_t)vx_key_id(key) + row0;
          out_keys[o] = (key & 0xFFFFFFFF00000000ull) | (uint64_t)(0xFFFFFFFFu - (uint32_t)gid);
          out_ids[o] = gid;
          out_scores[o] = vx_key_score(key);
        }
      }
    }
    __syncthreads();  // keys / s_red are reused by the next query
  }
}

// Per-shard maxima for the certificate's error bound: [0] max |x|, [1] max |bf16(x)|,
// [2] max |x - bf16(x)| over the shard's rows (float bits, atomicMax of non-negative floats).
__global__ void row_stats_kernel(const float* __restrict__ docs, int64_t n, int D,
                                 unsigned int* __restrict__ out_bits,
                                 const float* __restrict__ colscale) {
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  float b0 = 0.0f, b1 = 0.0f, b2 = 0.0f, b3 = 0.0f, b4 = 0.0f, nsum = 0.0f;
  for (int64_t r = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * wpb) {
    const float* x = docs + r * D;
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f, s4 = 0.0f;
    for (int c = lane; c < D; c += 32) {
      const float v = x[c];
      const float v16 = vx_bf16_bits_to_f32(vx_f32_to_bf16_bits(v));
      s0 = fmaf(v, v, s0);
      s1 = fmaf(v16, v16, s1);
      s2 = fmaf(v - v16, v - v16, s2);
      if (colscale) {  // s8 shadow with column scales: |x8| (integer) and |x - s x8|
        const float sc = colscale[c];
        const float q8 = sc > 0.0f ? (float)vx_quant8(v, sc) : 0.0f;
        s3 = fmaf(q8, q8, s3);
        s4 = fmaf(v - sc * q8, v - sc * q8, s4);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      s3 += __shfl_xor_sync(0xffffffffu, s3, o);
      s4 += __shfl_xor_sync(0xffffffffu, s4, o);
    }
    b0 = fmaxf(b0, sqrtf(s0));
    nsum += sqrtf(s0);
    b1 = fmaxf(b1, sqrtf(s1));
    b2 = fmaxf(b2, sqrtf(s2));
    b3 = fmaxf(b3, sqrtf(s3));
    b4 = fmaxf(b4, sqrtf(s4));
  }
  if (lane == 0) {
    atomicMax(&out_bits[0], __float_as_uint(b0 * 1.00001f));
    atomicMax(&out_bits[1], __float_as_uint(b1 * 1.00001f));
    atomicMax(&out_bits[2], __float_as_uint(b2 * 1.00001f));
    atomicAdd(reinterpret_cast<float*>(out_bits) + 7, nsum);  // sum of row norms (heuristics)
    if (colscale) {  // s x8 is rounded to fp32 here: 1e-3 of margin for the residual norm
      atomicMax(&out_bits[3], __float_as_uint(b3 * 1.00001f));  // integer squares: exact sum
      atomicMax(&out_bits[4], __float_as_uint(b4 * 1.001f));
    }
  }
}

// ------------------------------------------------------------------- host side
cudaError_t launch_rerank_wide(const float* docs, const float* fq, int D, const int* fidx,
                               const int* fcount, const uint64_t* part_all, int B, int GS,
                               int P_pairs, int P_single, int kc, int k, int64_t row0,
                               const float* xstats, int fmt, const float* qscale,
                               uint64_t* wkeys, uint64_t* out_keys, int64_t* out_ids,
                               float* out_scores, int* flags, cudaStream_t st,
                               const uint64_t* seed, int seed_ld) {
  const int M = P_single * kc;
  int kp2 = 16;
  while (kp2 < k) kp2 <<= 1;
  const size_t smem = ((size_t)((M + 1) & ~1) + kp2) * 8;  // staged keys + the top-k
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(wide_select_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // S CTAs per failing query (about one row per thread), W queries in flight; both loops
  // exit at once when the device-side count is 0 (the common case)
  const int S = (M + 255) / 256;
  const int W = B < 32 ? B : 32;
  wide_score_kernel<<<W * S, 256, (size_t)D * 4, st>>>(docs, fq, D, fidx, fcount, part_all, B,
                                                       GS, P_pairs, P_single, kc, S, wkeys);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  wide_select_kernel<<<W, 256, smem, st>>>(fq, D, fidx, fcount, part_all, B, GS, P_pairs,
                                           P_single, kc, k, row0, xstats, fmt, qscale, wkeys,
                                           out_keys, out_ids, out_scores, flags, seed, seed_ld);
  return cudaGetLastError();
}

size_t scan_tc_smem(int QT, int TD, int fmt, int* ns_out) {
  const int stage = QT * kTcStageUnit + TD * 128;
  (void)fmt;
  const size_t fixed = (size_t)QT * 128 * 16 * 8 + 16 + 1024;  // epilogue scratch
  int ns = 6;
  while (ns > 2 && (size_t)ns * stage + fixed + (2 * ns + 4) * 8 > 227 * 1024) --ns;
  *ns_out = ns;
  return (size_t)ns * stage + fixed + (size_t)(2 * ns + 4) * 8;
}

template <int QT, int TD>
static cudaError_t launch_tc(const CUtensorMap* tq, const CUtensorMap* tx, const ScanTcArgs& a,
                             int grid, size_t smem, cudaStream_t st) {
  // per-CTA list length: kc_of(fmt), or kSampleKC for the seed's sample pass
  const int kc = a.kc ? a.kc : kc_of(a.fmt);
  if (kc != kc_of(a.fmt) && kc != kSampleKC) return cudaErrorInvalidValue;
  auto kfn = kc == kSampleKC
                 ? (a.fmt == FMT_TF32 ? scan_tc_kernel<QT, TD, FMT_TF32, kSampleKC>
                                      : (a.fmt == FMT_I8 ? scan_tc_kernel<QT, TD, FMT_I8, kSampleKC>
                                                         : scan_tc_kernel<QT, TD, FMT_BF16, kSampleKC>))
                 : (a.fmt == FMT_TF32 ? scan_tc_kernel<QT, TD, FMT_TF32, kc_of(FMT_TF32)>
                                      : (a.fmt == FMT_I8 ? scan_tc_kernel<QT, TD, FMT_I8, kc_of(FMT_I8)>
                                                         : scan_tc_kernel<QT, TD, FMT_BF16, kc_of(FMT_BF16)>));
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TcCfg<QT, TD>::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kfn, *tq, *tx, a);
}

cudaError_t launch_scan_tc(int QT, int TD, const CUtensorMap* tq, const CUtensorMap* tx,
                           const ScanTcArgs& a, int grid, size_t smem, cudaStream_t st) {
  if (QT == 1 && TD == 128) return launch_tc<1, 128>(tq, tx, a, grid, smem, st);
  if (QT == 1 && TD == 256) return launch_tc<1, 256>(tq, tx, a, grid, smem, st);
  if (QT == 2 && TD == 128) return launch_tc<2, 128>(tq, tx, a, grid, smem, st);
  if (QT == 2 && TD == 256) return launch_tc<2, 256>(tq, tx, a, grid, smem, st);
  return cudaErrorInvalidValue;
}

// Staging: R rows per round in DC-float chunks (the largest multiple of 32 <= 192 dividing
// D), two chunk buffers.  Whole rows before (R = 16 / 32 rows per round, 2-4 CTAs per SM):
// s8 k' = 1024 at B = 1024 took 635 us at 3.6 TB/s with the CTAs' single computing warp the
// critical path (profiles/r01/README.md).  Now (ncu, same 1.96 GHz clock, B = 1024 s8
// k' = 1024, profiles/r01/rerank_chunks.txt): R = 64 / DC = 192 (two CTAs per SM) 519-539 us
// at 4.4 TB/s, R = 128 533-558, R = 256 / DC = 96 563-585, R = 192 / DC = 64 740-760.
// VX_DEBUG_RERANK_ROWS / _DC: timing experiments.
cudaError_t launch_rerank(const float* docs, const float* q, int D, uint64_t* cand, int B,
                          int kp, const uint64_t* part, int grid, int ldlists, int kc, int k,
                          int64_t row0, const float* xstats, int fmt, const float* qscale,
                          uint64_t* out_keys, int64_t* out_ids, float* out_scores, int* flags,
                          cudaStream_t st, int phase, const float* tau, uint64_t* hkeys,
                          float* lb, const uint64_t* seed, int seed_ld, const RerankFuse& fz) {
  if (fz.mlists && (fz.mM > kMergeSmemKeys || (fz.mM & 1) || fz.mM < kp))
    return cudaErrorInvalidValue;
  const size_t base = (size_t)((D + 3) & ~3) * 4 + (size_t)kp * 8;
  static const int env_rows = [] {
    const char* e = getenv("VX_DEBUG_RERANK_ROWS");
    return e ? atoi(e) : 0;
  }();
  static const int env_dc = [] {
    const char* e = getenv("VX_DEBUG_RERANK_DC");
    return e ? atoi(e) : 0;
  }();
  static const int env_bufs = [] {
    const char* e = getenv("VX_DEBUG_RERANK_BUFS");
    return e ? atoi(e) : 0;
  }();
  static const int env_pf = [] {
    const char* e = getenv("VX_DEBUG_RERANK_PF");
    return e ? atoi(e) : -1;
  }();
  const int head_all = phase == 0 && B <= 64 ? 1 : 0;
  const int S = fz.split > 1 && head_all && !fz.mlists ? fz.split : 1;
  if (fz.split > 1 && S == 1) return cudaErrorInvalidValue;  // split needs the standalone merge
  const int kslice = (kp + S - 1) / S;  // candidates one CTA re-scores (whole-set head)
  // one wave with an SM per CTA (B <= the SM count): each CTA may take the whole shared
  // memory, and twice the chain threads — a single query's 1024 rows were bound by 64 serial
  // fmaf chains and 64 small bulk copies per item (B = 1: 121 -> 67 us, B = 16: 172 -> 125 us
  // at 10M x 768 s8, profiles/r02/rerank/small_batch.txt)
  static const int num_sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  const bool sm_each = B * S <= num_sms;
  int NB = env_bufs >= 2 ? std::min(env_bufs, kRerankMaxBufs) : 2;
  int DC = env_dc > 0 && env_dc % 32 == 0 && D % env_dc == 0 ? env_dc : 192;
  while (DC > 32 && D % DC) DC -= 32;
  int R = env_rows > 0 ? std::min(env_rows, 256) : (sm_each ? 128 : 64);
  static const int env_smem_kb = [] {
    const char* e = getenv("VX_DEBUG_RERANK_SMEM_KB");
    return e ? atoi(e) : 0;
  }();
  auto smem_of = [&](int r) { return base + (size_t)NB * r * (DC + 4) * 4; };
  const size_t smem_cap =
      (size_t)(env_smem_kb > 0 ? std::min(env_smem_kb, 220) : (sm_each ? 220 : 110)) * 1024;
  while (R > 16 && smem_of(R) > smem_cap) R -= 16;  // default: two CTAs per SM
  size_t smem = smem_of(R);
  // small batch, latency-bound: ALL k' whole rows in one burst of bulk copies and one wait
  // (one round, one chunk), instead of the chunk stream
  // (Four 192-float chunks on four barriers instead, so the chains could start on the first
  // quarter, took the 100K-row B = 16 head from 4.0 to 7.9 us: four times the bulk copies.)
  if (head_all && env_dc == 0 && base + (size_t)kslice * (D + 4) * 4 <= 220 * 1024) {
    DC = D;
    R = kslice;
    NB = 2;  // one item: only buffer 0
    smem = base + (size_t)kslice * (D + 4) * 4;
  }
  // L2 prefetch distance in items beyond the staging window (packed into nbuf's high bits)
  const int PF = head_all ? 0 : std::min(env_pf >= 0 ? env_pf : 0, 15);
  smem = std::max(smem, base + (size_t)512 * 8);  // the final selection's survivors
  // the fused merge stages the lists and its selection in the row buffers
  if (fz.mlists)
    smem = std::max(smem, base + (size_t)(((fz.mM + 1) & ~1) + kRerankMergeSel + kRerankMergeFilter) * 8);
  cudaError_t e = cudaFuncSetAttribute(rerank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  // programmatic dependent launch: opt-in (VX_PDL=1).  Measured on the 100K-row B = 16 stage
  // it made the step slower (93 vs 88 us: the early CTAs' wait + the dependency flush cost
  // more than the launch latency they hide), and within noise on the 10M-row stage.
  static const bool no_pdl = getenv("VX_PDL") == nullptr || getenv("VX_DEBUG_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B * S);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, rerank_kernel, docs, q, D, cand, kp, part, grid, ldlists, kc,
                            k, row0, xstats, fmt, qscale, out_keys, out_ids, out_scores, flags, R,
                            DC, phase, tau, hkeys, lb, seed, seed_ld, head_all, NB | (PF << 4),
                            fz);
}

// ------------------------------------------------------------------- sharded threshold tau
// all[G][B][k]: every shard's head exact scores (rerank phase 1; -inf = empty) — distinct
// documents, so tau[b] = the largest v with count(all >= v) >= k is <= the global exact k-th.
__global__ void __launch_bounds__(256)
    shard_tau_kernel(const float* __restrict__ all, int G, int B, int k, float* __restrict__ tau) {
  __shared__ float s_v[1024];
  __shared__ float s_w[8];
  const int b = blockIdx.x;
  const int n = G * k;  // <= 1024 (G <= 8, k <= 128)
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    s_v[i] = all[((size_t)(i / k) * B + b) * k + (i % k)];
  __syncthreads();
  float best = -INFINITY;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = s_v[i];
    if (!(v > -INFINITY)) continue;
    int cnt = 0;
    for (int j = 0; j < n; ++j) cnt += s_v[j] >= v ? 1 : 0;
    if (cnt >= k) best = fmaxf(best, v);
  }
  for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = s_w[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, s_w[w]);
    tau[b] = m;
  }
}

__global__ void fill_neg_inf_kernel(float* __restrict__ v, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] = -INFINITY;
}

cudaError_t launch_shard_tau(const float* all, int G, int B, int k, float* tau, cudaStream_t st) {
  if (G * k > 1024) {  // beyond the kernel's smem list: no threshold (every shard re-ranks its
                       // whole candidate set; still exact, just no pruning)
    fill_neg_inf_kernel<<<(B + 255) / 256, 256, 0, st>>>(tau, B);
    return cudaGetLastError();
  }
  shard_tau_kernel<<<B, 256, 0, st>>>(all, G, B, k, tau);
  return cudaGetLastError();
}

cudaError_t launch_row_stats(const float* docs, int64_t n, int D, unsigned int* out_bits,
                             cudaStream_t st, const float* colscale) {
  cudaError_t e = cudaMemsetAsync(out_bits, 0, 20, st);  // [0..4]; [5] = the s8 doc factor
  if (e == cudaSuccess) e = cudaMemsetAsync(out_bits + 7, 0, 4, st);  // [7] = sum of |x|
  if (e != cudaSuccess) return e;
  int64_t blocks = (n + 7) / 8;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  row_stats_kernel<<<(int)blocks, 256, 0, st>>>(docs, n, D, out_bits, colscale);
  return cudaGetLastError();
}

}  // namespace vx
