// scan_tc2.cu — K2 for B > 128: the coarse tensor-core scan on CTA PAIRS
// (tcgen05.mma.cta_group::2, cluster of 2 on one TPC), 256 x QG queries per pass.
//
// One pair owns a TD-document tile (TD = 256 / QG) and QG query groups of 256.  CTA r stages,
// per K-chunk, the 128 query rows [256g + 128r, +128) of every group g (A) and documents
// [tile*TD + r*TD/2, +TD/2) (B) in ITS smem.  Per k-step the leader issues QG MMAs of
// M=256 x N=TD — MMA g reads group g's A rows of both CTAs and the B rows of both CTAs —
// into TMEM columns [(buf*QG + g)*TD, +TD) = documents of the tile (contiguous).  Each
// CTA's TMEM receives its 128 query rows.  Two accumulator buffers either way (512 columns),
// so the epilogue of one tile overlaps the MMAs of the next.
//   QG = 1 (128 < B <= 256): 256-document tiles, 4 epilogue warps.
//   QG = 2 (B > 256, VX_OPT_SCAN_PAIRS = 2): 128-document tiles, 8 epilogue warps (two per
//          SM sub-partition: twice the latency hiding for the divergent selection); every
//          document byte read from HBM feeds 512 queries — half the HBM traffic per query.
//
// Pipeline / synchronisation (a 2-SM UMMA pipeline, written out):
//   full[s]   leader-only, count 1: leader producer arrive.expect_tx(both CTAs' bytes); both
//             CTAs' TMA (.cta_group::2) complete_tx on the leader's barrier.
//   empty[s]  both CTAs, count 1: the leader's tcgen05.commit multicast to both.
//   tfull[b]  both CTAs, count 1: commit multicast after the tile's last chunk.
//   tempty[b] leader-only, count 2 x 4QG: every epilogue warp of both CTAs (the peer remotely).
// Warps: 0 document producer, 1 MMA issuer (+ TMEM allocator), 2 query producer,
//        3 .. 3+4QG-1 epilogue (group g = warps 3+4g .. 6+4g; warp w reads TMEM lanes
//        32*(w%4) .. +31).  Epilogue: thread = query, vx_select.cuh (group-max filter,
//        register-resident KC-list).
#include <cuda_runtime.h>
#include <math.h>

#include <type_traits>

#include "vx_internal.cuh"
#include "vx_ptx.cuh"
#include "vx_select.cuh"

namespace vx {

constexpr int kP2Unit = 16384;        // 128 rows x 128 B
constexpr int kP2SmemLimit = 227 * 1024;

template <int QG>
struct P2Cfg {
  static constexpr int TD = 256 / QG;                    // documents per pair tile
  static constexpr int NBUF = 2;                         // accumulator buffers (512 columns)
  static constexpr int kCols = 512;
  static constexpr int kBUnit = TD / 2 * 128;            // per CTA: TD/2 document rows x 128 B
  static constexpr int kEpiWarps = 4 * QG;
  static constexpr int kThreads = (3 + kEpiWarps) * 32;
  static constexpr int kAStage = QG * kP2Unit;           // per CTA: QG query blocks
  static constexpr int kNA = QG == 1 ? 4 : 3;            // query stages (L2-resident: short)
  static constexpr int kScratch = kEpiWarps * 32 * 64 * 4;  // 64 words per epilogue thread
};

// Separate rings for A (queries, from L2) and B (documents, from HBM): the document ring
// gets the remaining smem, so each SM keeps ~100-128 KB of HBM reads in flight.
template <int QG>
static size_t p2_smem(int nb) {
  using C = P2Cfg<QG>;
  return (size_t)C::kNA * C::kAStage + (size_t)nb * C::kBUnit + C::kScratch +
         (size_t)(2 * C::kNA + 2 * nb + 4) * 8 + 16 + 1024;
}

template <int QG, int FMT, int KC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P2Cfg<QG>::kThreads, 1)
    scan_tc2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tx,
                    const ScanTcArgs a) {
  using C = P2Cfg<QG>;
  constexpr int TD = C::TD, NA = C::kNA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int nb = a.ns;  // document stages
  uint8_t* ringA = smem;
  uint8_t* ringB = smem + (size_t)NA * C::kAStage;
  uint32_t* scratch_base = reinterpret_cast<uint32_t*>(ringB + (size_t)nb * C::kBUnit);  // [64][32*EW]
  uint64_t* fullA = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(scratch_base) + C::kScratch);
  uint64_t* emptyA = fullA + NA;
  uint64_t* fullB = emptyA + NA;
  uint64_t* emptyB = fullB + nb;
  uint64_t* tfull = emptyB + nb;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_idx_uniform(), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // K-chunk = one 128-byte swizzle atom: 32 fp32 (tf32), 64 bf16, 128 s8
  constexpr int cw = FMT == FMT_TF32 ? 32 : (FMT == FMT_I8 ? 128 : 64);
  const int nch = a.D / cw;
  const uint32_t n_local = a.n_local;
  const int ntiles = (int)((n_local + TD - 1) / TD);
  uint64_t kt_c0 = 0, kt_g0 = 0;
  ktimer_begin(a.ktimer, kt_c0, kt_g0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tx);
    for (int i = 0; i < NA; ++i) {
      mbar_init(&fullA[i], 1);
      mbar_init(&emptyA[i], 1);
    }
    for (int i = 0; i < nb; ++i) {
      mbar_init(&fullB[i], 1);
      mbar_init(&emptyB[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * C::kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, C::kCols);
  tc_fence_before();
  cluster_sync();  // barrier inits + TMEM allocation visible pair-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 || warp == 2) {
    // ------------------------------------------------ TMA producers (both CTAs):
    // warp 0 streams document blocks, warp 2 query blocks, each with its own ring; the
    // whole warp walks the ring (warp-uniform state), one elected lane issues the copies
    const bool docs = warp == 0;
    const uint64_t pol = docs ? policy_evict_first() : policy_evict_last();
    const int nst = docs ? nb : NA;
    uint64_t* fullR = docs ? fullB : fullA;
    uint64_t* emptyR = docs ? emptyB : emptyA;
    uint8_t* ring = docs ? ringB : ringA;
    const int sbytes = docs ? C::kBUnit : C::kAStage;
    const uint32_t bytes_pair = 2u * (uint32_t)sbytes;
    const uint32_t fb0 = mapa_shared(smem_u32(fullR), 0);  // the leader's full barriers
    int s = 0;
    uint32_t ph = 0;
    for (int tile = pair; tile < ntiles; tile += npairs) {
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&emptyR[s], ph ^ 1);
        // timing experiments (dbg bits 2/4): after the first pass over the ring, stop
        // streaming documents / queries and let the MMA reuse the staged data
        const bool skip = (a.dbg_no_select & (docs ? 2 : 4)) && (tile != pair);
        __syncwarp();
        if (elect_one()) {
          const uint32_t fb = fb0 + (uint32_t)(s * 8);
          if (leader) mbar_expect_tx(&fullR[s], skip ? 0u : bytes_pair);
          uint8_t* st = ring + (size_t)s * sbytes;
          if (skip) {
          } else if (docs) {
            tma_load_2d_pair(st, &tx, fb, c * cw, tile * TD + (int)rank * (TD / 2), pol);
          } else {
#pragma unroll
            for (int g = 0; g < QG; ++g)
              tma_load_2d_pair(st + g * kP2Unit, &tq, fb, c * cw, g * 256 + (int)rank * 128, pol);
          }
        }
        __syncwarp();
        if (++s == nst) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    // Producer tail: the leader's multicast commits to our empty barriers must all have
    // landed before this CTA exits (a late arrive would hit the next kernel's smem).
    for (int i = 0; i < nst; ++i) {
      mbar_wait(&emptyR[s], ph ^ 1);
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA, whole warp)
    // The warp walks the pipeline together (all lanes wait on the barriers) and one elected
    // lane issues: loop state stays warp-uniform, so descriptors live in uniform registers
    // and each MMA is a single UTCHMMA — a single-thread loop paid R2UR waterfalls per
    // MMA and could not keep up with a 2-SM M=256 x N=256 MMA (128 cycles each).
    if (leader) {
      constexpr uint32_t idesc = make_idesc_fmt(FMT, 256u, (uint32_t)TD);
      const uint64_t da0 = umma_desc_sw128(smem_u32(ringA));
      const uint64_t db0 = umma_desc_sw128(smem_u32(ringB));
      int sa = 0, sb = 0, buf = 0;
      uint32_t pa = 0, pb = 0, bph = 0;
      for (int tile = pair; tile < ntiles; tile += npairs) {
        mbar_wait(&tempty[buf], bph ^ 1);
        tc_fence_after();
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&fullA[sa], pa);
          mbar_wait(&fullB[sb], pb);
          tc_fence_after();
          __syncwarp();
          if (elect_one()) {
            // descriptor start address is addr >> 4: stage / group / K-step offsets add
            const uint64_t da = da0 + (uint64_t)(sa * (C::kAStage >> 4));
            const uint64_t db = db0 + (uint64_t)(sb * (C::kBUnit >> 4));
            // dbg bit 8 (timing experiments): stream + commit without issuing the MMAs
            if (!(a.dbg_no_select & 8) || tile == pair)
#pragma unroll
              for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int g = 0; g < QG; ++g)
                  mma_pair_k<FMT>(tmem_base + (uint32_t)((buf * QG + g) * TD),
                                   da + (uint64_t)(g * (kP2Unit >> 4) + 2 * j), db + 2 * j, idesc,
                                   (c | j) != 0 ? 1u : 0u);
            mma_commit_pair(&emptyA[sa], 0x3);
            mma_commit_pair(&emptyB[sb], 0x3);
          }
          __syncwarp();
          if (++sa == NA) {
            sa = 0;
            pa ^= 1;
          }
          if (++sb == nb) {
            sb = 0;
            pb ^= 1;
          }
        }
        if (elect_one()) mma_commit_pair(&tfull[buf], 0x3);
        __syncwarp();
        if (++buf == C::NBUF) {
          buf = 0;
          bph ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (both CTAs): thread = query
    const int e = warp - 3;                    // 0 .. 4QG-1
    const int g = e >> 2;                      // query group
    const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
    const int m = quad * 32 + lane;            // row of this CTA's 128 queries of group g
    const int q = g * 256 + (int)rank * 128 + m;  // query within the launch
    uint32_t* scratch = scratch_base + (e * 32 + lane);  // [64][32*EW]
    constexpr int SS = C::kEpiWarps * 32;             // scratch row stride
    const uint32_t te_leader = mapa_shared(smem_u32(&tempty[0]), 0);
    uint64_t L[KC];
#pragma unroll
    for (int j = 0; j < KC; ++j) L[j] = 0ull;
    // admission threshold: the query's seed, else -inf
    float thr = q < a.B ? seed_thr(a.seed, a.seed_ld, q) : -INFINITY;
    if (a.dbg_no_select & 16) thr = 2e9f;  // timing only: the filter's fast path alone
    int buf = 0;
    uint32_t bph = 0;
    for (int tile = pair; tile < ntiles; tile += npairs) {
      mbar_wait(&tfull[buf], bph);
      tc_fence_after();
      const uint32_t col = tmem_base + (uint32_t)((buf * QG + g) * TD) + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
      for (int cc = 0; cc < TD / 64; ++cc) {
        uint32_t r[64];
        tmem_ld64(col + cc * 64, r);
        tmem_ld_wait();
        if (cc == TD / 64 - 1) {
          // the tile's last chunk is in registers: hand the accumulator buffer back to the
          // MMA now, not after the selection — the next-but-one tile's MMAs overlap it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(te_leader + (uint32_t)(buf * 8));
        }
        if (q >= a.B || (a.dbg_no_select & 1)) continue;
        const uint32_t doc0 = (uint32_t)tile * TD + cc * 64;  // columns map to docs 1:1
        admit<FMT, KC, 64>(r, doc0, n_local, scratch, SS, L, thr);
      }
      if (++buf == C::NBUF) {
        buf = 0;
        bph ^= 1;
      }
    }
    if (q < a.B) {
      // per-query stride = gridDim.x lists (the single-CTA kernel's layout): every query
      // group of a batch shares one layout, so one merge / re-rank launch covers the batch
      uint64_t* out = a.part + ((size_t)q * gridDim.x + pair) * KC;
#pragma unroll
      for (int j = 0; j < KC; ++j) out[j] = L[j];
    }
  }
  tc_fence_before();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  ktimer_end(a.ktimer, kt_c0, kt_g0);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::kCols);
  }
}

size_t scan_tc2_smem(int QG, int* ns_out) {
  int nb = 8;
  auto sz = [&](int n) { return QG == 2 ? p2_smem<2>(n) : p2_smem<1>(n); };
  while (nb > 2 && sz(nb) > (size_t)kP2SmemLimit) --nb;
  *ns_out = nb;
  return sz(nb);
}

cudaError_t launch_scan_tc2(int QG, const CUtensorMap* tq, const CUtensorMap* tx,
                            const ScanTcArgs& a, int grid, size_t smem, cudaStream_t st) {
  if (grid < 2 || (grid & 1) || (QG != 1 && QG != 2)) return cudaErrorInvalidValue;
  // per-pair list length: kc_of(fmt), or kSampleKC for the seed's sample pass
  const int kc = a.kc ? a.kc : kc_of(a.fmt);
  if (kc != kc_of(a.fmt) && kc != kSampleKC) return cudaErrorInvalidValue;
  auto pick = [&](auto qg) {
    constexpr int Q = decltype(qg)::value;
    if (kc == kSampleKC)
      return a.fmt == FMT_TF32 ? scan_tc2_kernel<Q, FMT_TF32, kSampleKC>
                               : (a.fmt == FMT_I8 ? scan_tc2_kernel<Q, FMT_I8, kSampleKC>
                                                  : scan_tc2_kernel<Q, FMT_BF16, kSampleKC>);
    return a.fmt == FMT_TF32 ? scan_tc2_kernel<Q, FMT_TF32, kc_of(FMT_TF32)>
                             : (a.fmt == FMT_I8 ? scan_tc2_kernel<Q, FMT_I8, kc_of(FMT_I8)>
                                                : scan_tc2_kernel<Q, FMT_BF16, kc_of(FMT_BF16)>);
  };
  auto kfn = QG == 2 ? pick(std::integral_constant<int, 2>{}) : pick(std::integral_constant<int, 1>{});
  const int threads = QG == 2 ? P2Cfg<2>::kThreads : P2Cfg<1>::kThreads;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kfn<<<grid, threads, smem, st>>>(*tq, *tx, a);
  return cudaGetLastError();
}

}  // namespace vx
