// vx_stage.cu — the per-batch retrieval stage behind the C-ABI (include/vortex_b200.h):
// local certified top-k (tensor-core coarse scan or exact K1 scan, merge, exact re-rank,
// certificate levels 2-3), MaxSim, the two-phase NCCL shard exchange, CUDA graphs per stage
// part, the device-pointer entry points, model load (vx_prepare) and vx_sync.
//
// The stage a deployment registers as the search operator (reference: ComponentFn,
// proj/include/vortex/runtime.hpp:179; invoked by Runtime::complete_batch,
// runtime.hpp:656-672) runs, per batch of B queries:
//   part 1: [broadcast queries] -> K2 coarse scan + per-CTA top-16 -> K3 merge to k'
//           -> K2b exact re-rank + certificate (-> K2c / K1 on failure)
//           -> [gather k x G keys to rank 0 -> K3 merge]
//   part 2: [broadcast tokens + winners] -> K4 MaxSim (owned winners) -> [max-reduce]
//           -> order by MaxSim
// Shard mode mirrors the reference's key->shard placement (kvs.hpp:160-175): contiguous
// document ranges, a document's row and its token block on one GPU.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "vx_handle.cuh"

// Exact path: K1 scan + merge: d_q [B][D] -> keys (global ids) / ids / scores [B][k]
// the device-side launch timer of kind i (VX_DEBUG_NO_KTIMER: none — A/B timing of the
// timers' own cost only)
static vx::KTimer* ktimer_of(vx_index* h, int i) {
  static const bool off = getenv("VX_DEBUG_NO_KTIMER") != nullptr;
  return off ? nullptr : h->d_ktimer + i;
}

static vx_status local_topk_f32(vx_index* h, const float* d_q, int B, int k, uint64_t* keys,
                                int64_t* ids, float* scores, cudaStream_t st,
                                const int* d_count = nullptr) {
  const int D = h->desc.dim;
  const int kcap = kcap_of(k);
  const int grid = h->grid;
  // queries per launch: the largest bucket whose smem plan fits (big k / big D shrink it)
  int gmax = 32, ns0 = 0, cap0 = 0;
  while (gmax > 1 && !vx::scan_f32_smem(gmax, D, kcap, &ns0, &cap0)) gmax >>= 1;
  // device-count launch (certificate fallback): ONE launch loops over the query groups on
  // the device, sized by the count; host-sized batches launch one kernel per group
  const int step = d_count ? B : gmax;
  for (int g0 = 0; g0 < B; g0 += step) {
    const int Bg = std::min(step, B - g0);
    const int bucket = d_count ? gmax : vx::scan_f32_bucket(Bg);
    int ns = 0, cap = 0;
    size_t smem = vx::scan_f32_smem(bucket, D, kcap, &ns, &cap);
    if (!smem) return fail(VX_ERR_UNSUPPORTED, "scan config (B=%d, D=%d, k=%d) exceeds smem", Bg, D, k);
    vx::ScanF32Args a;
    a.q = d_q + (size_t)g0 * D;
    a.B = Bg;
    a.D = D;
    a.n_local = (uint32_t)h->n_local;
    a.kcap = kcap;
    a.cap = cap;
    a.ns = ns;
    a.part = h->d_part + (size_t)g0 * grid * kcap;
    a.d_count = d_count;
    a.g0 = g0;
    a.ktimer = d_count ? nullptr : ktimer_of(h, vx::KT_F32);
    if (g0 == 0 && !d_count) CU_TRY(record_scan_ev(h, h->tev[0], st));
    CU_TRY(vx::launch_scan_f32(bucket, &h->tmap_docs, a, grid, smem, st));
    count_launch(h);
  }
  if (!d_count) CU_TRY(record_scan_ev(h, h->tev[1], st));
  CU_TRY(vx::launch_merge_topk(h->d_part, B, grid * kcap, k, h->row0, keys, ids, scores, st,
                               d_count));
  count_launch(h);
  return VX_OK;
}

// candidates the TC pass hands to the exact re-rank
// k' = 4 next_pow2(k) in [64, 256] (VX_OPT_KPRIME overrides, up to 512).  256 is the
// measured sweet spot for bf16 at k = 100: with 16-entry per-pair lists, k' = 512 fails
// certificate 1 for ~13% of queries (a pair holding >= 16 of the top-512), k' = 256 for
// ~0.03% (profiles/cert_rate.py, profiles/r01/cert_rate.jsonl).
// The s8 pass's error bound is ~4x the bf16 one (residual norms of 7-bit integers vs 8-bit
// mantissas), so its candidate set is 8 next_pow2(k) in [128, 1024] with 32-entry lists.
// Sharded (G shards, the tau exchange on): what a shard must certify is its share of the
// candidates that can reach the GLOBAL top-k — certificate 2 holds when the shard's k'-th
// coarse key + E is below tau, and a shard's (k'/G)-th best coarse key sits at the same
// quantile of its N/G rows as the k'-th of the whole index.  So a shard takes k'/G (not below
// 2 next_pow2(k): the head re-scores k rows): s8 k = 100 -> 512 at G = 2, 256 at G >= 4 — the
// fused merge, the exact-key sort and the list certificate shrink with it (the level-2 and
// level-3 fallbacks still catch a query whose shard was unusually dense).
static int kprime_of(const vx_index* h, int k, int fmt) {
  if (h->kprime) return std::max(h->kprime, next_pow2(k));
  int kp = fmt == vx::FMT_I8 ? std::min(1024, std::max(128, 8 * next_pow2(k)))
                             : std::min(256, std::max(64, 4 * next_pow2(k)));
  if (h->nranks > 1) kp = std::max(std::min(kp, 2 * next_pow2(k)), kp / next_pow2(h->nranks));
  return kp;
}

// coarse operand format of the tensor-core pass for this handle
// AUTO takes the s8 pass (a quarter of the fp32 bytes, twice the bf16 tensor rate; measured
// 10M x 768 B=1024 stage 8.99 ms vs 13.5 ms bf16 — profiles/r01/README.md) when
//  * the shard's one-scale quantisation is tight enough for the certificate to hold at
//    k' = 8 next_pow2(k): max |x - sx x8| <= 3 % of the mean row norm (synthetic rows ~1 %,
//    Gaussian rows ~1.5 %) — an outlier coordinate inflates the shared scale, widens the
//    error bound E and would push queries to the exact re-scan;
//  * the shard is long enough for the pass to amortise filling the 32-key lists: >= 16
//    tiles per CTA (100K x 768, B=16: s8 0.093 ms vs bf16 0.063 ms — the first tiles insert
//    every document).
// Otherwise bf16.
constexpr float kI8AutoMaxRelResidual = 0.03f;
constexpr int kI8AutoMinTilesPerCta = 16;

// AUTO's runtime check of the s8 pass (called with the device's certificate counters: fc[1]
// level-2 and fc[3] level-3 running totals).  The static test above (quantisation residual vs
// row norms) cannot see the QUERIES: with anisotropic rows (a few dimensions carrying most of
// the spread — include/vx_synth.h dist 1) the s8 bound E exceeds the score gaps and every
// query falls through to the exact re-scan (measured: 587 ms per 1024-query batch instead of
// 7.5).  When, over >= 16 queries, more than 1/8 needed the re-scan or half the wide
// re-rank (the isotropic headline: ~0.5 % level 2, no re-scans), AUTO leaves s8 for the bf16 pass (whose relative per-element error does not care
// about the anisotropy) until the shard is re-uploaded.  Results are exact either way.
void maybe_demote_i8(vx_index* h, const int* fc, uint64_t queries) {
  if (h->coarse != VX_COARSE_AUTO || h->i8_demoted || coarse_fmt(h) != vx::FMT_I8) {
    h->cert_seen_q = queries;
    h->cert_seen_l2 = (uint64_t)fc[1];
    h->cert_seen_l3 = (uint64_t)fc[3];
    return;
  }
  const uint64_t dq = queries - h->cert_seen_q;
  if (dq < 16) return;
  const uint64_t l2 = (uint64_t)fc[1] - h->cert_seen_l2, l3 = (uint64_t)fc[3] - h->cert_seen_l3;
  if (l3 * 8 > dq || l2 * 2 > dq) {
    h->i8_demoted = true;
    drop_graphs(h);  // the captured stages bake the s8 choice in
  }
  h->cert_seen_q = queries;
  h->cert_seen_l2 = (uint64_t)fc[1];
  h->cert_seen_l3 = (uint64_t)fc[3];
}

int coarse_fmt(const vx_index* h) {
  if (h->coarse == VX_COARSE_I8 && h->docs8) return vx::FMT_I8;
  if (h->coarse == VX_COARSE_AUTO && h->docs8 && !h->i8_demoted &&
      h->n_local >= (int64_t)256 * h->num_sms * kI8AutoMinTilesPerCta &&
      h->xstats_host[4] <= kI8AutoMaxRelResidual * h->xstats_host[7] / (float)std::max<int64_t>(1, h->n_local))
    return vx::FMT_I8;
  if (h->coarse == VX_COARSE_TF32 || !h->docs16) return vx::FMT_TF32;
  return vx::FMT_BF16;
}

static bool tc_eligible(const vx_index* h, int B, int k) {
  (void)h;
  (void)B;
  return k <= 128;
}

// Tensor-core path: K2 coarse scan (top-16/32 per CTA) -> K3 merge to top-k' -> K2b exact
// re-rank + certificate -> exact re-scan of any query whose certificate failed.
// Sharded threshold exchange: every rank contributes B x k exact scores of distinct
// documents (lb; -inf = empty); tau[b] = the k-th largest of the union is <= the global
// exact k-th.  All ranks call it at the same point of the stage.
static vx_status shard_tau(vx_index* h, const float* lb, int B, int k, cudaStream_t st,
                           bool want_tau) {
  NCCL_TRY(nccl().AllGather(lb, h->d_lball, (size_t)B * k, ncclFloat32, h->comm, st));
  if (!want_tau) return VX_OK;
  CU_TRY(vx::launch_shard_tau(h->d_lball, h->nranks, B, k, h->d_tau, st));
  count_launch(h);
  return VX_OK;
}

static vx_status local_topk_tc(vx_index* h, const float* d_q, int B, int k, uint64_t* keys,
                               int64_t* ids, float* scores, cudaStream_t st) {
  const int D = h->desc.dim;
  const int grid = h->grid;
  const int fmt = coarse_fmt(h);
  const bool bf16 = fmt == vx::FMT_BF16, i8 = fmt == vx::FMT_I8;
  const int kp = kprime_of(h, k, fmt);
  const int KC = vx::kc_of(fmt);  // per-CTA list length
  if (D % (i8 ? 128 : (bf16 ? 64 : 32))) return fail(VX_ERR_UNSUPPORTED, "TC scan: D %d", D);
  if (kp > 1024) return fail(VX_ERR_UNSUPPORTED, "k' %d > 1024", kp);
  CU_TRY(record_scan_ev(h, h->tev[0], st));
  if (bf16) {
    CU_TRY(vx::launch_to_bf16(d_q, h->d_q16, (int64_t)B * D, st));
    count_launch(h);
  } else if (i8) {
    CU_TRY(vx::launch_rows_to_i8(d_q, B, D,
                                 reinterpret_cast<const float*>(h->d_xnorm) + vx::kXstatColScale,
                                 h->d_q8, h->d_qs8, st));
    count_launch(h);
  }
  // queries per pass over the index: 512 (default, CTA pairs with two query groups on
  // 128-document tiles: half the HBM traffic per query, two epilogue warps per SM
  // sub-partition; measured 10M x 768 B=1024: s8 6.05 ms vs 7.40, bf16 11.7 vs 15.8 with
  // 256-query passes — profiles/r01/README.md); VX_OPT_SCAN_PAIRS = 1: 256 (one group on
  // 256-document tiles); 0: the single-CTA kernels (QT = 2 x 128)
  const bool pairs = h->use_pairs && grid % 2 == 0;
  const int GS = (pairs && h->use_pairs == 2) ? 512 : 256;
  const int ldp = grid * KC;
  auto lists_per_query = [&](int r) {
    return (pairs && std::min(GS, B - r) > 128) ? grid / 2 : grid;
  };
  // Admission-threshold seeds.  A query's empty list admits every document of the first
  // tiles and ~KC ln(n/KC) in all, and with 32 queries per epilogue warp any passing lane
  // sends the warp down the insertion path: a selection cost that does not shrink with the
  // shard (512-query s8 passes, threshold pinned above every score vs the real selection:
  // 10M rows 2.45 vs 2.92 ms, 2.5M 0.59 vs 0.92, 1.25M 0.28 vs 0.57 —
  // profiles/r01/decomp_seed.jsonl).  So the same kernel first scans a strided
  // 1/kSeedStride row sample of the shard (its tensor map skips rows) with kSampleKC-key
  // lists (short lists keep the sample's own fill cheap: 34 us vs 124 us with 32-key lists
  // at 2.5M rows), the lists merge to each query's kSeedM best keys, and the full pass starts
  // admitting at the kSeedM-th: expected shard rank kSeedM x kSeedStride = 2048 >= k' for
  // every k <= 128; it lands above the k'-th coarse score with probability
  // P(Poisson(k'/64) >= 32) ~ 1e-4 at k' = 1024 (measured: m = 16 sent 1-9 % of the queries
  // to the exact re-scan, m = 32 none — profiles/r01/seed_m.jsonl).  Documents below the
  // seed never enter a list; the re-rank certificate bounds them by the seed (rerank_kernel,
  // wide_select_kernel), so results are unchanged.  10M x 768 s8 B = 1024: scan 5.95 ->
  // 5.24 ms; one shard of 4 / 8: 1.89 -> 1.49, 1.18 -> 0.84 ms (seed_stage2.jsonl).
  constexpr int kSeedLd = 32;
  const int kSeedStride = h->dbg_seed_stride ? h->dbg_seed_stride : 64;
  const int kSeedM = h->dbg_seed_m ? h->dbg_seed_m : 32;
  const int64_t n_sample = h->n_local / kSeedStride;
  const bool seeded = h->scan_seed && n_sample >= 8192;
  // the sample's lists: the upper part of d_part (the level-2 scratch, free until then)
  uint64_t* sample_lists = h->d_part + (size_t)h->desc.max_batch * grid * 32;
  auto scan_pass = [&](bool sample) -> vx_status {
    for (int g0 = 0; g0 < B; g0 += GS) {
      const int Bg = std::min(GS, B - g0);
      const bool on_pairs = pairs && Bg > 128;
      const int QT = Bg <= 128 ? 1 : 2;
      const int QG = on_pairs && Bg > 256 ? 2 : 1;
      const int TD1 = h->scan_tile ? h->scan_tile : 256;
      // small batch on the single-CTA kernel: replicate the queries over the 128 A-tile rows
      // so every epilogue lane selects (ScanTcArgs::rep): 16 rows x 8, 32 x 4, 64 x 2
      const int rep = (!on_pairs && QT == 1 && TD1 == 256 && !h->dbg_no_rep)
                          ? (Bg <= 16 ? 8 : (Bg <= 32 ? 4 : (Bg <= 64 ? 2 : 1)))
                          : 1;
      const int a_rows = on_pairs ? 128 : (rep > 1 ? 128 / rep : (QT == 1 ? ((Bg + 7) & ~7) : 128));
      CUtensorMap tq;
      // the coarse query copies span whole A tiles (kQueryPadRows rows past the batch are
      // allocated): no out-of-bounds TMA fill — a 1-query pass with 15 filled rows per
      // 16-row box took 1.58 ms at 10M rows against 1.10 ms at 16 queries
      const uint64_t qext = on_pairs ? (uint64_t)QG * 256  // a pass: QG groups of 2 x 128 rows
                                     : (uint64_t)((Bg + a_rows - 1) / a_rows) * a_rows;
      const uint64_t qrows = std::min<uint64_t>((uint64_t)(B - g0) + kQueryPadRows, qext);
      if (bf16)
        VX_TRY(make_tmap_2d(&tq, h->d_q16 + (size_t)g0 * D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                            std::max<uint64_t>(qrows, (uint64_t)Bg), D, 64, (uint32_t)a_rows));
      else if (i8)
        VX_TRY(make_tmap_2d(&tq, h->d_q8 + (size_t)g0 * D, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1,
                            std::max<uint64_t>(qrows, (uint64_t)Bg), D, 128, (uint32_t)a_rows));
      else
        VX_TRY(make_tmap_2d(&tq, d_q + (size_t)g0 * D, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                            (uint64_t)Bg, D, 32, (uint32_t)a_rows));
      vx::ScanTcArgs a;
      a.n_local = (uint32_t)(sample ? n_sample : h->n_local);
      a.D = D;
      a.B = Bg;
      a.a_rows = a_rows;
      a.fmt = fmt;
      a.dbg_no_select = h->dbg_tc_bits;  // timing experiments only (VX_DEBUG_TC_NOSELECT)
      a.kc = sample ? vx::kSampleKC : 0;
      a.rep = rep;
      a.ktimer = ktimer_of(h, sample ? vx::KT_SAMPLE : vx::KT_SCAN);
      a.part = sample ? sample_lists + (size_t)g0 * grid * vx::kSampleKC : h->d_part + (size_t)g0 * ldp;
      a.seed = (seeded && !sample) ? h->d_seedk + (size_t)g0 * kSeedLd + (kSeedM - 1) : nullptr;
      a.seed_ld = kSeedLd;
      // the first pass after the query conversion launches as its programmatic dependent
      static const bool no_scan_pdl = getenv("VX_DEBUG_NO_SCAN_PDL") != nullptr;  // A/B only
      a.pdl = (!no_scan_pdl && !on_pairs && g0 == 0 && (sample || !seeded) && (bf16 || i8)) ? 1 : 0;
      // 128-document pair tiles (QG = 2) load 64-row document boxes per CTA
      const CUtensorMap* tx;
      if (QG == 2)
        tx = i8 ? &h->tmap_docs8_h : (bf16 ? &h->tmap_docs16_h : &h->tmap_docs_h);
      else
        tx = i8 ? &h->tmap_docs8 : (bf16 ? &h->tmap_docs16 : &h->tmap_docs);
      CUtensorMap txs;  // the sample: every kSeedStride-th row, same boxes
      if (sample) {
        const uint32_t rows = QG == 2 ? 64 : 128;
        if (i8)
          VX_TRY(make_tmap_2d(&txs, h->docs8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1,
                              (uint64_t)n_sample, D, 128, rows, (uint64_t)kSeedStride * D));
        else if (bf16)
          VX_TRY(make_tmap_2d(&txs, h->docs16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                              (uint64_t)n_sample, D, 64, rows, (uint64_t)kSeedStride * D));
        else
          VX_TRY(make_tmap_2d(&txs, h->docs, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                              (uint64_t)n_sample, D, 32, rows, (uint64_t)kSeedStride * D));
        tx = &txs;
      }
      if (on_pairs) {
        // 128 < B: CTA pairs (cta_group::2), 256 documents x 256 QG queries per pair tile
        int ns2 = 0;
        const size_t smem2 = vx::scan_tc2_smem(QG, &ns2);
        a.ns = ns2;
        CU_TRY(vx::launch_scan_tc2(QG, &tq, tx, a, grid, smem2, st));
      } else {
        // 256-document tiles halve the per-document query re-streaming from L2 (measured:
        // B=128 bf16 2.31 ms vs 3.78 ms with 128; B=256 3.9 ms vs 4.36 ms) — profiles/r01/
        const int TD = TD1;
        int ns = 0;
        size_t smem = vx::scan_tc_smem(QT, TD, fmt, &ns);
        if (h->dbg_tc_stages) {  // timing experiments only (VX_DEBUG_TC_STAGES)
          const int want = h->dbg_tc_stages;
          if (want >= 2 && want < ns) {
            smem -= (size_t)(ns - want) * (QT * 16384 + TD * 128 + 16);
            ns = want;
          }
        }
        a.ns = ns;
        // timing experiments only: per-CTA phase stamps of the full pass, summarised on stderr
        static const bool trace = getenv("VX_DEBUG_SCAN_TRACE") != nullptr;
        static uint64_t* d_trace = nullptr;
        if (trace && !sample) {
          if (!d_trace) CU_TRY(cudaMalloc(&d_trace, (size_t)1024 * 16 * 8));
          CU_TRY(cudaMemsetAsync(d_trace, 0, (size_t)grid * 16 * 8, st));
          a.trace = d_trace;
        }
        CU_TRY(vx::launch_scan_tc(QT, TD, &tq, tx, a, grid, smem, st));
        if (trace && !sample) {
          std::vector<uint64_t> tr((size_t)grid * 16);
          CU_TRY(cudaStreamSynchronize(st));
          CU_TRY(cudaMemcpy(tr.data(), d_trace, tr.size() * 8, cudaMemcpyDeviceToHost));
          uint64_t t0 = ~0ull;
          for (int c = 0; c < grid; ++c) t0 = std::min(t0, tr[(size_t)c * 16]);
          const char* names[16] = {"entry", "setup", "first-stage", "last-mma", "epilogue", "end", "end(w2)", "acc-ready", "mb-written", "after-nbar", "merged", "pre-fence", "pre-sync", "epi(w3)", "epi(w4)", "epi(w5)"};
          fprintf(stderr, "[scan trace] B=%d n=%lld grid=%d (us after the first CTA entry: min / median / max)\n",
                  Bg, (long long)a.n_local, grid);
          for (int f = 0; f < 16; ++f) {
            std::vector<double> v;
            for (int c = 0; c < grid; ++c)
              if (tr[(size_t)c * 16 + f]) v.push_back((tr[(size_t)c * 16 + f] - t0) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, "  %-12s %8.2f %8.2f %8.2f\n", names[f], v.front(), v[v.size() / 2], v.back());
          }
        }
      }
      count_launch(h);
    }
    return VX_OK;
  };
  // merge each query's P lists (stride grid lists) to its best kout keys — one launch per
  // run of query groups with the same P (the whole batch when every group ran on CTA pairs)
  auto merge_lists = [&](const uint64_t* lists, int kc, int kout, uint64_t* out,
                         int ldout) -> vx_status {
    const int64_t ld = (int64_t)grid * kc;
    for (int r0 = 0; r0 < B;) {
      const int P = lists_per_query(r0);
      int r1 = r0;
      while (r1 < B && lists_per_query(r1) == P) r1 += GS;
      r1 = std::min(r1, B);
      CU_TRY(vx::launch_merge_topk(lists + (size_t)r0 * ld, r1 - r0, P * kc, kout, 0,
                                   out + (size_t)r0 * ldout, nullptr, nullptr, st, nullptr, ld,
                                   ldout, P, kc));
      count_launch(h);
      r0 = r1;
    }
    return VX_OK;
  };
  if (seeded) {
    VX_TRY(scan_pass(true));
    VX_TRY(merge_lists(sample_lists, vx::kSampleKC, kSeedM, h->d_seedk, kSeedLd));
  }
  VX_TRY(scan_pass(false));
  if (h->nranks > 1 && h->rank == 0) CU_TRY(record_ext(h->pev[5], st));
  // each query's seed key (the certificate bounds what it dropped), stride kSeedLd
  const uint64_t* seed_keys = seeded ? h->d_seedk + (kSeedM - 1) : nullptr;
  CU_TRY(record_scan_ev(h, h->tev[1], st));
  // Certificate failures, entirely on device (no host round trip: the stage stays
  // capturable in one CUDA graph; every launch below exits at once when its count is 0):
  //   level 2: compact the failing queries, re-rank all their list entries above the
  //            deepest truncation point (rerank_wide_kernel) — no index access;
  //   level 3: the queries that still fail are re-scanned exactly (K1 sized by the device
  //            count) and scattered back.
  int* cnt2 = h->d_fcount;      // [count, running total] of level-2 queries
  int* cnt3 = h->d_fcount + 2;  // [count, running total] of exact re-scans
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CU_TRY(cudaStreamIsCapturing(st, &cap));
  const bool captured = cap == cudaStreamCaptureStatusActive;
  // Captured (CUDA graph): the compaction sets a conditional handle, and levels 2-3 are the
  // body of an IF node — a batch whose queries all pass certificate 1 (the common case)
  // replays no level-2/3 launches at all (six ~2.5 us empty launches at B = 16, 100K rows).
  static const bool no_cond = getenv("VX_DEBUG_NO_COND") != nullptr;  // A/B timing only
  cudaGraphConditionalHandle hc = 0;
  if (captured && !no_cond) {
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CU_TRY(cudaStreamGetCaptureInfo(st, &cap, nullptr, &g, &deps, &ndeps));
    CU_TRY(cudaGraphConditionalHandleCreate(&hc, g, 0, cudaGraphCondAssignDefault));
  }
  // exact re-rank (per run of query groups with the same P, so the 2-per-SM re-rank CTAs pack
  // full waves), with the K3 merge of each query's lists to its coarse top-k' fused in front
  // (no merge launch, no candidate round trip) and the compaction of the batch's certificate
  // failures in the last CTA of the last launch (no compaction launch).  Sharded: phase 1
  // re-scores each query's k best coarse candidates, the shards all-gather those exact scores
  // (shard_tau: tau <= the global exact k-th), phase 2 re-ranks only the candidates that can
  // still reach the GLOBAL top-k
  const bool sharded = h->nranks > 1;
  static const bool no_fuse = getenv("VX_DEBUG_NO_FUSE_MERGE") != nullptr;  // A/B timing only
  // small batch (the whole candidate set is the head, launch_rerank: B <= 64) with a large
  // k': S CTAs per query, one wave — a single CTA per query was bound by its serial chains
  // and small bulk copies (B = 1: 1024 rows in one CTA, 69 us of a 97 us re-rank).  The merge
  // then runs as its own launch (every CTA of a query reads the sorted candidates).
  static const bool no_split = getenv("VX_DEBUG_NO_RERANK_SPLIT") != nullptr;  // A/B only
  int split = 1;
  if (!sharded && !no_split && B <= 64 && kp >= 256 &&
      (int64_t)h->desc.max_batch * h->grid * 224 >= (int64_t)B * kp)
    split = std::max(1, std::min(16, h->num_sms / B));
  // (small batches take the merge as its own launch too: fused into the re-rank CTA, whose
  // shared memory holds the whole candidate set, it took ~11 us of a 100K-row B = 16 step
  // against ~5 us + a launch standalone — profiles/r02/rank/fuse_small_batch.txt)
  const bool fuse_merge = !no_fuse && split == 1 && B > 64 &&
                          (int64_t)h->grid * KC <= vx::kMergeSmemKeys;
  if (!fuse_merge) VX_TRY(merge_lists(h->d_part, KC, kp, h->d_ckeys, kp));
  float* lb = reinterpret_cast<float*>(h->d_send);
  for (int pass = sharded ? 1 : 0; pass <= (sharded ? 2 : 0); ++pass) {
    if (pass == 2) VX_TRY(shard_tau(h, lb, B, k, st, true));
    for (int r0 = 0; r0 < B;) {
      const int P = lists_per_query(r0);
      int r1 = r0;
      while (r1 < B && lists_per_query(r1) == P) r1 += GS;
      r1 = std::min(r1, B);
      vx::RerankFuse fz;
      fz.ktimer = ktimer_of(h, vx::KT_RERANK);
      if (split > 1) {
        fz.split = split;
        fz.ekeys = h->d_part + (size_t)h->desc.max_batch * grid * 32;  // the level-2 scratch
        fz.qctr = h->d_qctr;
      }
      // G > 2 shards: each re-scores 2k/G head rows before the tau exchange instead of k (the
      // union of G x 2k/G head scores still holds k distinct exact scores, so tau stays a lower
      // bound of the global k-th; the local bound L is dropped and tau alone prunes the tail)
      if (sharded && h->nranks > 2)
        fz.head = std::min(k, std::max(16, (2 * k + h->nranks - 1) / h->nranks));
      static const bool no_filter = getenv("VX_DEBUG_NO_MERGE_FILTER") != nullptr;
      fz.filter = no_filter ? 0 : 1;
      if (fuse_merge && pass <= 1) {
        fz.mlists = h->d_part + (size_t)r0 * ldp;
        fz.mM = P * KC;
        fz.mld = ldp;
      }
      if (pass != 1 && r1 == B) {
        fz.ctr = h->d_ctr;
        fz.flags_all = h->d_flags;
        fz.Ball = B;
        fz.qall = d_q;
        fz.fidx = h->d_fidx;
        fz.fcount = cnt2;
        fz.fq = h->d_fq;
        fz.cond = (unsigned long long)hc;
        fz.use_cond = captured && !no_cond ? 1 : 0;
      }
      static const bool rtrace = getenv("VX_DEBUG_RERANK_TRACE") != nullptr;
      static uint64_t* d_rtrace = nullptr;
      if (rtrace) {
        if (!d_rtrace) CU_TRY(cudaMalloc(&d_rtrace, (size_t)8192 * 8 * 8));
        CU_TRY(cudaMemsetAsync(d_rtrace, 0, (size_t)(r1 - r0) * 8 * 8, st));
        fz.trace = d_rtrace;
      }
      CU_TRY(vx::launch_rerank(h->docs, d_q + (size_t)r0 * D, D, h->d_ckeys + (size_t)r0 * kp,
                               r1 - r0, kp, h->d_part + (size_t)r0 * ldp, P, grid, KC, k,
                               h->row0, reinterpret_cast<const float*>(h->d_xnorm), fmt,
                               i8 ? h->d_qs8 + r0 : nullptr, keys + (size_t)r0 * k,
                               ids + (size_t)r0 * k, scores + (size_t)r0 * k, h->d_flags + r0,
                               st, pass, pass == 2 ? h->d_tau + r0 : nullptr,
                               sharded ? h->d_hkeys + (size_t)r0 * k : nullptr,
                               lb + (size_t)r0 * k,
                               seed_keys ? seed_keys + (size_t)r0 * kSeedLd : nullptr, kSeedLd,
                               fz));
      count_launch(h);
      if (rtrace) {  // per-CTA phase spans (us): median / max over the launch's CTAs
        std::vector<uint64_t> tr((size_t)(r1 - r0) * 8);
        CU_TRY(cudaStreamSynchronize(st));
        CU_TRY(cudaMemcpy(tr.data(), d_rtrace, tr.size() * 8, cudaMemcpyDeviceToHost));
        const char* names[7] = {"norms", "dependency", "merge", "head", "tail", "sort", "cert+out"};
        uint64_t t0 = ~0ull, t1 = 0;
        for (int c = 0; c < r1 - r0; ++c) {
          t0 = std::min(t0, tr[(size_t)c * 8]);
          t1 = std::max(t1, tr[(size_t)c * 8 + 7]);
        }
        fprintf(stderr, "[rerank trace] pass %d B=%d kp=%d: launch span %.1f us; per CTA (median / max):",
                pass, r1 - r0, kp, (t1 - t0) * 1e-3);
        for (int f = 0; f < 7; ++f) {
          std::vector<double> v;
          for (int c = 0; c < r1 - r0; ++c) {
            const uint64_t a0 = tr[(size_t)c * 8 + f], a1 = tr[(size_t)c * 8 + f + 1];
            if (a0 && a1 && a1 >= a0) v.push_back((a1 - a0) * 1e-3);
          }
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          fprintf(stderr, " %s %.2f/%.2f", names[f], v[v.size() / 2], v.back());
        }
        fprintf(stderr, "\n");
      }
      r0 = r1;
    }
  }
  if (sharded && h->rank == 0) CU_TRY(record_ext(h->pev[6], st));
  // wide-key scratch: the upper part of d_part (the lists use B x grid x KC <= B x grid x 32
  // of its B x grid x 256 entries; the level-3 re-scan writes d_part only after level 2)
  uint64_t* wkeys = h->d_part + (size_t)h->desc.max_batch * grid * 32;
  auto chain = [&](cudaStream_t cs, bool count) -> vx_status {  // levels 2 and 3
    CU_TRY(vx::launch_rerank_wide(h->docs, h->d_fq, D, h->d_fidx, cnt2, h->d_part, B, GS,
                                  pairs ? grid / 2 : 0, grid, KC, k, h->row0,
                                  reinterpret_cast<const float*>(h->d_xnorm), fmt,
                                  i8 ? h->d_qs8 : nullptr, wkeys, keys, ids, scores, h->d_flags, cs,
                                  seed_keys, kSeedLd));
    CU_TRY(vx::launch_cert_compact(h->d_flags, B, d_q, D, h->d_fidx, cnt3, h->d_fq, cs));
    uint64_t* fk = h->d_ckeys;  // reuse: [B][k] (k <= 256)
    int64_t* fi = h->d_out_ids;
    float* fs = h->d_out_ms;
    const uint64_t before = h->st.kernel_launches;
    VX_TRY(local_topk_f32(h, h->d_fq, B, k, fk, fi, fs, cs, cnt3));
    CU_TRY(vx::launch_cert_scatter(h->d_fidx, cnt3, B, k, fk, fi, fs, keys, ids, scores, cs));
    if (count) count_launch(h, 4);
    else h->st.kernel_launches = before;  // conditional body: runs only on a failure
    return VX_OK;
  };
  // eager: every launch below exits at once when its device-side count is 0
  if (!captured || no_cond) return chain(st, true);
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CU_TRY(cudaStreamGetCaptureInfo(st, &cap, nullptr, &g, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CU_TRY(cudaGraphAddNode(&node, g, deps, ndeps, &cp));
  CU_TRY(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CU_TRY(cudaStreamBeginCaptureToGraph(h->stream_cond, body, nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal));
  const vx_status bs = chain(h->stream_cond, false);
  cudaGraph_t out = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(h->stream_cond, &out);
  VX_TRY(bs);
  CU_TRY(ee);
  return VX_OK;
}

static vx_status local_topk(vx_index* h, const float* d_q, int B, int k, uint64_t* keys,
                            int64_t* ids, float* scores, cudaStream_t st) {
  const bool tc = h->scan_algo == VX_SCAN_TC ||
                  (h->scan_algo == VX_SCAN_AUTO && tc_eligible(h, B, k));
  if (tc) {
    if (!tc_eligible(h, B, k)) return fail(VX_ERR_UNSUPPORTED, "tensor-core scan needs k <= 128");
    return local_topk_tc(h, d_q, B, k, keys, ids, scores, st);
  }
  VX_TRY(local_topk_f32(h, d_q, B, k, keys, ids, scores, st));
  // the exact path needs no threshold, but takes part in the exchange whenever a tensor-
  // core rank could be waiting in it (k <= 128), so mixed paths never deadlock
  if (h->nranks > 1 && tc_eligible(h, B, k)) VX_TRY(shard_tau(h, scores, B, k, st, false));
  return VX_OK;
}

// Does the tensor-core MaxSim take the fp32-faithful hi/lo query split for nq tokens?
// (AUTO / TC: yes when nq <= 64; VX_MAXSIM_TC_BF16Q: tokens rounded to bf16.)
static bool maxsim_split(const vx_index* h, int nq) {
  return !h->tokens32 && (h->maxsim_algo == VX_MAXSIM_AUTO || h->maxsim_algo == VX_MAXSIM_TC) &&
         nq <= vx::kMaxSimSplitMaxNq &&
         vx::maxsim_tc_supported(nq, h->desc.tok_per_doc, h->desc.tok_dim);
}

vx_status run_maxsim(vx_index* h, const float* d_qtok, int B, int nq, const int64_t* d_cand,
                     int C, float* d_out, cudaStream_t st, int64_t id_lo, int64_t id_hi,
                     const uint16_t* d_qtok16) {
  if (!has_tokens(h)) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  vx::MaxSimArgs a;
  a.qtok = d_qtok;
  a.qtok16 = d_qtok16;
  a.cand = d_cand;
  a.table = h->tokens;
  a.table32 = h->tokens32;
  a.T = h->desc.tok_blocks;
  a.B = B;
  a.nq = nq;
  a.C = C;
  a.Nd = h->desc.tok_per_doc;
  a.d = h->desc.tok_dim;
  a.out = d_out;
  a.id_lo = id_lo;
  a.id_hi = id_hi;
  if (h->nranks > 1 && id_hi - id_lo < h->desc.n_docs)
    a.own_frac = (float)((double)(id_hi - id_lo) / (double)h->desc.n_docs);
  a.ktimer = ktimer_of(h, vx::KT_MAXSIM);
  const bool tc = !h->tokens32 && h->maxsim_algo != VX_MAXSIM_CC &&
                  vx::maxsim_tc_supported(nq, a.Nd, a.d);
  if ((h->maxsim_algo == VX_MAXSIM_TC || h->maxsim_algo == VX_MAXSIM_TC_BF16Q) && !tc)
    return fail(VX_ERR_UNSUPPORTED, "tensor-core MaxSim unsupported for nq=%d Nd=%d d=%d", nq, a.Nd, a.d);
  a.split = maxsim_split(h, nq) ? 1 : 0;
  a.lo_off = (int64_t)B * nq * a.d;  // the shard exchange's two-plane layout
  if (h->tokens32) {
    if (nq > 32 || a.Nd > 128 || (a.d & 3))
      return fail(VX_ERR_UNSUPPORTED, "fp32 token store MaxSim: nq <= 32, Nd <= 128, d %% 4 == 0");
    CU_TRY(vx::launch_maxsim_f32(a, st));
  } else if (tc) {
    CU_TRY(vx::launch_maxsim_tc(&h->tmap_tok, a, st));
  } else {
    CU_TRY(vx::launch_maxsim(a, st));
  }
  count_launch(h);
  return VX_OK;
}

// ---------------------------------------------------------------- shard exchange

// recv [G][B][k] keys -> [B][G*k] (reusing d_part) for the merge
__global__ void transpose_shard_kernel(const uint64_t* recv, int G, int B, int k, uint64_t* keys) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int total = G * B * k;
  if (i < total) {
    int g = i / (B * k), r = i - g * B * k, b = r / k, j = r - b * k;
    keys[(size_t)b * G * k + g * k + j] = recv[i];
  }
}

// The stage in two parts, shared by rank 0 and the shard ranks:
//   part 1 (core_topk): the certified local top-k by inner product into h->d_keys/d_ids/d_ip;
//     G > 1, phase 1: every shard's local top-k KEYS -> rank 0 (grouped send/recv, 8 B per
//     candidate: a key carries the exact fp32 score and the global id), rank 0 merges to
//     the global top-k in the same buffers;
//   part 2 (core_rescore): MaxSim of the top-k, output order (MaxSim desc, id asc).
//     G > 1, phase 2: rank 0 broadcasts the query tokens and the B x k global winners, each
//     shard computes MaxSim only for the winners it owns (others -INF, no token loads), an
//     NCCL max-reduce to rank 0 assembles the scores.  Every shard does 1/G of the MaxSim
//     work (rescoring each shard's whole local top-k would cost every GPU the full B x k).
// The split lets the host API upload the query tokens while part 1 runs (they are only
// read by part 2).
vx_status core_topk(vx_index* h, const float* d_q, int B, int k, cudaStream_t st) {
  VX_TRY(local_topk(h, d_q, B, k, h->d_keys, h->d_ids, h->d_ip, st));
  if (h->nranks == 1) return VX_OK;
  const int n = B * k;
  const bool root = h->rank == 0;
  if (root) CU_TRY(record_ext(h->pev[2], st));
  const size_t bytes = (size_t)n * 8;
  uint64_t* recv = reinterpret_cast<uint64_t*>(h->d_recv);
  NCCL_TRY(nccl().GroupStart());
  if (root) {
    for (int r = 0; r < h->nranks; ++r) {
      if (r == 0)
        CU_TRY(cudaMemcpyAsync(recv, h->d_keys, bytes, cudaMemcpyDeviceToDevice, st));
      else
        NCCL_TRY(nccl().Recv(recv + (size_t)r * n, bytes, ncclUint8, r, h->comm, st));
    }
  } else {
    NCCL_TRY(nccl().Send(h->d_keys, bytes, ncclUint8, 0, h->comm, st));
  }
  NCCL_TRY(nccl().GroupEnd());
  if (!root) return VX_OK;
  const int G = h->nranks;
  transpose_shard_kernel<<<(G * n + 255) / 256, 256, 0, st>>>(recv, G, B, k, h->d_part);
  count_launch(h);
  CU_TRY(cudaGetLastError());
  // keys already carry global ids: id_base 0
  // the shards' top-k lists are each descending: G lists of k keys
  CU_TRY(vx::launch_merge_topk(h->d_part, B, G * k, k, 0, h->d_keys, h->d_ids, h->d_ip, st,
                               nullptr, 0, 0, G, k));
  count_launch(h);
  CU_TRY(record_ext(h->pev[3], st));
  return VX_OK;
}

static vx_status gather_order(vx_index* h, int B, int k, int n, int64_t* d_ids, float* d_ip,
                              float* d_ms, cudaStream_t st);

// d_qtok: rank 0's query tokens (ignored on the shard ranks, which receive them)
vx_status core_rescore(vx_index* h, const float* d_qtok, int B, int nq, int k,
                              int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st) {
  if (h->nranks == 1) {
    VX_TRY(run_maxsim(h, d_qtok, B, nq, h->d_ids, k, h->d_ms, st));
    CU_TRY(vx::launch_order_by(h->d_ms, h->d_ids, h->d_ip, B, k, d_ids, d_ip, d_ms, st));
    count_launch(h);
    return VX_OK;
  }
  const int n = B * k;
  const bool root = h->rank == 0;
  // the tokens travel in the MaxSim operand format: bf16 hi + lo planes for the fp32-faithful
  // tensor-core kernel (the fp32 bytes), else one bf16 plane (the kernels round fp32 tokens
  // with the same RNE anyway, so the scores are unchanged) — half the broadcast bytes
  const int64_t ntok = (int64_t)B * nq * h->desc.tok_dim;
  if (h->tokens32) {
    // fp32 token store: the fp32 query tokens travel as they are (the CUDA-core MaxSim keeps
    // them unrounded), into every rank's d_qtok
    if (root && d_qtok != h->d_qtok)
      CU_TRY(cudaMemcpyAsync(h->d_qtok, d_qtok, (size_t)ntok * 4, cudaMemcpyDeviceToDevice, st));
    NCCL_TRY(nccl().GroupStart());
    NCCL_TRY(nccl().Broadcast(h->d_qtok, h->d_qtok, (size_t)ntok, ncclFloat32, 0, h->comm, st));
    NCCL_TRY(nccl().Broadcast(h->d_ids, h->d_ids, (size_t)n, ncclInt64, 0, h->comm, st));
    NCCL_TRY(nccl().GroupEnd());
    if (root) CU_TRY(record_ext(h->pev[7], st));
    VX_TRY(run_maxsim(h, h->d_qtok, B, nq, h->d_ids, k, h->d_ms, st, h->row0,
                      h->row0 + h->n_local));
    if (root) CU_TRY(record_ext(h->pev[8], st));
    return gather_order(h, B, k, n, d_ids, d_ip, d_ms, st);
  }
  const int64_t nplanes = maxsim_split(h, nq) ? 2 : 1;
  if (root) {
    if (nplanes == 2)
      CU_TRY(vx::launch_split_bf16(d_qtok, h->d_qtok16, ntok, st));
    else
      CU_TRY(vx::launch_to_bf16(d_qtok, h->d_qtok16, ntok, st));
    count_launch(h);
  }
  NCCL_TRY(nccl().GroupStart());
  NCCL_TRY(nccl().Broadcast(h->d_qtok16, h->d_qtok16, (size_t)(ntok * nplanes) * 2, ncclUint8, 0,
                            h->comm, st));
  NCCL_TRY(nccl().Broadcast(h->d_ids, h->d_ids, (size_t)n, ncclInt64, 0, h->comm, st));
  NCCL_TRY(nccl().GroupEnd());
  if (root) CU_TRY(record_ext(h->pev[7], st));
  VX_TRY(run_maxsim(h, nullptr, B, nq, h->d_ids, k, h->d_ms, st, h->row0, h->row0 + h->n_local,
                    h->d_qtok16));
  if (root) CU_TRY(record_ext(h->pev[8], st));
  return gather_order(h, B, k, n, d_ids, d_ip, d_ms, st);
}

// every winner has one owner (the others hold -inf): the shards' score arrays go to rank 0 in
// one grouped send / receive step and the order kernel takes their max (no NCCL max-reduce)
static vx_status gather_order(vx_index* h, int B, int k, int n, int64_t* d_ids, float* d_ip,
                              float* d_ms, cudaStream_t st) {
  const bool root = h->rank == 0;
  const int G = h->nranks;
  float* ms_all = reinterpret_cast<float*>(h->d_recv);  // [G][B][k] on rank 0 (phase 1 is done)
  NCCL_TRY(nccl().GroupStart());
  if (root) {
    CU_TRY(cudaMemcpyAsync(ms_all, h->d_ms, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    for (int r = 1; r < G; ++r)
      NCCL_TRY(nccl().Recv(ms_all + (size_t)r * n, (size_t)n, ncclFloat32, r, h->comm, st));
  } else {
    NCCL_TRY(nccl().Send(h->d_ms, (size_t)n, ncclFloat32, 0, h->comm, st));
  }
  NCCL_TRY(nccl().GroupEnd());
  if (!root) return VX_OK;
  CU_TRY(vx::launch_order_by(ms_all, h->d_ids, h->d_ip, B, k, d_ids, d_ip, d_ms, st, G, (size_t)n));
  count_launch(h);
  return VX_OK;
}

// CUDA-graph mode (VX_OPT_GRAPHS): each part for one (B, k[, nq]) is captured once and
// replayed — one launch per part instead of ~12 kernels, no host work between the kernels
// (the batcher hands each batch to the graphs of its size, north star (e)).  The graphs read
// the handle's fixed input buffers and write its fixed output buffers; user pointers are copied
// in/out around the replay.  The first batch of a shape runs the part eagerly (it also sets
// the kernels' smem attributes) and captures it for the next ones.
// Sharded (G > 1): EVERY rank captures the same parts — part 1 = the NCCL broadcast of the
// queries + the local certified top-k with its threshold all-gather + the key gather to rank
// 0; part 2 = the token / winner broadcast, the owner MaxSim and the max-reduce — so the
// collectives inside the graphs match rank for rank.  Only the 16-byte batch header travels
// outside a graph (the shard ranks need B to pick the graph).
enum { PART_TOPK = 1, PART_RESCORE = 2 };

static vx_status part_body(vx_index* h, int part, int B, int nq, int k, cudaStream_t st) {
  if (part == PART_TOPK) {
    CU_TRY(record_ev(h, h->tev[2], st));
    if (h->nranks > 1) {
      NCCL_TRY(nccl().Broadcast(h->d_q, h->d_q, (size_t)B * h->desc.dim, ncclFloat32, 0, h->comm, st));
      if (h->rank == 0) CU_TRY(record_ext(h->pev[1], st));
    }
    VX_TRY(core_topk(h, h->d_q, B, k, st));
  } else {
    VX_TRY(core_rescore(h, h->rank == 0 ? h->d_qtok : nullptr, B, nq, k, h->d_out_ids,
                        h->d_out_ip, h->d_out_ms, st));
  }
  CU_TRY(record_ev(h, h->tev[3], st));
  return VX_OK;
}

static uint64_t part_key(int part, int B, int nq, int k) {
  return ((uint64_t)part << 48) | ((uint64_t)B << 24) | ((uint64_t)k << 12) |
         (uint64_t)(part == PART_RESCORE ? nq : 0);
}

vx_status run_part(vx_index* h, int part, int B, int nq, int k, cudaStream_t st) {
  const uint64_t key = part_key(part, B, nq, k);
  cudaEvent_t* used;
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    CU_TRY(cudaGraphLaunch(it->second.exec, st));
    h->st.kernel_launches += it->second.launches;
    h->st.graph_replays += 1;
    used = h->gev;
    h->step_ev_valid = it->second.events;
  } else {
    VX_TRY(part_body(h, part, B, nq, k, st));
    h->step_ev_valid = true;
    // capture on the handle's stream after the eager run completes (capture records, it
    // does not execute; sharded, every rank captures at the same batch)
    CU_TRY(cudaStreamSynchronize(st));
    const uint64_t before = h->st.kernel_launches;
    h->tev = h->gev;  // the graph records its own (external) events
    h->graph_events = false;
    CU_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    vx_status s = part_body(h, part, B, nq, k, h->stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    h->tev = h->ev;
    const int launches = (int)(h->st.kernel_launches - before);
    h->st.kernel_launches = before;
    if (s != VX_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    if (e != cudaSuccess) return fail(VX_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(VX_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    h->graphs[key] = {ex, launches, h->graph_events};
    used = h->ev;  // this call's timing: the eager run
  }
  if (part == PART_TOPK) h->ev_start = used;
  h->ev_end = used;
  return VX_OK;
}

static void stage_done(vx_index* h, int B);

// One GPU, graphs on: the whole stage (top-k [+ MaxSim and order]) as ONE graph captured
// against the caller's buffers (vx_index::io_graphs).  *done = false: not taken (sharded,
// graphs off, first sighting of these buffers, or the per-shape budget spent) — the caller
// runs the two-part path with its copies.
vx_status stage_direct(vx_index* h, int op, const float* d_q, const float* d_qtok, int B, int nq,
                       int k, int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st,
                       bool* done) {
  *done = false;
  if (!h->use_graphs || h->nranks > 1) return VX_OK;
  // d_out_ids / d_out_ms are the certificate chain's level-3 scratch: never the direct outputs
  if ((void*)d_ids == (void*)h->d_out_ids || (void*)d_ip == (void*)h->d_out_ms ||
      (void*)d_ms == (void*)h->d_out_ms)
    return VX_OK;
  const bool rescore = op == OP_RESCORE;
  vx_index::IoKey key{part_key(rescore ? 4 : 3, B, nq, k),
                      {(uintptr_t)d_q, (uintptr_t)d_qtok, (uintptr_t)d_ids, (uintptr_t)d_ip,
                       (uintptr_t)d_ms}};
  auto it = h->io_graphs.find(key);
  if (it == h->io_graphs.end()) {
    int& per = h->io_per_shape[key.shape];
    if (per >= vx_index::kIoGraphsPerShape) return VX_OK;
    int& seen = h->io_seen[key];
    if (seen++ == 0) {
      if (h->io_seen.size() > 64) h->io_seen.clear();  // bounded: one-off buffers
      return VX_OK;
    }
    // capture (the eager run of this shape already happened on the first sighting)
    CU_TRY(cudaStreamSynchronize(st));
    CU_TRY(cudaStreamSynchronize(h->stream));
    const uint64_t before = h->st.kernel_launches;
    h->tev = h->gev;
    h->graph_events = false;
    CU_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    vx_status s = VX_OK;
    {
      cudaStream_t cs = h->stream;
      s = record_ev(h, h->tev[2], cs) == cudaSuccess ? VX_OK : fail(VX_ERR_CUDA, "event");
      if (s == VX_OK) {
        if (rescore) {
          s = core_topk(h, d_q, B, k, cs);
          if (s == VX_OK) s = core_rescore(h, d_qtok, B, nq, k, d_ids, d_ip, d_ms, cs);
        } else {
          s = local_topk(h, d_q, B, k, h->d_keys, d_ids, d_ip, cs);
        }
      }
      if (s == VX_OK && record_ev(h, h->tev[3], cs) != cudaSuccess) s = fail(VX_ERR_CUDA, "event");
    }
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    h->tev = h->ev;
    const int launches = (int)(h->st.kernel_launches - before);
    h->st.kernel_launches = before;
    if (s != VX_OK) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    if (e != cudaSuccess) return fail(VX_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(VX_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
    it = h->io_graphs.emplace(key, vx_index::GraphEntry{ex, launches, h->graph_events}).first;
    h->io_seen.erase(key);
    ++per;
  }
  // the capture stream and the caller's stream: the replay runs on the caller's
  CU_TRY(cudaGraphLaunch(it->second.exec, st));
  h->st.kernel_launches += it->second.launches;
  h->st.graph_replays += 1;
  h->ev_start = h->ev_end = h->gev;
  h->step_ev_valid = it->second.events;
  h->stream_last = st;
  stage_done(h, B);
  *done = true;
  return VX_OK;
}

// Rank 0 entry, part 1: announce the batch to the shards (header), then broadcast + top-k.
vx_status stage_begin(vx_index* h, int op, const float* d_q, int B, int nq, int k,
                      cudaStream_t st) {
  if (h->nranks > 1) {
    if (h->rank != 0) return fail(VX_ERR_STATE, "only rank 0 issues searches; call vx_shard_serve");
    h->h_hdr[0] = op;
    h->h_hdr[1] = B;
    h->h_hdr[2] = k;
    h->h_hdr[3] = nq;
    CU_TRY(cudaEventRecord(h->pev[0], st));
    CU_TRY(cudaMemcpyAsync(h->d_hdr, h->h_hdr, 16, cudaMemcpyHostToDevice, st));
    NCCL_TRY(nccl().Broadcast(h->d_hdr, h->d_hdr, 4, ncclInt32, 0, h->comm, st));
  }
  if (h->use_graphs) {
    if (d_q != h->d_q)
      CU_TRY(cudaMemcpyAsync(h->d_q, d_q, (size_t)B * h->desc.dim * 4, cudaMemcpyDeviceToDevice,
                             st));
    VX_TRY(run_part(h, PART_TOPK, B, nq, k, st));
  } else {
    CU_TRY(record_ev(h, h->tev[2], st));
    if (h->nranks > 1) {
      NCCL_TRY(nccl().Broadcast(d_q, h->d_q, (size_t)B * h->desc.dim, ncclFloat32, 0, h->comm, st));
      CU_TRY(cudaEventRecord(h->pev[1], st));
    }
    VX_TRY(core_topk(h, h->nranks > 1 ? h->d_q : d_q, B, k, st));
    CU_TRY(record_ev(h, h->tev[3], st));
    h->ev_start = h->ev_end = h->ev;
    h->step_ev_valid = true;
  }
  return VX_OK;
}

static void stage_done(vx_index* h, int B) {
  if (h->stream_last && h->stream_last != h->stream) {  // the caller's stream: vx_sync waits
    cudaEventRecord(h->ev_done, h->stream_last);
    h->done_pending = true;
  }
  if (h->nranks > 1 && h->rank == 0) {
    cudaEventRecord(h->pev[4], h->stream_last);
    h->phases_pending = true;
  }
  h->timing_pending = true;
  h->st.batches += 1;
  h->st.queries += B;
}

// part 2 of a search (no rescore): the top-k by inner product to the caller's buffers
vx_status stage_search_out(vx_index* h, int B, int k, int64_t* d_ids, float* d_ip,
                                  cudaStream_t st) {
  const size_t n = (size_t)B * k;
  CU_TRY(cudaMemcpyAsync(d_ids, h->d_ids, n * 8, cudaMemcpyDeviceToDevice, st));
  CU_TRY(cudaMemcpyAsync(d_ip, h->d_ip, n * 4, cudaMemcpyDeviceToDevice, st));
  h->stream_last = st;
  stage_done(h, B);
  return VX_OK;
}

// part 2 of the fused stage: MaxSim rescore + order into the caller's buffers
vx_status stage_finish(vx_index* h, const float* d_qtok, int B, int nq, int k,
                              int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st) {
  if (h->use_graphs) {
    if (d_qtok != h->d_qtok)
      CU_TRY(cudaMemcpyAsync(h->d_qtok, d_qtok, (size_t)B * nq * h->desc.tok_dim * 4,
                             cudaMemcpyDeviceToDevice, st));
    VX_TRY(run_part(h, PART_RESCORE, B, nq, k, st));
    const size_t n = (size_t)B * k;
    if (d_ids != h->d_out_ids)
      CU_TRY(cudaMemcpyAsync(d_ids, h->d_out_ids, n * 8, cudaMemcpyDeviceToDevice, st));
    if (d_ip != h->d_out_ip)
      CU_TRY(cudaMemcpyAsync(d_ip, h->d_out_ip, n * 4, cudaMemcpyDeviceToDevice, st));
    if (d_ms != h->d_out_ms)
      CU_TRY(cudaMemcpyAsync(d_ms, h->d_out_ms, n * 4, cudaMemcpyDeviceToDevice, st));
  } else {
    VX_TRY(core_rescore(h, d_qtok, B, nq, k, d_ids, d_ip, d_ms, st));
    CU_TRY(record_ev(h, h->tev[3], st));
    h->ev_end = h->ev;
  }
  h->stream_last = st;
  stage_done(h, B);
  return VX_OK;
}

extern "C" vx_status vx_search_dev(vx_index* h, const float* d_q, int32_t B, int32_t k,
                                   int64_t* d_ids, float* d_scores, void* stream) {
  if (!h || !d_q || !d_ids || !d_scores) return fail(VX_ERR_INVALID, "null argument");
  VX_TRY(check_batch(h, B, k));
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = pick_stream(h, stream);
  bool done = false;
  VX_TRY(stage_direct(h, OP_SEARCH, d_q, nullptr, B, 0, k, d_ids, d_scores, nullptr, st, &done));
  if (done) return VX_OK;
  VX_TRY(stage_begin(h, OP_SEARCH, d_q, B, 0, k, st));
  return stage_search_out(h, B, k, d_ids, d_scores, st);
}

extern "C" vx_status vx_search_rescore_dev(vx_index* h, const float* d_q, const float* d_qtok,
                                           int32_t B, int32_t nq, int32_t k, int64_t* d_ids,
                                           float* d_ip, float* d_ms, void* stream) {
  if (!h || !d_q || !d_qtok || !d_ids || !d_ip || !d_ms) return fail(VX_ERR_INVALID, "null argument");
  VX_TRY(check_batch(h, B, k));
  if (!has_tokens(h)) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = pick_stream(h, stream);
  bool done = false;
  VX_TRY(stage_direct(h, OP_RESCORE, d_q, d_qtok, B, nq, k, d_ids, d_ip, d_ms, st, &done));
  if (done) return VX_OK;
  VX_TRY(stage_begin(h, OP_RESCORE, d_q, B, nq, k, st));
  return stage_finish(h, d_qtok, B, nq, k, d_ids, d_ip, d_ms, st);
}

extern "C" vx_status vx_maxsim_dev(vx_index* h, const float* d_qtok, int32_t B, int32_t nq,
                                   const int64_t* d_cand, int32_t C, float* d_out, void* stream) {
  if (!h || !d_qtok || !d_cand || !d_out) return fail(VX_ERR_INVALID, "null argument");
  if (B < 1 || B > h->desc.max_batch || C < 1) return fail(VX_ERR_INVALID, "B %d C %d", B, C);
  CU_TRY(cudaSetDevice(h->device));
  return run_maxsim(h, d_qtok, B, nq, d_cand, C, d_out, pick_stream(h, stream));
}

extern "C" vx_status vx_prepare(vx_index* h, int32_t op, int32_t k, int32_t nq, int32_t b_max) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (op != VX_PREPARE_SEARCH && op != VX_PREPARE_RESCORE) return fail(VX_ERR_INVALID, "op %d", op);
  VX_TRY(check_batch(h, b_max, k));
  const bool rescore = op == VX_PREPARE_RESCORE;
  if (rescore && (!has_tokens(h) || nq < 1 || nq > h->desc.max_qtok))
    return fail(VX_ERR_INVALID, "rescore needs a token store and 1 <= nq <= max_qtok");
  if (!h->use_graphs) return VX_OK;
  if (h->nranks > 1 && h->rank != 0)
    return fail(VX_ERR_STATE, "vx_prepare is issued by rank 0 (the shard ranks capture in vx_shard_serve)");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  // realistic inputs (generator rows), so every eager run takes the certified fast path
  CU_TRY(vx::launch_synth_rows(h->d_q, 0x5eedull, 0, b_max, h->desc.dim, st));
  if (rescore)
    CU_TRY(vx::launch_synth_rows(h->d_qtok, 0x5eed1ull, 0, (int64_t)b_max * nq, h->desc.tok_dim, st));
  const vx_stats saved = h->st;
  for (int B = 1; B <= b_max; ++B) {
    const bool have1 = h->graphs.count(part_key(PART_TOPK, B, 0, k)) != 0;
    const bool have2 = !rescore || h->graphs.count(part_key(PART_RESCORE, B, nq, k)) != 0;
    if (have1 && have2) continue;
    if (h->nranks > 1) {
      // a real (synthetic) batch through the protocol: the shard ranks, serving, run and
      // capture their parts of it at the same batch
      VX_TRY(stage_begin(h, rescore ? OP_RESCORE : OP_SEARCH, h->d_q, B, nq, k, st));
      if (rescore)
        VX_TRY(stage_finish(h, h->d_qtok, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
      else
        VX_TRY(stage_search_out(h, B, k, h->d_out_ids, h->d_out_ip, st));
      continue;
    }
    if (!have1) VX_TRY(run_part(h, PART_TOPK, B, 0, k, st));
    if (!have2) VX_TRY(run_part(h, PART_RESCORE, B, nq, k, st));
  }
  CU_TRY(cudaStreamSynchronize(st));
  h->st = saved;  // preload work is not serving work
  VX_TRY(ktimer_reset(h));
  h->timing_pending = false;
  h->phases_pending = false;
  return VX_OK;
}

extern "C" vx_status vx_sync(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  CU_TRY(cudaSetDevice(h->device));
  // the certificate counters and the device timers come back with the wait itself (one async
  // copy into pinned memory each, one synchronize: two blocking cudaMemcpy calls here took
  // ~15-20 us of every host-API batch)
  if (h->done_pending) {
    CU_TRY(cudaStreamWaitEvent(h->stream, h->ev_done, 0));
    h->done_pending = false;
  }
  uint8_t* hs = static_cast<uint8_t*>(h->h_sync);
  CU_TRY(cudaMemcpyAsync(hs, h->d_fcount, 16 + sizeof(vx::KTimer) * vx::KT_N,
                         cudaMemcpyDeviceToHost, h->stream));  // counters + timers: adjacent
  CU_TRY(cudaStreamSynchronize(h->stream));
  if (h->timing_pending) {
    cudaEvent_t* E = h->ev_start;
    cudaEvent_t* F = h->ev_end;
    if (h->step_ev_valid) CU_TRY(cudaEventSynchronize(F[3]));
    float a = 0, b = 0;
    if (!h->step_ev_valid) {
      h->st.last_step_ms = -1.0f;  // a replay without stage events (VX_OPT_STAGE_EVENTS 0)
      h->st.last_scan_ms = -1.0f;
    } else if (cudaEventElapsedTime(&b, E[2], F[3]) == cudaSuccess) {
      // the scan span: events on eager runs, else the scan kernels' device timers
      if (!(h->scan_ev_valid && cudaEventElapsedTime(&a, h->ev[0], h->ev[1]) == cudaSuccess))
        a = -1.0f;
      h->st.last_scan_ms = a;
      h->st.last_step_ms = b;
      if (a >= 0) h->st.scan_ms_total += a;
      h->st.step_ms_total += b;
      h->st.timed_batches += 1;
    }
    h->scan_ev_valid = false;
    h->timing_pending = false;
    if (h->phases_pending) {
      for (int i = 0; i < 4; ++i) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, h->pev[i], h->pev[i + 1]) == cudaSuccess)
          h->st.phase_ms[i] = ms;
      }
      // finer: bcast done -> scan done -> re-rank done -> local done; gather done -> phase-2
      // bcast done -> MaxSim done -> end
      const int from[6] = {1, 5, 6, 3, 7, 8}, to[6] = {5, 6, 2, 7, 8, 4};
      for (int i = 0; i < 6; ++i) {
        float ms = -1.0f;
        if (cudaEventElapsedTime(&ms, h->pev[from[i]], h->pev[to[i]]) != cudaSuccess) ms = -1.0f;
        h->st.phase_detail_ms[i] = ms;
      }
      h->phases_pending = false;
    }
    int fc[4] = {0, 0, 0, 0};  // certificate levels counted on device
    memcpy(fc, hs, 16);
    h->st.cert_level2 = (uint64_t)fc[1];
    h->st.cert_fallbacks = (uint64_t)fc[3];
    maybe_demote_i8(h, fc, h->st.queries);
  }
  vx::KTimer kt[vx::KT_N];  // device-side launch timers (every launch since the last reset)
  memcpy(kt, hs + 16, sizeof kt);
  for (int i = 0; i < 4; ++i) {  // the ABI's four kinds
    h->st.kt_launches[i] = kt[i].launches;
    h->st.kt_ms[i] = (double)kt[i].total_ns * 1e-6;
    h->st.kt_sm_mhz[i] = kt[i].clk_ns ? (double)kt[i].clk_cycles * 1e3 / (double)kt[i].clk_ns : 0.0;
  }
  h->st.kt_rerank_launches = kt[vx::KT_RERANK].launches;
  h->st.kt_rerank_ms = (double)kt[vx::KT_RERANK].total_ns * 1e-6;
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < vx::KT_N; ++i)
    if (kt[i].launches && kt[i].last_start < t0) t0 = kt[i].last_start;
  for (int i = 0; i < vx::KT_N; ++i) {
    const bool on = kt[i].launches && t0 != ~0ull;
    h->st.kt_last_us[2 * i] = on ? (double)(kt[i].last_start - t0) * 1e-3 : 0.0;
    h->st.kt_last_us[2 * i + 1] = on ? (double)(kt[i].last_end - t0) * 1e-3 : 0.0;
  }
  h->st.kt_origin_ns = t0 != ~0ull ? t0 : 0ull;
  cudaGetLastError();
  return VX_OK;
}

