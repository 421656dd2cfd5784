// vx_ptx.cuh — sm_100a PTX helpers: mbarriers, TMA (cp.async.bulk[.tensor]),
// tcgen05 (TMEM alloc / MMA / commit / ld), UMMA descriptors, warp top-k helpers.
// Bitfield layouts follow the PTX ISA tcgen05 "shared memory descriptor" and
// "instruction descriptor" tables (cross-checked against CUTLASS 4.5
// cute/arch/mma_sm100_desc.hpp, vendored under flashinfer/data/cutlass).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "vx_internal.cuh"  // FMT_* operand formats

#define VX_DEV __device__ __forceinline__

namespace vx {

VX_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

VX_DEV uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

VX_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
VX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
VX_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
VX_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

VX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
VX_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
VX_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
VX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---------------------------------------------------------------- TMA
VX_DEV void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 2-D tiled tensor load into smem, completion via mbarrier transaction bytes.
VX_DEV void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1,
                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// Programmatic dependent launch: a kernel launched with the PDL attribute may start while its
// predecessor still runs; pdl_wait() blocks until the predecessor grid has completed and its
// memory is visible (a no-op without the attribute); pdl_trigger() lets the dependent grid be
// scheduled as soon as every CTA of this grid has issued it (or exited).
VX_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
VX_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
// L2 prefetch of one 128-byte line (no register result, fire and forget).
VX_DEV void prefetch_l2(const void* g) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(reinterpret_cast<uint64_t>(g)));
}
// 1-D bulk copy global -> smem (16 B aligned, size multiple of 16).
VX_DEV void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Per-thread 16-byte async copy global -> smem (L1 bypass), grouped completion.
VX_DEV void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(reinterpret_cast<uint64_t>(gsrc))
               : "memory");
}
VX_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
VX_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
VX_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
VX_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- named barriers
VX_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- tcgen05
// TMEM allocation: executed by one full warp; writes the TMEM base address to smem.
VX_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
VX_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
VX_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
VX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32 (fp32 operands, TF32 math, fp32 accumulate)
VX_DEV void mma_tf32_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::f16 (bf16/fp16 operands, fp32 accumulate)
VX_DEV void mma_f16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
VX_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread.
VX_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 32 lanes x 32 bit, 32 consecutive columns -> 32 registers per thread.
VX_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
VX_DEV void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}
VX_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major operand, SWIZZLE_128B canonical layout:
// rows of 128 B, 8-row core groups 1024 B apart (SBO), LBO unused (=1), version 1.
VX_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);          // start address [0,14)
  d |= (uint64_t)1u << 16;                              // LBO (ignored for swizzled K-major)
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;        // SBO [32,46)
  d |= (uint64_t)1u << 46;                              // version = 1 (sm_100)
  d |= (uint64_t)2u << 61;                              // layout: SWIZZLE_128B
  return d;
}

// Instruction descriptor (kind::f16 / kind::tf32): fp32 accumulate, A/B K-major.
//   c_format [4,6)=1 (F32); a_format [7,10); b_format [10,13); n_dim [17,23)=N>>3;
//   m_dim [24,29)=M>>4.   Formats: 0=F16, 1=BF16, 2=TF32.
__host__ __device__ constexpr uint32_t make_idesc(uint32_t fmt, uint32_t M, uint32_t N) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// ---------------------------------------------------------------- clusters / CTA pairs
VX_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
VX_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`
VX_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Default .release.cta semantics (as CUTLASS's ClusterBarrier::arrive): the arrive only has
// to order this thread's completed tcgen05.ld (tcgen05.fence::before_thread_sync) before the
// peer's MMA, not publish generic memory at cluster scope — .release.cluster compiled to
// MEMBAR.ALL.GPU + ERRBAR, ~15 % of the scan epilogue's stall samples.
VX_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// TMA load issued by either CTA of a pair; completion bytes go to the mbarrier at
// `bar_cluster_addr` (the leader's), data to this CTA's smem.
VX_DEV void tma_load_2d_pair(void* smem_dst, const void* tmap, uint32_t bar_cluster_addr, int32_t c0,
                             int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes."
      "L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar_cluster_addr), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
VX_DEV void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
VX_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// 2-SM MMA (issued by the pair's leader): A rows split across the two CTAs (M = 256), B rows
// (the N dimension) split across the two CTAs; D: each CTA's TMEM holds its 128 rows.
VX_DEV void mma_pair(uint32_t kind_tf32, uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                     uint32_t idesc, uint32_t accumulate) {
  if (kind_tf32)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// kind::i8 (s8 x s8, exact s32 accumulate; K = 32 per instruction = the same 32 bytes of K
// per row as bf16's K = 16)
VX_DEV void mma_i8_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
VX_DEV void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Instruction descriptor per format: f32 accumulate for bf16 / tf32, s32 for s8 x s8.
//   c_format [4,6) (1 = F32, 2 = S32); a/b_format [7,10)/[10,13) (BF16 = 1, TF32 = 2;
//   for kind::i8: 1 = signed 8-bit).
__host__ __device__ constexpr uint32_t make_idesc_fmt(int fmt, uint32_t M, uint32_t N) {
  return fmt == FMT_I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24))
                       : make_idesc(fmt == FMT_TF32 ? 2u : 1u, M, N);
}

// Compile-time operand kind (no per-MMA runtime select in the issue loop).
template <int FMT>
VX_DEV void mma_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                   uint32_t accumulate) {
  if constexpr (FMT == FMT_TF32)
    mma_tf32_ss(d_tmem, adesc, bdesc, idesc, accumulate);
  else if constexpr (FMT == FMT_I8)
    mma_i8_ss(d_tmem, adesc, bdesc, idesc, accumulate);
  else
    mma_f16_ss(d_tmem, adesc, bdesc, idesc, accumulate);
}
template <int FMT>
VX_DEV void mma_pair_k(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                       uint32_t accumulate) {
  if constexpr (FMT == FMT_I8)
    mma_i8_pair(d_tmem, adesc, bdesc, idesc, accumulate);
  else
    mma_pair(FMT == FMT_TF32 ? 1u : 0u, d_tmem, adesc, bdesc, idesc, accumulate);
}
// TMEM accumulator word -> coarse score (s32 products are exact; |sum| < 2^24 converts exactly)
template <int FMT>
VX_DEV float acc_score(uint32_t w) {
  if constexpr (FMT == FMT_I8)
    return __int2float_rn((int)w);
  else
    return __uint_as_float(w);
}
// Max of a 32-column accumulator chunk as a score, as a balanced tree; for s32 accumulators the
// max is taken on the integers (IMNMX) and only the winner is converted — the per-chunk filter
// of the scan epilogues runs on every column, so this is their common-case cost.
template <int FMT>
VX_DEV float chunk_max32(const uint32_t (&r)[32]) {
  if constexpr (FMT == FMT_I8) {
    int m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = max((int)r[2 * i], (int)r[2 * i + 1]);
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1)
#pragma unroll
      for (int i = 0; i < s; ++i) m[i] = max(m[i], m[i + s]);
    return __int2float_rn(m[0]);
  } else {
    float m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) m[i] = fmaxf(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1)
#pragma unroll
      for (int i = 0; i < s; ++i) m[i] = fmaxf(m[i], m[i + s]);
    return m[0];
  }
}
// Warp index the compiler can prove warp-uniform (so role branches and the MMA issue loop
// live on the uniform datapath instead of per-thread registers + R2UR waterfalls).
VX_DEV int warp_idx_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

// Commit the leader's MMAs to the mbarrier at the same offset in every CTA of `mask`.
VX_DEV void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// ---------------------------------------------------------------- warp top-k helpers
// In-smem bitonic sort (descending) of n = power of two u64 keys by one warp.
VX_DEV void warp_bitonic_desc(uint64_t* buf, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = lane; i < (n >> 1); i += 32) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc = (lo & size) == 0;
        uint64_t a = buf[lo], b = buf[hi];
        if ((a < b) == desc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncwarp();
    }
  }
}

// ---- device-side launch timing (KTimer, vx_internal.cuh); thread 0 of every CTA
VX_DEV uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// every CTA's start; the launch's is their minimum (a reduction, no return)
VX_DEV void ktimer_begin(KTimer* t, uint64_t& c0, uint64_t& g0) {
  if (!t || threadIdx.x != 0) return;
  g0 = gtimer_ns();
  c0 = clock64();
  atomicMin(&t->start, (unsigned long long)g0);
}
// after the CTA's last work (its final barrier).  The end stamp is a reduction (no return);
// the arrival is ONE acquire-release atomic (it publishes this CTA's stamp and, for the last
// CTA, acquires everyone's); the last CTA's fold issues its two loads together and only
// reductions / relaxed stores after them.
VX_DEV void ktimer_end(KTimer* t, uint64_t c0, uint64_t g0) {
  if (!t || threadIdx.x != 0) return;
  const uint64_t g1 = gtimer_ns(), c1 = clock64();
  atomicMax(&t->end, (unsigned long long)g1);
  if (blockIdx.x == 0) {
    atomicAdd(&t->clk_cycles, (unsigned long long)(c1 - c0));
    atomicAdd(&t->clk_ns, (unsigned long long)(g1 - g0));
  }
  const unsigned long long n = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
  unsigned long long prev;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(prev) : "l"(&t->done) : "memory");
  if (prev == n - 1) {  // last CTA: fold this launch, re-arm the slot
    unsigned long long s, e;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%2];\n\tld.relaxed.gpu.global.u64 %1, [%3];"
                 : "=l"(s), "=l"(e) : "l"(&t->start), "l"(&t->end) : "memory");
    atomicAdd(&t->total_ns, e - s);
    atomicAdd(&t->launches, 1ull);
    asm volatile(
        "st.relaxed.gpu.global.u64 [%0], %1;\n\tst.relaxed.gpu.global.u64 [%2], %3;\n\t"
        "st.relaxed.gpu.global.u64 [%4], %5;\n\tst.relaxed.gpu.global.u64 [%6], %7;\n\t"
        "st.relaxed.gpu.global.u64 [%8], %9;"
        :: "l"(&t->last_start), "l"(s), "l"(&t->last_end), "l"(e), "l"(&t->start), "l"(~0ull),
           "l"(&t->end), "l"(0ull), "l"(&t->done), "l"(0ull) : "memory");
  }
}

}  // namespace vx
