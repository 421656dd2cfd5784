// vx_api.cu — the C-ABI (include/vortex_b200.h), part 1: NCCL loading, errors, tensor maps,
// index handles (device memory, streams, events), options and stats, index / token data,
// the host-buffer operators, the live batcher (vx_serve_trace) and the shard communicator.
// The per-batch stage itself is vx_stage.cu.  No CPU fallback: every entry point fails loudly
// without a usable device.
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "vx_batcher.hpp"
#include "vx_handle.cuh"

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = getenv("VX_NCCL_LIB");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
#define SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(Broadcast, "ncclBroadcast");
    SYM(Reduce, "ncclReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast &&
             api.Reduce && api.AllGather && api.Send && api.Recv && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
  });
  return api;
}

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

vx_status fail(vx_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

// ---------------------------------------------------------------- tensor maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// 2-D row-major matrix [rows][cols] of `elem` bytes, box {box_cols, box_rows}, 128B swizzle.
vx_status make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt,
                              int elem, uint64_t rows, uint64_t cols, uint32_t box_cols,
                              uint32_t box_rows, uint64_t pitch) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(VX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {(pitch ? pitch : cols) * (uint64_t)elem};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VX_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return VX_OK;
}

extern "C" int32_t vx_abi_version(void) { return VX_ABI_VERSION; }
extern "C" const char* vx_last_error(void) { return g_err.c_str(); }

extern "C" vx_status vx_index_create(const vx_index_desc* d, vx_index** out) {
  if (!d || !out) return fail(VX_ERR_INVALID, "null argument");
  *out = nullptr;
  if (d->n_docs < 1 || d->n_docs >= (int64_t)0xFFFFFFFFll)
    return fail(VX_ERR_INVALID, "n_docs must be in [1, 2^32-1)");
  if (d->dim < 32 || d->dim > 4096 || d->dim % 32)
    return fail(VX_ERR_INVALID, "dim must be a multiple of 32 in [32, 4096]");
  if (d->n_shards < 1 || d->shard < 0 || d->shard >= d->n_shards)
    return fail(VX_ERR_INVALID, "bad shard %d of %d", d->shard, d->n_shards);
  if (d->max_batch < 1 || d->max_k < 1 || d->max_k > 256)
    return fail(VX_ERR_INVALID, "max_batch >= 1 and 1 <= max_k <= 256 required");
  if (d->tok_per_doc < 0 || (d->tok_per_doc > 0 && (d->tok_dim < 16 || d->tok_dim % 16 ||
                                                    d->tok_blocks < 1 || d->max_qtok < 1 ||
                                                    d->max_qtok > 128)))
    return fail(VX_ERR_INVALID, "bad token-store shape");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(VX_ERR_CUDA, "no CUDA device visible (the B200 path has no CPU fallback)");
  if (d->device < 0 || d->device >= ndev) return fail(VX_ERR_INVALID, "device %d", d->device);
  cudaDeviceProp prop;
  CU_TRY(cudaGetDeviceProperties(&prop, d->device));
  if (prop.major != 10)
    return fail(VX_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", d->device,
                prop.major, prop.minor);
  vx_index* h = new vx_index();
  h->desc = *d;
  h->device = d->device;
  h->num_sms = prop.multiProcessorCount;
  h->row0 = (d->n_docs * d->shard) / d->n_shards;
  h->n_local = (d->n_docs * (d->shard + 1)) / d->n_shards - h->row0;
  vx_status s = VX_OK;
  auto cleanup = [&](vx_status e) {
    vx_index_destroy(h);
    return e;
  };
  if (const char* e = getenv("VX_DEBUG_TC_NOSELECT")) h->dbg_tc_bits = atoi(e);
  if (const char* e = getenv("VX_DEBUG_TC_STAGES")) h->dbg_tc_stages = atoi(e);
  if (const char* e = getenv("VX_DEBUG_NO_REP")) h->dbg_no_rep = atoi(e);
  if (const char* e = getenv("VX_DEBUG_SEED_M")) h->dbg_seed_m = std::min(32, std::max(1, atoi(e)));
  if (getenv("VX_DEBUG_NO_SEED")) h->scan_seed = 0;  // timing experiments only
  if (const char* e = getenv("VX_DEBUG_SEED_STRIDE")) h->dbg_seed_stride = std::min(1024, std::max(8, atoi(e)));
  if (cudaSetDevice(h->device) != cudaSuccess) return cleanup(fail(VX_ERR_CUDA, "cudaSetDevice"));
  if (h->n_local < 1) return cleanup(fail(VX_ERR_INVALID, "empty shard"));
#define ALLOC(ptr, bytes)                                                              \
  do {                                                                                 \
    cudaError_t _e = cudaMalloc((void**)&(ptr), (bytes));                              \
    if (_e != cudaSuccess)                                                             \
      return cleanup(fail(VX_ERR_OOM, "cudaMalloc %zu bytes: %s", (size_t)(bytes),       \
                          cudaGetErrorString(_e)));                                    \
  } while (0)
  const size_t D = d->dim, B = d->max_batch, K = d->max_k;
  ALLOC(h->docs, (size_t)h->n_local * D * 4);
  if (d->tok_per_doc > 0)
  {
    if (d->flags & VX_FLAG_TOKENS_F32)
      ALLOC(h->tokens32, (size_t)d->tok_blocks * d->tok_per_doc * d->tok_dim * 4);
    else
      ALLOC(h->tokens, (size_t)d->tok_blocks * d->tok_per_doc * d->tok_dim * 2);
  }
  h->grid = h->num_sms;
  ALLOC(h->d_q, B * D * 4);
  if (d->tok_per_doc > 0) ALLOC(h->d_qtok, B * d->max_qtok * d->tok_dim * 4);
  if (d->tok_per_doc > 0 && d->n_shards > 1)  // bf16 hi + lo planes (shard exchange)
    ALLOC(h->d_qtok16, 2 * B * d->max_qtok * d->tok_dim * 2);
  ALLOC(h->d_part, B * (size_t)h->grid * 256 * 8);
  ALLOC(h->d_keys, B * K * 8);
  ALLOC(h->d_ids, B * K * 8);
  ALLOC(h->d_ip, B * K * 4);
  ALLOC(h->d_ms, B * K * 4);
  ALLOC(h->d_out_ids, B * K * 8);
  ALLOC(h->d_out_ip, B * K * 4);
  ALLOC(h->d_out_ms, B * K * 4);
  ALLOC(h->d_send, B * K * 8);
  if (d->n_shards > 1 && d->shard == 0)
    ALLOC(h->d_recv, (size_t)d->n_shards * B * K * 8);
  if (d->n_shards > 1) {  // the sharded re-rank threshold (all-gathered lower bounds)
    ALLOC(h->d_lball, (size_t)d->n_shards * B * K * 4);
    ALLOC(h->d_tau, B * 4);
    ALLOC(h->d_hkeys, B * K * 8);
  }
  ALLOC(h->d_hdr, 16);
  ALLOC(h->d_ckeys, B * 1024 * 8);
  ALLOC(h->d_seedk, B * 32 * 8);
  ALLOC(h->d_flags, B * 4);
  ALLOC(h->d_xnorm, (8 + D) * 4);  // shard statistics + the s8 column scales
  ALLOC(h->d_colmax, D * 4);
  ALLOC(h->d_fq, B * D * 4);
  ALLOC(h->d_fidx, B * 4);
  // the certificate counters and the device timers in one allocation: vx_sync returns both
  // with one copy
  ALLOC(h->d_fcount, 16 + sizeof(vx::KTimer) * vx::KT_N);
  h->d_ktimer = reinterpret_cast<vx::KTimer*>(reinterpret_cast<uint8_t*>(h->d_fcount) + 16);
  ALLOC(h->d_ctr, 16);
  ALLOC(h->d_qctr, (size_t)B * 4);
  // bf16 shadow for the coarse scan: K-chunks of 64 bf16 (one 128-byte swizzle atom), so
  // D % 64 == 0; otherwise the coarse scan reads the fp32 rows as TF32 (32-wide chunks)
  if (!(d->flags & VX_FLAG_NO_BF16_SHADOW) && D % 64 == 0) {
    ALLOC(h->docs16, (size_t)h->n_local * D * 2);
    // + kQueryPadRows rows: the scan's query tensor map always spans whole A tiles (rows past
    // the batch are real memory, not TMA out-of-bounds fills — those made a 1-query 10M-row
    // scan 1.58 ms against 1.10 ms at 16 queries; profiles/r02/small_batch/)
    ALLOC(h->d_q16, (B + kQueryPadRows) * D * 2);
  }
  // s8 shadow: K-chunks of 128 s8, and |s32 dot| < 2^24 (exact fp32 keys) needs D <= 1024
  if (!(d->flags & VX_FLAG_NO_I8_SHADOW) && D % 128 == 0 && D <= 1024) {
    ALLOC(h->docs8, (size_t)h->n_local * D);
    ALLOC(h->d_q8, (B + kQueryPadRows) * D);
    ALLOC(h->d_qs8, B * 4);
  }
#undef ALLOC
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->stream_cond, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->tok_ev, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(fail(VX_ERR_CUDA, "stream create"));
  for (auto& e : h->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(VX_ERR_CUDA, "event create"));
  for (auto& e : h->gev)
    if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(VX_ERR_CUDA, "event create"));
  for (auto& e : h->pev)
    if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(VX_ERR_CUDA, "event create"));
  h->h_stage_bytes = B * D * 4 + (d->tok_per_doc > 0 ? B * d->max_qtok * d->tok_dim * 4 : 0) +
                     B * K * 16 + 64;
  if (cudaMallocHost(&h->h_stage, h->h_stage_bytes) != cudaSuccess)
    return cleanup(fail(VX_ERR_OOM, "pinned staging"));
  if (cudaMallocHost((void**)&h->h_hdr, 32) != cudaSuccess)  // [4] header + [4] cert counters
    return cleanup(fail(VX_ERR_OOM, "pinned header"));
  if (cudaMallocHost((void**)&h->h_flags, B * 4) != cudaSuccess)
    return cleanup(fail(VX_ERR_OOM, "pinned flags"));
  if (cudaMallocHost(&h->h_sync, 16 + sizeof(vx::KTimer) * vx::KT_N) != cudaSuccess)
    return cleanup(fail(VX_ERR_OOM, "pinned sync mirror"));
  if (cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(fail(VX_ERR_CUDA, "event create"));
  if ((h->d_q16 && cudaMemset(h->d_q16, 0, (size_t)(B + kQueryPadRows) * D * 2) != cudaSuccess) ||
      (h->d_q8 && cudaMemset(h->d_q8, 0, (size_t)(B + kQueryPadRows) * D) != cudaSuccess))
    return cleanup(fail(VX_ERR_CUDA, "memset"));
  if (cudaMemset(h->d_xnorm, 0, (8 + D) * 4) != cudaSuccess || cudaMemset(h->d_fcount, 0, 16) != cudaSuccess || cudaMemset(h->d_ctr, 0, 16) != cudaSuccess || cudaMemset(h->d_qctr, 0, (size_t)B * 4) != cudaSuccess ||
      ktimer_reset(h) != VX_OK)
    return cleanup(fail(VX_ERR_CUDA, "memset"));
  if (h->tokens) {
    s = make_tmap_2d(&h->tmap_tok, h->tokens, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     (uint64_t)d->tok_blocks * d->tok_per_doc, (uint64_t)d->tok_dim, 64,
                     (uint32_t)std::min(d->tok_per_doc, 256));
    if (s != VX_OK) return cleanup(s);
  }
  for (int half = 0; half < 2; ++half) {  // 128-row boxes, and 64-row boxes (QG = 2 tiles)
    const uint32_t rows = half ? 64 : 128;
    s = make_tmap_2d(half ? &h->tmap_docs_h : &h->tmap_docs, h->docs,
                     CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)h->n_local, D, 32, rows);
    if (s != VX_OK) return cleanup(s);
    if (h->docs16) {
      s = make_tmap_2d(half ? &h->tmap_docs16_h : &h->tmap_docs16, h->docs16,
                       CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)h->n_local, D, 64, rows);
      if (s != VX_OK) return cleanup(s);
    }
    if (h->docs8) {
      s = make_tmap_2d(half ? &h->tmap_docs8_h : &h->tmap_docs8, h->docs8,
                       CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)h->n_local, D, 128, rows);
      if (s != VX_OK) return cleanup(s);
    }
  }
  *out = h;
  return VX_OK;
}

extern "C" vx_status vx_index_destroy(vx_index* h) {
  if (!h) return VX_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  // graphs first: captured NCCL operations hold references on the communicator, and
  // destroying it under live graphs hangs
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
  h->graphs.clear();
  for (auto& kv : h->io_graphs) cudaGraphExecDestroy(kv.second.exec);
  h->io_graphs.clear();
  if (h->comm) nccl().CommDestroy(h->comm);
  void* ptrs[] = {h->docs,  h->tokens, h->tokens32, h->d_q,      h->d_qtok,    h->d_part, h->d_keys,
                  h->d_ids, h->d_ip,      h->d_ms,     h->d_out_ids, h->d_out_ip,
                  h->d_out_ms, h->d_send, h->d_recv, h->d_hdr, h->d_ckeys, h->d_seedk, h->d_flags,
                  h->d_xnorm, h->d_fq, h->docs16, h->d_q16, h->d_fidx, h->d_fcount,
                  h->d_qtok16, h->docs8, h->d_q8, h->d_qs8, h->d_lball, h->d_tau, h->d_hkeys,
                  h->d_colmax, h->d_ctr, h->d_qctr};  // (d_ktimer lives in d_fcount's allocation)
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->h_stage) cudaFreeHost(h->h_stage);
  if (h->h_hdr) cudaFreeHost(h->h_hdr);
  if (h->h_flags) cudaFreeHost(h->h_flags);
  if (h->h_sync) cudaFreeHost(h->h_sync);
  if (h->ev_done) cudaEventDestroy(h->ev_done);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->gev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->pev)
    if (e) cudaEventDestroy(e);
  if (h->tok_ev) cudaEventDestroy(h->tok_ev);
  if (h->stream2) cudaStreamDestroy(h->stream2);
  if (h->stream_cond) cudaStreamDestroy(h->stream_cond);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return VX_OK;
}

extern "C" vx_status vx_index_shard_range(const vx_index* h, int64_t* row0, int64_t* n_local) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (row0) *row0 = h->row0;
  if (n_local) *n_local = h->n_local;
  return VX_OK;
}

static vx_status refresh_shadows(vx_index* h, int64_t row_off, int64_t nrows);

extern "C" vx_status vx_set_option(vx_index* h, int32_t option, int64_t value) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  drop_graphs(h);  // every option below changes what a captured stage would run
  switch (option) {
    case VX_OPT_SCAN:
      if (value != VX_SCAN_AUTO && value != VX_SCAN_F32 && value != VX_SCAN_TC)
        return fail(VX_ERR_INVALID, "scan algorithm %lld", (long long)value);
      h->scan_algo = (int)value;
      return VX_OK;
    case VX_OPT_GRID:
      if (value < 0 || value > h->num_sms) return fail(VX_ERR_INVALID, "grid %lld", (long long)value);
      h->grid = value == 0 ? h->num_sms : (int)value;
      return VX_OK;
    case VX_OPT_STAGE_EVENTS:
      if (value != 0 && value != 1) return fail(VX_ERR_INVALID, "stage events %lld", (long long)value);
      h->stage_events = value == 1;
      return VX_OK;
    case VX_OPT_KPRIME:
      if (value != 0 && (value < 16 || value > 1024 || (value & (value - 1))))
        return fail(VX_ERR_INVALID, "kprime %lld (0 or a power of two in [16, 1024])", (long long)value);
      h->kprime = (int)value;
      return VX_OK;
    case VX_OPT_I8_SCALE:
      if (value != 0 && value != 1) return fail(VX_ERR_INVALID, "i8 scale %lld", (long long)value);
      if (h->i8_per_column != (int)value) {
        h->i8_per_column = (int)value;
        if (h->docs8) VX_TRY(refresh_shadows(h, 0, 0));  // re-quantise the shard
        CU_TRY(cudaStreamSynchronize(h->stream));
      }
      return VX_OK;
    case VX_OPT_SCAN_SEED:
      if (value != 0 && value != 1) return fail(VX_ERR_INVALID, "scan seed %lld", (long long)value);
      h->scan_seed = (int)value;
      return VX_OK;
    case VX_OPT_SCAN_PAIRS:
      if (value < 0 || value > 2) return fail(VX_ERR_INVALID, "pairs %lld", (long long)value);
      h->use_pairs = (int)value;
      return VX_OK;
    case VX_OPT_SCAN_TILE:
      if (value != 0 && value != 128 && value != 256)
        return fail(VX_ERR_INVALID, "scan tile %lld (0, 128 or 256)", (long long)value);
      h->scan_tile = (int)value;
      return VX_OK;
    case VX_OPT_COARSE:
      if (value != VX_COARSE_AUTO && value != VX_COARSE_TF32 && value != VX_COARSE_BF16 &&
          value != VX_COARSE_I8)
        return fail(VX_ERR_INVALID, "coarse format %lld", (long long)value);
      if (value == VX_COARSE_BF16 && !h->docs16)
        return fail(VX_ERR_STATE, "no bf16 shadow (VX_FLAG_NO_BF16_SHADOW or D %% 64 != 0)");
      if (value == VX_COARSE_I8 && !h->docs8)
        return fail(VX_ERR_STATE, "no s8 shadow (VX_FLAG_NO_I8_SHADOW, D %% 128 != 0 or D > 1024)");
      h->coarse = (int)value;
      return VX_OK;
    case VX_OPT_MAXSIM:
      if (value != VX_MAXSIM_AUTO && value != VX_MAXSIM_CC && value != VX_MAXSIM_TC &&
          value != VX_MAXSIM_TC_BF16Q)
        return fail(VX_ERR_INVALID, "maxsim algorithm %lld", (long long)value);
      if ((value == VX_MAXSIM_TC || value == VX_MAXSIM_TC_BF16Q) && h->tokens &&
          !vx::maxsim_tc_supported(h->desc.max_qtok, h->desc.tok_per_doc, h->desc.tok_dim))
        return fail(VX_ERR_UNSUPPORTED, "tensor-core MaxSim needs Nd in {64,128,256}, d in {64,128}");
      if ((value == VX_MAXSIM_TC || value == VX_MAXSIM_TC_BF16Q) && h->tokens32)
        return fail(VX_ERR_UNSUPPORTED, "the fp32 token store runs the CUDA-core MaxSim");
      h->maxsim_algo = (int)value;
      return VX_OK;
    case VX_OPT_GRAPHS:
      if (value != 0 && value != 1) return fail(VX_ERR_INVALID, "graphs %lld", (long long)value);
      h->use_graphs = value == 1;
      return VX_OK;
    default:
      return fail(VX_ERR_INVALID, "unknown option %d", option);
  }
}

extern "C" vx_status vx_get_option(const vx_index* h, int32_t option, int64_t* value) {
  if (!h || !value) return fail(VX_ERR_INVALID, "null argument");
  switch (option) {
    case VX_OPT_SCAN: *value = h->scan_algo; return VX_OK;
    case VX_OPT_GRID: *value = h->grid; return VX_OK;
    case VX_OPT_GRAPHS: *value = h->use_graphs ? 1 : 0; return VX_OK;
    case VX_OPT_MAXSIM: *value = h->maxsim_algo; return VX_OK;
    case VX_OPT_SCAN_TILE: *value = h->scan_tile; return VX_OK;
    case VX_OPT_SCAN_PAIRS: *value = h->use_pairs; return VX_OK;
    case VX_OPT_KPRIME: *value = h->kprime; return VX_OK;
    case VX_OPT_SCAN_SEED: *value = h->scan_seed; return VX_OK;
    case VX_OPT_I8_SCALE: *value = h->i8_per_column; return VX_OK;
    case VX_OPT_STAGE_EVENTS: *value = h->stage_events ? 1 : 0; return VX_OK;
    case VX_OPT_COARSE: {
      const int f = coarse_fmt(h);
      *value = f == vx::FMT_I8 ? VX_COARSE_I8 : (f == vx::FMT_TF32 ? VX_COARSE_TF32 : VX_COARSE_BF16);
      return VX_OK;
    }
    default: return fail(VX_ERR_INVALID, "unknown option %d", option);
  }
}

extern "C" vx_status vx_get_stats(const vx_index* h, vx_stats* out) {
  if (!h || !out) return fail(VX_ERR_INVALID, "null argument");
  *out = h->st;
  return VX_OK;
}
extern "C" vx_status vx_reset_stats(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaStreamSynchronize(h->stream));
  CU_TRY(cudaMemset(h->d_fcount, 0, 16));
  VX_TRY(ktimer_reset(h));
  h->cert_seen_q = h->cert_seen_l2 = h->cert_seen_l3 = 0;
  h->st = vx_stats{};
  return VX_OK;
}

// After the fp32 rows of the shard changed: the coarse-scan shadows and the shard maxima the
// certificate bounds with.  The s8 scale is shard-wide, so the whole s8 shadow is rebuilt.
static vx_status refresh_shadows(vx_index* h, int64_t row_off, int64_t nrows) {
  const int64_t D = h->desc.dim;
  drop_graphs(h);  // the AUTO coarse format and the certificate inputs may change
  float* colscale = reinterpret_cast<float*>(h->d_xnorm) + vx::kXstatColScale;
  if (h->docs8) {
    // column scales, then the shadow; the s8 coarse units' document factor xstats[5] = 1
    // (the scales ride on the query side, vx::launch_rows_to_i8)
    CU_TRY(vx::launch_to_i8_shadow(h->docs, h->n_local, (int)D, h->docs8, h->d_colmax, colscale,
                                   h->i8_per_column, h->stream));
    h->i8_demoted = false;  // a new shard: AUTO may take the s8 pass again
    const float one = 1.0f;
    CU_TRY(cudaMemcpyAsync(h->d_xnorm + 5, &one, 4, cudaMemcpyHostToDevice, h->stream));
    CU_TRY(cudaStreamSynchronize(h->stream));  // `one` is a host stack value
    count_launch(h, 3);
  }
  CU_TRY(vx::launch_row_stats(h->docs, h->n_local, (int)D, h->d_xnorm, h->stream,
                              h->docs8 ? colscale : nullptr));
  count_launch(h);
  if (h->docs16 && nrows > 0) {
    CU_TRY(vx::launch_to_bf16(h->docs + row_off * D, h->docs16 + row_off * D, nrows * D,
                              h->stream));
    count_launch(h);
  }
  // host copy of the shard maxima for the AUTO coarse-format choice (coarse_fmt); the callers
  // synchronise the stream before returning
  CU_TRY(cudaMemcpyAsync(h->xstats_host, h->d_xnorm, sizeof(h->xstats_host),
                         cudaMemcpyDeviceToHost, h->stream));
  return VX_OK;
}

extern "C" vx_status vx_index_synth(vx_index* h, uint64_t seed) {
  return vx_index_synth_dist(h, seed, 0);
}

extern "C" vx_status vx_index_synth_dist(vx_index* h, uint64_t seed, int32_t dist) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (dist != 0 && dist != 1) return fail(VX_ERR_INVALID, "dist %d (0 isotropic, 1 anisotropic)", dist);
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(vx::launch_synth_rows(h->docs, seed, h->row0, h->n_local, h->desc.dim, h->stream,
                               (uint32_t)dist));
  count_launch(h);
  VX_TRY(refresh_shadows(h, 0, h->n_local));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_index_upload(vx_index* h, const float* rows, int64_t row0, int64_t n) {
  if (!h || (!rows && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (row0 < h->row0 || n < 0 || row0 + n > h->row0 + h->n_local)
    return fail(VX_ERR_INVALID, "rows [%lld,%lld) outside shard [%lld,%lld)", (long long)row0,
                (long long)(row0 + n), (long long)h->row0, (long long)(h->row0 + h->n_local));
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(h->docs + (row0 - h->row0) * h->desc.dim, rows,
                         (size_t)n * h->desc.dim * 4, cudaMemcpyHostToDevice, h->stream));
  // the TC certificate needs the shard maxima and the coarse shadows: recompute
  VX_TRY(refresh_shadows(h, row0 - h->row0, n));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_index_download(const vx_index* h, float* rows, int64_t row0, int64_t n) {
  if (!h || (!rows && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (row0 < h->row0 || n < 0 || row0 + n > h->row0 + h->n_local)
    return fail(VX_ERR_INVALID, "rows outside shard");
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(rows, h->docs + (row0 - h->row0) * h->desc.dim,
                         (size_t)n * h->desc.dim * 4, cudaMemcpyDeviceToHost, h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_download(const vx_index* h, uint16_t* tok, int64_t blk0, int64_t n) {
  if (!h || (!tok && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no bf16 token store");
  if (blk0 < 0 || n < 0 || blk0 + n > h->desc.tok_blocks)
    return fail(VX_ERR_INVALID, "token blocks out of range");
  const size_t blk = (size_t)h->desc.tok_per_doc * h->desc.tok_dim;
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(tok, h->tokens + blk0 * blk, n * blk * 2, cudaMemcpyDeviceToHost,
                         h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_synth(vx_index* h, uint64_t seed) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (!has_tokens(h)) return fail(VX_ERR_STATE, "index has no token store");
  CU_TRY(cudaSetDevice(h->device));
  if (h->tokens32)  // the same generator, unrounded (the bf16 store holds its RNE)
    CU_TRY(vx::launch_synth_rows(h->tokens32, seed, 0,
                                 (int64_t)h->desc.tok_blocks * h->desc.tok_per_doc,
                                 h->desc.tok_dim, h->stream));
  else
    CU_TRY(vx::launch_synth_tokens(h->tokens, seed, 0, h->desc.tok_blocks, h->desc.tok_per_doc,
                                   h->desc.tok_dim, h->stream));
  count_launch(h);
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_upload_f32(vx_index* h, const float* tok, int64_t blk0, int64_t n) {
  if (!h || (!tok && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens32) return fail(VX_ERR_STATE, "index has no fp32 token store");
  if (blk0 < 0 || n < 0 || blk0 + n > h->desc.tok_blocks)
    return fail(VX_ERR_INVALID, "token blocks out of range");
  const size_t blk = (size_t)h->desc.tok_per_doc * h->desc.tok_dim;
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(h->tokens32 + blk0 * blk, tok, n * blk * 4, cudaMemcpyHostToDevice,
                         h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_download_f32(const vx_index* h, float* tok, int64_t blk0, int64_t n) {
  if (!h || (!tok && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens32) return fail(VX_ERR_STATE, "index has no fp32 token store");
  if (blk0 < 0 || n < 0 || blk0 + n > h->desc.tok_blocks)
    return fail(VX_ERR_INVALID, "token blocks out of range");
  const size_t blk = (size_t)h->desc.tok_per_doc * h->desc.tok_dim;
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(tok, h->tokens32 + blk0 * blk, n * blk * 4, cudaMemcpyDeviceToHost,
                         h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_upload(vx_index* h, const uint16_t* tok, int64_t blk0, int64_t n) {
  if (!h || (!tok && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no bf16 token store");
  if (blk0 < 0 || n < 0 || blk0 + n > h->desc.tok_blocks)
    return fail(VX_ERR_INVALID, "token blocks out of range");
  const size_t blk = (size_t)h->desc.tok_per_doc * h->desc.tok_dim;
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(h->tokens + blk0 * blk, tok, n * blk * 2, cudaMemcpyHostToDevice,
                         h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

// ---------------------------------------------------------------- host-buffer API
// Host staging of a batch: one copy into the handle's pinned buffer, either from one
// contiguous [B][row] array or gathered from B row pointers (e.g. straight out of the
// runtime's query payloads, so the operator adapter copies each query exactly once).
static void gather_rows(uint8_t* dst, const float* base, const float* const* rows, int B,
                        size_t row_bytes) {
  if (rows)
    for (int i = 0; i < B; ++i) memcpy(dst + (size_t)i * row_bytes, rows[i], row_bytes);
  else
    memcpy(dst, base, (size_t)B * row_bytes);
}

// Page-locked host memory (cudaMallocHost / cudaHostRegister): the DMA engines read / write
// it directly, so the host API skips the staging memcpy — at B = 1024 the 16.8 MB of fp32
// query tokens took ~1 ms of host memcpy per batch.  The WHOLE range [p, p + bytes) must lie
// inside one page-locked allocation (a buffer straddling two pinned allocations with pageable
// memory between them is not DMA-safe); anything else goes through the staging buffer.
typedef CUresult (*PFN_ptrAttr)(void*, CUpointer_attribute, CUdeviceptr);
static PFN_ptrAttr get_ptr_attr() {
  static PFN_ptrAttr fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_ptrAttr>(p);
  });
  return fn;
}

// Ranges already verified (a few per thread: the callers' long-lived I/O buffers) skip the
// three driver queries per buffer (~2 us each call, three buffers a batch).  A stale entry
// (the allocation freed, the range reused as pageable memory) is harmless: cudaMemcpyAsync
// stages pageable memory itself, and every host-API call synchronizes before returning.
struct PinnedRange {
  uintptr_t start = 0;
  size_t size = 0;
};
static thread_local PinnedRange t_pinned[8];
static thread_local int t_pinned_next = 0;

static bool is_pinned(const void* p, size_t bytes) {
  if (!p || !bytes) return false;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  for (const PinnedRange& r : t_pinned)
    if (r.size && a >= r.start && a + bytes <= r.start + r.size) return true;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type != cudaMemoryTypeHost) return false;
  PFN_ptrAttr fn = get_ptr_attr();
  if (!fn) return false;
  CUdeviceptr start = 0;
  size_t size = 0;
  const CUdeviceptr dp = (CUdeviceptr)(uintptr_t)(at.devicePointer ? at.devicePointer : p);
  if (fn(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, dp) != CUDA_SUCCESS ||
      fn(&size, CU_POINTER_ATTRIBUTE_RANGE_SIZE, dp) != CUDA_SUCCESS)
    return false;
  // the range is reported in the allocation's device address space; p's offset into it is
  // the same in host and device views
  if (!((uint64_t)dp >= (uint64_t)start && (uint64_t)dp + bytes <= (uint64_t)start + size))
    return false;
  PinnedRange& r = t_pinned[t_pinned_next++ & 7];
  r.start = a - (uintptr_t)((uint64_t)dp - (uint64_t)start);  // the allocation, host view
  r.size = size;
  return true;
}

// source of a batch upload: the caller's contiguous pinned buffer itself, else the rows
// gathered into the handle's pinned staging
static const void* upload_src(vx_index* h, uint8_t* stage, const float* base,
                              const float* const* rows, int B, size_t row_bytes) {
  if (!rows && is_pinned(base, (size_t)B * row_bytes)) return base;
  gather_rows(stage, base, rows, B, row_bytes);
  h->st.host_staged_bytes += (uint64_t)B * row_bytes;
  return stage;
}

// device -> host result copy: straight into a pinned destination, else via the staging
// (*deferred set: memcpy after the sync)
static cudaError_t download(vx_index* h, void* dst, uint8_t* stage, const void* src, size_t bytes,
                            cudaStream_t st, bool* deferred) {
  *deferred = !is_pinned(dst, bytes);
  if (*deferred) h->st.host_staged_bytes += bytes;
  return cudaMemcpyAsync(*deferred ? static_cast<void*>(stage) : dst, src, bytes,
                         cudaMemcpyDeviceToHost, st);
}

static bool rows_ok(const float* const* rows, int B) {
  for (int i = 0; i < B; ++i)
    if (!rows[i]) return false;
  return true;
}

// A failed call may have left a DMA from / to the caller's own (pinned) buffers in flight:
// drain both streams before returning the error, so the caller may free them at once.
static vx_status drained(vx_index* h, vx_status s) {
  if (s != VX_OK) {
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->stream2) cudaStreamSynchronize(h->stream2);
    cudaGetLastError();
  }
  return s;
}

static vx_status host_search(vx_index* h, const float* q, const float* const* q_rows, int32_t B,
                             int32_t k, int64_t* ids, float* scores) {
  VX_TRY(check_batch(h, B, k));
  if (q_rows && !rows_ok(q_rows, B)) return fail(VX_ERR_INVALID, "null query row");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t qrow = (size_t)h->desc.dim * 4, qb = (size_t)B * qrow;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  CU_TRY(cudaMemcpyAsync(h->d_q, upload_src(h, stage, q, q_rows, B, qrow), qb,
                         cudaMemcpyHostToDevice, st));
  // the direct graph writes the stage's own result buffers (d_ids / d_ip: the certificate
  // chain uses d_out_* as level-3 scratch), the two-part path copies them to d_out_*
  bool done = false;
  VX_TRY(stage_direct(h, OP_SEARCH, h->d_q, nullptr, B, 0, k, h->d_ids, h->d_ip, nullptr, st,
                      &done));
  if (!done) {
    VX_TRY(stage_begin(h, OP_SEARCH, h->d_q, B, 0, k, st));
    VX_TRY(stage_search_out(h, B, k, h->d_out_ids, h->d_out_ip, st));
  }
  const size_t n = (size_t)B * k;
  bool d_ids, d_sc;
  CU_TRY(download(h, ids, stage, done ? h->d_ids : h->d_out_ids, n * 8, st, &d_ids));
  CU_TRY(download(h, scores, stage + n * 8, done ? h->d_ip : h->d_out_ip, n * 4, st, &d_sc));
  VX_TRY(vx_sync(h));
  if (d_ids) memcpy(ids, stage, n * 8);
  if (d_sc) memcpy(scores, stage + n * 8, n * 4);
  return VX_OK;
}

extern "C" vx_status vx_search(vx_index* h, const float* q, int32_t B, int32_t k, int64_t* ids,
                               float* scores) {
  if (!h || !q || !ids || !scores) return fail(VX_ERR_INVALID, "null argument");
  return drained(h, host_search(h, q, nullptr, B, k, ids, scores));
}

extern "C" vx_status vx_search_rows(vx_index* h, const float* const* q_rows, int32_t B, int32_t k,
                                    int64_t* ids, float* scores) {
  if (!h || !q_rows || !ids || !scores) return fail(VX_ERR_INVALID, "null argument");
  return drained(h, host_search(h, nullptr, q_rows, B, k, ids, scores));
}

static vx_status host_maxsim(vx_index* h, const float* qtok, int32_t B, int32_t nq,
                             const int64_t* cand, int32_t C, float* out) {
  if (!has_tokens(h)) return fail(VX_ERR_STATE, "index has no token store");
  if (B < 1 || B > h->desc.max_batch || C < 1 || C > h->desc.max_k)
    return fail(VX_ERR_INVALID, "B %d / C %d outside [1,%d] / [1,%d]", B, C, h->desc.max_batch,
                h->desc.max_k);
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t tb = (size_t)B * nq * h->desc.tok_dim * 4, cb = (size_t)B * C * 8;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  CU_TRY(cudaMemcpyAsync(h->d_qtok, upload_src(h, stage, qtok, nullptr, B, tb / B), tb,
                         cudaMemcpyHostToDevice, st));
  const void* csrc = cand;
  if (!is_pinned(cand, cb)) {
    memcpy(stage + tb, cand, cb);
    h->st.host_staged_bytes += cb;
    csrc = stage + tb;
  }
  CU_TRY(cudaMemcpyAsync(h->d_out_ids, csrc, cb, cudaMemcpyHostToDevice, st));
  VX_TRY(run_maxsim(h, h->d_qtok, B, nq, h->d_out_ids, C, h->d_out_ms, st));
  bool d_out;
  CU_TRY(download(h, out, stage, h->d_out_ms, (size_t)B * C * 4, st, &d_out));
  VX_TRY(vx_sync(h));
  if (d_out) memcpy(out, stage, (size_t)B * C * 4);
  return VX_OK;
}

extern "C" vx_status vx_maxsim(vx_index* h, const float* qtok, int32_t B, int32_t nq,
                               const int64_t* cand, int32_t C, float* out) {
  if (!h || !qtok || !cand || !out) return fail(VX_ERR_INVALID, "null argument");
  return drained(h, host_maxsim(h, qtok, B, nq, cand, C, out));
}

static vx_status host_search_rescore(vx_index* h, const float* q, const float* const* q_rows,
                                     const float* qtok, const float* const* tok_rows, int32_t B,
                                     int32_t nq, int32_t k, int64_t* ids, float* ip, float* ms) {
  VX_TRY(check_batch(h, B, k));
  if (!has_tokens(h)) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  if ((q_rows && !rows_ok(q_rows, B)) || (tok_rows && !rows_ok(tok_rows, B)))
    return fail(VX_ERR_INVALID, "null query row");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t qrow = (size_t)h->desc.dim * 4, trow = (size_t)nq * h->desc.tok_dim * 4;
  const size_t qb = (size_t)B * qrow, tb = (size_t)B * trow;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  CU_TRY(cudaMemcpyAsync(h->d_q, upload_src(h, stage, q, q_rows, B, qrow), qb,
                         cudaMemcpyHostToDevice, st));
  VX_TRY(stage_begin(h, OP_RESCORE, h->d_q, B, nq, k, st));
  // the query tokens are only read by part 2: (stage and) upload them while part 1 runs
  CU_TRY(cudaMemcpyAsync(h->d_qtok, upload_src(h, stage + qb, qtok, tok_rows, B, trow), tb,
                         cudaMemcpyHostToDevice, h->stream2));
  CU_TRY(cudaEventRecord(h->tok_ev, h->stream2));
  CU_TRY(cudaStreamWaitEvent(st, h->tok_ev, 0));
  VX_TRY(stage_finish(h, h->d_qtok, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
  const size_t n = (size_t)B * k;
  bool d_ids, d_ip, d_ms;
  CU_TRY(download(h, ids, stage, h->d_out_ids, n * 8, st, &d_ids));
  CU_TRY(download(h, ip, stage + n * 8, h->d_out_ip, n * 4, st, &d_ip));
  CU_TRY(download(h, ms, stage + n * 12, h->d_out_ms, n * 4, st, &d_ms));
  VX_TRY(vx_sync(h));
  if (d_ids) memcpy(ids, stage, n * 8);
  if (d_ip) memcpy(ip, stage + n * 8, n * 4);
  if (d_ms) memcpy(ms, stage + n * 12, n * 4);
  return VX_OK;
}

extern "C" vx_status vx_search_rescore(vx_index* h, const float* q, const float* qtok, int32_t B,
                                       int32_t nq, int32_t k, int64_t* ids, float* ip,
                                       float* ms) {
  if (!h || !q || !qtok || !ids || !ip || !ms) return fail(VX_ERR_INVALID, "null argument");
  return drained(h, host_search_rescore(h, q, nullptr, qtok, nullptr, B, nq, k, ids, ip, ms));
}

extern "C" vx_status vx_search_rescore_rows(vx_index* h, const float* const* q_rows,
                                            const float* const* tok_rows, int32_t B, int32_t nq,
                                            int32_t k, int64_t* ids, float* ip, float* ms) {
  if (!h || !q_rows || !tok_rows || !ids || !ip || !ms) return fail(VX_ERR_INVALID, "null argument");
  return drained(h, host_search_rescore(h, nullptr, q_rows, nullptr, tok_rows, B, nq, k, ids, ip, ms));
}

// ---------------------------------------------------------------- comm
extern "C" vx_status vx_comm_unique_id(uint8_t out_id[128]) {
  if (!out_id) return fail(VX_ERR_INVALID, "null argument");
  if (!nccl().ok) return fail(VX_ERR_NCCL, "libnccl.so.2 not loadable (set VX_NCCL_LIB)");
  ncclUniqueId id;
  NCCL_TRY(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
  memcpy(out_id, &id, 128);
  return VX_OK;
}

extern "C" vx_status vx_comm_init(vx_index* h, const uint8_t id[128], int32_t nranks,
                                  int32_t rank) {
  if (!h || !id) return fail(VX_ERR_INVALID, "null argument");
  if (nranks != h->desc.n_shards || rank != h->desc.shard)
    return fail(VX_ERR_INVALID, "comm (%d of %d) must match shard (%d of %d)", rank, nranks,
                h->desc.shard, h->desc.n_shards);
  if (h->comm) return fail(VX_ERR_STATE, "comm already initialised");
  if (!nccl().ok) return fail(VX_ERR_NCCL, "libnccl.so.2 not loadable (set VX_NCCL_LIB)");
  CU_TRY(cudaSetDevice(h->device));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  NCCL_TRY(nccl().CommInitRank(&h->comm, nranks, uid, rank));
  h->nranks = nranks;
  h->rank = rank;
  return VX_OK;
}

// The shard ranks' serve loop.  Per batch the host must learn the 16-byte header (B picks
// the graph), so it waits for the header broadcast — polling an event instead of a blocking
// stream sync (the wake-up of a yielding sync was tens of us per batch) — then launches the
// batch's parts: the captured graphs of its shape (VX_OPT_GRAPHS; the first batch of a shape
// runs eagerly and captures, like rank 0), else the eager stage.
extern "C" vx_status vx_shard_serve(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (!h->comm || h->rank == 0) return fail(VX_ERR_STATE, "vx_shard_serve is for ranks != 0");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  for (;;) {
    NCCL_TRY(nccl().Broadcast(h->d_hdr, h->d_hdr, 4, ncclInt32, 0, h->comm, st));
    CU_TRY(cudaMemcpyAsync(h->h_hdr, h->d_hdr, 16, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaMemcpyAsync(h->h_hdr + 4, h->d_fcount, 16, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaEventRecord(h->tok_ev, st));
    cudaError_t q;
    while ((q = cudaEventQuery(h->tok_ev)) == cudaErrorNotReady) {
    }
    CU_TRY(q);
    const int op = h->h_hdr[0], B = h->h_hdr[1], k = h->h_hdr[2], nq = h->h_hdr[3];
    maybe_demote_i8(h, h->h_hdr + 4, h->st.queries);  // this shard's certificate record so far
    if (op == OP_STOP) return VX_OK;
    if (B < 1 || B > h->desc.max_batch || k < 1 || k > h->desc.max_k)
      return fail(VX_ERR_STATE, "bad batch header %d/%d/%d", op, B, k);
    if (op == OP_RESCORE && (nq < 1 || nq > h->desc.max_qtok))
      return fail(VX_ERR_STATE, "bad batch header nq %d", nq);
    if (h->use_graphs) {
      VX_TRY(run_part(h, 1 /*PART_TOPK*/, B, op == OP_RESCORE ? nq : 0, k, st));
      if (op == OP_RESCORE) VX_TRY(run_part(h, 2 /*PART_RESCORE*/, B, nq, k, st));
    } else {
      NCCL_TRY(nccl().Broadcast(h->d_q, h->d_q, (size_t)B * h->desc.dim, ncclFloat32, 0, h->comm, st));
      VX_TRY(core_topk(h, h->d_q, B, k, st));
      if (op == OP_RESCORE)  // phase 2: receives the tokens + winners, MaxSim on owned winners
        VX_TRY(core_rescore(h, nullptr, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
    }
    h->st.batches += 1;
    h->st.queries += B;
  }
}

extern "C" vx_status vx_shard_stop(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (!h->comm || h->rank != 0) return fail(VX_ERR_STATE, "vx_shard_stop is for rank 0");
  CU_TRY(cudaSetDevice(h->device));
  h->h_hdr[0] = OP_STOP;
  h->h_hdr[1] = h->h_hdr[2] = h->h_hdr[3] = 0;
  CU_TRY(cudaMemcpyAsync(h->d_hdr, h->h_hdr, 16, cudaMemcpyHostToDevice, h->stream));
  NCCL_TRY(nccl().Broadcast(h->d_hdr, h->d_hdr, 4, ncclInt32, 0, h->comm, h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}
