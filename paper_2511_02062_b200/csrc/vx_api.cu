// vx_api.cu — the C-ABI (include/vortex_b200.h): index handles, device memory,
// streams, the per-batch stage pipeline and the NCCL shard exchange.
//
// The stage a deployment registers as the search operator (reference:
// ComponentFn, proj/include/vortex/runtime.hpp:179; invoked by
// Runtime::complete_batch, runtime.hpp:656-672) runs, per batch of B queries:
//   [H2D queries]  -> K1 scan + per-CTA top-k  -> K3 merge (local top-k)
//   -> K4 MaxSim of the local top-k -> [NCCL gather k x G to rank 0 -> merge]
//   -> order by MaxSim -> [D2H]
// Shard mode mirrors the reference's key->shard placement (kvs.hpp:160-175):
// contiguous document ranges, a document's row and its token block on one GPU.
// No CPU fallback: every entry point fails loudly without a usable device.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vortex_b200.h"
#include "vx_batcher.hpp"
#include "vx_internal.cuh"

// ---------------------------------------------------------------- NCCL (loaded lazily)
// NCCL is dlopen'ed on first use instead of linked: a host process (e.g. PyTorch) may
// already carry its own libnccl.so.2, and two copies under one soname break each other.
// Order: an already-loaded libnccl.so.2, $VX_NCCL_LIB, then the system library.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok = false;
};

static NcclApi& nccl() {
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
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast &&
             api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  return api;
}

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

static vx_status fail(vx_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CU_TRY(expr)                                                                     \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(_e == cudaErrorMemoryAllocation ? VX_ERR_OOM : VX_ERR_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(_e), __FILE__, __LINE__);                    \
  } while (0)

#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      return fail(VX_ERR_NCCL, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(_r), __FILE__, \
                  __LINE__);                                                              \
  } while (0)

#define VX_TRY(expr)                 \
  do {                               \
    vx_status _s = (expr);           \
    if (_s != VX_OK) return _s;      \
  } while (0)

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
static vx_status make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt,
                              int elem, uint64_t rows, uint64_t cols, uint32_t box_cols,
                              uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return fail(VX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * (uint64_t)elem};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VX_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return VX_OK;
}

// ---------------------------------------------------------------- handle

struct vx_index {
  vx_index_desc desc{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  int64_t row0 = 0, n_local = 0;
  float* docs = nullptr;
  uint16_t* tokens = nullptr;
  CUtensorMap tmap_docs{};
  CUtensorMap tmap_tok{};
  uint16_t* docs16 = nullptr;    // bf16 shadow of the shard (coarse scan), may be null
  CUtensorMap tmap_docs16{};
  uint16_t* d_q16 = nullptr;     // [maxB][D] bf16 queries for the bf16 coarse scan
  int coarse = VX_COARSE_AUTO;
  int scan_tile = 0;             // documents per tensor-core tile (0 = auto)
  int kprime = 0;                // TC candidate set size k' (0 = auto; VX_OPT_KPRIME)
  int dbg_tc_bits = 0;           // timing-experiment knobs, read once from the environment at
  int dbg_tc_stages = 0;         //   create: VX_DEBUG_TC_NOSELECT (bit mask), VX_DEBUG_TC_STAGES
  int use_pairs = 1;             // CTA-pair scan for B > 128: 0 off, 1 on, 2 on + 512-query
                                 // passes (VX_OPT_SCAN_PAIRS)
  // options
  int scan_algo = VX_SCAN_AUTO;
  int maxsim_algo = VX_MAXSIM_AUTO;
  int grid = 0;
  // workspace
  float* d_q = nullptr;          // [maxB][D]
  float* d_qtok = nullptr;       // [maxB][maxNq][d]
  uint16_t* d_qtok16 = nullptr;  // bf16 copy for the shard exchange (half the broadcast bytes)
  uint64_t* d_part = nullptr;    // [maxB][grid][256]
  uint64_t* d_keys = nullptr;    // [maxB][maxK]
  int64_t* d_ids = nullptr;      // [maxB][maxK]
  float* d_ip = nullptr;         // [maxB][maxK]
  float* d_ms = nullptr;         // [maxB][maxK]
  int64_t* d_out_ids = nullptr;  // [maxB][maxK]
  float* d_out_ip = nullptr;
  float* d_out_ms = nullptr;
  void* d_send = nullptr;        // [maxB][maxK] x 8 B scratch (rank 0: the reduced MaxSim)
  void* d_recv = nullptr;        // [G][maxB][maxK] gathered keys (rank 0)
  int32_t* d_hdr = nullptr;      // [4]
  uint64_t* d_ckeys = nullptr;   // [maxB][512] merged coarse keys (TC path)
  int* d_flags = nullptr;        // [maxB] certificate failures (TC path)
  unsigned int* d_xnorm = nullptr;  // [3] row-norm maxima of the shard (float bits, row_stats)
  float* d_fq = nullptr;         // [maxB][D] queries gathered for the exact fallback
  int* d_fidx = nullptr;         // [maxB] flagged query indices
  int* d_fcount = nullptr;       // [2] flagged count of the last batch, running total
  // pinned host staging
  void* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  int32_t* h_hdr = nullptr;
  int* h_flags = nullptr;
  // comm
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // stats
  vx_stats st{};
  cudaEvent_t ev[4] = {};        // eager-path timing events: scan begin/end, stage begin/end
  cudaEvent_t gev[4] = {};       // the same, recorded by captured graph nodes
  cudaEvent_t* tev = ev;         // events the code being issued records into
  cudaEvent_t* ev_start = ev;    // last batch: the array holding scan begin/end + stage begin
  cudaEvent_t* ev_end = ev;      //   ... and the one holding the stage end (read by vx_sync)
  cudaStream_t stream_last = nullptr;  // stream of the last batch's final part
  cudaStream_t stream2 = nullptr;      // host API: query-token upload overlapping part 1
  cudaEvent_t tok_ev = nullptr;
  cudaEvent_t pev[5] = {};       // sharded rank 0 phases: start, bcast done, local done,
  bool phases_pending = false;   //   gather done, end
  bool timing_pending = false;
  // CUDA graphs per (op, B, k, nq)
  struct GraphEntry {
    cudaGraphExec_t exec;
    int launches;
  };
  bool use_graphs = false;
  std::map<uint64_t, GraphEntry> graphs;
};

static void count_launch(vx_index* h, int n = 1) { h->st.kernel_launches += n; }

// Timing events: inside a stream capture they must be EXTERNAL event nodes, or the graph only
// uses them for internal ordering and never records them for the host to read.
static cudaError_t record_ev(vx_index* h, cudaEvent_t e, cudaStream_t st) {
  return cudaEventRecordWithFlags(e, st,
                                  h->tev == h->gev ? cudaEventRecordExternal : cudaEventRecordDefault);
}

extern "C" int32_t vx_abi_version(void) { return VX_ABI_VERSION; }
extern "C" const char* vx_last_error(void) { return g_err.c_str(); }

static int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
static int kcap_of(int k) { return std::max(16, next_pow2(k)); }

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
    ALLOC(h->tokens, (size_t)d->tok_blocks * d->tok_per_doc * d->tok_dim * 2);
  h->grid = h->num_sms;
  ALLOC(h->d_q, B * D * 4);
  if (d->tok_per_doc > 0) ALLOC(h->d_qtok, B * d->max_qtok * d->tok_dim * 4);
  if (d->tok_per_doc > 0 && d->n_shards > 1) ALLOC(h->d_qtok16, B * d->max_qtok * d->tok_dim * 2);
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
  ALLOC(h->d_hdr, 16);
  ALLOC(h->d_ckeys, B * 512 * 8);
  ALLOC(h->d_flags, B * 4);
  ALLOC(h->d_xnorm, 16);
  ALLOC(h->d_fq, B * D * 4);
  ALLOC(h->d_fidx, B * 4);
  ALLOC(h->d_fcount, 16);
  // bf16 shadow for the coarse scan: K-chunks of 64 bf16 (one 128-byte swizzle atom), so
  // D % 64 == 0; otherwise the coarse scan reads the fp32 rows as TF32 (32-wide chunks)
  if (!(d->flags & VX_FLAG_NO_BF16_SHADOW) && D % 64 == 0) {
    ALLOC(h->docs16, (size_t)h->n_local * D * 2);
    ALLOC(h->d_q16, B * D * 2);
  }
#undef ALLOC
  if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&h->stream2, cudaStreamNonBlocking) != cudaSuccess ||
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
  if (cudaMallocHost((void**)&h->h_hdr, 16) != cudaSuccess)
    return cleanup(fail(VX_ERR_OOM, "pinned header"));
  if (cudaMallocHost((void**)&h->h_flags, B * 4) != cudaSuccess)
    return cleanup(fail(VX_ERR_OOM, "pinned flags"));
  if (cudaMemset(h->d_xnorm, 0, 16) != cudaSuccess || cudaMemset(h->d_fcount, 0, 16) != cudaSuccess)
    return cleanup(fail(VX_ERR_CUDA, "memset"));
  if (h->tokens) {
    s = make_tmap_2d(&h->tmap_tok, h->tokens, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     (uint64_t)d->tok_blocks * d->tok_per_doc, (uint64_t)d->tok_dim, 64,
                     (uint32_t)std::min(d->tok_per_doc, 256));
    if (s != VX_OK) return cleanup(s);
  }
  s = make_tmap_2d(&h->tmap_docs, h->docs, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                   (uint64_t)h->n_local, D, 32, 128);
  if (s != VX_OK) return cleanup(s);
  if (h->docs16) {
    s = make_tmap_2d(&h->tmap_docs16, h->docs16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     (uint64_t)h->n_local, D, 64, 128);
    if (s != VX_OK) return cleanup(s);
  }
  *out = h;
  return VX_OK;
}

extern "C" vx_status vx_index_destroy(vx_index* h) {
  if (!h) return VX_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->comm) nccl().CommDestroy(h->comm);
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
  void* ptrs[] = {h->docs,  h->tokens,    h->d_q,      h->d_qtok,    h->d_part, h->d_keys,
                  h->d_ids, h->d_ip,      h->d_ms,     h->d_out_ids, h->d_out_ip,
                  h->d_out_ms, h->d_send, h->d_recv, h->d_hdr, h->d_ckeys, h->d_flags,
                  h->d_xnorm, h->d_fq, h->docs16, h->d_q16, h->d_fidx, h->d_fcount,
                  h->d_qtok16};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->h_stage) cudaFreeHost(h->h_stage);
  if (h->h_hdr) cudaFreeHost(h->h_hdr);
  if (h->h_flags) cudaFreeHost(h->h_flags);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->gev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->pev)
    if (e) cudaEventDestroy(e);
  if (h->tok_ev) cudaEventDestroy(h->tok_ev);
  if (h->stream2) cudaStreamDestroy(h->stream2);
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

extern "C" vx_status vx_set_option(vx_index* h, int32_t option, int64_t value) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
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
    case VX_OPT_KPRIME:
      if (value != 0 && (value < 16 || value > 512 || (value & (value - 1))))
        return fail(VX_ERR_INVALID, "kprime %lld (0 or a power of two in [16, 512])", (long long)value);
      h->kprime = (int)value;
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
      if (value != VX_COARSE_AUTO && value != VX_COARSE_TF32 && value != VX_COARSE_BF16)
        return fail(VX_ERR_INVALID, "coarse format %lld", (long long)value);
      if (value == VX_COARSE_BF16 && !h->docs16)
        return fail(VX_ERR_STATE, "index created with VX_FLAG_NO_BF16_SHADOW");
      h->coarse = (int)value;
      return VX_OK;
    case VX_OPT_MAXSIM:
      if (value != VX_MAXSIM_AUTO && value != VX_MAXSIM_CC && value != VX_MAXSIM_TC)
        return fail(VX_ERR_INVALID, "maxsim algorithm %lld", (long long)value);
      if (value == VX_MAXSIM_TC && h->tokens &&
          !vx::maxsim_tc_supported(h->desc.max_qtok, h->desc.tok_per_doc, h->desc.tok_dim))
        return fail(VX_ERR_UNSUPPORTED, "tensor-core MaxSim needs Nd in {64,128,256}, d in {64,128}");
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
  h->st = vx_stats{};
  return VX_OK;
}

extern "C" vx_status vx_index_synth(vx_index* h, uint64_t seed) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(vx::launch_synth_rows(h->docs, seed, h->row0, h->n_local, h->desc.dim, h->stream));
  count_launch(h);
  CU_TRY(vx::launch_row_stats(h->docs, h->n_local, h->desc.dim, h->d_xnorm, h->stream));
  count_launch(h);
  if (h->docs16) {
    CU_TRY(vx::launch_to_bf16(h->docs, h->docs16, h->n_local * h->desc.dim, h->stream));
    count_launch(h);
  }
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
  // the TC certificate needs an upper bound on the row norms: recompute over the shard
  CU_TRY(vx::launch_row_stats(h->docs, h->n_local, h->desc.dim, h->d_xnorm, h->stream));
  count_launch(h);
  if (h->docs16 && n > 0) {
    const size_t off = (size_t)(row0 - h->row0) * h->desc.dim;
    CU_TRY(vx::launch_to_bf16(h->docs + off, h->docs16 + off, n * h->desc.dim, h->stream));
    count_launch(h);
  }
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
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
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
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(vx::launch_synth_tokens(h->tokens, seed, 0, h->desc.tok_blocks, h->desc.tok_per_doc,
                                 h->desc.tok_dim, h->stream));
  count_launch(h);
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

extern "C" vx_status vx_tokens_upload(vx_index* h, const uint16_t* tok, int64_t blk0, int64_t n) {
  if (!h || (!tok && n > 0)) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  if (blk0 < 0 || n < 0 || blk0 + n > h->desc.tok_blocks)
    return fail(VX_ERR_INVALID, "token blocks out of range");
  const size_t blk = (size_t)h->desc.tok_per_doc * h->desc.tok_dim;
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaMemcpyAsync(h->tokens + blk0 * blk, tok, n * blk * 2, cudaMemcpyHostToDevice,
                         h->stream));
  CU_TRY(cudaStreamSynchronize(h->stream));
  return VX_OK;
}

// ---------------------------------------------------------------- pipeline pieces

static cudaStream_t pick_stream(vx_index* h, void* s) {
  return s ? reinterpret_cast<cudaStream_t>(s) : h->stream;
}

static vx_status check_batch(vx_index* h, int32_t B, int32_t k) {
  if (B < 1 || B > h->desc.max_batch)
    return fail(VX_ERR_INVALID, "batch %d outside [1, %d]", B, h->desc.max_batch);
  if (k < 1 || k > h->desc.max_k) return fail(VX_ERR_INVALID, "k %d outside [1, %d]", k, h->desc.max_k);
  return VX_OK;
}

// Exact path: K1 scan + merge: d_q [B][D] -> keys (global ids) / ids / scores [B][k]
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
    if (g0 == 0 && !d_count) CU_TRY(record_ev(h, h->tev[0], st));
    CU_TRY(vx::launch_scan_f32(bucket, &h->tmap_docs, a, grid, smem, st));
    count_launch(h);
  }
  if (!d_count) CU_TRY(record_ev(h, h->tev[1], st));
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
static int kprime_of(const vx_index* h, int k) {
  if (h->kprime) return std::max(h->kprime, next_pow2(k));
  return std::min(256, std::max(64, 4 * next_pow2(k)));
}

static bool tc_eligible(const vx_index* h, int B, int k) {
  (void)h;
  (void)B;
  return k <= 128;
}

// Tensor-core path: K2 coarse scan (top-16 per CTA) -> K3 merge to top-k' -> K2b exact
// re-rank + certificate -> exact re-scan of any query whose certificate failed.
static vx_status local_topk_tc(vx_index* h, const float* d_q, int B, int k, uint64_t* keys,
                               int64_t* ids, float* scores, cudaStream_t st) {
  const int D = h->desc.dim;
  const int grid = h->grid;
  const int kp = kprime_of(h, k);
  const bool bf16 = h->docs16 && h->coarse != VX_COARSE_TF32;
  if (D % (bf16 ? 64 : 32)) return fail(VX_ERR_UNSUPPORTED, "TC scan: D %d", D);
  CU_TRY(record_ev(h, h->tev[0], st));
  if (bf16) {
    CU_TRY(vx::launch_to_bf16(d_q, h->d_q16, (int64_t)B * D, st));
    count_launch(h);
  }
  // queries per pass over the index: 256 (CTA pairs, or the single-CTA kernel's QT = 2 x
  // 128); VX_OPT_SCAN_PAIRS = 2 feeds 512 queries per pass on CTA pairs (QG = 2: a single
  // TMEM buffer for both groups, so the epilogue no longer overlaps the MMA — measured
  // slower than two QG = 1 passes at 10M x 768, profiles/r01/README.md)
  const bool pairs = h->use_pairs && grid % 2 == 0;
  const int GS = (pairs && h->use_pairs == 2) ? 512 : 256;
  for (int g0 = 0; g0 < B; g0 += GS) {
    const int Bg = std::min(GS, B - g0);
    const bool on_pairs = pairs && Bg > 128;
    const int QT = Bg <= 128 ? 1 : 2;
    const int a_rows = on_pairs ? 128 : (QT == 1 ? ((Bg + 7) & ~7) : 128);
    CUtensorMap tq;
    if (bf16)
      VX_TRY(make_tmap_2d(&tq, h->d_q16 + (size_t)g0 * D, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                          (uint64_t)Bg, D, 64, (uint32_t)a_rows));
    else
      VX_TRY(make_tmap_2d(&tq, d_q + (size_t)g0 * D, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                          (uint64_t)Bg, D, 32, (uint32_t)a_rows));
    vx::ScanTcArgs a;
    a.n_local = (uint32_t)h->n_local;
    a.D = D;
    a.B = Bg;
    a.a_rows = a_rows;
    a.fmt = bf16 ? 1 : 2;
    a.dbg_no_select = 0;
    a.dbg_no_select = h->dbg_tc_bits;  // timing experiments only (VX_DEBUG_TC_NOSELECT)
    a.part = h->d_part + (size_t)g0 * grid * vx::kTcListLen;
    if (on_pairs) {
      // 128 < B: CTA pairs (cta_group::2), 256 documents x 256 QG queries per pair tile
      const int QG = Bg > 256 ? 2 : 1;
      int ns2 = 0;
      const size_t smem2 = vx::scan_tc2_smem(QG, &ns2);
      a.ns = ns2;
      CU_TRY(vx::launch_scan_tc2(QG, &tq, bf16 ? &h->tmap_docs16 : &h->tmap_docs, a, grid,
                                 smem2, st));
    } else {
      // 256-document tiles halve the per-document query re-streaming from L2 (measured: B=128
      // bf16 2.31 ms vs 3.78 ms with 128; B=256 3.9 ms vs 4.36 ms) — profiles/r01/
      const int TD = h->scan_tile ? h->scan_tile : 256;
      int ns = 0;
      size_t smem = vx::scan_tc_smem(QT, TD, &ns);
      if (h->dbg_tc_stages) {  // timing experiments only (VX_DEBUG_TC_STAGES)
        const int want = h->dbg_tc_stages;
        if (want >= 2 && want < ns) {
          smem -= (size_t)(ns - want) * (QT * 16384 + TD * 128 + 16);
          ns = want;
        }
      }
      a.ns = ns;
      CU_TRY(vx::launch_scan_tc(QT, TD, &tq, bf16 ? &h->tmap_docs16 : &h->tmap_docs, a, grid,
                                smem, st));
    }
    count_launch(h);
  }
  CU_TRY(record_ev(h, h->tev[1], st));
  // merge each query's lists (P per query, stride grid lists) to the coarse top-k', exact
  // re-rank — one launch each per run of query groups with the same P (the whole batch
  // when every group ran on CTA pairs), so the 2-per-SM re-rank CTAs pack full waves
  const int ldp = grid * vx::kTcListLen;
  for (int r0 = 0; r0 < B;) {
    const int P = (pairs && std::min(GS, B - r0) > 128) ? grid / 2 : grid;
    int r1 = r0;
    while (r1 < B && ((pairs && std::min(GS, B - r1) > 128) ? grid / 2 : grid) == P) r1 += GS;
    r1 = std::min(r1, B);
    const int Bn = r1 - r0;
    const uint64_t* part = h->d_part + (size_t)r0 * ldp;
    uint64_t* ck = h->d_ckeys + (size_t)r0 * kp;
    CU_TRY(vx::launch_merge_topk(part, Bn, P * vx::kTcListLen, kp, 0, ck, nullptr, nullptr, st,
                                 nullptr, ldp));
    count_launch(h);
    CU_TRY(vx::launch_rerank(h->docs, d_q + (size_t)r0 * D, D, ck, Bn, kp, part, P, grid, k,
                             h->row0,
                             reinterpret_cast<const float*>(h->d_xnorm), bf16 ? 1 : 0,
                             keys + (size_t)r0 * k, ids + (size_t)r0 * k,
                             scores + (size_t)r0 * k, h->d_flags + r0, st));
    count_launch(h);
    r0 = r1;
  }
  // Certificate failures, entirely on device (no host round trip: the stage stays
  // capturable in one CUDA graph; every launch below exits at once when its count is 0):
  //   level 2: compact the failing queries, re-rank all their list entries above the
  //            deepest truncation point (rerank_wide_kernel) — no index access;
  //   level 3: the queries that still fail are re-scanned exactly (K1 sized by the device
  //            count) and scattered back.
  int* cnt2 = h->d_fcount;      // [count, running total] of level-2 queries
  int* cnt3 = h->d_fcount + 2;  // [count, running total] of exact re-scans
  CU_TRY(vx::launch_cert_compact(h->d_flags, B, d_q, D, h->d_fidx, cnt2, h->d_fq, st));
  count_launch(h);
  CU_TRY(vx::launch_rerank_wide(h->docs, h->d_fq, D, h->d_fidx, cnt2, h->d_part, B, GS,
                                pairs ? grid / 2 : 0, grid, k, h->row0,
                                reinterpret_cast<const float*>(h->d_xnorm), bf16 ? 1 : 0, keys,
                                ids, scores, h->d_flags, st));
  count_launch(h);
  CU_TRY(vx::launch_cert_compact(h->d_flags, B, d_q, D, h->d_fidx, cnt3, h->d_fq, st));
  count_launch(h);
  uint64_t* fk = h->d_ckeys;  // reuse: [B][k] (k <= 256)
  int64_t* fi = h->d_out_ids;
  float* fs = h->d_out_ms;
  VX_TRY(local_topk_f32(h, h->d_fq, B, k, fk, fi, fs, st, cnt3));
  CU_TRY(vx::launch_cert_scatter(h->d_fidx, cnt3, B, k, fk, fi, fs, keys, ids, scores, st));
  count_launch(h);
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
  return local_topk_f32(h, d_q, B, k, keys, ids, scores, st);
}

static vx_status run_maxsim(vx_index* h, const float* d_qtok, int B, int nq, const int64_t* d_cand,
                            int C, float* d_out, cudaStream_t st, int64_t id_lo = 0,
                            int64_t id_hi = INT64_MAX, const uint16_t* d_qtok16 = nullptr) {
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  vx::MaxSimArgs a;
  a.qtok = d_qtok;
  a.qtok16 = d_qtok16;
  a.cand = d_cand;
  a.table = h->tokens;
  a.T = h->desc.tok_blocks;
  a.B = B;
  a.nq = nq;
  a.C = C;
  a.Nd = h->desc.tok_per_doc;
  a.d = h->desc.tok_dim;
  a.out = d_out;
  a.id_lo = id_lo;
  a.id_hi = id_hi;
  const bool tc = h->maxsim_algo != VX_MAXSIM_CC &&
                  vx::maxsim_tc_supported(nq, a.Nd, a.d);
  if (h->maxsim_algo == VX_MAXSIM_TC && !tc)
    return fail(VX_ERR_UNSUPPORTED, "tensor-core MaxSim unsupported for nq=%d Nd=%d d=%d", nq, a.Nd, a.d);
  if (tc)
    CU_TRY(vx::launch_maxsim_tc(&h->tmap_tok, a, st));
  else
    CU_TRY(vx::launch_maxsim(a, st));
  count_launch(h);
  return VX_OK;
}

// ---------------------------------------------------------------- shard exchange
enum { OP_STOP = 0, OP_SEARCH = 1, OP_RESCORE = 2 };

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
static vx_status core_topk(vx_index* h, const float* d_q, int B, int k, cudaStream_t st) {
  VX_TRY(local_topk(h, d_q, B, k, h->d_keys, h->d_ids, h->d_ip, st));
  if (h->nranks == 1) return VX_OK;
  const int n = B * k;
  const bool root = h->rank == 0;
  if (root) CU_TRY(cudaEventRecord(h->pev[2], st));
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
  CU_TRY(vx::launch_merge_topk(h->d_part, B, G * k, k, 0, h->d_keys, h->d_ids, h->d_ip, st));
  count_launch(h);
  CU_TRY(cudaEventRecord(h->pev[3], st));
  return VX_OK;
}

// d_qtok: rank 0's query tokens (ignored on the shard ranks, which receive them)
static vx_status core_rescore(vx_index* h, const float* d_qtok, int B, int nq, int k,
                              int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st) {
  if (h->nranks == 1) {
    VX_TRY(run_maxsim(h, d_qtok, B, nq, h->d_ids, k, h->d_ms, st));
    CU_TRY(vx::launch_order_by(h->d_ms, h->d_ids, h->d_ip, B, k, d_ids, d_ip, d_ms, st));
    count_launch(h);
    return VX_OK;
  }
  const int n = B * k;
  const bool root = h->rank == 0;
  // the tokens travel as bf16 (the MaxSim operand precision: the kernels round fp32 tokens
  // with the same RNE anyway, so the scores are unchanged) — half the broadcast bytes
  const int64_t ntok = (int64_t)B * nq * h->desc.tok_dim;
  if (root) {
    CU_TRY(vx::launch_to_bf16(d_qtok, h->d_qtok16, ntok, st));
    count_launch(h);
  }
  NCCL_TRY(nccl().GroupStart());
  NCCL_TRY(nccl().Broadcast(h->d_qtok16, h->d_qtok16, (size_t)ntok * 2, ncclUint8, 0, h->comm, st));
  NCCL_TRY(nccl().Broadcast(h->d_ids, h->d_ids, (size_t)n, ncclInt64, 0, h->comm, st));
  NCCL_TRY(nccl().GroupEnd());
  VX_TRY(run_maxsim(h, nullptr, B, nq, h->d_ids, k, h->d_ms, st, h->row0, h->row0 + h->n_local,
                    h->d_qtok16));
  float* ms_all = reinterpret_cast<float*>(h->d_send);  // [B][k] on rank 0
  NCCL_TRY(nccl().Reduce(h->d_ms, ms_all, (size_t)n, ncclFloat32, ncclMax, 0, h->comm, st));
  if (!root) return VX_OK;
  CU_TRY(vx::launch_order_by(ms_all, h->d_ids, h->d_ip, B, k, d_ids, d_ip, d_ms, st));
  count_launch(h);
  return VX_OK;
}

// CUDA-graph mode (VX_OPT_GRAPHS, single GPU): each part for one (B, k[, nq]) is captured
// once and replayed — one launch per part instead of ~12 kernels, no host work between the
// kernels (the batcher hands each batch to the graphs of its size, north star (e)).  The
// graphs read the handle's fixed input buffers and write its fixed output buffers; user
// pointers are copied in/out around the replay.  The first batch of a shape runs the part
// eagerly (it also sets the kernels' smem attributes) and captures it for the next ones.
enum { PART_TOPK = 1, PART_RESCORE = 2 };

static vx_status part_body(vx_index* h, int part, int B, int nq, int k, cudaStream_t st) {
  if (part == PART_TOPK) {
    CU_TRY(record_ev(h, h->tev[2], st));
    VX_TRY(core_topk(h, h->d_q, B, k, st));
  } else {
    VX_TRY(core_rescore(h, h->d_qtok, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
  }
  CU_TRY(record_ev(h, h->tev[3], st));
  return VX_OK;
}

static uint64_t part_key(int part, int B, int nq, int k) {
  return ((uint64_t)part << 48) | ((uint64_t)B << 24) | ((uint64_t)k << 12) |
         (uint64_t)(part == PART_RESCORE ? nq : 0);
}

static vx_status run_part(vx_index* h, int part, int B, int nq, int k, cudaStream_t st) {
  const uint64_t key = part_key(part, B, nq, k);
  cudaEvent_t* used;
  auto it = h->graphs.find(key);
  if (it != h->graphs.end()) {
    CU_TRY(cudaGraphLaunch(it->second.exec, st));
    h->st.kernel_launches += it->second.launches;
    h->st.graph_replays += 1;
    used = h->gev;
  } else {
    VX_TRY(part_body(h, part, B, nq, k, st));
    // capture on the handle's stream after the eager run completes (capture records, it
    // does not execute)
    CU_TRY(cudaStreamSynchronize(st));
    const uint64_t before = h->st.kernel_launches;
    h->tev = h->gev;  // the graph records its own (external) events
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
    h->graphs[key] = {ex, launches};
    used = h->ev;  // this call's timing: the eager run
  }
  if (part == PART_TOPK) h->ev_start = used;
  h->ev_end = used;
  return VX_OK;
}

// Rank 0 entry, part 1: announce the batch to the shards (header, queries), then top-k.
static vx_status stage_begin(vx_index* h, int op, const float* d_q, int B, int nq, int k,
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
    NCCL_TRY(nccl().Broadcast(d_q, h->d_q, (size_t)B * h->desc.dim, ncclFloat32, 0, h->comm, st));
    CU_TRY(cudaEventRecord(h->pev[1], st));
  }
  if (h->use_graphs && h->nranks == 1) {
    if (d_q != h->d_q)
      CU_TRY(cudaMemcpyAsync(h->d_q, d_q, (size_t)B * h->desc.dim * 4, cudaMemcpyDeviceToDevice,
                             st));
    VX_TRY(run_part(h, PART_TOPK, B, nq, k, st));
  } else {
    CU_TRY(record_ev(h, h->tev[2], st));
    VX_TRY(core_topk(h, d_q, B, k, st));
    CU_TRY(record_ev(h, h->tev[3], st));
    h->ev_start = h->ev_end = h->ev;
  }
  return VX_OK;
}

static void stage_done(vx_index* h, int B) {
  if (h->nranks > 1 && h->rank == 0) {
    cudaEventRecord(h->pev[4], h->stream_last);
    h->phases_pending = true;
  }
  h->timing_pending = true;
  h->st.batches += 1;
  h->st.queries += B;
}

// part 2 of a search (no rescore): the top-k by inner product to the caller's buffers
static vx_status stage_search_out(vx_index* h, int B, int k, int64_t* d_ids, float* d_ip,
                                  cudaStream_t st) {
  const size_t n = (size_t)B * k;
  CU_TRY(cudaMemcpyAsync(d_ids, h->d_ids, n * 8, cudaMemcpyDeviceToDevice, st));
  CU_TRY(cudaMemcpyAsync(d_ip, h->d_ip, n * 4, cudaMemcpyDeviceToDevice, st));
  h->stream_last = st;
  stage_done(h, B);
  return VX_OK;
}

// part 2 of the fused stage: MaxSim rescore + order into the caller's buffers
static vx_status stage_finish(vx_index* h, const float* d_qtok, int B, int nq, int k,
                              int64_t* d_ids, float* d_ip, float* d_ms, cudaStream_t st) {
  if (h->use_graphs && h->nranks == 1) {
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
  VX_TRY(stage_begin(h, OP_SEARCH, d_q, B, 0, k, st));
  return stage_search_out(h, B, k, d_ids, d_scores, st);
}

extern "C" vx_status vx_search_rescore_dev(vx_index* h, const float* d_q, const float* d_qtok,
                                           int32_t B, int32_t nq, int32_t k, int64_t* d_ids,
                                           float* d_ip, float* d_ms, void* stream) {
  if (!h || !d_q || !d_qtok || !d_ids || !d_ip || !d_ms) return fail(VX_ERR_INVALID, "null argument");
  VX_TRY(check_batch(h, B, k));
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = pick_stream(h, stream);
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
  if (rescore && (!h->tokens || nq < 1 || nq > h->desc.max_qtok))
    return fail(VX_ERR_INVALID, "rescore needs a token store and 1 <= nq <= max_qtok");
  if (!h->use_graphs || h->nranks > 1) return VX_OK;
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  // realistic inputs (generator rows), so every eager run takes the certified fast path
  CU_TRY(vx::launch_synth_rows(h->d_q, 0x5eedull, 0, b_max, h->desc.dim, st));
  if (rescore)
    CU_TRY(vx::launch_synth_rows(h->d_qtok, 0x5eed1ull, 0, (int64_t)b_max * nq, h->desc.tok_dim, st));
  const vx_stats saved = h->st;
  for (int B = 1; B <= b_max; ++B) {
    if (!h->graphs.count(part_key(PART_TOPK, B, 0, k)))
      VX_TRY(run_part(h, PART_TOPK, B, 0, k, st));
    if (rescore && !h->graphs.count(part_key(PART_RESCORE, B, nq, k)))
      VX_TRY(run_part(h, PART_RESCORE, B, nq, k, st));
  }
  CU_TRY(cudaStreamSynchronize(st));
  h->st = saved;  // preload work is not serving work
  h->timing_pending = false;
  return VX_OK;
}

extern "C" vx_status vx_sync(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  CU_TRY(cudaSetDevice(h->device));
  CU_TRY(cudaStreamSynchronize(h->stream));
  if (h->timing_pending) {
    cudaEvent_t* E = h->ev_start;
    cudaEvent_t* F = h->ev_end;
    CU_TRY(cudaEventSynchronize(F[3]));
    float a = 0, b = 0;
    if (cudaEventElapsedTime(&a, E[0], E[1]) == cudaSuccess &&
        cudaEventElapsedTime(&b, E[2], F[3]) == cudaSuccess) {
      h->st.last_scan_ms = a;
      h->st.last_step_ms = b;
      h->st.scan_ms_total += a;
      h->st.step_ms_total += b;
      h->st.timed_batches += 1;
    }
    h->timing_pending = false;
    if (h->phases_pending) {
      for (int i = 0; i < 4; ++i) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, h->pev[i], h->pev[i + 1]) == cudaSuccess)
          h->st.phase_ms[i] = ms;
      }
      h->phases_pending = false;
    }
    int fc[4] = {0, 0, 0, 0};  // certificate levels counted on device
    CU_TRY(cudaMemcpy(fc, h->d_fcount, 16, cudaMemcpyDeviceToHost));
    h->st.cert_level2 = (uint64_t)fc[1];
    h->st.cert_fallbacks = (uint64_t)fc[3];
  }
  cudaGetLastError();
  return VX_OK;
}

// ---------------------------------------------------------------- host-buffer API
extern "C" vx_status vx_search(vx_index* h, const float* q, int32_t B, int32_t k, int64_t* ids,
                               float* scores) {
  if (!h || !q || !ids || !scores) return fail(VX_ERR_INVALID, "null argument");
  VX_TRY(check_batch(h, B, k));
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t qb = (size_t)B * h->desc.dim * 4;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  memcpy(stage, q, qb);
  CU_TRY(cudaMemcpyAsync(h->d_q, stage, qb, cudaMemcpyHostToDevice, st));
  VX_TRY(stage_begin(h, OP_SEARCH, h->d_q, B, 0, k, st));
  VX_TRY(stage_search_out(h, B, k, h->d_out_ids, h->d_out_ip, st));
  int64_t* hid = reinterpret_cast<int64_t*>(stage);
  float* hsc = reinterpret_cast<float*>(stage + (size_t)B * k * 8);
  CU_TRY(cudaMemcpyAsync(hid, h->d_out_ids, (size_t)B * k * 8, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaMemcpyAsync(hsc, h->d_out_ip, (size_t)B * k * 4, cudaMemcpyDeviceToHost, st));
  VX_TRY(vx_sync(h));
  memcpy(ids, hid, (size_t)B * k * 8);
  memcpy(scores, hsc, (size_t)B * k * 4);
  return VX_OK;
}

extern "C" vx_status vx_maxsim(vx_index* h, const float* qtok, int32_t B, int32_t nq,
                               const int64_t* cand, int32_t C, float* out) {
  if (!h || !qtok || !cand || !out) return fail(VX_ERR_INVALID, "null argument");
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  if (B < 1 || B > h->desc.max_batch || C < 1 || C > h->desc.max_k)
    return fail(VX_ERR_INVALID, "B %d / C %d outside [1,%d] / [1,%d]", B, C, h->desc.max_batch,
                h->desc.max_k);
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t tb = (size_t)B * nq * h->desc.tok_dim * 4, cb = (size_t)B * C * 8;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  memcpy(stage, qtok, tb);
  CU_TRY(cudaMemcpyAsync(h->d_qtok, stage, tb, cudaMemcpyHostToDevice, st));
  memcpy(stage + tb, cand, cb);
  CU_TRY(cudaMemcpyAsync(h->d_out_ids, stage + tb, cb, cudaMemcpyHostToDevice, st));
  VX_TRY(run_maxsim(h, h->d_qtok, B, nq, h->d_out_ids, C, h->d_out_ms, st));
  CU_TRY(cudaMemcpyAsync(stage, h->d_out_ms, (size_t)B * C * 4, cudaMemcpyDeviceToHost, st));
  VX_TRY(vx_sync(h));
  memcpy(out, stage, (size_t)B * C * 4);
  return VX_OK;
}

extern "C" vx_status vx_search_rescore(vx_index* h, const float* q, const float* qtok, int32_t B,
                                       int32_t nq, int32_t k, int64_t* ids, float* ip,
                                       float* ms) {
  if (!h || !q || !qtok || !ids || !ip || !ms) return fail(VX_ERR_INVALID, "null argument");
  VX_TRY(check_batch(h, B, k));
  if (!h->tokens) return fail(VX_ERR_STATE, "index has no token store");
  if (nq < 1 || nq > h->desc.max_qtok) return fail(VX_ERR_INVALID, "nq %d", nq);
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t qb = (size_t)B * h->desc.dim * 4, tb = (size_t)B * nq * h->desc.tok_dim * 4;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  memcpy(stage, q, qb);
  CU_TRY(cudaMemcpyAsync(h->d_q, stage, qb, cudaMemcpyHostToDevice, st));
  VX_TRY(stage_begin(h, OP_RESCORE, h->d_q, B, nq, k, st));
  // the query tokens are only read by part 2: stage + upload them while part 1 runs
  memcpy(stage + qb, qtok, tb);
  CU_TRY(cudaMemcpyAsync(h->d_qtok, stage + qb, tb, cudaMemcpyHostToDevice, h->stream2));
  CU_TRY(cudaEventRecord(h->tok_ev, h->stream2));
  CU_TRY(cudaStreamWaitEvent(st, h->tok_ev, 0));
  VX_TRY(stage_finish(h, h->d_qtok, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
  const size_t n = (size_t)B * k;
  CU_TRY(cudaMemcpyAsync(stage, h->d_out_ids, n * 8, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaMemcpyAsync(stage + n * 8, h->d_out_ip, n * 4, cudaMemcpyDeviceToHost, st));
  CU_TRY(cudaMemcpyAsync(stage + n * 12, h->d_out_ms, n * 4, cudaMemcpyDeviceToHost, st));
  VX_TRY(vx_sync(h));
  memcpy(ids, stage, n * 8);
  memcpy(ip, stage + n * 8, n * 4);
  memcpy(ms, stage + n * 12, n * 4);
  return VX_OK;
}

// ---------------------------------------------------------------- live batcher
// Wall-clock mode of the opportunistic batcher (vx_batcher.hpp) with this handle as the
// stage's executor — the "live" mode the reference reserves but does not implement
// (proj/include/vortex/config.hpp:43).  One batch in flight: the GPU stage is a serial
// resource exactly like exec::Instance::busy_until (executor.hpp:44-59).
extern "C" vx_status vx_serve_trace(vx_index* h, const uint64_t* arrivals_us, int64_t n,
                                    int32_t cap, const float* queries, const float* qtok,
                                    int32_t nq, int32_t k, int64_t* ids, double* latency_us,
                                    int64_t* batch_of, int64_t* n_batches) {
  if (!h || (n > 0 && (!arrivals_us || !queries || !latency_us)))
    return fail(VX_ERR_INVALID, "null argument");
  if (cap < 1 || cap > h->desc.max_batch) return fail(VX_ERR_INVALID, "cap %d", cap);
  VX_TRY(check_batch(h, cap, k));
  const bool rescore = qtok != nullptr;
  if (rescore && (!h->tokens || nq < 1 || nq > h->desc.max_qtok))
    return fail(VX_ERR_INVALID, "query tokens need a token store and 1 <= nq <= max_qtok");
  for (int64_t i = 1; i < n; ++i)
    if (arrivals_us[i] < arrivals_us[i - 1]) return fail(VX_ERR_INVALID, "arrivals not sorted");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  const size_t D = h->desc.dim, td = rescore ? (size_t)h->desc.tok_dim : 0;
  uint8_t* stage = static_cast<uint8_t*>(h->h_stage);
  vx::OpportunisticBatcher bat(cap);
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto now_us = [&] {
    return (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(clk::now() - t0).count();
  };
  int64_t next = 0, nb = 0;
  while (next < n || bat.queued() > 0) {
    uint64_t t = now_us();
    if (bat.queued() == 0 && next < n && arrivals_us[next] > t) {
      // idle: wait for the next planned arrival (spin the last 200 us for precision)
      while ((t = now_us()) + 200 < arrivals_us[next])
        std::this_thread::sleep_for(std::chrono::microseconds(100));
      while ((t = now_us()) < arrivals_us[next]) {
      }
    }
    while (next < n && arrivals_us[next] <= t) bat.arrive(next++);
    std::vector<int64_t> batch = bat.maybe_dispatch();
    if (batch.empty()) continue;
    const int B = (int)batch.size();
    // gather the batch's payloads (host ingress) -> pinned staging -> HBM
    for (int i = 0; i < B; ++i) memcpy(stage + i * D * 4, queries + batch[i] * D, D * 4);
    CU_TRY(cudaMemcpyAsync(h->d_q, stage, (size_t)B * D * 4, cudaMemcpyHostToDevice, st));
    if (rescore) {
      uint8_t* ts = stage + (size_t)B * D * 4;
      const size_t tb = (size_t)nq * td * 4;
      for (int i = 0; i < B; ++i) memcpy(ts + i * tb, qtok + batch[i] * nq * td, tb);
      CU_TRY(cudaMemcpyAsync(h->d_qtok, ts, (size_t)B * tb, cudaMemcpyHostToDevice, st));
    }
    VX_TRY(stage_begin(h, rescore ? OP_RESCORE : OP_SEARCH, h->d_q, B, nq, k, st));
    if (rescore)
      VX_TRY(stage_finish(h, h->d_qtok, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
    else
      VX_TRY(stage_search_out(h, B, k, h->d_out_ids, h->d_out_ip, st));
    int64_t* hid = reinterpret_cast<int64_t*>(stage);
    CU_TRY(cudaMemcpyAsync(hid, h->d_out_ids, (size_t)B * k * 8, cudaMemcpyDeviceToHost, st));
    VX_TRY(vx_sync(h));
    const uint64_t done = now_us();
    for (int i = 0; i < B; ++i) {
      const int64_t q = batch[i];
      latency_us[q] = (double)done - (double)arrivals_us[q];
      if (batch_of) batch_of[q] = nb;
      if (ids) memcpy(ids + q * k, hid + (size_t)i * k, (size_t)k * 8);
    }
    ++nb;
    bat.complete();
  }
  if (n_batches) *n_batches = nb;
  return VX_OK;
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

extern "C" vx_status vx_shard_serve(vx_index* h) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  if (!h->comm || h->rank == 0) return fail(VX_ERR_STATE, "vx_shard_serve is for ranks != 0");
  CU_TRY(cudaSetDevice(h->device));
  cudaStream_t st = h->stream;
  for (;;) {
    NCCL_TRY(nccl().Broadcast(h->d_hdr, h->d_hdr, 4, ncclInt32, 0, h->comm, st));
    CU_TRY(cudaMemcpyAsync(h->h_hdr, h->d_hdr, 16, cudaMemcpyDeviceToHost, st));
    CU_TRY(cudaStreamSynchronize(st));
    const int op = h->h_hdr[0], B = h->h_hdr[1], k = h->h_hdr[2], nq = h->h_hdr[3];
    if (op == OP_STOP) return VX_OK;
    if (B < 1 || B > h->desc.max_batch || k < 1 || k > h->desc.max_k)
      return fail(VX_ERR_STATE, "bad batch header %d/%d/%d", op, B, k);
    if (op == OP_RESCORE && (nq < 1 || nq > h->desc.max_qtok))
      return fail(VX_ERR_STATE, "bad batch header nq %d", nq);
    NCCL_TRY(nccl().Broadcast(h->d_q, h->d_q, (size_t)B * h->desc.dim, ncclFloat32, 0, h->comm, st));
    VX_TRY(core_topk(h, h->d_q, B, k, st));
    if (op == OP_RESCORE)  // phase 2: receives the tokens + winners, MaxSim on owned winners
      VX_TRY(core_rescore(h, nullptr, B, nq, k, h->d_out_ids, h->d_out_ip, h->d_out_ms, st));
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
