// vx_live.cu — live (wall-clock) serving: the opportunistic batcher (vx_batcher.hpp, the
// policy of Runtime::maybe_dispatch, proj/include/vortex/runtime.hpp:617-654) driving real GPU
// stages — the "live" mode the reference reserves but does not implement
// (proj/include/vortex/config.hpp:43).  One host thread serves R members (replica mode: the
// full index on each of R GPUs), routed at ingress by the reference's power-of-two-choices
// (Runtime::pick_member, runtime.hpp:522-536, outstanding = routed minus completed,
// runtime.hpp:299, :668; draws from std::mt19937_64(seed) as sim::Rng::below, sim.hpp:86-89).
//
// Each member is a serial resource (exec::Instance::busy_until, executor.hpp:44-59): at most
// one batch in flight, dispatched the moment the member is idle with min(queued, cap) oldest
// queries.  The batch is decided at dispatch, but its DATA moves earlier: while batch n
// computes, the queries queued behind it are gathered into pinned staging and DMA'd (copy
// engine, second stream) into the member's other device input buffer, so at dispatch only the
// rows that arrived since are left to upload.  Two pinned + two device buffers per member
// alternate between consecutive batches (batch n-1's uses are complete before batch n is
// dispatched).  Results come back by DMA into pinned memory; completion is observed by
// polling an event, so the host keeps admitting, routing and pre-staging meanwhile.
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <random>
#include <thread>
#include <vector>

#include "vx_batcher.hpp"
#include "vx_handle.cuh"

namespace {

struct Member {
  vx_index* h = nullptr;
  vx::OpportunisticBatcher bat{1};
  bool busy = false;
  std::vector<int64_t> cur;
  int outstanding = 0;     // routed here and not completed (pick_member's load signal)
  int nextbuf = 0;         // input buffer the next batch uses
  int staged = 0;          // queue-head queries already staged into nextbuf
  uint8_t* pin[2] = {nullptr, nullptr};  // pinned: [cap][D] f32 queries, then [cap][nq][td] tokens
  float* dq[2] = {nullptr, nullptr};     // device copies of the same
  float* dt[2] = {nullptr, nullptr};
  int64_t* res = nullptr;                // pinned [cap][k] ids
  cudaStream_t up = nullptr;             // H2D (copy engine)
  cudaEvent_t up_ev = nullptr, done = nullptr;
};

}  // namespace

static void free_member(Member& m) {
  if (!m.h) return;
  cudaSetDevice(m.h->device);
  if (m.up) cudaStreamSynchronize(m.up);
  if (m.h->stream) cudaStreamSynchronize(m.h->stream);
  for (int i = 0; i < 2; ++i) {
    if (m.pin[i]) cudaFreeHost(m.pin[i]);
    if (m.dq[i]) cudaFree(m.dq[i]);
    if (m.dt[i]) cudaFree(m.dt[i]);
  }
  if (m.res) cudaFreeHost(m.res);
  if (m.up_ev) cudaEventDestroy(m.up_ev);
  if (m.done) cudaEventDestroy(m.done);
  if (m.up) cudaStreamDestroy(m.up);
}

extern "C" vx_status vx_serve_trace_replicas(
    vx_index* const* handles, int32_t R, const uint64_t* arrivals_us, int64_t n, int32_t cap,
    const float* queries, const float* qtok, int32_t nq, int32_t k, uint64_t seed,
    int32_t* instance_of, uint64_t* dispatch_us, uint64_t* complete_us, uint64_t* admit_seq,
    uint64_t* dispatch_seq, uint64_t* complete_seq, int64_t* ids, double* latency_us,
    int64_t* batch_of, int64_t* n_batches) {
  if (!handles || R < 1 || (n > 0 && (!arrivals_us || !queries || !latency_us)))
    return fail(VX_ERR_INVALID, "null argument");
  const bool rescore = qtok != nullptr;
  const int32_t D = handles[0]->desc.dim;
  const int32_t td = rescore ? handles[0]->desc.tok_dim : 0;
  for (int r = 0; r < R; ++r) {
    vx_index* h = handles[r];
    if (!h) return fail(VX_ERR_INVALID, "null handle %d", r);
    if (h->nranks > 1) return fail(VX_ERR_STATE, "replica members are whole-index handles");
    if (h->desc.dim != D || (rescore && h->desc.tok_dim != td))
      return fail(VX_ERR_INVALID, "replicas must share the index shape");
    if (cap < 1 || cap > h->desc.max_batch) return fail(VX_ERR_INVALID, "cap %d", cap);
    VX_TRY(check_batch(h, cap, k));
    if (rescore && (!has_tokens(h) || nq < 1 || nq > h->desc.max_qtok))
      return fail(VX_ERR_INVALID, "query tokens need a token store and 1 <= nq <= max_qtok");
  }
  for (int64_t i = 1; i < n; ++i)
    if (arrivals_us[i] < arrivals_us[i - 1]) return fail(VX_ERR_INVALID, "arrivals not sorted");
  const size_t qrow = (size_t)D * 4, trow = rescore ? (size_t)nq * td * 4 : 0;
  std::vector<Member> mem(R);
  auto cleanup = [&](vx_status s) {
    for (auto& m : mem) free_member(m);
    return s;
  };
  // errors past this point release the members' buffers
#define LIVE_TRY(expr)                  \
  do {                                  \
    const vx_status _s = (expr);        \
    if (_s != VX_OK) return cleanup(_s); \
  } while (0)
#define LIVE_CU(expr)                                                                        \
  do {                                                                                       \
    const cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                                   \
      return cleanup(fail(VX_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                          __LINE__));                                                        \
  } while (0)
  for (int r = 0; r < R; ++r) {
    Member& m = mem[r];
    m.h = handles[r];
    m.bat = vx::OpportunisticBatcher(cap);
    if (cudaSetDevice(m.h->device) != cudaSuccess) return cleanup(fail(VX_ERR_CUDA, "device"));
    bool ok = cudaStreamCreateWithFlags(&m.up, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&m.up_ev, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming) == cudaSuccess &&
              cudaMallocHost((void**)&m.res, (size_t)cap * k * 8) == cudaSuccess;
    for (int i = 0; i < 2 && ok; ++i)
      ok = cudaMallocHost((void**)&m.pin[i], (size_t)cap * (qrow + trow)) == cudaSuccess &&
           cudaMalloc((void**)&m.dq[i], (size_t)cap * qrow) == cudaSuccess &&
           (!rescore || cudaMalloc((void**)&m.dt[i], (size_t)cap * trow) == cudaSuccess);
    if (!ok) return cleanup(fail(VX_ERR_OOM, "live buffers"));
  }
  // the reference's pick_member over members 0..R-1 (all active)
  std::mt19937_64 gen(seed);
  auto below = [&](uint64_t m) { return std::uniform_int_distribution<uint64_t>(0, m - 1)(gen); };
  auto pick = [&]() -> int {
    if (R == 1) return 0;
    uint64_t a = below((uint64_t)R);
    uint64_t b = below((uint64_t)R - 1);
    if (b >= a) ++b;
    const int ia = (int)a, ib = (int)b;
    if (mem[ia].outstanding != mem[ib].outstanding)
      return mem[ia].outstanding < mem[ib].outstanding ? ia : ib;
    return ia < ib ? ia : ib;
  };
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto now_us = [&] {
    return (uint64_t)std::chrono::duration_cast<std::chrono::microseconds>(clk::now() - t0).count();
  };
  // Threads: the calling thread is the ingress (routes each arrival at its planned time); each
  // member has its own dispatcher thread (completion, dispatch, pre-staging on its GPU).  One
  // host thread serving every member was the bottleneck at R > 1 (4 members: 335 K q/s at
  // p99 <= 10 ms, below one member's 549 K — small batches, ~10 CUDA calls and a row gather per
  // dispatch, all serialised).  The reference's single event loop is kept where it matters:
  // every routing decision, dispatch snapshot and completion takes `mu` together with the
  // global sequence number, so the event order the replay tests check is one total order.
  std::mutex mu;
  uint64_t seq = 0;
  std::atomic<int64_t> remaining(n);
  std::atomic<bool> stop(false), failed(false);
  std::string err_msg;
  vx_status err_code = VX_OK;
  auto record_error = [&](vx_status code) {
    std::lock_guard<std::mutex> g(mu);
    if (!failed.exchange(true)) {
      err_code = code;
      err_msg = vx_last_error();  // thread-local in the failing thread
    }
  };
  const int stage_chunk = std::max(8, std::min(64, cap / 16));
  int64_t nb_total = 0;
  // rows [i0, i1) of the queue snapshot `rows` -> member m's next input buffer (gather + DMA)
  auto stage_rows = [&](Member& m, const int64_t* rows, int i0, int i1) -> vx_status {
    if (i1 <= i0) return VX_OK;
    uint8_t* p = m.pin[m.nextbuf];
    for (int i = i0; i < i1; ++i) {
      const int64_t q = rows[i - i0];
      memcpy(p + (size_t)i * qrow, queries + q * D, qrow);
      if (rescore) memcpy(p + (size_t)cap * qrow + (size_t)i * trow, qtok + q * (int64_t)nq * td, trow);
    }
    CU_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(m.dq[m.nextbuf]) + (size_t)i0 * qrow,
                           p + (size_t)i0 * qrow, (size_t)(i1 - i0) * qrow, cudaMemcpyHostToDevice,
                           m.up));
    if (rescore)
      CU_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(m.dt[m.nextbuf]) + (size_t)i0 * trow,
                             p + (size_t)cap * qrow + (size_t)i0 * trow, (size_t)(i1 - i0) * trow,
                             cudaMemcpyHostToDevice, m.up));
    return VX_OK;
  };
  auto member_loop = [&](int r) {
    Member& m = mem[r];
    if (cudaSetDevice(m.h->device) != cudaSuccess) {
      fail(VX_ERR_CUDA, "cudaSetDevice");
      record_error(VX_ERR_CUDA);
      return;
    }
    std::vector<int64_t> snap;
    std::vector<int64_t> batch;
    while (!stop.load(std::memory_order_relaxed) && !failed.load(std::memory_order_relaxed)) {
      bool progressed = false;
      if (m.busy) {
        const cudaError_t q = cudaEventQuery(m.done);
        if (q == cudaSuccess) {  // complete_batch (runtime.hpp:656-672)
          const uint64_t tc = now_us();
          const int B = (int)m.cur.size();
          uint64_t cs;
          {
            std::lock_guard<std::mutex> g(mu);
            cs = seq++;
            m.outstanding -= B;
            m.bat.complete();
          }
          for (int i = 0; i < B; ++i) {
            const int64_t qq = m.cur[i];
            latency_us[qq] = (double)tc - (double)arrivals_us[qq];
            if (complete_us) complete_us[qq] = tc;
            if (complete_seq) complete_seq[qq] = cs;
            if (ids) memcpy(ids + qq * k, m.res + (size_t)i * k, (size_t)k * 8);
          }
          m.busy = false;
          remaining.fetch_sub(B);
          progressed = true;
        } else if (q != cudaErrorNotReady) {
          fail(VX_ERR_CUDA, "live batch: %s", cudaGetErrorString(q));
          record_error(VX_ERR_CUDA);
          return;
        }
      }
      if (!m.busy) {  // maybe_dispatch (runtime.hpp:617-654): snapshot + sequence number
        int B = 0, pre = m.staged;
        uint64_t ds = 0;
        {
          std::lock_guard<std::mutex> g(mu);
          if (m.bat.queued() > 0) {
            B = (int)std::min<size_t>(m.bat.queued(), (size_t)cap);
            snap.clear();
            for (int i = pre; i < B; ++i) snap.push_back(m.bat.queued_at((size_t)i));
            batch = m.bat.maybe_dispatch();
            ds = seq++;
          }
        }
        if (B > 0) {
          vx_status s = stage_rows(m, snap.data(), pre, B);
          const uint64_t td_us = now_us();
          for (int64_t qq : batch) {
            if (dispatch_us) dispatch_us[qq] = td_us;
            if (dispatch_seq) dispatch_seq[qq] = ds;
          }
          vx_index* h = m.h;
          cudaStream_t st = h->stream;
          if (s == VX_OK && (cudaEventRecord(m.up_ev, m.up) != cudaSuccess ||
                             cudaStreamWaitEvent(st, m.up_ev, 0) != cudaSuccess))
            s = fail(VX_ERR_CUDA, "live: staging event");
          if (s == VX_OK)
            s = stage_begin(h, rescore ? OP_RESCORE : OP_SEARCH, m.dq[m.nextbuf], B, nq, k, st);
          if (s == VX_OK)
            s = rescore ? stage_finish(h, m.dt[m.nextbuf], B, nq, k, h->d_out_ids, h->d_out_ip,
                                       h->d_out_ms, st)
                        : stage_search_out(h, B, k, h->d_out_ids, h->d_out_ip, st);
          if (s == VX_OK &&
              (cudaMemcpyAsync(m.res, h->d_out_ids, (size_t)B * k * 8, cudaMemcpyDeviceToHost,
                               st) != cudaSuccess ||
               cudaEventRecord(m.done, st) != cudaSuccess))
            s = fail(VX_ERR_CUDA, "live: result copy");
          if (s != VX_OK) {
            record_error(s);
            return;
          }
          {
            std::lock_guard<std::mutex> g(mu);
            const int64_t id = nb_total++;
            if (batch_of)
              for (int64_t qq : batch) batch_of[qq] = id;
          }
          m.cur.swap(batch);
          m.busy = true;
          m.nextbuf ^= 1;
          m.staged = 0;
          progressed = true;
        }
      }
      if (m.busy) {  // pre-stage the queries queued behind the running batch, in chunks
        int target = 0;
        {
          std::lock_guard<std::mutex> g(mu);
          target = (int)std::min<size_t>(m.bat.queued(), (size_t)cap);
          if (target - m.staged >= stage_chunk) {
            snap.clear();
            for (int i = m.staged; i < target; ++i) snap.push_back(m.bat.queued_at((size_t)i));
          } else {
            target = m.staged;
          }
        }
        if (target > m.staged) {
          const vx_status s = stage_rows(m, snap.data(), m.staged, target);
          if (s != VX_OK) {
            record_error(s);
            return;
          }
          m.staged = target;
          progressed = true;
        }
      }
      if (!progressed) std::this_thread::yield();
    }
  };
  std::vector<std::thread> workers;
  for (int r = 0; r < R; ++r) workers.emplace_back(member_loop, r);
  // ingress: route every arrival at its planned time (runtime.hpp:289-290 tags at submit)
  for (int64_t next = 0; next < n && !failed.load();) {
    uint64_t t = now_us();
    if (arrivals_us[next] > t) {
      while ((t = now_us()) + 200 < arrivals_us[next] && !failed.load())
        std::this_thread::sleep_for(std::chrono::microseconds(100));
      while ((t = now_us()) < arrivals_us[next]) {
      }
    }
    std::lock_guard<std::mutex> g(mu);
    while (next < n && arrivals_us[next] <= t) {
      const int r = pick();
      ++mem[r].outstanding;
      mem[r].bat.arrive(next);
      if (instance_of) instance_of[next] = r;
      if (admit_seq) admit_seq[next] = seq++;
      ++next;
    }
  }
  while (remaining.load() > 0 && !failed.load()) std::this_thread::yield();
  stop.store(true);
  for (auto& w : workers) w.join();
  if (failed.load()) return cleanup(fail(err_code, "%s", err_msg.c_str()));
  if (n_batches) *n_batches = nb_total;
  for (auto& m : mem) {
    LIVE_CU(cudaSetDevice(m.h->device));
    LIVE_TRY(vx_sync(m.h));
  }
#undef LIVE_TRY
#undef LIVE_CU
  return cleanup(VX_OK);
}

extern "C" vx_status vx_serve_trace(vx_index* h, const uint64_t* arrivals_us, int64_t n,
                                    int32_t cap, const float* queries, const float* qtok,
                                    int32_t nq, int32_t k, int64_t* ids, double* latency_us,
                                    int64_t* batch_of, int64_t* n_batches) {
  if (!h) return fail(VX_ERR_INVALID, "null handle");
  vx_index* hs[1] = {h};
  return vx_serve_trace_replicas(hs, 1, arrivals_us, n, cap, queries, qtok, nq, k, 7, nullptr,
                                 nullptr, nullptr, nullptr, nullptr, nullptr, ids, latency_us,
                                 batch_of, n_batches);
}
