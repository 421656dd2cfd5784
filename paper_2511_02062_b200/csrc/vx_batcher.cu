// vx_batcher.cu — virtual-clock replay of the opportunistic batcher (no GPU), the C-ABI
// vx_batcher_simulate.  The same OpportunisticBatcher drives the live GPU mode
// (vx_serve_trace in vx_api.cu).  Event semantics follow the reference simulator:
//   SimExecutor::execute_batch: end = start + micros(L(b) * 1000)  (executor.hpp:172-182,
//   the cast truncates toward zero), completion fires at `end`; arrivals at the same
//   instant run first (they were scheduled earlier, sim.hpp:19-24 FIFO tie order).
#include <stdint.h>

#include <cmath>
#include <random>
#include <string>

#include "../../include/vortex_b200.h"
#include "vx_batcher.hpp"

extern "C" vx_status vx_batcher_simulate(const uint64_t* arrivals_us, int64_t n, int32_t cap,
                                         const int32_t* knot_batch, const double* knot_ms,
                                         int32_t n_knots, int64_t* batch_of,
                                         uint64_t* dispatch_us, uint64_t* complete_us,
                                         int64_t* n_batches) {
  if (n < 0 || cap < 1 || n_knots < 1 || !knot_batch || !knot_ms || (n > 0 && !arrivals_us))
    return VX_ERR_INVALID;
  vx::LatencyProfile prof;
  for (int i = 0; i < n_knots; ++i) {
    if (knot_batch[i] < 1 || (i > 0 && knot_batch[i] <= knot_batch[i - 1])) return VX_ERR_INVALID;
    prof.b.push_back(knot_batch[i]);
    prof.ms.push_back(knot_ms[i]);
  }
  for (int64_t i = 1; i < n; ++i)
    if (arrivals_us[i] < arrivals_us[i - 1]) return VX_ERR_INVALID;
  vx::OpportunisticBatcher bat(cap);
  int64_t next = 0, nb = 0;
  uint64_t end = 0;
  std::vector<int64_t> cur;
  auto dispatch = [&](uint64_t now) {
    std::vector<int64_t> b = bat.maybe_dispatch();
    if (b.empty()) return;  // executing (or nothing queued): the in-flight batch stays `cur`
    cur.swap(b);
    end = now + (uint64_t)(prof.latency_ms((int)cur.size()) * 1000.0);
    for (int64_t q : cur) {
      if (batch_of) batch_of[q] = nb;
      if (dispatch_us) dispatch_us[q] = now;
    }
    ++nb;
  };
  while (next < n || bat.executing()) {
    const bool arrival_first = next < n && (!bat.executing() || arrivals_us[next] <= end);
    if (arrival_first) {
      const uint64_t now = arrivals_us[next];
      bat.arrive(next++);
      dispatch(now);
    } else {
      for (int64_t q : cur)
        if (complete_us) complete_us[q] = end;
      bat.complete();
      dispatch(end);
    }
  }
  if (n_batches) *n_batches = nb;
  return VX_OK;
}

// Replica mode: R members of one stage, each its own opportunistic batcher, and the
// reference's routing in front of them (Runtime::pick_member, runtime.hpp:522-536):
// power-of-two-choices on `outstanding` (tags issued minus stage completions,
// runtime.hpp:299, :668), ties to the lower index, two draws per query from the runtime's
// mt19937_64 (sim.hpp:80-89 Rng::below = std::uniform_int_distribution over
// std::mt19937_64, seeded with RuntimeOptions::seed = 7, runtime.hpp:188) — the same
// standard-library types, so the draws are identical.  With R = 1 no draw is made.
extern "C" vx_status vx_batcher_simulate_replicas(
    const uint64_t* arrivals_us, int64_t n, int32_t replicas, int32_t cap,
    const int32_t* knot_batch, const double* knot_ms, int32_t n_knots, uint64_t seed,
    int32_t* instance_of, uint64_t* dispatch_us, uint64_t* complete_us, int64_t* n_batches) {
  if (n < 0 || replicas < 1 || cap < 1 || n_knots < 1 || !knot_batch || !knot_ms ||
      (n > 0 && !arrivals_us))
    return VX_ERR_INVALID;
  vx::LatencyProfile prof;
  for (int i = 0; i < n_knots; ++i) {
    if (knot_batch[i] < 1 || (i > 0 && knot_batch[i] <= knot_batch[i - 1])) return VX_ERR_INVALID;
    prof.b.push_back(knot_batch[i]);
    prof.ms.push_back(knot_ms[i]);
  }
  for (int64_t i = 1; i < n; ++i)
    if (arrivals_us[i] < arrivals_us[i - 1]) return VX_ERR_INVALID;
  const int R = replicas;
  std::vector<vx::OpportunisticBatcher> bat(R, vx::OpportunisticBatcher(cap));
  std::vector<std::vector<int64_t>> cur(R);
  std::vector<uint64_t> end(R, 0), seq(R, 0);
  std::vector<int> outstanding(R, 0);
  std::mt19937_64 gen(seed);
  auto below = [&](uint64_t m) { return std::uniform_int_distribution<uint64_t>(0, m - 1)(gen); };
  auto pick = [&]() -> int {
    if (R == 1) return 0;
    uint64_t a = below((uint64_t)R);
    uint64_t b = below((uint64_t)R - 1);
    if (b >= a) ++b;
    const int ia = (int)a, ib = (int)b;
    if (outstanding[ia] != outstanding[ib]) return outstanding[ia] < outstanding[ib] ? ia : ib;
    return ia < ib ? ia : ib;
  };
  int64_t next = 0, nb = 0;
  uint64_t order = 0;  // dispatch sequence: equal completion instants run in dispatch order
  auto dispatch = [&](int r, uint64_t now) {
    std::vector<int64_t> b = bat[r].maybe_dispatch();
    if (b.empty()) return;
    cur[r].swap(b);
    end[r] = now + (uint64_t)(prof.latency_ms((int)cur[r].size()) * 1000.0);
    seq[r] = order++;
    for (int64_t q : cur[r]) {
      if (instance_of) instance_of[q] = r;
      if (dispatch_us) dispatch_us[q] = now;
    }
    ++nb;
  };
  for (;;) {
    int rc = -1;  // earliest completing replica (ties: dispatch order)
    for (int r = 0; r < R; ++r)
      if (bat[r].executing() && (rc < 0 || end[r] < end[rc] || (end[r] == end[rc] && seq[r] < seq[rc])))
        rc = r;
    if (next >= n && rc < 0) break;
    if (next < n && (rc < 0 || arrivals_us[next] <= end[rc])) {
      const uint64_t now = arrivals_us[next];
      const int r = pick();
      ++outstanding[r];
      bat[r].arrive(next++);
      dispatch(r, now);
    } else {
      for (int64_t q : cur[rc]) {
        if (complete_us) complete_us[q] = end[rc];
        --outstanding[rc];
      }
      bat[rc].complete();
      dispatch(rc, end[rc]);
    }
  }
  if (n_batches) *n_batches = nb;
  return VX_OK;
}

// Open-loop arrival schedule (bench::arrival_times, proj/include/vortex/bench.hpp:54-67):
// poisson: t += Exp(rate / 1e6) gaps drawn from std::mt19937_64(seed) through
// std::exponential_distribution<double> (sim.hpp:95-98); constant: t = start + i * 1e6/rate;
// each time rounded with llround.  Same standard-library types as the reference, so the same
// seed gives the same trace.
extern "C" vx_status vx_arrival_times(double rate_qps, int64_t count, uint64_t seed,
                                      uint64_t start_us, int32_t poisson, uint64_t* out) {
  if (!(rate_qps > 0) || count < 0 || (count > 0 && !out)) return VX_ERR_INVALID;
  std::mt19937_64 gen(seed);
  const double gap_us = 1e6 / rate_qps;
  double t = (double)start_us;
  for (int64_t i = 0; i < count; ++i) {
    if (poisson)
      t += std::exponential_distribution<double>(rate_qps / 1e6)(gen);
    else
      t = (double)start_us + (double)i * gap_us;
    out[i] = (uint64_t)std::llround(t);
  }
  return VX_OK;
}
