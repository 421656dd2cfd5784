// vx_batcher.cu — virtual-clock replay of the opportunistic batcher (no GPU), the C-ABI
// vx_batcher_simulate.  The same OpportunisticBatcher drives the live GPU mode
// (vx_serve_trace in vx_api.cu).  Event semantics follow the reference simulator:
//   SimExecutor::execute_batch: end = start + micros(L(b) * 1000)  (executor.hpp:172-182,
//   the cast truncates toward zero), completion fires at `end`; arrivals at the same
//   instant run first (they were scheduled earlier, sim.hpp:19-24 FIFO tie order).
#include <stdint.h>

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
