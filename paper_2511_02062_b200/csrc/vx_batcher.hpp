// vx_batcher.hpp — the opportunistic, SLO-bounded batching policy of the reference
// (Runtime::maybe_dispatch, proj/include/vortex/runtime.hpp:617-654) for ONE stage member,
// clock-agnostic so the same code runs on a virtual clock (replay against a latency profile,
// checked against the reference runtime in oracle/_ref) and on the wall clock (live GPU mode).
//
// Policy, restated:
//  * arrivals append to a FIFO (runtime.hpp:613 m.queue.push_back);
//  * when the member is not executing and the queue is non-empty, dispatch
//    k = min(|queue|, cap) oldest queries — never wait to fill (runtime.hpp:630-634);
//  * completion clears `executing` and immediately re-runs the check (runtime.hpp:659, :671);
//  * same-timestamp order: every arrival is scheduled before any completion event
//    (bench.hpp:175-182 schedules the whole open-loop trace up front, sim.hpp:19-24 runs
//    equal timestamps FIFO), so an arrival at the completion instant joins the next batch.
//  * the cap is min(stage max_batch, replica max_batch) (runtime.hpp:631-632); the SLO bound
//    comes from choosing the replica cap as the largest profiled batch whose latency fits
//    the budget (planner.hpp:91-102 picks profile points under the cap).
#pragma once

#include <algorithm>
#include <cstdint>
#include <deque>
#include <vector>

namespace vx {

// Piecewise-linear latency profile L(b), proj/include/vortex/profile.hpp:90-109:
// below the first knot scale through it, between knots interpolate, past the last knot
// extrapolate with the last segment's slope.
struct LatencyProfile {
  std::vector<int> b;
  std::vector<double> ms;
  double latency_ms(int batch) const {
    const size_t n = b.size();
    const double x = batch;
    if (n == 1 || x <= b.front()) {
      if (n == 1 || x == b.front()) return ms.front();
      return ms.front() * x / b.front();
    }
    for (size_t i = 1; i < n; ++i)
      if (x <= b[i]) {
        const double t = (x - b[i - 1]) / double(b[i] - b[i - 1]);
        return ms[i - 1] + t * (ms[i] - ms[i - 1]);
      }
    const double slope = (ms[n - 1] - ms[n - 2]) / double(b[n - 1] - b[n - 2]);
    return ms[n - 1] + slope * (x - b[n - 1]);
  }
};

class OpportunisticBatcher {
 public:
  explicit OpportunisticBatcher(int cap) : cap_(cap < 1 ? 1 : cap) {}
  void arrive(int64_t qid) { queue_.push_back(qid); }
  bool executing() const { return executing_; }
  size_t queued() const { return queue_.size(); }
  int64_t queued_at(size_t i) const { return queue_[i]; }  // i-th oldest queued query
  // Returns the batch to dispatch now (empty if executing or nothing queued).
  std::vector<int64_t> maybe_dispatch() {
    std::vector<int64_t> batch;
    if (executing_ || queue_.empty()) return batch;
    const size_t k = std::min<size_t>(queue_.size(), (size_t)cap_);
    batch.assign(queue_.begin(), queue_.begin() + k);
    queue_.erase(queue_.begin(), queue_.begin() + k);
    executing_ = true;
    return batch;
  }
  void complete() { executing_ = false; }

 private:
  int cap_;
  bool executing_ = false;
  std::deque<int64_t> queue_;
};

}  // namespace vx
