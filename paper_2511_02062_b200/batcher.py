"""Opportunistic, SLO-bounded batcher (reference: Runtime::maybe_dispatch,
proj/include/vortex/runtime.hpp:617-654) — Python face of the native implementation in
csrc/vx_batcher.{hpp,cu} (virtual clock) and vx_serve_trace (wall clock, live GPU).

Also: the open-loop arrival trace (bench.hpp:54-67 semantics), nearest-rank percentiles
(bench.hpp:69-76), SLO miss rate (bench.hpp:78-83), the SLO-bounded cap (largest profiled
batch whose latency fits the budget; planner.hpp:91-102) and measured profile rows in the
reference's CSV schema (profile.hpp:24: model_id,instance_size_gb,batch_size,latency_ms,
throughput_qps,memory_gb).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from ._lib import FP, LP, check


def _arrivals(rate_qps: float, count: int, seed: int, start_us: int, poisson: bool) -> np.ndarray:
    out = np.empty(count, np.uint64)
    check(_lib.load().vx_arrival_times(float(rate_qps), count, seed, start_us, 1 if poisson else 0,
                                       out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def poisson_arrivals(rate_qps: float, count: int, seed: int = 42, start_us: int = 0) -> np.ndarray:
    """Open-loop Poisson arrivals in integer microseconds (bench.hpp:54-67): exponential gaps
    from std::mt19937_64(seed), exactly the reference's trace for the same seed."""
    return _arrivals(rate_qps, count, seed, start_us, True)


def constant_arrivals(rate_qps: float, count: int, start_us: int = 0) -> np.ndarray:
    return _arrivals(rate_qps, count, 0, start_us, False)


def peak(profile: dict[int, float], batch_cap: int | None = None) -> int:
    """ProfileTable::peak (profile.hpp:110-123): the throughput-peak batch (throughput =
    1000 b / L(b)) among the profiled batches <= batch_cap; ties resolve to the smaller batch."""
    best, best_tp = None, -1.0
    for b in sorted(profile):
        if batch_cap is not None and b > batch_cap:
            continue
        tp = 1000.0 * b / profile[b]
        if tp > best_tp:
            best, best_tp = b, tp
    if best is None:
        raise ValueError("no profiled batch within the cap")
    return best


def percentile(values, p: float) -> float:
    """Nearest rank: the ceil(p/100*n)-th smallest (bench.hpp:69-76)."""
    v = np.sort(np.asarray(values, np.float64))
    if v.size == 0:
        raise ValueError("percentile of empty sample")
    rank = min(max(math.ceil(p / 100.0 * v.size), 1), v.size)
    return float(v[rank - 1])


def slo_miss_rate(latencies_us, target_us: float) -> float:
    v = np.asarray(latencies_us, np.float64)
    if v.size == 0:
        raise ValueError("miss rate of empty sample")
    return float((v > target_us).mean())


def slo_cap(profile: dict[int, float], slo_ms: float, stage_max_batch: int | None = None) -> int:
    """Largest profiled batch whose latency fits the SLO budget (and the stage cap)."""
    ok = [b for b, ms in profile.items() if ms <= slo_ms and (stage_max_batch is None or b <= stage_max_batch)]
    return max(ok) if ok else 1


def profile_rows(model_id: str, size_gb: float, profile: dict[int, float], memory_gb: float) -> str:
    out = "model_id,instance_size_gb,batch_size,latency_ms,throughput_qps,memory_gb\n"
    for b in sorted(profile):
        ms = profile[b]
        out += f"{model_id},{size_gb:g},{b},{ms:.6f},{1000.0 * b / ms:.3f},{memory_gb:.3f}\n"
    return out


def simulate(arrivals_us, cap: int, knots: dict[int, float]):
    """Virtual-clock replay (native).  Returns (batch_of, dispatch_us, complete_us)."""
    lib = _lib.load()
    a = np.ascontiguousarray(arrivals_us, np.uint64)
    n = a.shape[0]
    kb = np.array(sorted(knots), np.int32)
    km = np.array([knots[b] for b in sorted(knots)], np.float64)
    bo = np.empty(n, np.int64)
    du = np.empty(n, np.uint64)
    cu = np.empty(n, np.uint64)
    nb = C.c_int64()
    U64P = C.POINTER(C.c_uint64)
    check(lib.vx_batcher_simulate(a.ctypes.data_as(U64P), n, cap, kb.ctypes.data_as(C.POINTER(C.c_int32)),
                                  km.ctypes.data_as(C.POINTER(C.c_double)), kb.shape[0],
                                  bo.ctypes.data_as(LP), du.ctypes.data_as(U64P),
                                  cu.ctypes.data_as(U64P), C.byref(nb)))
    return bo, du, cu


def simulate_replicas(arrivals_us, replicas: int, cap: int, knots: dict[int, float],
                      seed: int = 7):
    """Replica mode on the virtual clock: `replicas` members behind the reference's
    power-of-two-choices router (runtime.hpp:522-536; seed 7 = RuntimeOptions::seed).
    Returns (instance_of, dispatch_us, complete_us, n_batches)."""
    lib = _lib.load()
    a = np.ascontiguousarray(arrivals_us, np.uint64)
    n = a.shape[0]
    kb = np.array(sorted(knots), np.int32)
    km = np.array([knots[b] for b in sorted(knots)], np.float64)
    io = np.empty(n, np.int32)
    du = np.empty(n, np.uint64)
    cu = np.empty(n, np.uint64)
    nb = C.c_int64()
    U64P = C.POINTER(C.c_uint64)
    check(lib.vx_batcher_simulate_replicas(
        a.ctypes.data_as(U64P), n, replicas, cap, kb.ctypes.data_as(C.POINTER(C.c_int32)),
        km.ctypes.data_as(C.POINTER(C.c_double)), kb.shape[0], seed,
        io.ctypes.data_as(C.POINTER(C.c_int32)), du.ctypes.data_as(U64P), cu.ctypes.data_as(U64P),
        C.byref(nb)))
    return io, du, cu, nb.value


def serve_trace(index, arrivals_us, cap: int, queries: np.ndarray, qtok: np.ndarray | None, k: int,
                want_ids: bool = False):
    """Live mode on the GPU: returns (latency_us, batch_of, ids or None)."""
    a = np.ascontiguousarray(arrivals_us, np.uint64)
    n = a.shape[0]
    q = np.ascontiguousarray(queries, np.float32)
    t = None if qtok is None else np.ascontiguousarray(qtok, np.float32)
    lat = np.empty(n, np.float64)
    bo = np.empty(n, np.int64)
    ids = np.empty((n, k), np.int64) if want_ids else None
    nb = C.c_int64()
    U64P = C.POINTER(C.c_uint64)
    check(index.lib.vx_serve_trace(index.handle, a.ctypes.data_as(U64P), n, cap, q.ctypes.data_as(FP),
                                   None if t is None else t.ctypes.data_as(FP),
                                   0 if t is None else t.shape[1], k,
                                   None if ids is None else ids.ctypes.data_as(LP),
                                   lat.ctypes.data_as(C.POINTER(C.c_double)), bo.ctypes.data_as(LP),
                                   C.byref(nb)))
    return lat, bo, ids


def serve_trace_replicas(indexes, arrivals_us, cap: int, queries: np.ndarray, qtok: np.ndarray | None,
                         k: int, seed: int = 7, want_ids: bool = False) -> dict:
    """Live replica mode (vx_serve_trace_replicas): R whole-index handles (one per GPU), queries
    routed at arrival by the reference's power of two choices (runtime.hpp:522-536).  Returns a
    dict of per-query arrays: latency_us, instance, dispatch_us, complete_us, admit_seq,
    dispatch_seq, complete_seq, batch_of (+ ids), and n_batches."""
    lib = _lib.load()
    a = np.ascontiguousarray(arrivals_us, np.uint64)
    n = a.shape[0]
    q = np.ascontiguousarray(queries, np.float32)
    t = None if qtok is None else np.ascontiguousarray(qtok, np.float32)
    R = len(indexes)
    hs = (C.c_void_p * R)(*[ix.handle.value for ix in indexes])
    out = {"latency_us": np.empty(n, np.float64), "instance": np.empty(n, np.int32),
           "dispatch_us": np.empty(n, np.uint64), "complete_us": np.empty(n, np.uint64),
           "admit_seq": np.empty(n, np.uint64), "dispatch_seq": np.empty(n, np.uint64),
           "complete_seq": np.empty(n, np.uint64),
           "batch_of": np.empty(n, np.int64)}
    ids = np.empty((n, k), np.int64) if want_ids else None
    nb = C.c_int64()
    U64P = C.POINTER(C.c_uint64)
    check(lib.vx_serve_trace_replicas(
        hs, R, a.ctypes.data_as(U64P), n, cap, q.ctypes.data_as(FP),
        None if t is None else t.ctypes.data_as(FP), 0 if t is None else t.shape[1], k, seed,
        out["instance"].ctypes.data_as(C.POINTER(C.c_int32)), out["dispatch_us"].ctypes.data_as(U64P),
        out["complete_us"].ctypes.data_as(U64P), out["admit_seq"].ctypes.data_as(U64P),
        out["dispatch_seq"].ctypes.data_as(U64P), out["complete_seq"].ctypes.data_as(U64P), None if ids is None else ids.ctypes.data_as(LP),
        out["latency_us"].ctypes.data_as(C.POINTER(C.c_double)), out["batch_of"].ctypes.data_as(LP),
        C.byref(nb)))
    out["n_batches"] = nb.value
    if want_ids:
        out["ids"] = ids
    return out
