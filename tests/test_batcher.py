"""The product batcher (csrc/vx_batcher.{hpp,cu}, virtual clock) against the REFERENCE
runtime's own decisions: committed fixtures produced by oracle/_ref (tests/golden/
make_batcher_golden.py) and, when the reference is mounted, fresh random traces run through
the reference binary.  Plus the reference's own batching test (test_runtime.cpp:246-268) and
the bench helpers (bench.hpp:54-83).  CPU only."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
DRIVER = ROOT / "oracle" / "_ref" / "vortex_ref_driver"


@pytest.fixture(scope="module")
def bat(vxlib):
    from paper_2511_02062_b200 import batcher
    return batcher


def fixtures():
    return json.loads((ROOT / "tests" / "golden" / "batcher_ref.json").read_text())


@pytest.mark.parametrize("case", fixtures(), ids=lambda c: c["name"])
def test_matches_reference_runtime_fixtures(bat, case):
    knots = {int(k): v for k, v in case["knots"].items()}
    b, d, c = bat.simulate(case["arrivals_us"], case["cap"], knots)
    assert b.tolist() == case["batch"]
    assert d.tolist() == case["dispatch_us"]
    assert c.tolist() == case["complete_us"]


def test_reference_opportunistic_batching_semantics(bat):
    # test_runtime.cpp:246-268: first arrival alone; 5 queued while busy -> one batch of 5;
    # 20 queued at once never exceed the cap of 8
    arr = [0] * 6
    b, _, _ = bat.simulate(arr, 8, {1: 10.0, 8: 40.0})
    sizes = np.bincount(b)
    assert sizes.tolist() == [1, 5]
    b, _, _ = bat.simulate([0] * 21, 8, {1: 10.0, 8: 40.0})
    assert np.bincount(b).max() <= 8 and np.bincount(b)[0] == 1


def test_fifo_order_and_conservation(bat):
    rng = np.random.default_rng(3)
    arr = np.sort(rng.integers(0, 1_000_000, 2000)).astype(np.uint64)
    b, d, c = bat.simulate(arr, 32, {1: 2.0, 32: 9.0})
    assert (np.diff(b) >= 0).all()              # FIFO: batches consume the queue in order
    assert (d >= arr).all() and (c > d).all()   # dispatched after arrival, done after dispatch
    assert len(np.unique(b)) == b.max() + 1     # every batch index used


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(6))
def test_random_traces_against_reference_binary(bat, seed):
    import sys
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    from make_batcher_golden import run_reference
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 700))
    rate = float(rng.choice([10.0, 200.0, 5000.0, 50000.0]))
    arr = np.rint(np.cumsum(rng.exponential(1e6 / rate, n))).astype(np.int64)
    if seed % 2:
        arr[rng.integers(0, n, n // 3)] = arr[0]  # duplicate timestamps
        arr = np.sort(arr)
    cap = int(rng.integers(1, 300))
    kb = np.unique(rng.integers(1, 400, int(rng.integers(1, 5))))
    knots = {int(b): float(0.5 + b * rng.uniform(0.01, 2.0)) for b in kb}
    ms = np.cumsum([knots[b] for b in sorted(knots)])  # monotone latencies
    knots = {b: float(m) for b, m in zip(sorted(knots), ms)}
    rb, rd, rc = run_reference(arr.tolist(), cap, knots)
    b, d, c = bat.simulate(arr, cap, knots)
    assert b.tolist() == rb and d.tolist() == rd and c.tolist() == rc


def replica_fixtures():
    return json.loads((ROOT / "tests" / "golden" / "batcher_replicas_ref.json").read_text())


@pytest.mark.parametrize("case", replica_fixtures(), ids=lambda c: c["name"])
def test_replica_routing_matches_reference_fixtures(bat, case):
    # Runtime::pick_member (runtime.hpp:522-536) in front of per-member batchers
    knots = {int(k): v for k, v in case["knots"].items()}
    i, d, c, _ = bat.simulate_replicas(case["arrivals_us"], case["replicas"], case["cap"], knots)
    assert i.tolist() == case["instance"]
    assert d.tolist() == case["dispatch_us"]
    assert c.tolist() == case["complete_us"]


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", range(6))
def test_random_replica_traces_against_reference_binary(bat, seed):
    import sys
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    from make_batcher_golden import run_reference_replicas
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 1500))
    R = int(rng.integers(1, 9))
    rate = float(rng.choice([50.0, 2000.0, 40000.0]))
    arr = np.rint(np.cumsum(rng.exponential(1e6 / rate, n))).astype(np.int64)
    if seed % 2:
        arr[rng.integers(0, n, n // 3)] = arr[0]
        arr = np.sort(arr)
    cap = int(rng.integers(1, 200))
    knots = {1: float(rng.uniform(0.5, 5.0)), 64: float(rng.uniform(6.0, 20.0))}
    ri, rd, rc = run_reference_replicas(arr.tolist(), R, cap, knots)
    i, d, c, _ = bat.simulate_replicas(arr, R, cap, knots)
    assert i.tolist() == ri and d.tolist() == rd and c.tolist() == rc


@pytest.mark.parametrize("case", json.loads((ROOT / "tests" / "golden" / "arrivals_ref.json").read_text()),
                         ids=lambda c: f"{c['kind']}_{c['rate_qps']}")
def test_arrival_traces_match_reference_fixtures(bat, case):
    # bench::arrival_times (bench.hpp:54-67) from sim::Rng(seed) (sim.hpp:80-98)
    if case["kind"] == "poisson":
        t = bat.poisson_arrivals(case["rate_qps"], case["count"], case["seed"], case["start_us"])
    else:
        t = bat.constant_arrivals(case["rate_qps"], case["count"], case["start_us"])
    assert t.tolist() == case["times"]


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("seed", [0, 5, 42, 2**40 + 3])
def test_poisson_traces_against_reference_binary(bat, seed):
    import sys
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    from make_batcher_golden import run_reference_arrivals
    for rate, n in [(10.0, 50), (1e5, 4000)]:
        assert bat.poisson_arrivals(rate, n, seed).tolist() == run_reference_arrivals(rate, n, seed, "poisson")


def test_profile_peak(bat):
    # ProfileTable::peak (profile.hpp:110-123): max throughput, ties to the smaller batch
    prof = {1: 125.0, 4: 400.0}                     # modelD: 8 vs 10 q/s -> 4
    assert bat.peak(prof) == 4 and bat.peak(prof, batch_cap=3) == 1
    assert bat.peak({1: 10.0, 2: 20.0, 4: 50.0}) == 1   # 100 = 100 > 80: tie -> smaller
    with pytest.raises(ValueError):
        bat.peak({8: 1.0}, batch_cap=4)


def test_bench_helpers(bat):
    # bench.hpp:69-83 semantics
    assert bat.percentile(list(range(1, 101)), 95) == 95.0
    assert bat.percentile([3, 1, 2], 50) == 2.0
    assert bat.slo_miss_rate([100, 300, 200, 201], 200) == 0.5
    a = bat.constant_arrivals(10, 5, start_us=1000)
    assert a.tolist() == [1000, 101000, 201000, 301000, 401000]  # test_bench.cpp:108-113
    p = bat.poisson_arrivals(100, 10000, seed=42)
    gap = (int(p[-1]) - int(p[0])) / (len(p) - 1)
    assert abs(gap - 10000.0) < 500.0                            # test_bench.cpp:115-125
    assert (bat.poisson_arrivals(100, 50, seed=42) == bat.poisson_arrivals(100, 50, seed=42)).all()


def test_slo_cap_and_profile_rows(bat):
    prof = {1: 4.8, 16: 5.1, 64: 5.8, 128: 6.1, 256: 8.7}
    assert bat.slo_cap(prof, 6.0) == 64
    assert bat.slo_cap(prof, 200.0) == 256
    assert bat.slo_cap(prof, 200.0, stage_max_batch=4) == 1
    rows = bat.profile_rows("modelD", 180, prof, 40.0).splitlines()
    assert rows[0] == "model_id,instance_size_gb,batch_size,latency_ms,throughput_qps,memory_gb"
    assert rows[2].startswith("modelD,180,16,5.1")


@pytest.mark.skipif(not DRIVER.exists(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("csv", ["profiles/r01/modelD_b200_profile.csv", "profiles/r02/modelD_b200_profile.csv"])
def test_measured_profile_round_trips_through_reference_profile_table(bat, csv, tmp_path):
    """The B200 stage's measured rows (profiles/emit_profile.py, batcher.profile_rows) are read
    by the REFERENCE's ProfileTable::from_csv_file (profile.hpp:42-61): its latency_ms
    interpolation (profile.hpp:90-109) returns the rows at the knots and interpolates between
    them as the restatement does, and its peak (profile.hpp:110-123) is batcher.peak's."""
    import subprocess
    path = ROOT / csv
    if not path.exists():
        pytest.skip(f"{csv} not produced yet")
    rows = [ln.split(",") for ln in path.read_text().splitlines()[1:] if ln.strip()]
    prof = {int(r[2]): float(r[3]) for r in rows}
    size = rows[0][1]
    bmax = max(prof) + 100
    for cap in (max(prof), 64, 4):
        out = subprocess.run([str(DRIVER), "profile", str(path), "modelD", size, str(bmax), str(cap)],
                             check=True, capture_output=True, text=True).stdout.split("\n")
        lat = {int(a.split()[1]): float(a.split()[2]) for a in out if a.startswith("lat")}
        peak = [a for a in out if a.startswith("peak")][0].split()
        assert int(peak[1]) == bat.peak(prof, batch_cap=cap)
    knots = sorted(prof)
    for b in range(1, bmax + 1):
        if b in prof:
            assert lat[b] == prof[b]
        elif b < knots[0]:
            assert lat[b] == pytest.approx(prof[knots[0]] * b / knots[0], rel=1e-12)
        elif b <= knots[-1]:
            assert lat[b] == pytest.approx(float(np.interp(b, knots, [prof[x] for x in knots])), rel=1e-12)
    # and a profile written by batcher.profile_rows round-trips at the knots (6 decimals)
    p2 = {1: 1.234567, 8: 1.5, 64: 2.75, 1024: 7.125}
    f = tmp_path / "p.csv"
    f.write_text(bat.profile_rows("modelD", 180.0, p2, 62.3))
    out = subprocess.run([str(DRIVER), "profile", str(f), "modelD", "180", "1024", "1024"],
                         check=True, capture_output=True, text=True).stdout.split("\n")
    lat = {int(a.split()[1]): float(a.split()[2]) for a in out if a.startswith("lat")}
    assert all(lat[b] == pytest.approx(v, abs=1e-6) for b, v in p2.items())
