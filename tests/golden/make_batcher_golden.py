"""Golden fixtures for the batcher, produced by the REFERENCE runtime itself
(oracle/_ref/vortex_ref_driver, compiled from /root/reference/proj/include by oracle/Makefile).

Each case: an arrival trace (us), the stage cap, profile knots; expected per query
(batch index, dispatch us, completion us) as the reference's Runtime + SimExecutor
produce them (runtime.hpp:617-672, executor.hpp:172-182, profile.hpp:90-109).
Run:  make -C oracle ref && python tests/golden/make_batcher_golden.py
"""
from __future__ import annotations

import json
import subprocess
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
DRIVER = HERE.parents[1] / "oracle" / "_ref" / "vortex_ref_driver"


def run_reference(arrivals, cap: int, knots: dict[int, float]):
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(str(int(a)) for a in arrivals) + "\n")
        path = f.name
    ks = ",".join(f"{b}:{ms!r}" for b, ms in sorted(knots.items()))
    out = subprocess.run([str(DRIVER), "batcher", path, str(cap), ks], check=True,
                         capture_output=True, text=True).stdout
    rows = sorted(tuple(int(x) for x in ln.split()) for ln in out.strip().splitlines())
    return [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]


def run_reference_replicas(arrivals, replicas: int, cap: int, knots: dict[int, float]):
    """The reference runtime with `replicas` members routed by Runtime::pick_member."""
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("\n".join(str(int(a)) for a in arrivals) + "\n")
        path = f.name
    ks = ",".join(f"{b}:{ms!r}" for b, ms in sorted(knots.items()))
    out = subprocess.run([str(DRIVER), "replicas", path, str(cap), ks, str(replicas)], check=True,
                         capture_output=True, text=True).stdout
    rows = sorted(tuple(int(x) for x in ln.split()) for ln in out.strip().splitlines())
    return [r[1] for r in rows], [r[2] for r in rows], [r[3] for r in rows]


def run_reference_arrivals(rate_qps: float, count: int, seed: int, kind: str, start_us: int = 0):
    out = subprocess.run([str(DRIVER), "arrivals", repr(float(rate_qps)), str(count), str(seed), kind,
                          str(start_us)], check=True, capture_output=True, text=True).stdout
    return [int(x) for x in out.split()]


def replica_cases():
    rng = np.random.default_rng(12)
    gpu = {1: 4.8, 16: 5.1, 64: 5.8, 128: 6.1, 256: 8.7}
    modeld = {1: 125.0, 4: 400.0}
    out = []
    pois = np.rint(np.cumsum(rng.exponential(1e6 / 40000.0, 4000))).astype(np.int64).tolist()
    out.append(("poisson_40kqps_gpu_4replicas_cap128", pois, 4, 128, gpu))
    pois = np.rint(np.cumsum(rng.exponential(1e6 / 30.0, 300))).astype(np.int64).tolist()
    out.append(("poisson_30qps_modelD_3replicas_cap4", pois, 3, 4, modeld))
    out.append(("simultaneous_8replicas", [0] * 50 + [1000] * 50, 8, 16, gpu))
    return out


def cases():
    rng = np.random.default_rng(11)
    modeld = {1: 125.0, 4: 400.0}                       # profiles.csv:17-22
    models = {1: 100.0, 8: 200.0, 16: 320.0, 32: 640.0}  # profiles.csv:24-27
    gpu = {1: 4.8, 16: 5.1, 64: 5.8, 128: 6.1, 256: 8.7}  # measured B200 stage (bench sweep)
    out = []
    out.append(("test_runtime_opportunistic", [0, 0, 0, 0, 0, 0], 8, {1: 10.0, 8: 40.0}))
    out.append(("completion_instant_ties", [0, 125000, 125000, 525000, 525001, 741666], 4, modeld))
    out.append(("constant_10qps_modelD", list(range(0, 3_000_000, 100_000)), 4, modeld))
    pois = np.rint(np.cumsum(rng.exponential(1e6 / 60.0, 400))).astype(np.int64).tolist()
    out.append(("poisson_60qps_modelS_cap16", pois, 16, models))
    burst = sorted(rng.integers(0, 50_000, 300).tolist())
    out.append(("burst_300_gpu_cap256", burst, 256, gpu))
    pois2 = np.rint(np.cumsum(rng.exponential(1e6 / 20000.0, 5000))).astype(np.int64).tolist()
    out.append(("poisson_20kqps_gpu_cap128", pois2, 128, gpu))
    frac = {1: 0.3333, 3: 1.0001, 7: 2.5}
    out.append(("fractional_ms_truncation", list(range(0, 20_000, 700)), 7, frac))
    return out


def main() -> None:
    fixtures = []
    for name, arr, cap, knots in cases():
        b, d, c = run_reference(arr, cap, knots)
        fixtures.append({"name": name, "arrivals_us": arr, "cap": cap,
                         "knots": {str(k): v for k, v in knots.items()},
                         "batch": b, "dispatch_us": d, "complete_us": c})
    (HERE / "batcher_ref.json").write_text(json.dumps(fixtures))
    rep = []
    for name, arr, R, cap, knots in replica_cases():
        i, d, c = run_reference_replicas(arr, R, cap, knots)
        rep.append({"name": name, "arrivals_us": arr, "replicas": R, "cap": cap,
                    "knots": {str(k): v for k, v in knots.items()},
                    "instance": i, "dispatch_us": d, "complete_us": c})
    (HERE / "batcher_replicas_ref.json").write_text(json.dumps(rep))
    arr = [{"rate_qps": r, "count": n, "seed": sd, "kind": kd, "start_us": st,
            "times": run_reference_arrivals(r, n, sd, kd, st)}
           for r, n, sd, kd, st in [(60.0, 500, 42, "poisson", 0), (20000.0, 3000, 7, "poisson", 1234),
                                    (333.0, 100, 1, "constant", 50)]]
    (HERE / "arrivals_ref.json").write_text(json.dumps(arr))
    print("wrote", len(fixtures), "cases")


if __name__ == "__main__":
    main()
