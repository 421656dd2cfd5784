#!/usr/bin/env python3
"""Benchmark of the B200 retrieval stage (BASELINE.json metric: retrieval queries/sec at
p99 batch latency <= SLO, 1/2/4/8 B200, % HBM/tensor roofline).

Workload (BASELINE.json configs[2], the sharded headline config): a 10M x 768 fp32
synthetic index partitioned across N GPUs, top-100 exact inner-product retrieval plus
PreFLMR MaxSim re-scoring (32 query tokens x 128 doc tokens x dim 128, bf16 token store),
batches of B queries.  One "step" = one batch through the stage.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Prints ONE JSON line on rank 0 (contract in the task statement).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)
BF16_FALLBACK_TFLOPS = 1590.0
METRIC = "retrieval queries/sec at p99 batch latency <= SLO"


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "src": "measured", "sm_max_mhz": d.get("sm_max_mhz"),
                "bf16_tflops": d.get("bf16_tflops", BF16_FALLBACK_TFLOPS),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d.get("bf16_tflops", BF16_FALLBACK_TFLOPS))}
    return {"hbm_gbs": HBM_FALLBACK_GBS, "src": "fallback", "sm_max_mhz": 1965.0,
            "bf16_tflops": BF16_FALLBACK_TFLOPS, "bf16_tflops_sustained": BF16_FALLBACK_TFLOPS}


def scan_roofline(pk: dict, *, tc: bool, bf16: bool, n_local: int, D: int, B: int, k: int,
                  scan_ms: float) -> dict:
    """Both ceilings of the candidate scan: HBM (the index bytes it streams +
    queries + results) and compute (2*B*N*D flops on the pipe that runs it).  `bound` is the
    one with the larger minimum time; achieved/peak/frac are reported for it, the other is kept
    alongside.  Tensor peak: MEASURED_PEAKS' sustained cuBLAS bf16 (the scan runs back to back
    inside a long step); TF32 = half of it (dense kind::tf32 rate); CUDA-core fp32 = 148 SMs x
    128 FMA/clk x 2 x max clock."""
    elem = 2 if bf16 else 4
    hbm_bytes = n_local * D * elem + B * D * elem + B * k * 12
    flops = 2.0 * B * n_local * D
    s = scan_ms / 1e3
    hbm = {"achieved": hbm_bytes / s / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "bytes_per_launch": hbm_bytes}
    hbm["frac"] = hbm["achieved"] / hbm["peak"]
    hbm["frac_of_8tbs"] = hbm["achieved"] / 8000.0
    if tc:
        peak_tf = pk["bf16_tflops_sustained"] * (1.0 if bf16 else 0.5)
        pipe = "tensor (tcgen05 kind::f16)" if bf16 else "tensor (tcgen05 kind::tf32)"
    else:
        peak_tf = 148 * 128 * 2 * (pk.get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
        pipe = "fp32 FMA (CUDA cores)"
    comp = {"achieved": flops / s / 1e12, "peak": peak_tf, "unit": "TFLOP/s", "pipe": pipe,
            "flops_per_launch": flops}
    comp["frac"] = comp["achieved"] / comp["peak"]
    if tc:
        comp["frac_of_burst"] = comp["achieved"] / (pk["bf16_tflops"] * (1.0 if bf16 else 0.5))
    t_hbm = hbm_bytes / (hbm["peak"] * 1e9)
    t_comp = flops / (comp["peak"] * 1e12)
    top = hbm if t_hbm >= t_comp else comp
    return {"bound": "hbm" if top is hbm else "tensor", "achieved": top["achieved"],
            "peak": top["peak"], "unit": top["unit"], "frac": top["frac"],
            "floor_ms": max(t_hbm, t_comp) * 1e3, "hbm": hbm, "compute": comp,
            "peak_src": pk["src"]}


def parse() -> argparse.Namespace:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-docs", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=768)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--nq", type=int, default=32)
    ap.add_argument("--tok-per-doc", type=int, default=128)
    ap.add_argument("--tok-dim", type=int, default=128)
    ap.add_argument("--tok-blocks", type=int, default=1 << 18)
    ap.add_argument("--slo-ms", type=float, default=200.0)
    ap.add_argument("--scan", choices=["auto", "f32", "tc"], default="auto")
    ap.add_argument("--coarse", choices=["auto", "tf32", "bf16"], default="auto",
                    help="operand format of the tensor-core candidate scan (exact fp32 re-rank either way)")
    ap.add_argument("--tile", type=int, default=0, choices=[0, 128, 256],
                    help="documents per tensor-core scan tile (0 = library default)")
    ap.add_argument("--pairs", type=int, default=-1, choices=[-1, 0, 1, 2],
                    help="CTA-pair (cta_group::2) scan for 128 < batch <= 256")
    ap.add_argument("--graphs", type=int, default=1, choices=[0, 1],
                    help="replay one captured CUDA graph per batch shape (single GPU)")
    ap.add_argument("--cpu-budget-s", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region
    (written to a file: a pipe would hold the lines in nvidia-smi's stdio buffer)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None
        self.path = Path(f"/tmp/vx_clocks_{os.getpid()}_{device}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100", "-f", str(self.path)],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.path.exists():
                self.rows = [[x.strip() for x in ln.split(",")]
                             for ln in self.path.read_text().splitlines() if ln.strip()]
                self.path.unlink()

    def summary(self) -> dict:
        ok = [r for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        sm = [float(r[1]) for r in ok]
        mx = [float(r[2]) for r in ok]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in ok for i in range(4) if r[5 + i].lower() == "active"})
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}
        if not ok and self.rows:
            out["raw"] = ",".join(self.rows[0])[:200]
        return out


# ----------------------------------------------------------------------------- CPU legs
def cpu_stage_time(args, n_rows: int, reps: int) -> dict:
    """Times the oracle port (fp32 AVX-512, all host cores) on a bounded sample of the
    workload and scales the scan linearly in N.  Test-infrastructure import, as allowed for
    the cpu_baseline / --impl reference legs only."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import vxoracle as o
    o.build()
    B, D, k = args.batch, args.dim, args.k
    X = o.synth_rows(42, 0, n_rows, D)
    Q = o.synth_rows(43, 0, B, D)
    qtok = o.synth_rows(44, 0, B * args.nq, args.tok_dim).reshape(B, args.nq, args.tok_dim)
    T = min(args.tok_blocks, 4096)
    table = o.synth_tokens(45, 0, T, args.tok_per_doc, args.tok_dim)
    t0 = time.perf_counter()
    for _ in range(reps):
        ids, _ = o.flat_topk(X, Q, k, mode=1)
    t_scan = (time.perf_counter() - t0) / reps
    rng = np.random.default_rng(7)
    cand = np.stack([rng.choice(args.n_docs, k, replace=False) for _ in range(B)]).astype(np.int64)
    t0 = time.perf_counter()
    o.maxsim(qtok, cand, table, mode=1)
    t_ms = time.perf_counter() - t0
    scale = args.n_docs / n_rows
    per_batch = t_scan * scale + t_ms
    return {"value": B / per_batch, "unit": "queries/s", "cores": o.threads(), "kind": "port",
            "sample": (f"{n_rows} of {args.n_docs} rows x {D} fp32, B={B}, k={k}, {reps} reps, scan "
                       f"time scaled x{scale:.1f} to the full index; + MaxSim of B x {k} candidates "
                       f"({args.nq}x{args.tok_per_doc}x{args.tok_dim} bf16) on {T} token blocks"),
            "batch_s": per_batch}


def cpu_sample_rows(args) -> tuple[int, int]:
    # ~budget seconds of CPU work: scan cost ~ rows*D*B FMAs at ~O(300) GFMA/s on 16 cores
    budget = args.cpu_budget_s
    rows = min(args.n_docs, 2_000_000)
    est = rows * args.dim * max(args.batch, 16) / 3e11
    reps = max(1, min(20, int(budget / max(est, 1e-3))))
    return rows, reps


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    import paper_2511_02062_b200 as vx
    from paper_2511_02062_b200 import build
    build.build()

    B, D, k, nq, td = args.batch, args.dim, args.k, args.nq, args.tok_dim
    idx = vx.Index(args.n_docs, D, device=local, n_shards=world, shard=rank,
                   tok_per_doc=args.tok_per_doc, tok_dim=td, tok_blocks=args.tok_blocks,
                   max_batch=B, max_k=k, max_qtok=nq)
    if args.graphs:
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
    if args.tile:
        idx.set_option(vx.VX_OPT_SCAN_TILE, args.tile)
    if args.pairs >= 0:
        idx.set_option(vx.VX_OPT_SCAN_PAIRS, args.pairs)
    if args.coarse != "auto":
        idx.set_option(vx.VX_OPT_COARSE, {"tf32": vx.VX_COARSE_TF32, "bf16": vx.VX_COARSE_BF16}[args.coarse])
    if args.scan != "auto":
        idx.set_option(vx.VX_OPT_SCAN, {"f32": vx.VX_SCAN_F32, "tc": vx.VX_SCAN_TC}[args.scan])
    idx.synth(42)
    idx.tokens_synth(45)
    if world > 1:
        uid = [vx.Index.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        idx.comm_init(uid[0], world, rank)

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)  # a real stream: the library launches on it, events see it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    from paper_2511_02062_b200 import synth

    def phase(fn=None):
        """Run one phase: rank 0 drives batches (fn); other ranks serve their shard until
        rank 0 sends stop.  Barriers bracket every phase."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        if rank == 0:
            r = fn()
            if world > 1:
                idx.shard_stop()
        else:
            t0 = time.perf_counter()
            idx.shard_serve()
            r = {"span_ms": (time.perf_counter() - t0) * 1e3}
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return r

    if rank == 0:
        q_h = synth.queries(B, D)
        qt_h = synth.query_tokens(B, nq, td)
        q = torch.from_numpy(q_h).to(dev)
        qt = torch.from_numpy(qt_h).to(dev)
        ids = torch.empty((B, k), dtype=torch.int64, device=dev)
        ip = torch.empty((B, k), dtype=torch.float32, device=dev)
        ms = torch.empty((B, k), dtype=torch.float32, device=dev)

    def step():
        idx.search_rescore_dev(q, qt, ids, ip, ms, k, stream=sp)

    def warm():
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        idx.sync()
        idx.reset_stats()
        return {}

    def timed():
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            idx.sync()  # samples the scan / stage device times of this batch
        torch.cuda.synchronize(dev)
        return {"lat": [a.elapsed_time(b) for a, b in evs], "span_ms": evs[0][0].elapsed_time(evs[-1][1]),
                "stats": idx.stats()}

    def end_to_end():
        # through the public host-buffer API: H2D of queries + tokens and D2H of results per step
        for _ in range(2):
            idx.search_rescore(q_h, qt_h, k)
        n_e2e = max(3, args.steps // 2)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            idx.search_rescore(q_h, qt_h, k)
        e2e_s = (time.perf_counter() - t0) / n_e2e
        return {"value": B / e2e_s, "unit": "queries/s",
                "h2d_bytes_per_step": B * D * 4 + B * nq * td * 4, "d2h_bytes_per_step": B * k * 16}

    phase(warm)
    with ClockSampler(local) as clk:  # sampling spans the timed phase (started before its barrier)
        result = phase(timed)
    result["clocks"] = clk.summary()
    # max over ranks of the timed span (rank 0: CUDA events; shard servers: their serve span)
    max_ms = result["span_ms"]
    if world > 1:
        t = torch.tensor([max_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
    e2e = None if args.no_e2e else phase(end_to_end)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        idx.close()
        return

    lat = result["lat"]
    st = result["stats"]
    p99 = float(np.percentile(lat, 99, method="inverted_cdf"))  # nearest rank (bench.hpp:69-76)
    value = B * args.steps / (max_ms / 1e3)
    mean_step = sum(lat) / len(lat)
    pk = peaks()
    scan_ms = st["scan_ms_total"] / max(1, st["timed_batches"])
    n_local = idx.n_local
    tc = args.scan == "tc" or (args.scan == "auto" and k <= 128)
    bf16 = tc and args.coarse != "tf32"
    roof = scan_roofline(pk, tc=tc, bf16=bf16, n_local=n_local, D=D, B=B, k=k, scan_ms=scan_ms)
    kernel_name = ((f"scan_tc_kernel (K2, tcgen05 {'kind::f16 on the bf16 shadow' if bf16 else 'kind::tf32'}"
                    " + fused top-k; exact fp32 re-rank)") if tc else "scan_f32_kernel (K1)")
    cpu = None
    if not args.no_cpu_baseline:
        rows, reps = cpu_sample_rows(args)
        c = cpu_stage_time(args, rows, reps)
        cpu = {k_: c[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
    out = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "p99_batch_ms": p99,
        "mean_batch_ms": mean_step,
        "slo_ms": args.slo_ms, "slo_met": p99 <= args.slo_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"sharded {args.n_docs // 1_000_000}Mx{D} fp32 flat-IP top-{k} + "
                               f"MaxSim rescore ({nq}x{args.tok_per_doc}x{td} bf16), batch {B}",
                   "n_docs": args.n_docs, "dim": D, "batch": B, "k": k, "shards": world,
                   "tok_blocks": args.tok_blocks, "l2": "index (GB) >> 126 MB L2: every step streams from HBM",
                   "scan": args.scan, "coarse": ("bf16" if bf16 else "tf32") if tc else None,
                   "exactness": "ids+scores bit-identical to the fp32 oracle (certified re-rank)"},
        "roofline": {**roof, "kernel": kernel_name, "scan_ms": scan_ms, "traffic": None},
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(st["kernel_launches"]),
        "root_phases_ms": ({"broadcast": st["phase_ms"][0], "local_stage": st["phase_ms"][1],
                            "gather": st["phase_ms"][2], "merge": st["phase_ms"][3]}
                           if world > 1 else None),
        "clocks": result["clocks"],
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    idx.close()


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rows, reps = cpu_sample_rows(args)
    c = cpu_stage_time(args, rows, max(1, reps // max(1, args.steps)))
    steps_s = c["batch_s"] * args.steps
    out = {
        "metric": METRIC, "impl": "reference", "value": c["value"], "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": c["batch_s"] * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"sharded {args.n_docs // 1_000_000}Mx{args.dim} fp32 flat-IP top-{args.k} + "
                               f"MaxSim rescore ({args.nq}x{args.tok_per_doc}x{args.tok_dim} bf16), batch {args.batch}",
                   "n_docs": args.n_docs, "dim": args.dim, "batch": args.batch, "k": args.k},
        "cpu_baseline": {k_: c[k_] for k_ in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": c["value"], "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": ("the reference contains no retrieval arithmetic (its search stage is a profiled "
                 "latency, proj/assets/profiles.csv:17-22); this arm times the oracle port of the "
                 "stage on the host cores"),
        "timed_s": steps_s,
    }
    print(json.dumps(out), flush=True)


def main() -> None:
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
