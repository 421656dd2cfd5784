#!/usr/bin/env python3
"""Benchmark of the B200 retrieval stage (BASELINE.json metric: retrieval queries/sec at
p99 batch latency <= SLO, 1/2/4/8 B200, % HBM/tensor roofline).

Default workload (BASELINE.json configs[2], the sharded headline config): a 10M x 768 fp32
synthetic index partitioned across N GPUs, top-100 exact inner-product retrieval plus
PreFLMR MaxSim re-scoring (32 query tokens x 128 doc tokens x dim 128, bf16 token store),
batches of B = 1024 queries (the batcher's cap under saturation: p99 batch latency ~15 ms
on one GPU, far inside the 200 ms SLO; per-GPU throughput is flat in B >= 256 because the
scan is tensor-bound there, and the larger batch amortises the per-batch exchange at N > 1).
One "step" = one batch through the stage.

The other configs run with --workload (one JSON line each, same keys):
    flat    configs[0]  100K x 768 top-10, batch 16 (L2 flushed between steps)
    maxsim  configs[1]  MaxSim of 64 queries x top-100 candidates (K4 alone)
    audio   configs[3]  1M x 1024 top-10, Poisson trace through the live batcher; value =
                        the best rate whose p99 <= SLO (default 10 ms)
    search  configs[4]  one point of the large-batch sweep (--batch 1..4096), search only

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


def scan_passes(tc: bool, B: int, pairs: int) -> tuple[int, int]:
    """(launches of the scan kernel per batch, queries per launch) for the stage's
    partitioning (vx_stage.cu local_topk_tc): CTA-pair passes of 512 queries (pairs = 2, the
    default) or 256 (pairs = 1) for B > 128, one single-CTA pass of <= 256 otherwise; the exact
    K1 scan (not tc) covers the batch in one launch."""
    if not tc:
        return 1, B
    gs = 512 if pairs in (-1, 2) and B > 256 else 256
    n = (B + gs - 1) // gs
    return n, min(B, gs)


def scan_roofline(pk: dict, *, tc: bool, coarse: str | None, n_local: int, D: int, B: int,
                  k: int, scan_ms: float, pairs: int = -1) -> dict:
    """Both ceilings of the candidate scan: HBM (the index bytes it streams +
    queries + results) and compute (2*B*N*D flops on the pipe that runs it).  `bound` is the
    one with the larger minimum time; achieved/peak/frac are reported for it, the other is kept
    alongside.  Tensor peak: MEASURED_PEAKS' burst cuBLAS bf16.  The sustained figure was
    measured with cuBLAS bf16 power-capped to a 1.3 GHz SM clock; the s8 scan draws less power
    and holds ~1.84 GHz through the step, so it beats that figure (frac_of_sustained > 1) —
    the burst rate is the honest ceiling for it.  TF32 = half of it (dense kind::tf32 rate); s8 = twice it (kind::i8
    issues M128xN256xK32 in the 128 cycles of a bf16 K16 MMA, profiles/r01/
    microbench_mma_rate_i8.log); CUDA-core fp32 = 148 SMs x 128 FMA/clk x 2 x max clock.
    coarse: "bf16" | "tf32" | "i8" for the tensor-core scan (None: the exact K1 scan)."""
    elem = {"bf16": 2, "i8": 1}.get(coarse, 4)
    # per launch (one pass over the shard for `bq` queries); the batch takes `launches`
    launches, bq = scan_passes(tc, B, pairs)
    hbm_bytes = n_local * D * elem + bq * D * elem + bq * k * 12
    flops = 2.0 * bq * n_local * D
    s = scan_ms / 1e3 / launches  # average launch duration
    hbm = {"achieved": hbm_bytes / s / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "bytes_per_launch": hbm_bytes}
    hbm["frac"] = hbm["achieved"] / hbm["peak"]
    hbm["frac_of_8tbs"] = hbm["achieved"] / 8000.0
    mult = {"bf16": 1.0, "tf32": 0.5, "i8": 2.0}.get(coarse, 0.0)
    if tc:
        peak_tf = pk["bf16_tflops"] * mult
        pipe = {"bf16": "tensor (tcgen05 kind::f16)", "tf32": "tensor (tcgen05 kind::tf32)",
                "i8": "tensor (tcgen05 kind::i8, TOP/s)"}[coarse]
    else:
        peak_tf = 148 * 128 * 2 * (pk.get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
        pipe = "fp32 FMA (CUDA cores)"
    comp = {"achieved": flops / s / 1e12, "peak": peak_tf, "unit": "TFLOP/s", "pipe": pipe,
            "flops_per_launch": flops}
    comp["frac"] = comp["achieved"] / comp["peak"]
    if tc:
        comp["frac_of_sustained"] = comp["achieved"] / (pk["bf16_tflops_sustained"] * mult)
        # datasheet dense figures (B200_PROFILING.md, context only): bf16 2250, tf32 1100,
        # 8-bit 4500 T(FL)OP/s
        comp["frac_of_nominal"] = comp["achieved"] / {"bf16": 2250.0, "tf32": 1100.0,
                                                      "i8": 4500.0}[coarse]
    t_hbm = hbm_bytes / (hbm["peak"] * 1e9)
    t_comp = flops / (comp["peak"] * 1e12)
    top = hbm if t_hbm >= t_comp else comp
    src = pk["src"]
    if top is comp and coarse in ("i8", "tf32"):
        src += (f" ({mult:g} x bf16_tflops: kind::{'i8' if coarse == 'i8' else 'tf32'} "
                f"issues {mult:g}x the MACs of a bf16 MMA per tensor cycle — "
                f"profiles/r01/microbench_mma_rate*.log)")
    return {"bound": "hbm" if top is hbm else "tensor", "achieved": top["achieved"],
            "peak": top["peak"], "unit": top["unit"], "frac": top["frac"],
            "floor_ms": max(t_hbm, t_comp) * 1e3 * launches, "hbm": hbm, "compute": comp,
            "launches": launches, "queries_per_launch": bq, "launch_ms": s * 1e3,
            "peak_src": src}


WORKLOADS = {
    # name: (BASELINE.json config, defaults)
    "stage": ("configs[2]: sharded 10M x 768 top-100 + MaxSim rescore (the headline)",
              dict(n_docs=10_000_000, dim=768, batch=1024, k=100, slo_ms=200.0)),
    "flat": ("configs[0]: flat IP top-10, 100K x 768 fp32, batch 1-32",
             dict(n_docs=100_000, dim=768, batch=16, k=10, slo_ms=200.0)),
    "maxsim": ("configs[1]: PreFLMR MaxSim, 32 q-tokens x top-100 x 128 doc tokens, dim 128, batch 1-64",
               dict(n_docs=10_000_000, dim=768, batch=64, k=100, slo_ms=200.0)),
    "audio": ("configs[3]: AudioQuery 1M x 1024 top-10, Poisson trace through the SLO-bounded batcher",
              dict(n_docs=1_000_000, dim=1024, batch=1024, k=10, slo_ms=10.0)),
    "search": ("configs[4]: large-batch sweep point, 10M x 768 top-100 search (no rescore)",
               dict(n_docs=10_000_000, dim=768, batch=256, k=100, slo_ms=200.0)),
}


def parse() -> argparse.Namespace:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="stage",
                    help="which BASELINE.json config to run (default: the headline, configs[2])")
    ap.add_argument("--n-docs", type=int, default=None)
    ap.add_argument("--dim", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--nq", type=int, default=32)
    ap.add_argument("--tok-per-doc", type=int, default=128)
    ap.add_argument("--tok-dim", type=int, default=128)
    ap.add_argument("--tok-blocks", type=int, default=1 << 18)
    ap.add_argument("--tok-f32", action="store_true",
                    help="fp32 doc-token store (SURVEY C2's fp32 variant): exact fp32 MaxSim on "
                         "the CUDA cores; default bf16 store")
    ap.add_argument("--slo-ms", type=float, default=None)
    ap.add_argument("--scan", choices=["auto", "f32", "tc"], default="auto")
    ap.add_argument("--coarse", choices=["auto", "tf32", "bf16", "i8"], default="auto",
                    help="operand format of the tensor-core candidate scan (exact fp32 re-rank either way)")
    ap.add_argument("--tile", type=int, default=0, choices=[0, 128, 256],
                    help="documents per tensor-core scan tile (0 = library default)")
    ap.add_argument("--pairs", type=int, default=-1, choices=[-1, 0, 1, 2],
                    help="CTA-pair (cta_group::2) scan for batch > 128 (2: 512 queries per pass)")
    ap.add_argument("--graphs", type=int, default=1, choices=[0, 1],
                    help="replay one captured CUDA graph per batch shape (single GPU)")
    ap.add_argument("--trace-s", type=float, default=0.5,
                    help="audio: seconds of Poisson arrivals per rate rung")
    ap.add_argument("--dist", choices=["iso", "aniso"], default="iso",
                    help="synthetic rows: isotropic, or anisotropic (power-law per-dimension scales "
                         "+ outlier dimensions, include/vx_synth.h dist 1) — index AND queries")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    for key, v in WORKLOADS[args.workload][1].items():
        if getattr(args, key) is None:
            setattr(args, key, v)
    return args


def workload_name(args) -> str:
    D, k, B = args.dim, args.k, args.batch
    n = (f"{args.n_docs // 1_000_000}M" if args.n_docs >= 1_000_000 else f"{args.n_docs // 1000}K")
    if getattr(args, "dist", "iso") == "aniso":
        n += " anisotropic"
    tok = f"{args.nq}x{args.tok_per_doc}x{args.tok_dim} bf16"
    return {
        "stage": f"sharded {n}x{D} fp32 flat-IP top-{k} + MaxSim rescore ({tok}), batch {B}",
        "flat": f"flat IP top-{k}, {n}x{D} fp32, batch {B}",
        "maxsim": f"MaxSim rescore of top-{k} candidates ({tok}), batch {B}",
        "audio": (f"AudioQuery {n}x{D} fp32 top-{k}, Poisson trace through the opportunistic "
                  f"batcher (cap {B}), p99 <= {args.slo_ms:g} ms"),
        "search": f"{'sharded ' if args.gpus > 1 else ''}{n}x{D} fp32 flat-IP top-{k} search, batch {B}",
    }[args.workload]


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
def _oracle():
    """Test-infrastructure import, allowed for the cpu_baseline / --impl reference legs only."""
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    import vxoracle as o
    o.build()
    return o


def mem_available_gb() -> float:
    try:
        for ln in Path("/proc/meminfo").read_text().splitlines():
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) / 2**20
    except OSError:
        pass
    return 0.0


def sample_rows(B: int, S: int) -> np.ndarray:
    """S query rows spread evenly over a batch of B (both 512-query passes of a 1024 batch)."""
    return np.unique(np.linspace(0, B - 1, min(S, B)).round().astype(np.int64))


def _compact_blocks(o, cand: np.ndarray, args):
    """The token blocks a candidate list touches (doc id -> block id mod T), generated from the
    same seed as the device store (untimed input preparation); returns (table, local ids)."""
    T = args.tok_blocks
    blk = np.where(cand >= 0, cand % T, 0)
    uniq, inv = np.unique(blk, return_inverse=True)
    if getattr(args, "tok_f32", False):  # the fp32 store: the generator's rows, unrounded
        table = np.stack([o.synth_rows(45, int(u) * args.tok_per_doc, args.tok_per_doc,
                                       args.tok_dim) for u in uniq])
    else:
        table = o.synth_token_blocks(45, uniq, args.tok_per_doc, args.tok_dim)
    return table, np.where(cand >= 0, inv.reshape(cand.shape), -1).astype(np.int64)


def cpu_check(args, world: int, gpu: dict, timed: bool) -> tuple[dict | None, dict]:
    """The oracle on a sample of the TIMED batch's own queries over the FULL index: checks the
    GPU step's outputs (tests/stagecheck.py bar) and, when `timed`, times the oracle's scan and
    MaxSim on the host cores (the cpu_baseline).  Index rows are generated chunk by chunk (the
    10M x 768 index never exists on the host); generation is untimed input preparation, like
    the GPU index fill."""
    o = _oracle()  # (also puts tests/ on the path for the checker)
    from stagecheck import check_ip_topk, check_stage
    wl, B, D, k = args.workload, args.batch, args.dim, args.k
    S = {"flat": B, "maxsim": B}.get(wl, 64)
    sel = sample_rows(B, S)
    t_scan = t_ms = 0.0
    reps = 1
    parity = {"queries_checked": int(len(sel)), "of_batch": B}
    try:
        if wl != "maxsim":
            Qs = gpu["q"][sel]
            if wl == "flat":  # 100K rows: resident; repeat the scan for a measurable time
                X = o.synth_rows(42, 0, args.n_docs, D, 1 if args.dist == "aniso" else 0)
                rid, rsc = o.flat_topk(X, Qs, k, mode=o.F32)
                t0 = time.perf_counter()
                while True:
                    o.flat_topk(X, Qs, k, mode=o.F32)
                    t_scan = time.perf_counter() - t0
                    if t_scan > 1.0 or reps >= 200:
                        break
                    reps += 1
                t_scan /= reps
            else:
                rid, rsc, t_scan = o.flat_topk_synth(42, args.n_docs, D, Qs, k, mode=o.F32,
                                                     dist=1 if args.dist == "aniso" else 0)
        if wl in ("stage", "maxsim"):
            qts = gpu["qt"][sel]
            cand = rid if wl == "stage" else gpu["cand"][sel]
            table, local = _compact_blocks(o, cand, args)
            t0 = time.perf_counter()
            o.maxsim(qts, local, table, mode=o.F32)
            t_ms = time.perf_counter() - t0
            truth = o.maxsim(qts, local, table, mode=o.F64_Q32 if not args.tok_f32 else o.F64)
        if wl == "stage":
            r = check_stage(gpu["ids"][sel], gpu["ip"][sel], gpu["ms"][sel], rid, rsc, truth)
            parity.update(r)
            parity["bar"] = ("IP ids + scores bit-equal to the oracle's in-order fp32 chains; MaxSim "
                             "<= 1e-5 rel (+1e-6) of the fp64 MaxSim of the fp32 query tokens; order "
                             "(MaxSim desc, id asc) equal to the oracle's except within-tolerance swaps")
        elif wl == "maxsim":
            err = np.abs(gpu["ms"][sel].astype(np.float64) - truth)
            assert (err <= 1e-5 * np.abs(truth) + 1e-6).all(), float(err.max())
            parity.update({"ms_max_abs_err": float(err.max()),
                           "ms_max_rel_err": float((err / np.abs(truth)).max()),
                           "bar": "<= 1e-5 rel (+1e-6) of the fp64 MaxSim of the fp32 query tokens"})
        else:
            for j, b in enumerate(sel):
                check_ip_topk(gpu["ids"][b], gpu["ip"][b], rid[j], rsc[j])
                assert np.array_equal(gpu["ids"][b], rid[j])  # order too: (score desc, id asc)
            parity["bar"] = "ids (in order) + scores bit-equal to the oracle's in-order fp32 chains"
        parity["ok"] = True
    except AssertionError as e:
        parity.update({"ok": False, "error": repr(e)[:300]})
    cpu = None
    if timed:
        parts = []
        if wl != "maxsim":
            parts.append(f"scan of {len(sel)} of the batch's {B} queries over all {args.n_docs} rows "
                         f"x {D} fp32, k={k}" + (f" ({reps} reps)" if reps > 1 else ""))
        if wl in ("stage", "maxsim"):
            parts.append(f"MaxSim of their {k if wl == 'stage' else gpu['cand'].shape[1]} candidates "
                         f"({args.nq}x{args.tok_per_doc}x{args.tok_dim}, bf16 doc tokens, "
                         f"{table.shape[0]} distinct blocks of the {args.tok_blocks}-block store)")
        cpu = {"value": len(sel) / (t_scan + t_ms), "unit": "queries/s", "cores": o.threads(),
               "kind": "port", "sample": "; ".join(parts) + " — the queries the GPU step was checked on",
               "batch_s": (t_scan + t_ms) * B / len(sel)}
    return cpu, parity


# ----------------------------------------------------------------------------- rooflines
def maxsim_roofline(pk: dict, *, B: int, C: int, nq: int, nd: int, d: int, ms: float,
                    f32: bool = False, mhz: float | None = None) -> dict:
    """K4 (MaxSim) ceilings: HBM bytes = the candidates' token blocks (bf16,
    or fp32 for the fp32 store) + query tokens + ids/scores; flops = 2*B*C*Nq*Nd*d (algorithmic;
    the tcgen05 tile issues M=128 rows, so the tensor pipe executes 128/Nq x that).  The fp32
    store runs on the CUDA cores: its compute ceiling is 148 SMs x 128 fp32 FMA/clk."""
    hbm_bytes = B * C * nd * d * (4 if f32 else 2) + B * nq * d * 4 + B * C * 12
    flops = 2.0 * B * C * nq * nd * d
    issued = 2.0 * B * C * 128 * nd * d
    s = ms / 1e3
    hbm = {"achieved": hbm_bytes / s / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "bytes_per_launch": hbm_bytes}
    hbm["frac"] = hbm["achieved"] / hbm["peak"]
    if f32:
        clk = (mhz or pk.get("sm_max_mhz") or 1965.0) * 1e6
        peak = 148 * 128 * 2 * clk / 1e12
        comp = {"achieved": flops / s / 1e12, "peak": peak, "unit": "TFLOP/s",
                "pipe": "fp32 FMA (CUDA cores) at the kernel's clock", "flops_per_launch": flops}
    else:
        comp = {"achieved": flops / s / 1e12, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "pipe": "tensor (tcgen05 kind::f16)", "flops_per_launch": flops,
                "issued_flops_per_launch": issued,
                "issued_frac": issued / s / 1e12 / pk["bf16_tflops"]}
    comp["frac"] = comp["achieved"] / comp["peak"]
    t_hbm, t_comp = hbm_bytes / (hbm["peak"] * 1e9), flops / (comp["peak"] * 1e12)
    top = hbm if t_hbm >= t_comp else comp
    return {"bound": "hbm" if top is hbm else "tensor", "achieved": top["achieved"],
            "peak": top["peak"], "unit": top["unit"], "frac": top["frac"],
            "floor_ms": max(t_hbm, t_comp) * 1e3, "hbm": hbm, "compute": comp,
            "peak_src": pk["src"]}


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
    from paper_2511_02062_b200 import build, synth
    build.build()

    wl = args.workload
    B, D, k, nq, td = args.batch, args.dim, args.k, args.nq, args.tok_dim
    sharded = wl in ("stage", "flat", "search") and world > 1   # else: independent replicas
    tokens = wl in ("stage", "maxsim")
    idx = vx.Index(args.n_docs, D, device=local, n_shards=world if sharded else 1,
                   shard=rank if sharded else 0,
                   tok_per_doc=args.tok_per_doc if tokens else 0, tok_dim=td,
                   tok_blocks=args.tok_blocks, max_batch=B, max_k=k, max_qtok=nq,
                   flags=(vx.VX_FLAG_NO_BF16_SHADOW if wl == "maxsim" else 0)
                   | (vx.VX_FLAG_TOKENS_F32 if (tokens and args.tok_f32) else 0))
    if args.graphs:
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
    if args.tile:
        idx.set_option(vx.VX_OPT_SCAN_TILE, args.tile)
    if args.pairs >= 0:
        idx.set_option(vx.VX_OPT_SCAN_PAIRS, args.pairs)
    if args.coarse != "auto":
        idx.set_option(vx.VX_OPT_COARSE, {"tf32": vx.VX_COARSE_TF32, "bf16": vx.VX_COARSE_BF16,
                                          "i8": vx.VX_COARSE_I8}[args.coarse])
    if args.scan != "auto":
        idx.set_option(vx.VX_OPT_SCAN, {"f32": vx.VX_SCAN_F32, "tc": vx.VX_SCAN_TC}[args.scan])
    rdist = 1 if args.dist == "aniso" else 0  # row distribution (vx_synth.h)
    if wl != "maxsim":
        idx.synth(42, dist=rdist)
    if tokens:
        idx.tokens_synth(45)
    if sharded:
        uid = [vx.Index.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        idx.comm_init(uid[0], world, rank)

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)  # a real stream: the library launches on it, events see it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    driver = rank == 0 or not sharded  # ranks that issue batches (shard servers only serve)

    def phase(fn):
        """One phase: driving ranks run fn; in sharded mode the other ranks serve their
        shard until rank 0 sends stop.  Barriers bracket every phase."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        if driver:
            r = fn()
            if sharded:
                idx.shard_stop()
        else:
            t0 = time.perf_counter()
            idx.shard_serve()
            r = {"span_ms": (time.perf_counter() - t0) * 1e3}
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        return r

    # ---- inputs (resident in HBM before the timed region) and the step of each workload
    flush_l2 = wl in ("flat", "maxsim")  # working set within a few x L2: flush between steps
    l2buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None
    l2sink = torch.zeros((), dtype=torch.int64, device=dev) if flush_l2 else None
    C = k
    if driver:
        q_h = synth.queries(B, D, seed=43 + 1000 * rank, dist=rdist) if wl != "maxsim" else None
        qt_h = synth.query_tokens(B, nq, td) if tokens else None
        rng = np.random.default_rng(7 + rank)
        cand_h = (np.stack([rng.choice(args.n_docs, C, replace=False) for _ in range(B)]).astype(np.int64)
                  if wl == "maxsim" else None)
        q = torch.from_numpy(q_h).to(dev) if q_h is not None else None
        qt = torch.from_numpy(qt_h).to(dev) if qt_h is not None else None
        cand = torch.from_numpy(cand_h).to(dev) if cand_h is not None else None
        # the e2e leg's host inputs live in page-locked memory (the contract's "pinned host
        # memory"; the library then DMAs them without its staging memcpy)
        pinned_keep = []

        def pinned(a):
            if a is None:
                return None
            t = torch.from_numpy(a).pin_memory()
            pinned_keep.append(t)
            return t.numpy()
        q_h, qt_h, cand_h = pinned(q_h), pinned(qt_h), pinned(cand_h)
        ids = torch.empty((B, k), dtype=torch.int64, device=dev)
        ip = torch.empty((B, k), dtype=torch.float32, device=dev)
        msc = torch.empty((B, k), dtype=torch.float32, device=dev)

    def step():
        if wl == "stage":
            idx.search_rescore_dev(q, qt, ids, ip, msc, k, stream=sp)
        elif wl == "maxsim":
            idx.maxsim_dev(qt, cand, msc, stream=sp)
        else:  # flat / search / audio's fixed-batch kernel measurement
            idx.search_dev(q, ids, ip, k, stream=sp)

    def warm():
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize(dev)
        idx.sync()
        idx.reset_stats()
        return {}

    def timed():
        # every step is enqueued without a host round trip in between (the host runs ahead, as
        # a serving loop does), so the event pairs see device time only; the kernels time
        # themselves on the device (vx_stats.kt_*: every launch, inside the graphs)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for a, b in evs:
            if l2buf is not None:
                # untimed, outside the event pair: write a buffer 2x the L2, then read it back so
                # the L2 holds CLEAN lines (after the write alone ~126 MB of dirty lines would be
                # written back to HBM inside the next timed step, on top of its own traffic)
                l2buf.zero_()
                l2sink.copy_(l2buf.view(torch.int32).sum())
            a.record(stream)
            step()
            b.record(stream)
        torch.cuda.synchronize(dev)
        idx.sync()
        lat = [a.elapsed_time(b) for a, b in evs]
        span = sum(lat) if l2buf is not None else evs[0][0].elapsed_time(evs[-1][1])
        return {"lat": lat, "span_ms": span, "stats": idx.stats()}

    def end_to_end():
        # through the public host-buffer API: H2D of the step's inputs, D2H of its results
        def call():
            if wl == "stage":
                idx.search_rescore(q_h, qt_h, k)
            elif wl == "maxsim":
                idx.maxsim(qt_h, cand_h)
            else:
                idx.search(q_h, k)
        for _ in range(2):
            call()
        n_e2e = max(3, args.steps // 2)
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            call()
        e2e_s = (time.perf_counter() - t0) / n_e2e
        h2d = {"stage": B * D * 4 + B * nq * td * 4, "maxsim": B * nq * td * 4 + B * C * 8}.get(wl, B * D * 4)
        d2h = {"stage": B * k * 16, "maxsim": B * C * 4}.get(wl, B * k * 12)
        return {"value": B / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h}

    def trace_ladder():
        # AudioQuery (configs[3]): ONE Poisson trace through the live opportunistic batcher
        # (vx_serve_trace_replicas: host payloads -> pinned double-buffered staging -> HBM); at
        # N GPUs rank 0 serves it with N replica members (one whole-index handle per GPU)
        # routed by the reference's power of two choices.  Raise the rate until p99 > SLO or
        # the stage saturates; report the best rate that meets the SLO.
        from paper_2511_02062_b200 import batcher
        if rank != 0:
            return {}
        members = [idx]
        for r in range(1, world):  # the other GPUs' replicas, driven from this host thread
            m = vx.Index(args.n_docs, D, device=r, max_batch=B, max_k=k)
            m.set_option(vx.VX_OPT_GRAPHS, 1)
            m.synth(42, dist=rdist)
            members.append(m)
        for m in members:
            m.prepare(k, B)  # model load: the graph of every batch size 1..cap, before serving
        pool = synth.queries(4096, D, seed=43, dist=rdist)
        def rung(rate):
            n = int(min(200_000, max(2000, rate * args.trace_s)))
            arr = batcher.poisson_arrivals(rate, n, seed=11)
            qs = pool[np.arange(n) % pool.shape[0]]
            o = batcher.serve_trace_replicas(members, arr, B, qs, None, k, seed=7)
            lat, bo = o["latency_us"], o["batch_of"]
            done = arr.astype(np.float64) + lat
            span_s = (done.max() - float(arr[0])) / 1e6
            nb = int(bo.max()) + 1
            r = {"rate_qps": rate, "queries": n, "achieved_qps": n / span_s,
                 "p99_ms": batcher.percentile(lat, 99.0) / 1e3,
                 "p50_ms": batcher.percentile(lat, 50.0) / 1e3, "batches": nb, "mean_batch": n / nb}
            r["ok"] = bool(r["p99_ms"] <= args.slo_ms and r["achieved_qps"] >= 0.9 * rate)
            rungs.append(r)
            return r

        # geometric ladder (x1.6) to the first rate that misses the SLO or saturates, then
        # bisect between the last good rate and it
        rungs, best, rate, bad = [], None, 2000.0, None
        for _ in range(18):
            r = rung(rate)
            if not r["ok"]:
                bad = rate
                break
            best = r
            rate *= 1.6
        if best is not None and bad is not None:
            lo, hi = best["rate_qps"], bad
            for _ in range(3):
                mid = 0.5 * (lo + hi)
                r = rung(mid)
                if r["ok"]:
                    best, lo = r, mid
                else:
                    hi = mid
        for m in members[1:]:
            m.close()
        return {"rungs": rungs, "best": best, "members": len(members)}

    ladder = None
    if wl == "audio":
        ladder = phase(trace_ladder)
    phase(warm)
    with ClockSampler(local) as clk:  # sampling spans the timed phase (started before its barrier)
        result = phase(timed)
    result["clocks"] = clk.summary()
    # the timed batch's outputs, for the oracle check after the e2e leg (rank 0)
    gpu_out = None
    if rank == 0:
        gpu_out = {"q": q_h, "qt": qt_h, "cand": cand_h,
                   "ids": ids.cpu().numpy() if wl != "maxsim" else None,
                   "ip": ip.cpu().numpy() if wl != "maxsim" else None,
                   "ms": msc.cpu().numpy() if tokens else None}
    # max over ranks of the timed span (rank 0: CUDA events; shard servers: their serve span)
    max_ms = result["span_ms"]
    if world > 1:
        t = torch.tensor([max_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
    e2e = None if (args.no_e2e or wl == "audio") else phase(end_to_end)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        idx.close()
        return

    lat = result["lat"]
    st = result["stats"]
    p99 = float(np.percentile(lat, 99, method="inverted_cdf"))  # nearest rank (bench.hpp:69-76)
    replicas = 1 if sharded else world
    value = replicas * B * args.steps / (max_ms / 1e3)
    mean_step = sum(lat) / len(lat)
    pk = peaks()
    n_local = idx.n_local
    tc = args.scan == "tc" or (args.scan == "auto" and k <= 128)
    coarse = (args.coarse if args.coarse != "auto" else idx.coarse_auto()) if tc else None
    bf16 = coarse == "bf16"
    def kt(i):  # device-side launch timer i: (launches, mean launch ms, SM MHz in-kernel)
        n = int(st["kt_launches"][i])
        return n, (st["kt_ms"][i] / n if n else None), (st["kt_sm_mhz"][i] or None)
    if wl == "maxsim":
        n_ms, ms_launch, ms_mhz = kt(3)
        kms = ms_launch if ms_launch else mean_step
        roof = maxsim_roofline(pk, B=B, C=C, nq=nq, nd=args.tok_per_doc, d=td, ms=kms,
                               f32=args.tok_f32, mhz=ms_mhz)
        kernel_name = ("maxsim_cc_kernel (K4', fp32 token store: exact in-order fp32 chains on "
                       "the CUDA cores)" if args.tok_f32 else
                       "maxsim_tc_kernel (K4, tcgen05 kind::f16, fused row-max + sum)")
        roof.update({"kernel": kernel_name, "kernel_ms": kms, "kernel_launches": n_ms,
                     "kernel_sm_mhz": ms_mhz, "traffic": None,
                     "timing": "device-side per-launch timer (first CTA start -> last CTA end)"})
    else:
        n_sc, sc_launch, sc_mhz = kt(0 if tc else 2)
        # per batch: the summed device time of its scan launches over the timed steps
        scan_ms = (st["kt_ms"][0 if tc else 2] / args.steps if sc_launch
                   else st["scan_ms_total"] / max(1, st["timed_batches"]))
        roof = scan_roofline(pk, tc=tc, coarse=coarse, n_local=n_local, D=D, B=B, k=k,
                             scan_ms=scan_ms, pairs=args.pairs)
        roof["timing"] = ("device-side per-launch timer over every timed launch (first CTA start -> "
                          "last CTA end, %globaltimer)" if sc_launch else "CUDA events")
        roof["kernel_launches"] = n_sc
        roof["kernel_sm_mhz"] = sc_mhz
        if tc and sc_mhz:
            # the tensor pipe's own ceiling at the clock the kernel ran at (tcgen05: 8192 bf16 /
            # 16384 s8 / 4096 tf32 MACs x2 per SM per cycle, profiles/r01/microbench_mma_rate*.log)
            per_clk = {"bf16": 8192, "i8": 16384, "tf32": 4096}[coarse] * 148
            roof["compute"]["peak_at_kernel_clock"] = per_clk * sc_mhz * 1e6 / 1e12
            roof["compute"]["frac_at_kernel_clock"] = (roof["compute"]["achieved"] /
                                                       roof["compute"]["peak_at_kernel_clock"])
        n_smp, smp_launch, _ = kt(1)
        if n_smp:
            roof["sample_pass_ms"] = smp_launch
        kinds = {"bf16": "kind::f16 on the bf16 shadow", "tf32": "kind::tf32",
                 "i8": "kind::i8 on the s8 shadow"}
        kernel_name = ((f"scan_tc{'2' if tc and B > 128 and args.pairs != 0 else ''}_kernel (K2, "
                        f"tcgen05 {kinds[coarse]} + fused top-k; exact fp32 re-rank)") if tc
                       else "scan_f32_kernel (K1)")
        fam = ("scan_tc2" if B > 128 and args.pairs != 0 else "scan_tc") if tc else "scan_f32"
        if fam == "scan_tc2" and roof["queries_per_launch"] > 256:
            fam = "scan_tc2_qg2"  # two query groups on 128-document tiles
        tkey = f"{fam}/{coarse or 'f32'}/{n_local}/{D}"
        tdb = ROOT / "profiles" / "r02" / "traffic.json"
        trec = json.loads(tdb.read_text()).get(tkey) if tdb.exists() else None
        roof.update({"kernel": kernel_name, "scan_ms": scan_ms,
                     "traffic": trec["dram_bytes"] if trec else None,
                     "traffic_src": trec["source"] if trec else None})
    cpu, parity = None, None
    if not args.no_cpu_baseline:
        # cpu_baseline (N = 1 only: rank 0's host cores) and, at every N, the oracle check of
        # the timed batch's own outputs over the full index
        c, parity = cpu_check(args, world, gpu_out, timed=world == 1)
        if c:
            cpu = {k_: c[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
    cfg = config_of(args, world)
    path = {"scan": "tc" if tc else "f32", "coarse": coarse,
            "maxsim": (("fp32 token store: exact in-order fp32 on the CUDA cores" if args.tok_f32
                        else "tcgen05 kind::f16, fp32 query tokens as bf16 hi+lo (nq <= 64)")
                       if tokens else None)}
    out = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "p99_batch_ms": p99,
        "mean_batch_ms": mean_step,
        "slo_ms": args.slo_ms, "slo_met": p99 <= args.slo_ms, "higher_is_better": True,
        "scaling": "strong" if sharded or world == 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": cfg, "path": path,
        "exactness": (("checked: " if parity.get("ok") else "CHECK FAILED: ") + parity["bar"]
                      if parity else "not checked (--no-cpu-baseline)"),
        "parity": parity,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(st["kernel_launches"]),
        # device-side kernel timers over the timed steps (first CTA start -> last CTA end per
        # launch) and the last step's kernel timeline: what the stage spends between kernels
        "kernel_ms_per_step": {
            "scan": st["kt_ms"][0] / args.steps, "sample": st["kt_ms"][1] / args.steps,
            "exact_scan": st["kt_ms"][2] / args.steps, "maxsim": st["kt_ms"][3] / args.steps,
            "rerank": st["kt_rerank_ms"] / args.steps},
        "last_step_timeline_us": {n: [round(st["kt_last_us"][2 * i], 2), round(st["kt_last_us"][2 * i + 1], 2)]
                                  for i, n in enumerate(["scan", "sample", "exact_scan", "maxsim", "rerank"])
                                  if st["kt_last_us"][2 * i + 1] > 0},
        "last_batch_device_ms": ({"stage": st["last_step_ms"], "scan_part": st["last_scan_ms"],
                                  "note": "CUDA events recorded by the stage itself"}
                                 if st["last_step_ms"] >= 0 else None),
        "cert_fallbacks": int(st["cert_fallbacks"]), "cert_level2": int(st["cert_level2"]),
        "root_phases_ms": ({"broadcast": st["phase_ms"][0], "local_stage": st["phase_ms"][1],
                            "gather_merge": st["phase_ms"][2],
                            "rescore_phase2": st["phase_ms"][3],
                            "detail": dict(zip(["local_scan", "local_rerank_tau", "local_rest",
                                                "p2_bcast", "p2_maxsim", "p2_reduce_order"],
                                               st["phase_detail_ms"]))}
                           if sharded else None),
        "clocks": result["clocks"],
    }
    if wl == "audio":
        b = ladder["best"]
        out["value"] = b["achieved_qps"] if b else 0.0  # the whole job: one trace over N members
        out["live_members"] = ladder["members"]
        out["p99_batch_ms"] = b["p99_ms"] if b else None
        out["slo_met"] = b is not None
        out["trace"] = ladder["rungs"]
        # the same rungs read against tighter / the reference's SLOs
        out["max_rate_by_slo_ms"] = {
            str(slo): max([r["achieved_qps"] for r in ladder["rungs"]
                           if r["p99_ms"] <= slo and r["achieved_qps"] >= 0.9 * r["rate_qps"]],
                          default=0.0)
            for slo in (5.0, 10.0, 20.0, 200.0, 500.0)}
        out["e2e"] = {"value": out["value"], "unit": "queries/s",
                      "h2d_bytes_per_step": int(round(b["mean_batch"] * D * 4)) if b else 0,
                      "d2h_bytes_per_step": int(round(b["mean_batch"] * k * 12)) if b else 0,
                      "note": "the trace itself runs through the host-buffer API (vx_serve_trace_replicas)"}
        out["fixed_batch_kernel"] = {"batch": B, "ms_per_step": max_ms / args.steps,
                                     "queries_per_s": value}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    idx.close()


def run_reference(args) -> None:
    """The reference arm: the CPU oracle port of the stage (the reference has no retrieval
    arithmetic of its own — its search stage is a profiled latency, profiles.csv:17-22) on
    this host's cores, all threads.  Each step = S of the batch's queries over the FULL index
    (resident in host memory when it fits, else generated chunk-wise with only the scan timed)
    + MaxSim of their top-k on the token store; exactly `steps` timed steps after `warmup`."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    o = _oracle()
    wl, B, D, k = args.workload, args.batch, args.dim, args.k
    S = min(B, {"flat": B, "maxsim": B, "audio": 32}.get(wl, 16))
    from paper_2511_02062_b200 import synth  # pure-numpy generator (no GPU library call)
    dist = 1 if args.dist == "aniso" else 0
    Qall = synth.queries(B, D, seed=43, dist=dist) if wl != "maxsim" else None
    QT = synth.query_tokens(B, args.nq, args.tok_dim) if wl in ("stage", "maxsim") else None
    rng = np.random.default_rng(7)
    CAND = (np.stack([rng.choice(args.n_docs, k, replace=False) for _ in range(B)]).astype(np.int64)
            if wl == "maxsim" else None)
    need_gb = args.n_docs * D * 4 / 2**30 if wl != "maxsim" else 0.0
    resident = need_gb < 0.6 * mem_available_gb()
    X = o.synth_rows(42, 0, args.n_docs, D, dist) if (resident and wl != "maxsim") else None
    steps_t = []
    for step in range(args.warmup + args.steps):
        sel = (np.arange(S) + step * S) % B  # walk through the batch
        t = 0.0
        if wl != "maxsim":
            if X is not None:
                t0 = time.perf_counter()
                rid, _ = o.flat_topk(X, Qall[sel], k, mode=o.F32)
                t += time.perf_counter() - t0
            else:
                rid, _, ts = o.flat_topk_synth(42, args.n_docs, D, Qall[sel], k, mode=o.F32, dist=dist)
                t += ts
        if wl in ("stage", "maxsim"):
            cand = rid if wl == "stage" else CAND[sel]
            table, local = _compact_blocks(o, cand, args)
            t0 = time.perf_counter()
            o.maxsim(QT[sel], local, table, mode=o.F32)
            t += time.perf_counter() - t0
        if step >= args.warmup:
            steps_t.append(t)
    step_s = sum(steps_t) / len(steps_t)
    value = S / step_s
    out = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if wl in ("stage", "flat", "search") else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(args, args.gpus),
        "sample_fraction": S / B,
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": o.threads(), "kind": "port",
                         "sample": (f"each step: {S} of the {B}-query batch over all {args.n_docs} rows x "
                                    f"{D} fp32 (index {'resident in host memory' if X is not None else 'generated chunk-wise, scan timed'})"
                                    + (f" + MaxSim of their top-{k} ({args.nq}x{args.tok_per_doc}x"
                                       f"{args.tok_dim}, bf16 doc tokens)" if wl in ("stage", "maxsim") else ""))},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("the reference contains no retrieval arithmetic (its search stage is a profiled "
                 "latency, proj/assets/profiles.csv:17-22); this arm times the oracle port of the "
                 "stage (fp32 AVX-512, in-order chains, all host threads) on the same workload"),
    }
    print(json.dumps(out), flush=True)


def config_of(args, world: int) -> dict:
    """The workload description both arms print (identical keys and values for one command)."""
    wl = args.workload
    sharded = wl in ("stage", "flat", "search") and world > 1
    cfg = {"workload": workload_name(args), "baseline_config": WORKLOADS[wl][0],
           "n_docs": args.n_docs, "dim": args.dim, "batch": args.batch, "k": args.k,
           "shards": world if sharded else 1, "replicas": 1 if sharded else world}
    if wl in ("stage", "maxsim"):
        cfg.update({"q_tokens": args.nq, "doc_tokens": args.tok_per_doc, "tok_dim": args.tok_dim,
                    "tok_blocks": args.tok_blocks,
                    "tok_store": "f32" if getattr(args, "tok_f32", False) else "bf16"})
    cfg["l2"] = ("L2 flushed between timed steps (untimed): a 256 MB buffer written, then read back so the L2 holds clean lines; value = sum of per-step event times"
                 if wl in ("flat", "maxsim") else "index (GB) >> 126 MB L2: every step streams from HBM")
    return cfg


def main() -> None:
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
