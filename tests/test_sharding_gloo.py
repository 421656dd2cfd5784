"""N > 1 host logic on CPU with gloo, world_size 2 (the GPU exchange uses NCCL).

What is tested is the sharded algorithm the stage runs across GPUs (vx_api.cu stage_core):
contiguous shard ranges [floor(N*g/G), floor(N*(g+1)/G)) (the affinity-group analog of
kvs.hpp:160-175), a per-shard exact top-k, a gather of k x G candidates to rank 0 and a
merge on (score desc, id asc) [phase 1]; then rank 0 broadcasts the global winners, each
shard computes MaxSim only for the winners it owns (-inf elsewhere) and a max-reduce to
rank 0 assembles the scores [phase 2].  Exactness: every global top-k member is in its
owner's local top-k, so rank 0's merge equals the single-index oracle, and every winner
has exactly one owner, so the max-reduce equals the single-index MaxSim.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def shard_range(N: int, G: int, g: int) -> tuple[int, int]:
    r0 = (N * g) // G
    return r0, (N * (g + 1)) // G - r0


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT / "oracle"))
    import vxoracle as o
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, D, B, k = 30_001, 64, 5, 17
    r0, n = shard_range(N, world, rank)
    X = o.synth_rows(42, r0, n, D)
    Q = o.synth_rows(43, 0, B, D)
    ids, sc = o.flat_topk(X, Q, k, mode=1, id_base=r0, threads=2)
    gathered = [None] * world
    dist.all_gather_object(gathered, (ids, sc))
    merged = np.zeros((B, k), np.int64)
    if rank == 0:
        allid = np.concatenate([g[0] for g in gathered], axis=1)
        allsc = np.concatenate([g[1] for g in gathered], axis=1)
        for b in range(B):
            order = np.lexsort((allid[b], -allsc[b]))[:k]
            merged[b] = allid[b][order]
    # phase 2: broadcast the winners, MaxSim on the owner, max-reduce to rank 0
    win = torch.from_numpy(merged)
    dist.broadcast(win, src=0)
    win = win.numpy()
    qtok = o.synth_rows(44, 0, B * 4, 32).reshape(B, 4, 32)
    table = o.synth_tokens(45, 0, 23, 8, 32)
    owned = np.where((win >= r0) & (win < r0 + n), win, -1)
    ms = torch.from_numpy(o.maxsim(qtok, owned, table, mode=1))
    dist.reduce(ms, dst=0, op=dist.ReduceOp.MAX)
    if rank == 0:
        Xf = o.synth_rows(42, 0, N, D)
        want, _ = o.flat_topk(Xf, Q, k, mode=1, threads=2)
        want_ms = o.maxsim(qtok, want, table, mode=1)
        q.put(bool(np.array_equal(merged, want)) and bool(np.array_equal(ms.numpy(), want_ms)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    for N in (1, 7, 10_000_000, 2**31 + 5):
        for G in (1, 2, 3, 4, 8):
            if N < G:
                continue
            spans = [shard_range(N, G, g) for g in range(G)]
            assert spans[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert spans[-1][0] + spans[-1][1] == N
            assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


def test_two_rank_gloo_two_phase_exchange_equals_global(oracle):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


def _tau_worker(rank: int, world: int, port: int, q) -> None:
    """The sharded re-rank (vx_stage.cu kprime_of / local_topk_tc, scan_tc.cu rerank_kernel
    phases 1-2, shard_tau_kernel) restated on CPU, as the GPU runs it: s8 coarse scores with the
    certificate's rigorous bound E; each shard keeps k'/G candidates (not below 2 next_pow2(k));
    phase 1 re-scores its head — the k best coarse candidates, 2k/G of them for G > 2 — EXACTLY
    and the shards all-gather those exact scores; tau = their k-th largest (k distinct
    documents score >= tau, so tau <= the global exact k-th); phase 2 re-ranks only the tail
    candidates with cscale c >= max(L, tau) - E (L = the head's minimum exact score when the
    head holds k rows) and certifies with `bound(T') < tau or exact k-th > bound(T')`; rank 0's
    merge must equal the single-index oracle."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(ROOT / "oracle"))
    import vxoracle as o
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, D, B, k = 40_000, 128, 6, 10

    def np2(x):
        p = 1
        while p < x:
            p <<= 1
        return p
    kp1 = min(1024, max(128, 8 * np2(k)))                    # the single-index s8 k'
    kp = max(min(kp1, 2 * np2(k)), kp1 // np2(world))        # the shard's k'/G
    kh = k if world <= 2 else min(k, max(16, (2 * k + world - 1) // world))
    kh = min(kh, kp)
    r0, n = shard_range(N, world, rank)
    X = o.synth_rows(42, r0, n, D).astype(np.float64)
    Q = o.synth_rows(43, 0, B, D).astype(np.float64)
    sx = np.abs(X).max() / 127.0
    X8 = np.clip(np.rint(X / sx), -127, 127)
    rx, xh = np.linalg.norm(X - X8 * sx, axis=1).max(), np.linalg.norm(X8 * sx, axis=1).max()
    sq = np.abs(Q).max(axis=1) / 127.0
    Q8 = np.clip(np.rint(Q / sq[:, None]), -127, 127)
    rq = np.linalg.norm(Q - Q8 * sq[:, None], axis=1)
    qh = np.linalg.norm(Q8 * sq[:, None], axis=1)
    E = (qh * rx + rq * xh + rq * rx) * 1.001 + 1e-9
    coarse = (Q8 @ X8.T) * (sq[:, None] * sx)          # cscale * s32 dot
    cand = np.argsort(-coarse, axis=1, kind="stable")[:, :kp]
    ccand = np.take_along_axis(coarse, cand, axis=1)
    Xe = o.synth_rows(42, r0, n, D)
    Qe = o.synth_rows(43, 0, B, D)

    def exact(b, rows):  # the in-order fp32 chains (VXO_F32), one row at a time
        return np.array([o.flat_topk(Xe[j:j + 1], Qe[b:b + 1], 1, mode=1)[1][0, 0] for j in rows],
                        np.float32)
    # phase 1: exact scores of the head, all-gathered
    head_ex = [exact(b, cand[b, :kh]) for b in range(B)]
    lb_np = np.full((B, k), -np.inf, np.float32)
    for b in range(B):
        lb_np[b, :kh] = head_ex[b]
    allb = [torch.zeros((B, k), dtype=torch.float32) for _ in range(world)]
    dist.all_gather(allb, torch.from_numpy(lb_np))
    tau = np.sort(np.concatenate([t.numpy() for t in allb], axis=1), axis=1)[:, ::-1][:, k - 1]
    ids = np.full((B, k), -1, np.int64)
    sc = np.full((B, k), -np.inf, np.float32)
    ok = True
    fetched = 0
    for b in range(B):
        L = float(head_ex[b].min()) if kh >= k else -np.inf
        lim = max(L, float(tau[b])) - E[b]
        tail = np.arange(kh, kp)
        tail = tail[ccand[b, tail] >= lim]                    # the pruned prefix (descending)
        keep = np.concatenate([cand[b, :kh], cand[b, tail]])
        ex = np.concatenate([head_ex[b], exact(b, cand[b, tail])])
        fetched += keep.size
        order = np.lexsort((keep, -ex))[:k]
        ids[b, :order.size] = keep[order] + r0
        sc[b, :order.size] = ex[order]
        bound = ccand[b, -1] + E[b]
        ok &= bool(bound < tau[b] or (order.size == k and ex[order[-1]] > bound))
    gathered = [None] * world
    dist.all_gather_object(gathered, (ids, sc, ok, fetched))
    if rank == 0:
        allid = np.concatenate([g[0] for g in gathered], axis=1)
        allsc = np.concatenate([g[1] for g in gathered], axis=1)
        merged = np.zeros((B, k), np.int64)
        for b in range(B):
            order = np.lexsort((allid[b], -allsc[b]))[:k]
            merged[b] = allid[b][order]
        want, _ = o.flat_topk(o.synth_rows(42, 0, N, D), o.synth_rows(43, 0, B, D), k, mode=1,
                              threads=2)
        certified = all(g[2] for g in gathered)
        q.put((certified, bool(np.array_equal(merged, want)), sum(g[3] for g in gathered)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_sharded_threshold_prunes_and_stays_exact(oracle, world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000 + 7 * world
    procs = [ctx.Process(target=_tau_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    certified, exact, fetched = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert certified and exact
    kp = max(min(128, 32), 128 // world)
    assert fetched < world * 6 * kp  # the threshold pruned candidates on the shards
