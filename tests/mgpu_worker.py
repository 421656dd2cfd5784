"""Rank body for tests/test_gpu_multi.py (launched with torch.distributed.run, one process
per GPU).  Rank 0 issues batches; ranks != 0 serve their shard; rank 0 checks the sharded
stage (NCCL broadcast of the batch, per-shard scan + MaxSim, k x G gather, merge) against
the oracle on the whole index.  Exit code 0 = parity."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> int:
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    import paper_2511_02062_b200 as vx
    N, D, B, k, nq, T = int(os.environ.get("VX_N", "300001")), 768, 9, 100, 32, 211
    idx = vx.Index(N, D, device=local, n_shards=world, shard=rank, tok_per_doc=128, tok_dim=128,
                   tok_blocks=T, max_batch=1024, max_k=128, max_qtok=nq)
    graphs = os.environ.get("VX_TEST_GRAPHS") == "1"
    if graphs:  # every rank: captured parts (NCCL collectives inside the graphs)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
    idx.synth(42)
    idx.tokens_synth(45)
    uid = [vx.Index.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    idx.comm_init(uid[0], world, rank)
    ok = True
    if rank == 0:
        import vxoracle as o
        from paper_2511_02062_b200 import synth
        Q = synth.rows(43, 0, B, D)
        qt = synth.query_tokens(B, nq, 128)
        if graphs:  # model load across the shards: every rank captures B = 1..9 (k = 100)
            idx.prepare(k, B, nq=nq)
        ids_s, sc_s = idx.search(Q, 10)
        if graphs:  # a second search of the same shape replays the captured graphs everywhere
            ids_s2, _ = idx.search(Q, 10)
            ok &= np.array_equal(ids_s, ids_s2)
        ids, ip, ms = idx.search_rescore(Q, qt, k)
        # a large batch: two 512-query CTA-pair passes on every shard, k = 100 (the headline
        # batch shape), checked in full including the output order
        QL = synth.rows(43, 1000, 1024, D)
        qtl = synth.query_tokens(1024, nq, 128, seed=46)
        ids_l, ip_l, ms_l = idx.search_rescore(QL, qtl, k)
        ids_l2, ip_l2, ms_l2 = idx.search_rescore(QL, qtl, k)  # deterministic across batches
        ok &= np.array_equal(ids_l, ids_l2) and np.array_equal(ms_l, ms_l2)
        # the s8 coarse pass on rank 0's shard (the headline's format; AUTO picks bf16 for these
        # short shards; options are per handle, so the other shards stay bf16 — a mixed stage
        # must be exact too): the per-shard candidate set k'/G and the tau-pruned tail
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_I8)
        ids_8, ip_8, ms_8 = idx.search_rescore(QL, qtl, k)
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_AUTO)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_F32)
        ids_f, sc_f = idx.search(Q[:3], 10)
        idx.shard_stop()
        from stagecheck import check_stage
        X = o.synth_rows(42, 0, N, D)
        rid, rsc = o.flat_topk(X, Q, 10, mode=1)
        ok &= np.array_equal(ids_s, rid) and np.array_equal(sc_s, rsc.astype(np.float32))
        ok &= np.array_equal(ids_f, rid[:3])
        table = o.synth_tokens(45, 0, T, 128, 128)
        try:
            for q_, t_, out in ((Q, qt, (ids, ip, ms)), (QL, qtl, (ids_l, ip_l, ms_l)),
                                (QL, qtl, (ids_8, ip_8, ms_8))):
                tid, tsc = o.flat_topk(X, q_, k, mode=1)
                tms = o.maxsim(t_, tid, table, mode=o.F64_Q32)
                r = check_stage(*out, tid, tsc, tms)
                print(f"rank0 B={q_.shape[0]}: {r}", flush=True)
        except AssertionError as e:
            print(f"rank0 stage check failed: {e!r}", flush=True)
            ok = False
        print(f"rank0 world={world} parity={'ok' if ok else 'FAIL'} stats={idx.stats()}", flush=True)
    else:
        idx.shard_serve()
        print(f"rank{rank} served {idx.stats()['batches']} batches", flush=True)
    dist.barrier()
    idx.close()
    # the fp32 token store across the shards (its phase 2 broadcasts the fp32 query tokens and
    # every owner runs the exact CUDA-core MaxSim): a small second index
    N2, T2 = 50_000, 61
    idx2 = vx.Index(N2, D, device=local, n_shards=world, shard=rank, tok_per_doc=128, tok_dim=128,
                    tok_blocks=T2, max_batch=16, max_k=16, max_qtok=nq,
                    flags=vx.VX_FLAG_TOKENS_F32)
    idx2.synth(42)
    idx2.tokens_synth(45)
    uid2 = [vx.Index.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid2, src=0)
    idx2.comm_init(uid2[0], world, rank)
    if rank == 0:
        import vxoracle as o
        from paper_2511_02062_b200 import synth
        from stagecheck import check_stage
        Q2 = synth.rows(43, 500, 5, D)
        qt2 = synth.query_tokens(5, nq, 128, seed=47)
        ids2, ip2, ms2 = idx2.search_rescore(Q2, qt2, 10)
        idx2.shard_stop()
        tab32 = o.synth_rows(45, 0, T2 * 128, 128).reshape(T2, 128, 128)
        rid2, rsc2 = o.flat_topk(o.synth_rows(42, 0, N2, D), Q2, 10, mode=1)
        try:
            check_stage(ids2, ip2, ms2, rid2, rsc2, o.maxsim(qt2, rid2, tab32, mode=o.F64))
            want = o.maxsim(qt2, ids2, tab32, mode=o.F32)
            ok &= bool(np.array_equal(ms2.astype(np.float64), want.astype(np.float32).astype(np.float64)))
            print(f"rank0 fp32 token store: ok={ok}", flush=True)
        except AssertionError as e:
            print(f"rank0 fp32 token store check failed: {e!r}", flush=True)
            ok = False
        print(f"rank0 world={world} parity={'ok' if ok else 'FAIL'} (fp32 store)", flush=True)
    else:
        idx2.shard_serve()
    dist.barrier()
    dist.destroy_process_group()
    idx2.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
