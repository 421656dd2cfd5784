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
                   tok_blocks=T, max_batch=300, max_k=128, max_qtok=nq)
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
        ids_s, sc_s = idx.search(Q, 10)
        ids, ip, ms = idx.search_rescore(Q, qt, k)
        # a large batch: CTA-pair passes (256 + 44 queries) on every shard, k = 100
        QL = synth.rows(43, 1000, 300, D)
        qtl = synth.query_tokens(300, nq, 128, seed=46)
        ids_l, ip_l, ms_l = idx.search_rescore(QL, qtl, k)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_F32)
        ids_f, sc_f = idx.search(Q[:3], 10)
        idx.shard_stop()
        X = o.synth_rows(42, 0, N, D)
        rid, rsc = o.flat_topk(X, Q, 10, mode=1)
        ok &= np.array_equal(ids_s, rid) and np.array_equal(sc_s, rsc.astype(np.float32))
        ok &= np.array_equal(ids_f, rid[:3])
        table = o.synth_tokens(45, 0, T, 128, 128)
        tid, tip, tms = o.search_rescore(X, Q, qt, table, k, mode=1)
        for b in range(B):
            ok &= sorted(ids[b].tolist()) == sorted(tid[b].tolist())
            lut = dict(zip(tid[b].tolist(), tms[b].tolist()))
            ok &= all(abs(lut[i] - m) <= 1e-5 * abs(lut[i]) for i, m in zip(ids[b].tolist(), ms[b].tolist()))
        lid, lip, lms = o.search_rescore(X, QL, qtl, table, k, mode=1)
        for b in range(300):
            ok &= sorted(ids_l[b].tolist()) == sorted(lid[b].tolist())
            lut = dict(zip(lid[b].tolist(), lip[b].tolist()))
            ok &= all(np.float32(lut[i]) == p for i, p in zip(ids_l[b].tolist(), ip_l[b].tolist()))
        print(f"rank0 world={world} parity={'ok' if ok else 'FAIL'} stats={idx.stats()}", flush=True)
    else:
        idx.shard_serve()
        print(f"rank{rank} served {idx.stats()['batches']} batches", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    idx.close()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
