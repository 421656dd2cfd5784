"""CUDA-graph mode (VX_OPT_GRAPHS): one captured graph per (op, B, k, nq) replayed for every
batch of that shape; results identical to the eager path, including the device-side exact
re-scan of certificate failures.  Runs on a B200."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


def test_graph_replay_matches_eager(vx, oracle):
    from paper_2511_02062_b200 import synth
    N, D, k, nq = 50_000, 768, 100, 32
    with vx.Index(N, D, tok_per_doc=128, tok_dim=128, tok_blocks=300, max_batch=64, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        want = {}
        for B in (1, 7, 64):
            Q = synth.rows(43, 1000 * B, B, D)
            qt = synth.query_tokens(B, nq, 128, seed=44 + B)
            want[B] = (Q, qt, idx.search_rescore(Q, qt, k))
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        idx.reset_stats()
        for rep in range(3):
            for B in (1, 7, 64):
                Q, qt, (ids, ip, ms) = want[B]
                gids, gip, gms = idx.search_rescore(Q, qt, k)
                assert np.array_equal(gids, ids) and np.array_equal(gip, ip) and np.array_equal(gms, ms)
        st = idx.stats()
    # first batch of each shape runs eagerly and captures; the stage is two graphs (top-k,
    # rescore), so each later batch replays 2
    assert st["graph_replays"] == 12
    assert st["batches"] == 9


def test_graph_mode_device_pointers(vx):
    import torch
    from paper_2511_02062_b200 import synth
    N, D, k, B = 30_000, 768, 10, 16
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        Q = synth.rows(43, 0, B, D)
        ref, _ = idx.search(Q, k)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        q = torch.from_numpy(Q).cuda()
        ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
        sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
        s = torch.cuda.Stream()
        for _ in range(4):
            ids.zero_()
            idx.search_dev(q, ids, sc, k, stream=s.cuda_stream)
            s.synchronize()
            assert np.array_equal(ids.cpu().numpy(), ref)


def test_graph_with_certificate_fallback(vx, oracle):
    N, D, B, k = 3000, 128, 4, 10
    X = oracle.synth_rows(42, 0, N, D)
    X[:600] = X[0]
    Q = np.stack([X[0], X[0], oracle.synth_rows(43, 0, 1, D)[0], X[5]])
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        for _ in range(3):
            ids, sc = idx.search(Q, k)
            rid, _ = oracle.flat_topk(X, Q, k, mode=1)
            assert np.array_equal(ids, rid)
        assert idx.stats()["cert_fallbacks"] >= 6


def test_prepare_precaptures_every_batch_size(vx, oracle):
    """vx_prepare (model load): after it, every batch size replays a graph on its first call
    and the results are the oracle's."""
    from paper_2511_02062_b200 import synth
    N, D, k, nq, bmax = 40_000, 256, 10, 8, 12
    X = oracle.synth_rows(42, 0, N, D)
    with vx.Index(N, D, tok_per_doc=64, tok_dim=64, tok_blocks=100, max_batch=bmax, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        idx.prepare(k, bmax)            # search graphs for B = 1..12
        idx.prepare(k, bmax, nq=nq)     # fused-stage graphs
        assert idx.stats()["batches"] == 0  # preload work is not serving work
        for B in (1, 5, 12):
            Q = synth.rows(43, 100 * B, B, D)
            ids, _ = idx.search(Q, k)
            assert np.array_equal(ids, oracle.flat_topk(X, Q, k, mode=1)[0])
            idx.search_rescore(Q, synth.query_tokens(B, nq, 64, seed=50 + B), k)
        st = idx.stats()
    assert st["graph_replays"] == 3 + 2 * 3 and st["batches"] == 6  # search 1 graph, stage 2


def test_direct_io_graphs_replay_against_caller_buffers(vx):
    """Single GPU, graphs on: from the second call with the same device buffers the whole stage
    is ONE graph captured against those buffers (no copies in or out); other buffers keep
    working and every result equals the eager path's."""
    import torch
    from paper_2511_02062_b200 import synth
    N, D, k, B, nq = 40_000, 768, 10, 8, 32
    with vx.Index(N, D, tok_per_doc=128, tok_dim=128, tok_blocks=300, max_batch=B, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        Q = synth.rows(43, 0, B, D)
        qt = synth.query_tokens(B, nq, 128, seed=44)
        ref_ids, ref_sc = idx.search(Q, k)
        r_ids, r_ip, r_ms = idx.search_rescore(Q, qt, k)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        q = torch.from_numpy(Q).cuda()
        qtd = torch.from_numpy(qt).cuda()
        s = torch.cuda.Stream()
        bufs = [(torch.empty((B, k), dtype=torch.int64, device="cuda"),
                 torch.empty((B, k), dtype=torch.float32, device="cuda"),
                 torch.empty((B, k), dtype=torch.float32, device="cuda")) for _ in range(2)]
        idx.reset_stats()
        for rep in range(4):
            for ids, sc, ms in bufs:
                ids.zero_(), sc.zero_(), ms.zero_()
                idx.search_dev(q, ids, sc, k, stream=s.cuda_stream)
                s.synchronize()
                assert np.array_equal(ids.cpu().numpy(), ref_ids)
                assert np.array_equal(sc.cpu().numpy(), ref_sc)
                ids.zero_(), sc.zero_(), ms.zero_()
                idx.search_rescore_dev(q, qtd, ids, sc, ms, k, stream=s.cuda_stream)
                s.synchronize()
                assert np.array_equal(ids.cpu().numpy(), r_ids)
                assert np.array_equal(sc.cpu().numpy(), r_ip)
                assert np.array_equal(ms.cpu().numpy(), r_ms)
        st = idx.stats()
    # per (op, buffers): call 1 eager + capture of the two-part graphs (or replay), call 2
    # captures the direct graph and replays it, calls 3-4 replay it
    assert st["batches"] == 16
    assert st["graph_replays"] >= 12
