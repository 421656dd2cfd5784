"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.  Runs on a B200.

Bar (BASELINE.json north_star):
  * exact scan: ids AND scores bit-identical to the oracle's VXO_F32 mode (same in-order
    fmaf chain per dot product, same (score desc, id asc) order); vs the fp64 truth, any id
    difference must be a tie within TIE_TOL and scores within 1e-4 relative;
  * MaxSim (bf16 doc tokens, fp32 accumulate): CUDA-core kernel (bf16-rounded query tokens)
    bit-identical to VXO_F32; the default tensor-core kernel (fp32 query tokens as bf16 hi +
    lo) within MS_RTOL of the fp64 MaxSim of the fp32 tokens (VXO_F64_Q32; tests/stagecheck.py).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TIE_TOL = 1e-6     # |s64(a) - s64(b)| under which two docs count as tied (fp32 noise ~1e-8)
SCORE_RTOL = 1e-4  # north-star bound for fp32-accumulated scores
MS_RTOL = 1e-5     # bf16-input MaxSim, fp32 accumulation vs fp64 of the same inputs


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


def ties_ok(ids_gpu, ids_ref, s64_lookup, kth_score):
    """ids may differ only where the differing docs are tied (fp64) with the k-th score."""
    a, b = set(ids_gpu.tolist()), set(ids_ref.tolist())
    for d in a ^ b:
        if abs(s64_lookup(d) - kth_score) > TIE_TOL:
            return False
    return True


def test_device_synth_bit_exact(vx, oracle):
    with vx.Index(5000, 768, tok_per_doc=16, tok_dim=64, tok_blocks=9) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        got = idx.download(0, 5000)
        want = oracle.synth_rows(42, 0, 5000, 768)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        assert np.array_equal(idx.tokens_download(0, 9), oracle.synth_tokens(45, 0, 9, 16, 64))


@pytest.mark.parametrize("N,D,B,k", [
    (1000, 64, 1, 1), (1000, 64, 5, 7), (4097, 128, 3, 10), (3000, 768, 4, 10),
    (100_000, 768, 16, 10), (20_000, 1024, 8, 100), (12_345, 768, 32, 100),
    (50_000, 256, 17, 128), (30_000, 768, 33, 256), (9_999, 768, 2, 64), (7, 32, 6, 5)])
def test_scan_bit_identical_to_oracle_f32(vx, oracle, N, D, B, k):
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=max(B, 1), max_k=max(k, 1)) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_F32)
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    valid = rid >= 0
    assert np.array_equal(sc[valid], rsc[valid].astype(np.float32))
    assert np.isneginf(sc[~valid]).all()
    # against the fp64 truth: ties within tolerance, scores within 1e-4 relative
    tid, tsc = oracle.flat_topk(X, Q, k, mode=0)
    for b in range(B):
        s64 = lambda d, b=b: float(np.dot(X[d].astype(np.float64), Q[b].astype(np.float64)))
        kth = tsc[b][min(k, N) - 1]
        assert ties_ok(ids[b][ids[b] >= 0], tid[b][tid[b] >= 0], s64, kth)
    v = tid >= 0
    np.testing.assert_allclose(sc[v], tsc[v], rtol=SCORE_RTOL, atol=1e-7)


def test_known_answer_ties(vx, golden):
    g = golden("kat_ties")
    X = np.zeros((6, 32), np.float32)
    X[:, :2] = g["X"]
    Q = np.zeros((2, 32), np.float32)
    Q[:, :2] = g["Q"]
    with vx.Index(6, 32, max_batch=2, max_k=4) as idx:
        idx.upload(X)
        ids, sc = idx.search(Q, 4)
    assert ids.tolist() == g["ids"].tolist()
    assert np.array_equal(sc, g["scores"].astype(np.float32))


def test_golden_fixture_ids(vx, oracle, golden):
    for name in ("ip_small", "ip_768", "ip_k100"):
        g = golden(name)
        N, D, B, k = (int(g[x]) for x in ("N", "D", "B", "k"))
        with vx.Index(N, D, max_batch=B, max_k=k) as idx:
            idx.synth(42)
            ids, sc = idx.search(oracle.synth_rows(43, 0, B, D), k)
        assert np.array_equal(ids, g["ids"]), name
        np.testing.assert_allclose(sc, g["scores"], rtol=SCORE_RTOL)


def test_edge_cases(vx, oracle):
    # k > N pads with -1/-INF; duplicate rows tie and resolve by id; zero query -> all ties
    X = oracle.synth_rows(42, 0, 40, 64)
    X[10] = X[3]
    X[20] = X[3]
    with vx.Index(40, 64, max_batch=4, max_k=64) as idx:
        idx.upload(X)
        ids, sc = idx.search(np.stack([X[3], np.zeros(64, np.float32)]), 50)
    assert ids[0, :3].tolist() == [3, 10, 20]
    assert (ids[:, 40:] == -1).all() and np.isneginf(sc[:, 40:]).all()
    assert ids[1, :40].tolist() == list(range(40))


def test_scan_rejects_bad_shapes(vx):
    with vx.Index(100, 64, max_batch=4, max_k=8) as idx:
        idx.synth(1)
        with pytest.raises(vx.VxError):
            idx.search(np.zeros((5, 64), np.float32), 4)
        with pytest.raises(vx.VxError):
            idx.search(np.zeros((1, 64), np.float32), 9)


def test_errors_are_reported_and_the_handle_stays_usable(vx, oracle):
    # every rejected call returns a status + message (no exception crosses the ABI, no
    # partial state): the next valid call on the same handle is exact
    N, D, k = 2000, 64, 8
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, 3, D)
    with vx.Index(N, D, tok_per_doc=16, tok_dim=64, tok_blocks=4, max_batch=4, max_k=k,
                  max_qtok=4) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        bad = [
            lambda: idx.set_option(vx.VX_OPT_KPRIME, 3),           # not a power of two
            lambda: idx.set_option(vx.VX_OPT_KPRIME, 2048),        # > 1024
            lambda: idx.set_option(vx.VX_OPT_SCAN_PAIRS, 5),
            lambda: idx.set_option(vx.VX_OPT_SCAN_TILE, 64),
            lambda: idx.set_option(999, 1),                        # unknown option
            lambda: idx.prepare(k, 5),                             # b_max > max_batch
            lambda: idx.search(Q, k + 1),                          # k > max_k
            lambda: idx.search_rescore(Q, np.zeros((3, 5, 64), np.float32), k),  # nq > max_qtok
            lambda: idx.upload(X[:10], row0=N - 5),                # outside the shard
            lambda: idx.maxsim(np.zeros((3, 4, 64), np.float32), np.zeros((3, k + 1), np.int64)),
        ]
        for f in bad:
            with pytest.raises(vx.VxError) as e:
                f()
            assert str(e.value).split(":", 1)[1].strip()  # a message, not just a code
        ids, sc = idx.search(Q, k)
    rid, _ = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)


def test_maxsim_matches_oracle(vx, oracle, golden):
    g = golden("maxsim_small")
    T, Nd, d = g["table"].shape
    with vx.Index(100, 32, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=4, max_k=8,
                  max_qtok=8) as idx:
        idx.tokens_upload(g["table"])
        out = idx.maxsim(g["qtok"], g["cand"])
    fin = np.isfinite(g["ms"])
    np.testing.assert_allclose(out[fin], g["ms"][fin], rtol=MS_RTOL)
    assert np.isneginf(out[~fin]).all()
    ref32 = oracle.maxsim(g["qtok"], g["cand"], g["table"], mode=1)
    assert np.array_equal(out[fin], ref32[fin].astype(np.float32))


@pytest.mark.parametrize("B,C", [(1, 100), (8, 100), (64, 100)])
def test_maxsim_preflmr_shape(vx, oracle, B, C):
    # PreFLMR config: 32 query tokens x 100 candidates x 128 doc tokens, dim 128
    T, Nd, d, nq = 257, 128, 128, 32
    rng = np.random.default_rng(B)
    cand = np.stack([rng.choice(10_000_000, C, replace=False) for _ in range(B)]).astype(np.int64)
    qtok = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    with vx.Index(1000, 32, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=B, max_k=C,
                  max_qtok=nq) as idx:
        idx.tokens_synth(45)
        out = idx.maxsim(qtok, cand)
    table = oracle.synth_tokens(45, 0, T, Nd, d)
    ref = oracle.maxsim(qtok, cand, table, mode=oracle.F64_Q32)
    np.testing.assert_allclose(out, ref, rtol=MS_RTOL, atol=1e-6)


def test_search_rescore_matches_oracle(vx, oracle):
    N, D, B, k, T, Nd, d, nq = 20_000, 768, 5, 100, 97, 128, 128, 32
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    qtok = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    table = oracle.synth_tokens(45, 0, T, Nd, d)
    with vx.Index(N, D, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=B, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        ids, ip, ms = idx.search_rescore(Q, qtok, k)
    from stagecheck import check_stage
    rid, rsc = oracle.flat_topk(X, Q, k, mode=oracle.F32)
    rms = oracle.maxsim(qtok, rid, table, mode=oracle.F64_Q32)
    check_stage(ids, ip, ms, rid, rsc, rms)  # ids, exact IP scores, MaxSim tolerance, order


def test_row_gather_api_equals_contiguous(vx, oracle):
    # vx_search_rows / vx_search_rescore_rows (payload row pointers, one host copy) give the
    # same results as the contiguous host API
    from paper_2511_02062_b200 import synth
    N, D, k, nq, B = 30_000, 256, 10, 8, 7
    with vx.Index(N, D, tok_per_doc=64, tok_dim=64, tok_blocks=40, max_batch=B, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        Q = synth.rows(43, 3, B, D)
        qt = synth.query_tokens(B, nq, 64)
        rows = [Q[i].copy() for i in range(B)]          # separate allocations
        trows = [qt[i].copy() for i in range(B)]
        assert all(np.array_equal(a, b) for a, b in zip(idx.search_rows(rows, k), idx.search(Q, k)))
        got = idx.search_rescore_rows(rows, trows, k)
        want = idx.search_rescore(Q, qt, k)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))


def test_pinned_host_buffers_equal_pageable(vx, oracle):
    # page-locked caller buffers are DMA'd directly (no staging memcpy, vx_api.cu upload_src /
    # download), pageable ones through the staging: same results either way, outputs included
    import torch
    from paper_2511_02062_b200 import synth
    N, D, k, nq, B = 30_000, 256, 10, 8, 7
    with vx.Index(N, D, tok_per_doc=64, tok_dim=64, tok_blocks=40, max_batch=B, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        Q = synth.rows(43, 3, B, D)
        qt = synth.query_tokens(B, nq, 64)
        Qp_t, qtp_t = torch.from_numpy(Q).pin_memory(), torch.from_numpy(qt).pin_memory()
        Qp, qtp = Qp_t.numpy(), qtp_t.numpy()
        assert all(np.array_equal(a, b) for a, b in zip(idx.search(Qp, k), idx.search(Q, k)))
        want = idx.search_rescore(Q, qt, k)
        got = idx.search_rescore(Qp, qtp, k)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))
        # pinned outputs through the C-ABI directly
        lib = idx.lib
        from paper_2511_02062_b200._lib import FP, LP
        ids_t = torch.empty((B, k), dtype=torch.int64).pin_memory()
        ip_t = torch.empty((B, k), dtype=torch.float32).pin_memory()
        ms_t = torch.empty((B, k), dtype=torch.float32).pin_memory()
        ids, ip, ms = ids_t.numpy(), ip_t.numpy(), ms_t.numpy()
        assert lib.vx_search_rescore(idx._h, Qp.ctypes.data_as(FP), qtp.ctypes.data_as(FP), B, nq, k,
                                     ids.ctypes.data_as(LP), ip.ctypes.data_as(FP),
                                     ms.ctypes.data_as(FP)) == 0
        assert np.array_equal(ids, want[0]) and np.array_equal(ip, want[1]) and np.array_equal(ms, want[2])


def test_component_payload_path(vx, oracle):
    N, D, k, T, Nd, d, nq = 5000, 768, 10, 31, 128, 128, 32
    Q = oracle.synth_rows(43, 0, 3, D)
    qtok = oracle.synth_rows(44, 0, 3 * nq, d).reshape(3, nq, d)
    with vx.Index(N, D, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=4, max_k=k,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        reg = vx.Registry()
        reg.register_component("modelD", vx.SearchComponent(idx, k))
        outs = reg.invoke("modelD", [vx.encode_query(Q[i], qtok[i]) for i in range(3)])
        ids, ip, ms = idx.search_rescore(Q, qtok, k)
    assert len(outs) == 3
    for i, p in enumerate(outs):
        r = vx.decode_result(p)
        assert r["id"].tolist() == ids[i].tolist()
        assert np.array_equal(r["ms"], ms[i])


def test_stats_count_launches(vx):
    with vx.Index(10_000, 128, max_batch=4, max_k=10) as idx:
        idx.synth(1)
        idx.reset_stats()
        idx.search(np.ones((4, 128), np.float32), 10)
        st = idx.stats()
    assert st["kernel_launches"] >= 2 and st["batches"] == 1 and st["queries"] == 4


# ------------------------------------------------------------------ tensor-core scan (K2)
@pytest.mark.parametrize("N,D,B,k", [
    (100_000, 768, 16, 10), (50_000, 768, 1, 1), (20_000, 1024, 8, 100), (12_345, 768, 32, 100),
    (30_000, 768, 128, 128), (40_000, 256, 129, 10), (25_000, 768, 256, 100), (9_000, 128, 300, 64),
    (4097, 64, 5, 7), (1000, 32, 3, 5)])
def test_tc_scan_bit_identical_to_oracle_f32(vx, oracle, N, D, B, k):
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        ids, sc = idx.search(Q, k)
        fallbacks = idx.stats()["cert_fallbacks"]
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    v = rid >= 0
    assert np.array_equal(sc[v], rsc[v].astype(np.float32))
    if N >= 10_000:
        assert fallbacks == 0


@pytest.mark.parametrize("pairs", [1, 2])
@pytest.mark.parametrize("coarse", ["bf16", "tf32", "i8"])
@pytest.mark.parametrize("N,D,B,k", [(60_000, 768, 512, 100), (30_001, 256, 257, 10),
                                     (20_000, 768, 700, 50), (10_000, 128, 1100, 16)])
def test_tc_pairs_large_batch_bit_identical(vx, oracle, N, D, B, k, coarse, pairs):
    # B > 256: several passes of the CTA-pair kernel (pairs=1: 256 queries per pass; pairs=2:
    # 512 per pass, two accumulator groups); results are still the exact oracle's
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, {"bf16": vx.VX_COARSE_BF16, "tf32": vx.VX_COARSE_TF32,
                                          "i8": vx.VX_COARSE_I8}[coarse])
        assert idx.coarse_auto() == coarse
        idx.set_option(vx.VX_OPT_SCAN_PAIRS, pairs)
        ids, sc = idx.search(Q, k)
        fallbacks = idx.stats()["cert_fallbacks"]
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    v = rid >= 0
    assert np.array_equal(sc[v], rsc[v].astype(np.float32))
    assert fallbacks <= B // 50


@pytest.mark.parametrize("pairs", [0, 1])
def test_tc_certificate_level2_wide_rerank(vx, oracle, pairs):
    # k' = k = 16 candidates: the first certificate (exact k-th > coarse k'-th + E) fails for
    # most queries; the wide re-rank over the full per-CTA lists (no index access) must
    # rescue them, exactly
    N, D, B, k = 100_000, 256, 200, 16
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_SCAN_PAIRS, pairs)
        idx.set_option(vx.VX_OPT_KPRIME, 16)
        ids, sc = idx.search(Q, k)
        st = idx.stats()
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    assert np.array_equal(sc, rsc.astype(np.float32))
    assert st["cert_level2"] >= B // 4
    assert st["cert_fallbacks"] <= st["cert_level2"] // 10


@pytest.mark.parametrize("B,k", [(40, 100), (70, 20)])
def test_tc_certificate_fallback_many_queries(vx, oracle, B, k):
    # most queries fail the certificate: the exact re-scan runs as ONE device-count launch
    # looping over several query groups on the device
    N, D = 3000, 128
    X = oracle.synth_rows(42, 0, N, D)
    X[:600] = X[0]
    Q = np.stack([X[0] if i % 7 else oracle.synth_rows(43, i, 1, D)[0] for i in range(B)])
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        for graphs in (0, 1, 1):
            idx.set_option(vx.VX_OPT_GRAPHS, graphs)
            ids, sc = idx.search(Q, k)
            rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
            assert np.array_equal(ids, rid)
            v = rid >= 0
            assert np.array_equal(sc[v], rsc[v].astype(np.float32))
        st = idx.stats()
    assert st["cert_fallbacks"] >= B // 2


@pytest.mark.parametrize("N,D,B,k", [
    (100_000, 768, 16, 10), (50_000, 768, 1, 1), (20_000, 1024, 8, 100), (12_345, 768, 32, 100),
    (30_000, 768, 128, 128), (40_000, 256, 129, 10), (25_000, 768, 256, 100), (4097, 128, 5, 7)])
def test_i8_coarse_bit_identical_to_oracle_f32(vx, oracle, N, D, B, k):
    # the s8 coarse pass (kind::i8, one scale per shard, per-query scales) only selects;
    # the certified exact re-rank makes ids and scores the oracle's
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_I8)
        ids, sc = idx.search(Q, k)
        st = idx.stats()
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    v = rid >= 0
    assert np.array_equal(sc[v], rsc[v].astype(np.float32))
    assert st["cert_fallbacks"] <= max(1, B // 20)


def test_i8_shadow_follows_uploads(vx, oracle):
    # the s8 scale is shard-wide: an upload that raises max|x| must requantise the shadow
    N, D, B, k = 3000, 128, 6, 10
    X = oracle.synth_rows(42, 0, N, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X)
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_I8)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        X[17] *= 3.0
        idx.upload(X[10:20], row0=10)
        Q = np.stack([X[17] / np.linalg.norm(X[17])] + [X[i] for i in (1, 2, 3, 4, 5)])
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid) and ids[0, 0] == 17


def test_tc_certificate_forces_exact_fallback(vx, oracle):
    # 600 identical rows + noise rows: coarse scores tie massively, the certificate cannot
    # separate the k-th from the candidate boundary -> exact re-scan, still exact results
    N, D, B, k = 3000, 128, 4, 10
    X = oracle.synth_rows(42, 0, N, D)
    X[:600] = X[0]
    Q = np.stack([X[0], X[0], oracle.synth_rows(43, 0, 1, D)[0], X[5]])
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        ids, sc = idx.search(Q, k)
        st = idx.stats()
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    assert st["cert_fallbacks"] >= 2
