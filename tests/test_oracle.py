"""The CPU oracle pinned against the golden fixtures (tests/golden/make_golden.py) and the
reference's own known answers (nearest-rank percentile, proj/tests/test_bench.cpp:60-91).
CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest


def test_generator_bit_exact(oracle, golden):
    g = golden("synth")
    for key, rows in g.items():
        _, s, d = key.split("_")
        seed, dim = int(s[1:]), int(d[1:])
        row0 = {"rows_s42_d768": 0, "rows_s43_d768": 0, "rows_s42_d1024": 9_999_996,
                "rows_s45_d128": 123456}[key]
        out = oracle.synth_rows(seed, row0, rows.shape[0], dim)
        assert out.view(np.uint32).tolist() == rows.view(np.uint32).tolist(), key
        norms = np.linalg.norm(out.astype(np.float64), axis=1)
        assert np.allclose(norms, 1.0, atol=1e-6)


def test_tokens_are_bf16_of_rows(oracle):
    tok = oracle.synth_tokens(45, 3, 2, 8, 64)
    rows = oracle.synth_rows(45, 3 * 8, 16, 64).reshape(2, 8, 64)
    u = rows.view(np.uint32).astype(np.uint64)
    rne = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(tok, rne)


@pytest.mark.parametrize("name", ["ip_small", "ip_768", "ip_k100"])
@pytest.mark.parametrize("mode", [0, 1])
def test_flat_topk_matches_golden(oracle, golden, name, mode):
    g = golden(name)
    N, D, B, k = (int(g[x]) for x in ("N", "D", "B", "k"))
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    ids, sc = oracle.flat_topk(X, Q, k, mode=mode)
    assert np.array_equal(ids, g["ids"])
    tol = 1e-12 if mode == 0 else 1e-6
    np.testing.assert_allclose(sc, g["scores"], rtol=0, atol=tol)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("threads", [1, 3, 0])
def test_known_answer_ties(oracle, golden, mode, threads):
    g = golden("kat_ties")
    ids, sc = oracle.flat_topk(g["X"], g["Q"], int(g["k"]), mode=mode, threads=threads)
    assert ids.tolist() == g["ids"].tolist()
    assert np.array_equal(sc, g["scores"])


def test_k_larger_than_n_pads(oracle):
    X = oracle.synth_rows(1, 0, 3, 32)
    Q = oracle.synth_rows(2, 0, 2, 32)
    ids, sc = oracle.flat_topk(X, Q, 5)
    assert (ids[:, 3:] == -1).all() and np.isneginf(sc[:, 3:]).all()
    assert sorted(ids[0, :3].tolist()) == [0, 1, 2]


def test_f32_mode_is_inorder_fma(oracle):
    X = oracle.synth_rows(42, 0, 50, 96)
    Q = oracle.synth_rows(43, 0, 3, 96)
    ids, sc = oracle.flat_topk(X, Q, 50, mode=1)
    for b in range(3):
        for j in range(50):
            acc = np.float32(0)
            x, q = X[ids[b, j]], Q[b]
            for t in range(96):  # fmaf == round(x*q + acc) with exact product: use f64
                acc = np.float32(np.float64(x[t]) * np.float64(q[t]) + np.float64(acc))
            assert np.float32(sc[b, j]) == acc


def test_maxsim_matches_golden(oracle, golden):
    g = golden("maxsim_small")
    out = oracle.maxsim(g["qtok"], g["cand"], g["table"], mode=0)
    np.testing.assert_allclose(out[np.isfinite(g["ms"])], g["ms"][np.isfinite(g["ms"])], rtol=1e-12)
    assert np.isneginf(out[1, 2])
    out32 = oracle.maxsim(g["qtok"], g["cand"], g["table"], mode=1)
    fin = np.isfinite(g["ms"])
    np.testing.assert_allclose(out32[fin], g["ms"][fin], rtol=1e-5)


def test_search_rescore_orders_by_maxsim(oracle):
    N, D, B, k, T, Nd, d, nq = 500, 64, 3, 20, 11, 8, 32, 4
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    table = oracle.synth_tokens(45, 0, T, Nd, d)
    qtok = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    ids, ip, ms = oracle.search_rescore(X, Q, qtok, table, k)
    tids, tsc = oracle.flat_topk(X, Q, k)
    for b in range(B):
        assert sorted(ids[b].tolist()) == sorted(tids[b].tolist())
        order = sorted(range(k), key=lambda i: (-ms[b, i], ids[b, i]))
        assert order == list(range(k))
        lut = dict(zip(tids[b].tolist(), tsc[b].tolist()))
        assert [lut[i] for i in ids[b].tolist()] == ip[b].tolist()


def test_percentile_reference_cases(oracle):
    # proj/tests/test_bench.cpp:60-69
    assert oracle.percentile([10], 5) == 10.0
    assert oracle.percentile([10], 95) == 10.0
    v = list(range(1, 101))
    assert oracle.percentile(v, 50) == 50.0
    assert oracle.percentile(v, 95) == 95.0
    assert oracle.percentile(v, 5) == 5.0
    assert oracle.percentile([3, 1, 2], 50) == 2.0
    assert math.isnan(oracle.percentile([], 50))
    rng = np.random.default_rng(9)
    for _ in range(50):
        s = rng.integers(0, 1000, size=int(rng.integers(1, 41))).astype(float)
        p = float(rng.integers(1, 100))
        r = oracle.percentile(s, p)
        rank = math.ceil(p / 100 * len(s))
        assert r in s and (s <= r).sum() >= rank and (s < r).sum() < rank


# ---- full-size helpers (chunked generation) and the fp32-query MaxSim truth

def test_flat_topk_synth_equals_whole_matrix(oracle):
    Q = oracle.synth_rows(43, 0, 5, 256)
    for mode in (oracle.F32, oracle.F64):
        ids, sc, t = oracle.flat_topk_synth(42, 30_001, 256, Q, 17, mode=mode, chunk=4096)
        wid, wsc = oracle.flat_topk(oracle.synth_rows(42, 0, 30_001, 256), Q, 17, mode=mode)
        assert np.array_equal(ids, wid) and np.array_equal(sc, wsc) and t > 0
    # an offset range (a shard's rows) reports global ids
    ids, _, _ = oracle.flat_topk_synth(42, 1000, 256, Q, 5, row0=7000, chunk=300)
    wid, _ = oracle.flat_topk(oracle.synth_rows(42, 7000, 1000, 256), Q, 5, mode=oracle.F32,
                              id_base=7000)
    assert np.array_equal(ids, wid)


def test_merge_topk_orders_and_pads(oracle):
    a_i = np.array([[5, 3, -1]]); a_s = np.array([[2.0, 1.0, -np.inf]])
    b_i = np.array([[4, 9, -1]]); b_s = np.array([[2.0, 0.5, -np.inf]])
    i, s = oracle.merge_topk(a_i, a_s, b_i, b_s, 5)
    assert i.tolist() == [[4, 5, 3, 9, -1]] and s[0, :4].tolist() == [2.0, 2.0, 1.0, 0.5]


def test_maxsim_synth_and_fp32_query_truth(oracle):
    T, Nd, d, B, nq, C = 37, 16, 64, 3, 5, 9
    table = oracle.synth_tokens(45, 0, T, Nd, d)
    assert np.array_equal(oracle.synth_token_blocks(45, [4, 0, 4, 36], Nd, d), table[[4, 0, 4, 36]])
    qt = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    cand = np.random.default_rng(1).integers(0, 10_000, (B, C)).astype(np.int64)
    cand[0, 3] = -1
    for mode in (oracle.F64, oracle.F32, oracle.F64_Q32):
        assert np.array_equal(oracle.maxsim(qt, cand, table, mode=mode),
                              oracle.maxsim_synth(qt, cand, 45, T, Nd, d, mode=mode))
    # VXO_F64_Q32 = numpy fp64 of the UNROUNDED query tokens
    want = np.empty((B, C))
    for b in range(B):
        for c in range(C):
            if cand[b, c] < 0:
                want[b, c] = -np.inf
                continue
            D = oracle.bf16_to_f32(table[cand[b, c] % T]).astype(np.float64)
            want[b, c] = (qt[b].astype(np.float64) @ D.T).max(axis=1).sum()
    got = oracle.maxsim(qt, cand, table, mode=oracle.F64_Q32)
    fin = np.isfinite(want)
    np.testing.assert_allclose(got[fin], want[fin], rtol=1e-12)
    assert np.isneginf(got[~fin]).all()
    # and it differs from the bf16-rounded-query truth by the rounding (~1e-3 relative)
    t16 = oracle.maxsim(qt, cand, table, mode=oracle.F64)
    assert np.abs(t16[fin] - got[fin]).max() > 1e-5


def test_stagecheck_accepts_near_ties_and_rejects_real_swaps():
    from stagecheck import check_stage_query
    rid = np.array([1, 2, 3]); rip = np.array([0.9, 0.8, 0.7])
    truth = np.array([5.0, 5.0 + 1e-7, 4.0])
    # GPU order 1 before 2 with its own MaxSim equal -> id asc; the truth swap is a near-tie
    r = check_stage_query(np.array([1, 2, 3]), np.float32(rip), np.array([5.0, 5.0, 4.0]), rid, rip, truth)
    assert r["order_swaps"] == 1
    with pytest.raises(AssertionError):  # a swap far outside the tolerance
        check_stage_query(np.array([3, 1, 2]), np.float32(rip[[2, 0, 1]]), np.array([5.0, 4.9, 4.8]),
                          rid, rip, np.array([5.0, 4.9, 5.0]))
    with pytest.raises(AssertionError):  # an IP score off by one ulp
        check_stage_query(np.array([1, 2, 3]), np.nextafter(np.float32(rip), 2), truth, rid, rip, truth)


def test_anisotropic_generator_matches_numpy_restatement(oracle):
    """vx_synth.h dist 1 (anisotropic): the C oracle, the numpy host generator and (on the GPU,
    tests/test_gpu_coarse.py) the device fill agree bit for bit."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2511_02062_b200 import synth
    for dist in (0, 1):
        a = oracle.synth_rows(42, 123_456, 40, 768, dist)
        b = synth.rows(42, 123_456, 40, 768, dist)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        assert np.allclose(np.linalg.norm(a.astype(np.float64), axis=1), 1.0, atol=1e-6)
    m = synth.mult(1, 768)
    assert m[0] == 33 and m[13] == 4 * 1 + 4 * 32 // 4 and m.min() == 1
    # the anisotropy the bench's --dist aniso runs on: leading dims ~20x the tail's spread
    a = oracle.synth_rows(42, 0, 2000, 768, 1)
    assert a[:, :4].std() > 15 * a[:, 400:].std()
