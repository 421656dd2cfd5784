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
