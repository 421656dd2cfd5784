"""The fp32 doc-token store (VX_FLAG_TOKENS_F32; SURVEY.md §8(d) C2's fp32 variant): MaxSim
runs as exact in-order fp32 chains on the CUDA cores with the query tokens unrounded, so every
MaxSim score is bit-identical to the oracle's VXO_F32 chains over the fp32 table (and within
1e-5 of fp64).  Runs on a B200."""
from __future__ import annotations

import numpy as np
import pytest

from stagecheck import check_stage

pytestmark = pytest.mark.gpu

N, D, NQ, ND, TD, T = 60_000, 768, 32, 128, 128, 97


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


@pytest.fixture(scope="module")
def table32(oracle):
    return oracle.synth_rows(45, 0, T * ND, TD).reshape(T, ND, TD)


def _index(vx, max_batch=16, k=10):
    idx = vx.Index(N, D, tok_per_doc=ND, tok_dim=TD, tok_blocks=T, max_batch=max_batch, max_k=100,
                   max_qtok=NQ, flags=vx.VX_FLAG_TOKENS_F32)
    idx.synth(42)
    idx.tokens_synth(45)
    return idx


def test_fp32_store_synth_upload_download(vx, table32):
    with _index(vx) as idx:
        assert idx.tokens_f32
        got = idx.tokens_download(0, T)
        assert got.dtype == np.float32 and np.array_equal(got, table32)  # the generator, unrounded
        rng = np.random.default_rng(3)
        blk = rng.standard_normal((5, ND, TD)).astype(np.float32)
        idx.tokens_upload(blk, 11)
        assert np.array_equal(idx.tokens_download(11, 5), blk)
        from paper_2511_02062_b200._lib import check
        with pytest.raises(vx.VxError):  # the bf16 entry points refuse an fp32 store
            check(idx.lib.vx_tokens_upload(idx._h, None, 0, 0))


@pytest.mark.parametrize("B", [1, 7, 16])
def test_fp32_store_maxsim_bit_exact(vx, oracle, table32, B):
    from paper_2511_02062_b200 import synth
    qt = synth.query_tokens(B, NQ, TD, seed=60 + B)
    rng = np.random.default_rng(B)
    cand = np.stack([rng.choice(N, 100, replace=False) for _ in range(B)]).astype(np.int64)
    cand[0, 5] = -1  # no candidate -> -inf
    with _index(vx) as idx:
        ms = idx.maxsim(qt, cand)
    want32 = oracle.maxsim(qt, cand, table32, mode=oracle.F32)
    want64 = oracle.maxsim(qt, cand, table32, mode=oracle.F64)
    assert np.array_equal(ms.astype(np.float64), want32.astype(np.float32).astype(np.float64))
    fin = np.isfinite(want64)
    assert np.all(np.abs(ms[fin] - want64[fin]) <= 1e-5 * np.abs(want64[fin]) + 1e-6)
    assert np.isneginf(ms[0, 5])


@pytest.mark.parametrize("graphs", [0, 1])
def test_fp32_store_stage_exact(vx, oracle, table32, graphs):
    from paper_2511_02062_b200 import synth
    B, k = 12, 10
    Q = synth.queries(B, D)
    qt = synth.query_tokens(B, NQ, TD, seed=71)
    with _index(vx) as idx:
        idx.set_option(vx.VX_OPT_GRAPHS, graphs)
        out = idx.search_rescore(Q, qt, k)
        out2 = idx.search_rescore(Q, qt, k)
    for a, b in zip(out, out2):
        assert np.array_equal(a, b)
    ids, ip, ms = out
    X = oracle.synth_rows(42, 0, N, D)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=oracle.F32)
    rms64 = oracle.maxsim(qt, rid, table32, mode=oracle.F64)
    check_stage(ids, ip, ms, rid, rsc, rms64)
    # bit-exact MaxSim against the oracle's fp32 chains of the fp32 tokens, row by row
    for b in range(B):
        want = oracle.maxsim(qt[b:b + 1], ids[b:b + 1], table32, mode=oracle.F32)[0]
        assert np.array_equal(ms[b].astype(np.float64), want.astype(np.float32).astype(np.float64))


def test_fp32_store_refuses_tensor_core_maxsim(vx):
    with _index(vx) as idx:
        with pytest.raises(vx.VxError):
            idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_TC)


@pytest.mark.parametrize("nq,nd,td", [(5, 64, 64), (32, 100, 128), (17, 128, 96)])
def test_fp32_store_partial_tiles(vx, oracle, nq, nd, td):
    """Query-token counts that are not a multiple of the 4-token register tile, doc blocks
    shorter than the 128-row tile, other token dims: still bit-identical."""
    from paper_2511_02062_b200 import synth
    N2, T2, B = 20_000, 37, 6
    table = oracle.synth_rows(45, 0, T2 * nd, td).reshape(T2, nd, td)
    qt = synth.query_tokens(B, nq, td, seed=81)
    rng = np.random.default_rng(nq)
    cand = np.stack([rng.choice(N2, 40, replace=False) for _ in range(B)]).astype(np.int64)
    with vx.Index(N2, 256, tok_per_doc=nd, tok_dim=td, tok_blocks=T2, max_batch=B, max_k=64,
                  max_qtok=32, flags=vx.VX_FLAG_TOKENS_F32) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        assert np.array_equal(idx.tokens_download(0, T2), table)
        ms = idx.maxsim(qt, cand)
    want = oracle.maxsim(qt, cand, table, mode=oracle.F32)
    assert np.array_equal(ms.astype(np.float64), want.astype(np.float32).astype(np.float64))
