"""Parity at the benched configurations themselves (BASELINE.json configs[0], [2], [3], [4]),
through the C-ABI, against the CPU oracle.  Runs on a B200.

The index of configs[2]/[4] (10M x 768 fp32 = 30.7 GB) never exists on the host: the oracle
generates its rows chunk by chunk (oracle/vxoracle.py flat_topk_synth) from the same
counter-based generator the device fill uses, and merges the per-chunk top-k lists.  The GPU
index is built exactly as bench.py builds it (device synth, seed 42; token store 2^18 blocks,
seed 45; CUDA graphs on; AUTO coarse format -> the s8 shadow with seeded admission thresholds,
512-query CTA-pair passes), and the queries are bench.py's (seed 43 rows, seed 44 tokens).

Bar (tests/stagecheck.py): inner-product ids as a set and every IP score bit-equal to the
oracle's VXO_F32; MaxSim within 1e-5 relative (+1e-6) of the fp64 MaxSim of the fp32 query
tokens; output order exact in the kernel's own keys and equal to the oracle's except swaps
inside that tolerance.
"""
from __future__ import annotations

import numpy as np
import pytest

from stagecheck import check_ip_topk, check_stage

pytestmark = pytest.mark.gpu

N10, D10, K10, NQ, ND, TD, TBLK = 10_000_000, 768, 100, 32, 128, 128, 1 << 18
# queries checked on the 10M index: every 16th of the headline batch (both 512-query passes),
# the first 16 (small-batch sweep points), every 64th of the 4096 batch
SEL10 = sorted(set(range(0, 1024, 16)) | set(range(16)) | set(range(0, 4096, 64)) | set(range(0, 256, 8)))


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


@pytest.fixture(scope="module")
def idx10m(vx):
    idx = vx.Index(N10, D10, tok_per_doc=ND, tok_dim=TD, tok_blocks=TBLK, max_batch=4096,
                   max_k=K10, max_qtok=NQ)
    idx.set_option(vx.VX_OPT_GRAPHS, 1)
    idx.synth(42)
    idx.tokens_synth(45)
    yield idx
    idx.close()


@pytest.fixture(scope="module")
def queries10m():
    from paper_2511_02062_b200 import synth
    return synth.queries(4096, D10, seed=43), synth.query_tokens(1024, NQ, TD)


@pytest.fixture(scope="module")
def oracle10m(oracle, queries10m):
    """Exact top-100 of the SEL10 queries over the full 10M-row synthetic index."""
    Q, _ = queries10m
    sel = np.array(SEL10)
    ids, sc, t = oracle.flat_topk_synth(42, N10, D10, Q[sel], K10, mode=oracle.F32)
    return {int(b): (ids[j], sc[j]) for j, b in enumerate(sel)}


def test_headline_config2_stage_exact_as_benched(vx, oracle, idx10m, queries10m, oracle10m):
    """configs[2]: 10M x 768, top-100 + MaxSim (32 x 128 x 128), B = 1024 — the bench step."""
    Q, qt = queries10m
    B = 1024
    assert idx10m.coarse_auto() == "i8"  # the s8 shadow + seeded pass the bench measures
    idx10m.reset_stats()
    first = idx10m.search_rescore(Q[:B], qt, K10)    # eager run + graph capture
    again = idx10m.search_rescore(Q[:B], qt, K10)    # graph replay (what the timed steps run)
    for a, b in zip(first, again):
        assert np.array_equal(a, b)
    st = idx10m.stats()
    assert st["graph_replays"] >= 1
    ids, ip, ms = again
    sel = np.arange(0, B, 16)
    rid = np.stack([oracle10m[int(b)][0] for b in sel])
    rip = np.stack([oracle10m[int(b)][1] for b in sel])
    rms = oracle.maxsim_synth(qt[sel], rid, 45, TBLK, ND, TD, mode=oracle.F64_Q32)
    r = check_stage(ids[sel], ip[sel], ms[sel], rid, rip, rms)
    print(f"configs[2] B=1024: {r['queries']} queries exact; MaxSim max rel err "
          f"{r['ms_max_rel_err']:.2e} (abs {r['ms_max_abs_err']:.2e}) vs fp64 of the fp32 "
          f"tokens; {r['order_swaps']} within-tolerance order swaps; cert level2 "
          f"{st['cert_level2']}, re-scans {st['cert_fallbacks']}")


def test_headline_bf16_query_tokens_error_is_stated(vx, oracle, idx10m, queries10m, oracle10m):
    """The bf16-rounded-query MaxSim (VX_MAXSIM_TC_BF16Q) is within 1e-5 of the fp64 MaxSim of
    the bf16-rounded tokens, and measurably NOT within it of the fp32-token truth — the error
    the default hi/lo split removes."""
    Q, qt = queries10m
    sel = np.arange(0, 1024, 64)
    rid = np.stack([oracle10m[int(b)][0] for b in sel])
    idx10m.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_TC_BF16Q)
    try:
        out = idx10m.maxsim(qt[sel], rid)
    finally:
        idx10m.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_AUTO)
    split = idx10m.maxsim(qt[sel], rid)
    t16 = oracle.maxsim_synth(qt[sel], rid, 45, TBLK, ND, TD, mode=oracle.F64)
    t32 = oracle.maxsim_synth(qt[sel], rid, 45, TBLK, ND, TD, mode=oracle.F64_Q32)
    np.testing.assert_allclose(out, t16, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(split, t32, rtol=1e-5, atol=1e-6)
    e16 = float(np.max(np.abs(out - t32) / np.abs(t32)))
    e32 = float(np.max(np.abs(split - t32) / np.abs(t32)))
    print(f"MaxSim rel err vs fp32-token truth: bf16 queries {e16:.2e}, hi/lo split {e32:.2e}")
    assert e16 > 10 * e32


@pytest.mark.parametrize("B", [1, 16, 64, 256, 4096])
def test_config4_sweep_points_exact(vx, idx10m, queries10m, oracle10m, B):
    """configs[4]: search-only sweep points on the 10M index, k = 100."""
    Q, _ = queries10m
    ids, sc = idx10m.search(Q[:B], K10)
    for b in [b for b in SEL10 if b < B]:
        rid, rsc = oracle10m[b]
        assert np.array_equal(ids[b], rid), b
        assert np.array_equal(sc[b], rsc.astype(np.float32)), b


@pytest.fixture(scope="module")
def idx1m(vx):
    idx = vx.Index(1_000_000, 1024, max_batch=1024, max_k=10)
    idx.set_option(vx.VX_OPT_GRAPHS, 1)
    idx.synth(42)
    yield idx
    idx.close()


def test_config3_audio_index_exact(vx, oracle, idx1m):
    """configs[3]: 1M x 1024, top-10 — fixed batches and a Poisson trace through the live
    batcher (variable batch sizes, each replaying its own captured graph)."""
    from paper_2511_02062_b200 import batcher, synth
    assert idx1m.coarse_auto() == "i8"
    Q = synth.queries(4096, 1024, seed=43)
    sel = np.arange(0, 4096, 32)
    rid, rsc, _ = oracle.flat_topk_synth(42, 1_000_000, 1024, Q[sel], 10, mode=oracle.F32)
    ids, sc = idx1m.search(Q[:1024], 10)
    for j, b in enumerate(sel[sel < 1024]):
        assert np.array_equal(ids[b], rid[j]) and np.array_equal(sc[b], rsc[j].astype(np.float32))
    idx1m.prepare(10, 1024)
    arr = batcher.poisson_arrivals(300_000.0, 4096, seed=11)
    lat, bo, tids = batcher.serve_trace(idx1m, arr, 1024, Q, None, 10, want_ids=True)
    sizes = np.bincount(bo)
    assert sizes.max() <= 1024 and len(set(sizes.tolist())) > 1  # several batch sizes
    assert np.array_equal(tids[sel], rid)


@pytest.mark.parametrize("B", [1, 2, 4, 8, 16, 32])
def test_config0_flat_exact_every_query(vx, oracle, B):
    """configs[0]: 100K x 768 top-10, batches of 1-32 (L2-sized shard: AUTO -> bf16)."""
    from paper_2511_02062_b200 import synth
    X = oracle.synth_rows(42, 0, 100_000, 768)
    Q = synth.queries(B, 768, seed=43)
    with vx.Index(100_000, 768, max_batch=32, max_k=10) as idx:
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        idx.synth(42)
        for _ in range(2):  # eager + capture, then the graph replay
            ids, sc = idx.search(Q, 10)
            rid, rsc = oracle.flat_topk(X, Q, 10, mode=oracle.F32)
            assert np.array_equal(ids, rid)
            assert np.array_equal(sc, rsc.astype(np.float32))
        for b in range(B):
            check_ip_topk(ids[b], sc[b], rid[b], rsc[b])
