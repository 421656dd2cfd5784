"""Both coarse formats of the tensor-core scan (TF32 on the fp32 rows, bf16 on the shadow)
return the oracle's exact answer: ids AND scores bit-identical to VXO_F32, because the coarse
pass only selects candidates and the certificate proves nothing outside them can enter the
top-k (else the query is re-scanned exactly).  Runs on a B200."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


@pytest.mark.parametrize("coarse", ["tf32", "bf16"])
@pytest.mark.parametrize("N,D,B,k", [
    (100_000, 768, 16, 10), (50_000, 768, 1, 100), (20_000, 1024, 64, 100), (30_000, 768, 200, 128),
    (12_345, 128, 7, 5), (4_000, 64, 300, 64)])
def test_coarse_formats_exact(vx, oracle, coarse, N, D, B, k):
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, {"tf32": vx.VX_COARSE_TF32, "bf16": vx.VX_COARSE_BF16}[coarse])
        ids, sc = idx.search(Q, k)
        fb = idx.stats()["cert_fallbacks"]
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    v = rid >= 0
    assert np.array_equal(sc[v], rsc[v].astype(np.float32))
    if N >= 20_000:
        assert fb == 0, f"{fb} certificate fallbacks"


def test_no_shadow_flag(vx, oracle):
    N, D, B, k = 10_000, 256, 4, 10
    with vx.Index(N, D, max_batch=B, max_k=k, flags=vx.VX_FLAG_NO_BF16_SHADOW) as idx:
        idx.synth(42)
        with pytest.raises(vx.VxError):
            idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_BF16)
        ids, _ = idx.search(oracle.synth_rows(43, 0, B, D), k)
    rid, _ = oracle.flat_topk(oracle.synth_rows(42, 0, N, D), oracle.synth_rows(43, 0, B, D), k, mode=1)
    assert np.array_equal(ids, rid)


def test_upload_refreshes_shadow(vx, oracle):
    # rows uploaded in two pieces; the bf16 shadow must follow every upload
    N, D, B, k = 6_000, 128, 5, 10
    X = oracle.synth_rows(7, 0, N, D)
    Q = oracle.synth_rows(8, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(1)
        idx.upload(X[:3000], 0)
        idx.upload(X[3000:], 3000)
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_BF16)
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)


def test_auto_coarse_follows_quantisation_quality(vx, oracle):
    # AUTO takes the s8 pass when the shard is long enough (>= 16 tiles of 256 rows per CTA)
    # and its per-column quantisation is tight (max residual norm <= 3 % of the mean row norm:
    # the synthetic rows are at ~1 %), bf16 when an outlier inflates a column scale so far that
    # the other rows lose that coordinate, or the shard is short — exact either way
    N, D, B, k = 700_000, 256, 24, 10
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X, 0)
        assert idx.coarse_auto() == "i8"
        ids, sc = idx.search(Q, k)
        rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
        assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))
        Xo = X.copy()
        Xo[123, 5] = 400.0  # one spike: the scale grows ~10^4 x, residuals ~ the row norms
        idx.upload(Xo[123:124], 123)
        assert idx.coarse_auto() == "bf16"
        ids, sc = idx.search(Q, k)
        rid, rsc = oracle.flat_topk(Xo, Q, k, mode=1)
        assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))
        idx.upload(X[123:124], 123)  # back to the tight scale
        assert idx.coarse_auto() == "i8"
    with vx.Index(50_000, D, max_batch=B, max_k=k) as idx:  # 1-2 tiles per CTA
        idx.synth(42)
        assert idx.coarse_auto() == "bf16"


def _clustered(rng, n, D, n_centers, spread):
    centers = rng.standard_normal((n_centers, D)).astype(np.float32)
    lab = rng.integers(0, n_centers, n)
    return (centers[lab] + spread * rng.standard_normal((n, D))).astype(np.float32), centers


@pytest.mark.parametrize("coarse", ["i8", "bf16"])
@pytest.mark.parametrize("spread", [0.05, 0.002])
def test_coarse_exact_on_clustered_near_duplicates(vx, oracle, coarse, spread):
    # near-duplicate documents (tight clusters, queries at the centres): the coarse error
    # bound E exceeds the gaps between many candidates, so certificates fail and the level-2
    # / level-3 paths carry the queries — the answer must still be the exact oracle's
    rng = np.random.default_rng(7)
    N, D, B, k = 700_000, 256, 48, 16
    X, centers = _clustered(rng, N, D, 300, spread)
    Q = (centers[rng.integers(0, 300, B)] + 0.01 * rng.standard_normal((B, D))).astype(np.float32)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X, 0)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, {"i8": vx.VX_COARSE_I8, "bf16": vx.VX_COARSE_BF16}[coarse])
        ids, sc = idx.search(Q, k)
        st = idx.stats()
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    assert np.array_equal(sc, rsc.astype(np.float32))
    if spread < 0.01:  # the tight case must have exercised the fallbacks
        assert st["cert_level2"] + st["cert_fallbacks"] > 0


@pytest.mark.parametrize("coarse", ["i8", "bf16"])
@pytest.mark.parametrize("B", [48, 300])
def test_seeded_scan_exact_and_equal_to_unseeded(vx, oracle, coarse, B):
    # shards of >= 512K rows seed each query's admission threshold from a 1/64 row sample
    # (VX_OPT_SCAN_SEED, vx_stage.cu local_topk_tc); the lists then skip every document below
    # the seed and the certificate bounds them by it — ids and scores must not move.
    # B = 300: the CTA-pair kernel with two query groups; 48: the single-CTA kernel
    N, D, k = 700_000, 256, 100
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    out = {}
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X, 0)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, {"i8": vx.VX_COARSE_I8, "bf16": vx.VX_COARSE_BF16}[coarse])
        assert idx.get_option(vx.VX_OPT_SCAN_SEED) == 1
        for seed in (1, 0):
            idx.set_option(vx.VX_OPT_SCAN_SEED, seed)
            out[seed] = idx.search(Q, k)
            assert idx.stats()["cert_fallbacks"] == 0
    for seed in (1, 0):
        assert np.array_equal(out[seed][0], rid)
        assert np.array_equal(out[seed][1], rsc.astype(np.float32))


@pytest.mark.parametrize("coarse", ["i8", "bf16"])
def test_seeded_scan_exact_when_the_sample_is_unrepresentative(vx, oracle, coarse):
    # every sampled row (row % 64 == 0) is scaled up 4x: the seed lands far above the k'-th
    # coarse score of the other rows, the lists miss documents that belong in the top-k, and
    # only the certificate's seed bound notices — the fallbacks must restore the exact answer
    N, D, B, k = 700_000, 256, 40, 50
    X = oracle.synth_rows(42, 0, N, D)
    X[::64] *= 4.0
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X, 0)
        idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
        idx.set_option(vx.VX_OPT_COARSE, {"i8": vx.VX_COARSE_I8, "bf16": vx.VX_COARSE_BF16}[coarse])
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid)
    assert np.array_equal(sc, rsc.astype(np.float32))


@pytest.mark.parametrize("B,k", [(24, 10), (300, 100)])
def test_anisotropic_rows_exact_and_auto_demotes_s8(vx, oracle, B, k):
    # power-law per-dimension scales + outlier dimensions (vx_synth.h dist 1), queries drawn
    # alike.  One s8 scale per shard: the residual test already sends AUTO to bf16.  Per-column
    # scales (VX_OPT_I8_SCALE = 1) pass the residual test (AUTO starts on s8), but folding them
    # into the query widens ITS error beyond the score gaps, so every query needs the exact
    # re-scan — results exact anyway — and the certificate record then demotes AUTO to bf16.
    N, D = 700_000, 768
    X = oracle.synth_rows(42, 0, N, D, 1)
    Q = oracle.synth_rows(43, 0, B, D, 1)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42, dist=1)
        assert np.array_equal(idx.download(1000, 64).view(np.uint32), X[1000:1064].view(np.uint32))
        assert idx.coarse_auto() == "bf16"  # static test: one shard scale is too coarse
        idx.set_option(vx.VX_OPT_I8_SCALE, 1)
        assert idx.coarse_auto() == "i8"
        ids, sc = idx.search(Q, k)
        assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))
        assert idx.coarse_auto() == "bf16"  # demoted by the certificate record
        st0 = idx.stats()
        ids, sc = idx.search(Q, k)
        st1 = idx.stats()
        assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))
        # the bf16 pass certifies (almost) every query: no exact re-scans
        assert st1["cert_fallbacks"] - st0["cert_fallbacks"] <= B // 50
        idx.synth(42, dist=0)  # a new shard resets the decision
        assert idx.coarse_auto() == "i8"
        idx.set_option(vx.VX_OPT_I8_SCALE, 0)
    print(f"anisotropic B={B}: s8 re-scans {st0['cert_fallbacks']}, then bf16 re-scans "
          f"{st1['cert_fallbacks'] - st0['cert_fallbacks']}")


def test_per_column_s8_scales_exact(vx, oracle):
    # VX_OPT_I8_SCALE = 1: column scales folded into the query; same exact results
    N, D, B, k = 700_000, 256, 40, 32
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_I8_SCALE, 1)
        idx.set_option(vx.VX_OPT_COARSE, vx.VX_COARSE_I8)
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(X, Q, k, mode=1)
    assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))


def test_outlier_row_switches_auto_to_bf16(vx, oracle):
    # a row 1000x longer than the rest inflates EVERY column scale: the other rows quantise
    # to ~0 and AUTO must leave s8
    N, D, B, k = 700_000, 256, 8, 10
    X = oracle.synth_rows(42, 0, N, D)
    Q = oracle.synth_rows(43, 0, B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.upload(X, 0)
        assert idx.coarse_auto() == "i8"
        Xo = X.copy()
        Xo[77] *= 1000.0
        idx.upload(Xo[77:78], 77)
        assert idx.coarse_auto() == "bf16"
        ids, sc = idx.search(Q, k)
    rid, rsc = oracle.flat_topk(Xo, Q, k, mode=1)
    assert np.array_equal(ids, rid) and np.array_equal(sc, rsc.astype(np.float32))
