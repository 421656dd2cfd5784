"""The small-batch re-rank split (RerankFuse::split: B <= 64 with k' >= 256 re-ranks each
query's whole candidate set over S = SMs / B CTAs; the query's last CTA selects, certifies
and writes) at slice sizes other than the benched ones, against the oracle.  s8 coarse on a
700K-row shard (AUTO picks s8 there), unseeded and seeded.  Runs on a B200."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, D = 700_000, 768


@pytest.fixture(scope="module")
def oracle_rows(oracle):
    return oracle.synth_rows(42, 0, N, D)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("B,k", [(3, 40), (5, 64), (33, 100), (64, 32), (1, 128)])
def test_split_rerank_bit_identical(vxlib, oracle, oracle_rows, B, k, seed):
    import paper_2511_02062_b200 as vx
    Q = oracle.synth_rows(43 + B, 0, B, D)
    with vx.Index(N, D, max_batch=64, max_k=128) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_SCAN_SEED, seed)
        assert idx.coarse_auto() == "i8"
        ids, sc = idx.search(Q, k)
        ids2, sc2 = idx.search(Q, k)  # the captured graph replays the same launches
        st = idx.stats()
    rid, rsc = oracle.flat_topk(oracle_rows, Q, k, mode=oracle.F32)
    assert np.array_equal(ids, rid) and np.array_equal(ids2, rid)
    assert np.array_equal(sc, rsc.astype(np.float32)) and np.array_equal(sc2, sc)
    assert st["cert_fallbacks"] == 0
