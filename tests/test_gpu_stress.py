"""Back-to-back kernels of different shapes in one process: every result re-checked.
Guards against cross-kernel interference (e.g. an async mbarrier arrive landing in the
next kernel's shared memory after a CTA exits).  Runs on a B200."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_alternating_shapes_stay_exact(vxlib, oracle):
    import paper_2511_02062_b200 as vx
    from paper_2511_02062_b200 import synth
    N, D, k, nq = 40_000, 256, 10, 32
    X = oracle.synth_rows(42, 0, N, D)
    shapes = [1, 200, 7, 256, 128, 3, 150]
    Qs = {B: synth.rows(43, 7 * B, B, D) for B in shapes}
    want = {B: oracle.flat_topk(X, Qs[B], k, mode=1)[0] for B in shapes}
    qt = synth.query_tokens(16, nq, 128)
    cand = np.arange(16 * 20, dtype=np.int64).reshape(16, 20) * 997 % N
    with vx.Index(N, D, tok_per_doc=128, tok_dim=128, tok_blocks=64, max_batch=256, max_k=20,
                  max_qtok=nq) as idx:
        idx.synth(42)
        idx.tokens_synth(45)
        ms_ref = idx.maxsim(qt, cand)
        for rep in range(4):
            for B in shapes:
                ids, _ = idx.search(Qs[B], k)
                assert np.array_equal(ids, want[B]), (rep, B)
                assert np.array_equal(idx.maxsim(qt, cand), ms_ref)
        assert idx.stats()["cert_fallbacks"] == 0
