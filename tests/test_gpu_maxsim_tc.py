"""Tensor-core MaxSim (K4, tcgen05 kind::f16) against the oracle.  Runs on a B200.

Stated tolerance (north star: "the stated tolerance must be reported for any bf16 path"):
doc tokens are stored bf16 (the data), products are exact in fp32, accumulation is fp32
inside the tensor core.
  * default (nq <= 64): the fp32 query tokens enter as bf16 hi + lo pairs; the result must be
    within MS_RTOL = 1e-5 relative (+1e-6) of the fp64 MaxSim of the FP32 query tokens
    (oracle VXO_F64_Q32);
  * VX_MAXSIM_TC_BF16Q (and nq > 64): query tokens rounded to bf16; within MS_RTOL of the
    fp64 MaxSim of the same bf16-rounded inputs (against the fp32 tokens ~1e-3 relative,
    tests/test_gpu_headline.py prints the measured figure).
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MS_RTOL = 1e-5


@pytest.fixture(scope="module")
def vx(vxlib):
    import paper_2511_02062_b200 as vx
    return vx


@pytest.mark.parametrize("B,C,nq,Nd,d,T", [
    (1, 100, 32, 128, 128, 257), (8, 100, 32, 128, 128, 1000), (64, 100, 32, 128, 128, 4096),
    (3, 7, 17, 128, 128, 11), (2, 40, 128, 128, 128, 50), (5, 33, 32, 64, 128, 64),
    (4, 20, 32, 256, 128, 30), (6, 50, 32, 128, 64, 99), (2, 1, 1, 64, 64, 3)])
@pytest.mark.parametrize("bf16q", [False, True])
def test_maxsim_tc_matches_oracle(vx, oracle, B, C, nq, Nd, d, T, bf16q):
    rng = np.random.default_rng(B * 1000 + C)
    cand = np.stack([rng.choice(10_000_000, C, replace=False) for _ in range(B)]).astype(np.int64)
    if C > 3:
        cand[0, 2] = -1
    qtok = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    with vx.Index(1000, 32, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=B, max_k=max(C, 1),
                  max_qtok=nq) as idx:
        idx.tokens_synth(45)
        idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_TC_BF16Q if bf16q else vx.VX_MAXSIM_TC)
        out = idx.maxsim(qtok, cand)
    table = oracle.synth_tokens(45, 0, T, Nd, d)
    split = not bf16q and nq <= 64
    ref = oracle.maxsim(qtok, cand, table, mode=oracle.F64_Q32 if split else oracle.F64)
    fin = np.isfinite(ref)
    np.testing.assert_allclose(out[fin], ref[fin], rtol=MS_RTOL, atol=1e-6)
    assert np.isneginf(out[~fin]).all()


def test_maxsim_tc_equals_cc_within_tolerance(vx, oracle):
    B, C, nq, Nd, d, T = 16, 100, 32, 128, 128, 2048
    rng = np.random.default_rng(5)
    cand = np.stack([rng.choice(1_000_000, C, replace=False) for _ in range(B)]).astype(np.int64)
    qtok = oracle.synth_rows(44, 0, B * nq, d).reshape(B, nq, d)
    with vx.Index(1000, 32, tok_per_doc=Nd, tok_dim=d, tok_blocks=T, max_batch=B, max_k=C,
                  max_qtok=nq) as idx:
        idx.tokens_synth(45)
        idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_TC_BF16Q)  # the same bf16 query tokens
        tc = idx.maxsim(qtok, cand)
        idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_CC)
        cc = idx.maxsim(qtok, cand)
    np.testing.assert_allclose(tc, cc, rtol=MS_RTOL)
