"""Checks of the fused stage's output (top-k by inner product, re-scored by MaxSim, ordered
MaxSim desc / id asc) against the oracle — shared by the GPU tests, smoke() and bench.py's
cpu_baseline leg (test infrastructure, like oracle/).

Stated tolerances (BASELINE.json north_star: ids identical except ties within tolerance, fp32
scores within 1e-4 relative, the tolerance of any bf16 path stated):
  * inner-product ids and scores: EXACT — the set of top-k ids and every score bit-equal to the
    oracle's VXO_F32 mode (the tensor-core scan only selects candidates; the reported scores
    are the exact in-order fp32 chains, certified);
  * MaxSim (default tensor-core kernel, fp32 query tokens entering as bf16 hi + lo pairs,
    bf16 doc-token store): |ms - truth| <= MS_RTOL |truth| + MS_ATOL where truth = the fp64
    MaxSim of the fp32 query tokens against the stored bf16 doc tokens (oracle VXO_F64_Q32);
  * output order: the GPU order is exactly (its own MaxSim desc, id asc), and against the
    oracle's order (truth desc, id asc) two entries may only be swapped when their truths
    differ by less than the MaxSim tolerance.
"""
from __future__ import annotations

import numpy as np

MS_RTOL = 1e-5
MS_ATOL = 1e-6


def ms_tol(truth: np.ndarray, rtol: float = MS_RTOL, atol: float = MS_ATOL) -> np.ndarray:
    return rtol * np.abs(truth) + atol


def check_ip_topk(ids, ip, ref_ids, ref_ip) -> None:
    """One query: the id set equals the oracle's and every score is bit-equal to its fp32."""
    v = ids >= 0
    rv = ref_ids >= 0
    assert sorted(ids[v].tolist()) == sorted(ref_ids[rv].tolist()), (ids, ref_ids)
    lut = dict(zip(ref_ids[rv].tolist(), ref_ip[rv].tolist()))
    for i, p in zip(ids[v].tolist(), ip[v].tolist()):
        assert np.float32(lut[i]) == np.float32(p), (i, p, lut[i])


def check_stage_query(ids, ip, ms, ref_ids, ref_ip, ref_ms, *, rtol=MS_RTOL, atol=MS_ATOL) -> dict:
    """One query of the fused stage.  ids/ip/ms: the GPU output in its order; ref_ids/ref_ip:
    the oracle's inner-product top-k (any order; ref_ip the exact fp32 chain values); ref_ms:
    the oracle's MaxSim truth for ref_ids.  Returns the measured MaxSim error and the number of
    adjacent positions whose order differs from the oracle's."""
    ids, ip, ms = np.asarray(ids), np.asarray(ip), np.asarray(ms)
    check_ip_topk(ids, ip, ref_ids, ref_ip)
    v = ids >= 0
    lut = dict(zip(np.asarray(ref_ids).tolist(), np.asarray(ref_ms).tolist()))
    iv, mv = ids[v], ms[v].astype(np.float64)
    truth = np.array([lut[i] for i in iv.tolist()], np.float64)
    err = np.abs(mv - truth)
    assert (err <= ms_tol(truth, rtol, atol)).all(), (err.max(), truth[err.argmax()])
    swaps = 0
    for j in range(len(iv) - 1):
        # the kernel's own order is exact: MaxSim desc, id asc
        assert mv[j] > mv[j + 1] or (mv[j] == mv[j + 1] and iv[j] < iv[j + 1]), (j, mv[j], mv[j + 1])
        # against the oracle's order: out of order only inside the tolerance
        ahead = truth[j] > truth[j + 1] or (truth[j] == truth[j + 1] and iv[j] < iv[j + 1])
        if not ahead:
            swaps += 1
            tol = ms_tol(truth[j:j + 2], rtol, atol).max()
            assert truth[j + 1] - truth[j] <= 2 * tol, (j, truth[j], truth[j + 1])
    assert not (v[1:] & ~v[:-1]).any()  # padding (-1) only after the real entries
    rel = float((err / np.maximum(np.abs(truth), 1e-30)).max()) if len(err) else 0.0
    return {"ms_max_abs_err": float(err.max()) if len(err) else 0.0, "ms_max_rel_err": rel,
            "order_swaps": swaps}


def check_stage(ids, ip, ms, ref_ids, ref_ip, ref_ms, **kw) -> dict:
    """All queries (rows); returns the worst errors and the total swap count."""
    out = {"ms_max_abs_err": 0.0, "ms_max_rel_err": 0.0, "order_swaps": 0, "queries": 0}
    for b in range(ids.shape[0]):
        r = check_stage_query(ids[b], ip[b], ms[b], ref_ids[b], ref_ip[b], ref_ms[b], **kw)
        out["ms_max_abs_err"] = max(out["ms_max_abs_err"], r["ms_max_abs_err"])
        out["ms_max_rel_err"] = max(out["ms_max_rel_err"], r["ms_max_rel_err"])
        out["order_swaps"] += r["order_swaps"]
        out["queries"] += 1
    return out
