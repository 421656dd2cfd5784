"""The device-side launch timers behind the bench's kernel times (vx_stats.kt_*: every launch,
inside CUDA graphs, folded by each launch's last CTA): launch counts, plausible durations and
clocks, and the last step's kernel order.  Runs on a B200."""
from __future__ import annotations

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("graphs", [0, 1])
def test_ktimers_count_and_order(vxlib, graphs):
    import paper_2511_02062_b200 as vx
    from paper_2511_02062_b200 import synth
    N, D, B, k, steps = 100_000, 768, 16, 10, 7
    Q = synth.queries(B, D)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_GRAPHS, graphs)
        for _ in range(3):
            idx.search(Q, k)
        idx.sync()
        idx.reset_stats()
        t0 = time.perf_counter()
        for _ in range(steps):
            idx.search(Q, k)
        idx.sync()
        wall_ms = (time.perf_counter() - t0) * 1e3
        s = idx.stats()
    # one tensor-core scan and one re-rank per batch, no sample pass (100K rows), no MaxSim
    assert s["kt_launches"][0] == steps
    assert s["kt_launches"][3] == 0
    assert s["kt_rerank_launches"] == steps
    scan_ms, rr_ms = s["kt_ms"][0], s["kt_rerank_ms"]
    assert 0 < scan_ms / steps < 1.0 and 0 < rr_ms / steps < 1.0
    assert scan_ms + rr_ms < wall_ms
    assert 300 < s["kt_sm_mhz"][0] < 2500
    tl = s["kt_last_us"]  # [kind][start, end], us after the earliest start
    scan, rerank = (tl[0], tl[1]), (tl[8], tl[9])
    assert scan[0] == 0.0 and scan[1] > 0
    assert scan[1] <= rerank[0] < rerank[1]
    assert s["kt_origin_ns"] > 0
    assert np.isfinite(scan_ms)


def test_sync_waits_for_the_callers_stream(vxlib):
    """vx_sync after a *_dev call on a caller's stream (no caller-side synchronize): it waits
    for that stream's work (an event recorded there) and the stats it returns count every
    launch; the direct-I/O graph's outputs are final when it returns."""
    import torch
    import paper_2511_02062_b200 as vx
    from paper_2511_02062_b200 import synth
    N, D, B, k, steps = 100_000, 768, 16, 10, 5
    dev = torch.device("cuda", 0)
    Q = synth.queries(B, D)
    q = torch.from_numpy(Q).to(dev)
    ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    ip = torch.empty((B, k), dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(dev)
    with vx.Index(N, D, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_GRAPHS, 1)
        want_ids, want_ip = idx.search(Q, k)
        for _ in range(3):  # first sighting eager, then the captured direct-I/O graph
            idx.search_dev(q, ids, ip, k, stream=st.cuda_stream)
        idx.sync()
        idx.reset_stats()
        for _ in range(steps):
            with torch.cuda.stream(st):
                ids.fill_(-7)
            idx.search_dev(q, ids, ip, k, stream=st.cuda_stream)
        idx.sync()  # no torch synchronize before it
        got_ids, got_ip = ids.cpu().numpy(), ip.cpu().numpy()
        s = idx.stats()
    assert s["kt_launches"][0] == steps and s["kt_rerank_launches"] == steps
    assert s["graph_replays"] == steps
    assert np.array_equal(got_ids, want_ids) and np.array_equal(got_ip, want_ip)
