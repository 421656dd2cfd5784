"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once — K1, K2 single-CTA + pairs (256/512 queries per pass), the
certificate levels, K4 tensor-core + CUDA-core MaxSim, graphs, the host-buffer stage."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_02062_b200 as vx  # noqa: E402
from paper_2511_02062_b200 import synth  # noqa: E402

N, D, k, nq = 20_000, 256, 10, 8
with vx.Index(N, D, tok_per_doc=64, tok_dim=64, tok_blocks=50, max_batch=600, max_k=20,
              max_qtok=nq) as idx:
    idx.synth(42)
    idx.tokens_synth(45)
    for B in (3, 200, 300):
        Q = synth.rows(43, B, B, D)
        idx.search(Q, k)
    idx.set_option(vx.VX_OPT_SCAN_PAIRS, 2)
    idx.search(synth.rows(43, 7, 520, D), k)
    idx.set_option(vx.VX_OPT_SCAN_PAIRS, 1)
    idx.set_option(vx.VX_OPT_KPRIME, 16)
    idx.search(synth.rows(43, 9, 64, D), 16)          # certificate level 2
    idx.set_option(vx.VX_OPT_KPRIME, 0)
    idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_F32)
    idx.search(synth.rows(43, 11, 9, D), k)           # K1
    idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_AUTO)
    qt = synth.query_tokens(16, nq, 64)
    cand = (np.arange(16 * 12, dtype=np.int64).reshape(16, 12) * 37) % N
    idx.maxsim(qt, cand)
    idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_CC)
    idx.maxsim(qt, cand)
    idx.set_option(vx.VX_OPT_MAXSIM, vx.VX_MAXSIM_AUTO)
    idx.set_option(vx.VX_OPT_GRAPHS, 1)
    for _ in range(2):
        idx.search_rescore(synth.rows(43, 5, 16, D), qt, k)
    print("sanitize case done", idx.stats()["cert_level2"], idx.stats()["cert_fallbacks"])

# seeded scans (shards >= 512K rows): the strided sample pass (4-key lists), the seed merge,
# the seeded full pass and the seed-bounded certificate — s8 and bf16, single-CTA and pairs
N2 = 600_000
with vx.Index(N2, D, max_batch=300, max_k=20) as idx:
    idx.synth(42)
    idx.set_option(vx.VX_OPT_SCAN, vx.VX_SCAN_TC)
    for co in (vx.VX_COARSE_I8, vx.VX_COARSE_BF16):
        idx.set_option(vx.VX_OPT_COARSE, co)
        for B in (40, 300):
            idx.search(synth.rows(43, 13, B, D), k)
    print("seeded case done", idx.stats()["cert_level2"], idx.stats()["cert_fallbacks"])
