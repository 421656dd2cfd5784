"""One fused stage (10M x 768 top-100 + MaxSim 32x128x128, one GPU, graphs off so every kernel
is its own launch) at batch B with a given coarse format, repeated a few times — the command
behind the per-kernel launch lists (ncu --metrics gpu__time_duration.sum) that break the stage
time into scan / merge / re-rank / certificate / MaxSim.  Prints the median stage time and the
certificate counters.
usage: python profiles/stage_kernels.py [coarse=bf16|i8|tf32] [B] [reps] [G]
G > 1: shard 0 of G on this one GPU (the per-shard share of a G-GPU stage; search only —
the MaxSim owner step needs the other ranks)."""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2511_02062_b200 as vx  # noqa: E402
from paper_2511_02062_b200 import synth  # noqa: E402

coarse = sys.argv[1] if len(sys.argv) > 1 else "i8"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
G = int(sys.argv[4]) if len(sys.argv) > 4 else 1
CO = {"bf16": vx.VX_COARSE_BF16, "tf32": vx.VX_COARSE_TF32, "i8": vx.VX_COARSE_I8}[coarse]
N, D, k, nq, td, Nd, T = 10_000_000, 768, 100, 32, 128, 128, 1 << 18
if G > 1:
    idx = vx.Index(N, D, n_shards=G, shard=0, max_batch=B, max_k=k)
    idx.synth(42)
else:
    idx = vx.Index(N, D, tok_per_doc=Nd, tok_dim=td, tok_blocks=T, max_batch=B, max_k=k, max_qtok=nq)
    idx.synth(42)
    idx.tokens_synth(45)
idx.set_option(vx.VX_OPT_COARSE, CO)
idx.set_option(vx.VX_OPT_SCAN_SEED, int(os.environ.get("VX_SCAN_SEED", "1")))
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
q = torch.from_numpy(synth.queries(B, D)).to(dev)
qt = torch.from_numpy(synth.query_tokens(B, nq, td)).to(dev)
ids = torch.empty((B, k), dtype=torch.int64, device=dev)
ip = torch.empty((B, k), dtype=torch.float32, device=dev)
ms = torch.empty((B, k), dtype=torch.float32, device=dev)
lat = []
for rep in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    if G > 1:
        idx.search_dev(q, ids, ip, k, stream=st.cuda_stream)
    else:
        idx.search_rescore_dev(q, qt, ids, ip, ms, k, stream=st.cuda_stream)
    b.record(st)
    b.synchronize()
    idx.sync()
    lat.append(a.elapsed_time(b))
s = idx.stats()
print(json.dumps({"coarse": idx.coarse_auto(), "seed": idx.get_option(vx.VX_OPT_SCAN_SEED), "B": B, "stage_ms": round(statistics.median(lat[1:]), 4),
                  "scan_ms": round(s["last_scan_ms"], 4), "level2": s["cert_level2"],
                  "rescans": s["cert_fallbacks"], "launches": s["kernel_launches"]}), flush=True)
idx.close()
