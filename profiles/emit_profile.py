"""Measured profile rows for the reference's planner: time the fused B200
stage (10M x 768 top-100 + MaxSim, one GPU, graphs on, inputs in HBM) at each profiled batch
size and write rows in the reference's profile CSV schema
(`model_id,instance_size_gb,batch_size,latency_ms,throughput_qps,memory_gb`,
proj/assets/profiles.csv; read by ProfileTable, profile.hpp:24,42-61) — replacing the
synthetic modelD rows (profiles.csv:17-22, 125 ms at b=1, 400 ms at b=4).
Also prints the SLO-bounded cap (planner.hpp:91-102) and the throughput peak
(profile.hpp:110-123) for the measured profile.

usage: python profiles/emit_profile.py [out.csv] [slo_ms]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2511_02062_b200 as vx  # noqa: E402
from paper_2511_02062_b200 import batcher, synth  # noqa: E402

out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r01" / "modelD_b200_profile.csv"
slo_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 200.0
N, D, k, nq, td, Nd, T = 10_000_000, 768, 100, 32, 128, 128, 1 << 18
BATCHES = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]
bmax = BATCHES[-1]
idx = vx.Index(N, D, tok_per_doc=Nd, tok_dim=td, tok_blocks=T, max_batch=bmax, max_k=k, max_qtok=nq)
idx.synth(42)
idx.tokens_synth(45)
idx.set_option(vx.VX_OPT_GRAPHS, 1)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
q = torch.from_numpy(synth.queries(bmax, D)).to(dev)
qt = torch.from_numpy(synth.query_tokens(bmax, nq, td)).to(dev)
ids = torch.empty((bmax, k), dtype=torch.int64, device=dev)
ip = torch.empty((bmax, k), dtype=torch.float32, device=dev)
ms = torch.empty((bmax, k), dtype=torch.float32, device=dev)
mem_gb = (N * D * (4 + 2 + 1) + T * Nd * td * 2) / 1e9  # fp32 rows + bf16 + s8 shadows + tokens
profile = {}
for B in BATCHES:
    lat = []
    for rep in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        idx.search_rescore_dev(q[:B], qt[:B], ids[:B], ip[:B], ms[:B], k, stream=st.cuda_stream)
        b.record(st)
        b.synchronize()
        if rep >= 2:  # the first batch of a shape captures its graphs
            lat.append(a.elapsed_time(b))
    profile[B] = statistics.median(lat)
    print(json.dumps({"batch": B, "latency_ms": round(profile[B], 4),
                      "throughput_qps": round(1000.0 * B / profile[B], 1)}), flush=True)
rows = batcher.profile_rows("modelD", 180.0, profile, mem_gb)
out.write_text(rows)  # header + one row per batch size
print(json.dumps({"csv": str(out), "slo_ms": slo_ms, "slo_cap": batcher.slo_cap(profile, slo_ms),
                  "peak_batch": batcher.peak(profile)}))
idx.close()
