"""BASELINE configs[4]: large-batch sweep on the 10M x 768 index, B = 1, 2, 4, ..., 4096 —
the HBM-streaming -> tcgen05-GEMM crossover.  One index, search only (top-100), graphs on,
inputs in HBM; per B: median stage time over 5 reps, the scan kernel time, and both
rooflines of the scan (bench.scan_roofline).  One JSON line per B.
usage: python profiles/batch_sweep.py [auto|bf16|tf32|i8] > profiles/r01/batch_sweep.jsonl"""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (roofline helpers)
import paper_2511_02062_b200 as vx  # noqa: E402
from paper_2511_02062_b200 import synth  # noqa: E402

N, D, k = 10_000_000, 768, 100
bmax = 4096
idx = vx.Index(N, D, max_batch=bmax, max_k=k)
idx.synth(42)
idx.set_option(vx.VX_OPT_GRAPHS, 1)
if len(sys.argv) > 1:
    idx.set_option(vx.VX_OPT_COARSE, {"auto": vx.VX_COARSE_AUTO, "bf16": vx.VX_COARSE_BF16,
                                      "tf32": vx.VX_COARSE_TF32, "i8": vx.VX_COARSE_I8}[sys.argv[1]])
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(dev)
torch.cuda.set_stream(st)
q = torch.from_numpy(synth.queries(bmax, D)).to(dev)
ids = torch.empty((bmax, k), dtype=torch.int64, device=dev)
sc = torch.empty((bmax, k), dtype=torch.float32, device=dev)
pk = bench.peaks()
B = 1
while B <= bmax:
    lat, scan = [], []
    for rep in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        idx.search_dev(q[:B], ids[:B], sc[:B], k, stream=st.cuda_stream)
        b.record(st)
        b.synchronize()
        idx.sync()
        if rep >= 2:
            lat.append(a.elapsed_time(b))
            scan.append(idx.stats()["last_scan_ms"])
    ms, sms = statistics.median(lat), statistics.median(scan)
    roof = bench.scan_roofline(pk, tc=True, coarse=idx.coarse_auto(), n_local=N, D=D, B=B, k=k,
                               scan_ms=sms)
    print(json.dumps({"batch": B, "stage_ms": round(ms, 4), "queries_per_s": round(1000.0 * B / ms, 1),
                      "scan_ms": round(sms, 4), "bound": roof["bound"], "frac": round(roof["frac"], 4),
                      "hbm_frac": round(roof["hbm"]["frac"], 4),
                      "tensor_frac": round(roof["compute"]["frac"], 4),
                      "passes": roof["launches"],
                      "cert_fallbacks": idx.stats()["cert_fallbacks"]}), flush=True)
    B *= 2
idx.close()
