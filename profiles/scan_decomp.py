"""Where the coarse scan's time goes: time the tensor-core scan kernel (idx.stats()["last_scan_ms"],
CUDA events around the launch) on the 10M x 768 index with parts of it disabled through the
VX_DEBUG_TC_NOSELECT bits (scan_tc.cu / scan_tc2.cu; debug only, results are garbage):
  1 = no selection (TMEM loads only), 2 / 4 = no doc / query streaming, 8 = no MMA,
  16 = admission threshold starts above every score (pair kernel: the filter's fast path only).
VX_DECOMP_N: index rows (default 10M; 2.5M = one shard of four).
One JSON line per (coarse, B, bits).  The bits are read when an index is created, so each
setting gets its own index.
usage: python profiles/scan_decomp.py [coarse=i8|bf16|tf32] [B,B,...] [bits,bits,...] [scan_pairs]"""
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
Bs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "128,256,1024").split(",")]
bits = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,1,7,9").split(",")]
pairs = int(sys.argv[4]) if len(sys.argv) > 4 else -1  # -1: the library default
CO = {"bf16": vx.VX_COARSE_BF16, "tf32": vx.VX_COARSE_TF32, "i8": vx.VX_COARSE_I8}[coarse]
N, D, k = int(os.environ.get("VX_DECOMP_N", 10_000_000)), 768, 100
bmax = max(Bs)
dev = torch.device("cuda", 0)
q = torch.from_numpy(synth.queries(bmax, D)).to(dev)
ids = torch.empty((bmax, k), dtype=torch.int64, device=dev)
sc = torch.empty((bmax, k), dtype=torch.float32, device=dev)
for bit in bits:
    os.environ["VX_DEBUG_TC_NOSELECT"] = str(bit)
    with vx.Index(N, D, max_batch=bmax, max_k=k) as idx:
        idx.synth(42)
        idx.set_option(vx.VX_OPT_COARSE, CO)
        idx.set_option(vx.VX_OPT_SCAN_SEED, int(os.environ.get("VX_SCAN_SEED", "1")))
        if pairs >= 0:
            idx.set_option(vx.VX_OPT_SCAN_PAIRS, pairs)
        for B in Bs:
            scan = []
            for rep in range(6):
                idx.search_dev(q[:B], ids[:B], sc[:B], k)
                idx.sync()
                if rep >= 2:
                    scan.append(idx.stats()["last_scan_ms"])
            print(json.dumps({"coarse": idx.coarse_auto(), "seed": idx.get_option(vx.VX_OPT_SCAN_SEED), "N": N, "B": B, "bits": bit, "scan_pairs": idx.get_option(vx.VX_OPT_SCAN_PAIRS),
                              "scan_ms": round(statistics.median(scan), 4)}), flush=True)
os.environ.pop("VX_DEBUG_TC_NOSELECT", None)
