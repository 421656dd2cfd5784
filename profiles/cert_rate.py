"""Certificate fallback rate of the tensor-core scan per shard (one GPU, shards evaluated one
at a time): for G in {1,2,4,8} and each shard g, search B queries on rows [gN/G, (g+1)N/G)
and count queries whose certificate failed (-> exact re-scan).  Sweeps k'.
usage: python profiles/cert_rate.py [N] [B] [k] [coarse=bf16|tf32|i8] [k',k',...] [G,G,...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_02062_b200 as vx  # noqa: E402
from paper_2511_02062_b200 import synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
coarse = sys.argv[4] if len(sys.argv) > 4 else "bf16"
KPS = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "256,512").split(",")]
GS = [int(x) for x in (sys.argv[6] if len(sys.argv) > 6 else "1,2,4,8").split(",")]
CO = {"bf16": vx.VX_COARSE_BF16, "tf32": vx.VX_COARSE_TF32, "i8": vx.VX_COARSE_I8}[coarse]
Q = synth.queries(B, 768)
for G in GS:
    for kp in KPS:
        fails = []
        t0 = time.time()
        for g in range(G):
            with vx.Index(N, 768, n_shards=G, shard=g, max_batch=B, max_k=k) as idx:
                idx.synth(42)
                idx.set_option(vx.VX_OPT_COARSE, CO)
                idx.set_option(vx.VX_OPT_KPRIME, kp)
                idx.search(Q, k)
                st = idx.stats()
                fails.append((st["cert_level2"], st["cert_fallbacks"]))
        print(json.dumps({"coarse": coarse, "G": G, "kprime": kp, "B": B, "k": k, "level2_and_rescans_per_shard": fails,
                          "s": round(time.time() - t0, 1)}), flush=True)
