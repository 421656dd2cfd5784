import sys, time, torch
sys.path.insert(0, '.')
import paper_2511_02062_b200 as vx
from paper_2511_02062_b200 import synth
B, k = 1024, 100
Q = synth.queries(B, 768)
for shard in (0, 1):
    with vx.Index(10_000_000, 768, n_shards=2, shard=shard, max_batch=B, max_k=k) as idx:
        idx.synth(42)
        q = torch.from_numpy(Q).cuda(); ids = torch.empty((B, k), dtype=torch.int64, device="cuda"); sc = torch.empty((B, k), device="cuda")
        s = torch.cuda.Stream(); torch.cuda.set_stream(s)
        for rep in range(4):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s); idx.search_dev(q, ids, sc, k, stream=s.cuda_stream); b.record(s); b.synchronize(); idx.sync()
            st = idx.stats()
            print(shard, rep, round(a.elapsed_time(b), 3), "scan", round(st["last_scan_ms"], 3), "fb", st["cert_fallbacks"])
