#!/bin/bash
# Full validation on a 4-GPU box: every GPU test (incl. multi-GPU), smoke, bench N=1 + the
# reference arm, scaling 2/4, AudioQuery at 1 and 4 members.
set -x
O=gpurun_out/${TAG:-f1}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_g1.json 2> $O/bench_g1.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
NS="2 4" BATCHES="1024" STEPS=30 timeout 1500 bash profiles/scaling.sh > $O/scaling.jsonl 2> $O/scaling.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload audio --steps 20 > $O/audio_g1.json 2> $O/audio_g1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 4 --workload audio --steps 20 > $O/audio_g4.json 2> $O/audio_g4.err
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
for f in $O/bench_g1.json $O/bench_ref.json $O/scaling.jsonl $O/audio_g1.json $O/audio_g4.json; do
python - $f <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: continue
    print(sys.argv[1].split('/')[-1], d.get("n_gpus"), round(d["value"]), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), d.get("p99_batch_ms"))
PY
done
