#!/bin/bash
# Headline stage at N = 1/2/4 GPUs and B = 1024 .. 4096 (per-batch fixed costs vs per-query).
set -x
O=gpurun_out/${TAG:-bs}
mkdir -p $O
NS="1 2 4" BATCHES="${BATCHES:-1024 2048 4096}" STEPS=20 timeout 2400 bash profiles/scaling.sh > $O/scaling.jsonl 2> $O/scaling.err
python - $O/scaling.jsonl <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    rp = d.get("root_phases_ms") or {}
    print(d["n_gpus"], d["config"]["batch"], round(d["value"]), round(d["ms_per_step"], 3), rp.get("detail"))
PY
