#!/bin/bash
# multi-GPU parity + scaling 2/4 at B = 1024 (+ 1 GPU reference line)
set -x
O=gpurun_out/${TAG:-mg2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > $O/pytest_multi.log 2>&1
NS="${NS:-1 2 4}" BATCHES="1024" STEPS=20 timeout 1500 bash profiles/scaling.sh > $O/scaling.jsonl 2> $O/scaling.err
tail -2 $O/pytest_multi.log
python - $O/scaling.jsonl <<'PY'
import json, sys
for l in open(sys.argv[1]):
    d = json.loads(l)
    rp = d.get("root_phases_ms") or {}
    det = rp.get("detail") or {}
    print(d["n_gpus"], d["config"]["batch"], round(d["value"]), round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in det.items()}, d.get("cert_level2"), d.get("cert_fallbacks"))
PY
