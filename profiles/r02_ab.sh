#!/bin/bash
# A/B on one box: programmatic dependent launch of the re-rank and graph event nodes (flat +
# headline, 1 GPU), then the 2-GPU headline with the finer root phases.
set -x
O=gpurun_out/${TAG:-ab}
mkdir -p $O
for v in "base:" "nopdl:VX_DEBUG_NO_PDL=1" "noev:VX_DEBUG_NO_GRAPH_EVENTS=1"; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 300 python bench.py --workload flat --steps 30 --no-cpu-baseline --no-e2e > $O/flat_$name.json 2>&1
  env $envs timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e > $O/stage_$name.json 2>&1
done
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus 2 --steps 20 --no-cpu-baseline > $O/stage_g2.json 2> $O/stage_g2.err
fi
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"] * 1e3, 1), d.get("last_batch_device_ms"), d.get("root_phases_ms"))
PY
done
