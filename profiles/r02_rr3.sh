#!/bin/bash
# Re-rank at three CTAs per SM (launch bounds 256 x 3: 80 registers, no spills) vs two:
# staging configurations under a 72 KB cap, headline bench, rerank kernel time per step.
O=gpurun_out/${TAG:-r3}; mkdir -p $O
for r in 1 2; do
  for cfg in "def:" "dc96:VX_DEBUG_RERANK_DC=96 VX_DEBUG_RERANK_SMEM_KB=72" "r32:VX_DEBUG_RERANK_SMEM_KB=72" "dc128:VX_DEBUG_RERANK_DC=128 VX_DEBUG_RERANK_SMEM_KB=72"; do
    n=${cfg%%:*}; e=${cfg#*:}
    env $e timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${n}_$r.json 2> $O/${n}_$r.err
  done
done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'r3')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), 'rerank', round(d['kernel_ms_per_step']['rerank'], 3), 'scan', round(d['kernel_ms_per_step']['scan'], 3))
    except Exception as e:
        print(f, 'ERR', e)
PY
