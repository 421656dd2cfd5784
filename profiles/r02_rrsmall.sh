#!/bin/bash
# Small-batch re-rank (10M x 768 s8, k' = 1024, one CTA per query): deeper staging and L2
# prefetch when a CTA has its SM to itself.
O=gpurun_out/${TAG:-rs}; mkdir -p $O
for b in 1 16; do
  for cfg in "def:" "nb4:VX_DEBUG_RERANK_BUFS=4 VX_DEBUG_RERANK_SMEM_KB=220" "pf4:VX_DEBUG_RERANK_PF=4" "pf8:VX_DEBUG_RERANK_PF=8" "nb4pf4:VX_DEBUG_RERANK_BUFS=4 VX_DEBUG_RERANK_SMEM_KB=220 VX_DEBUG_RERANK_PF=4"; do
    n=${cfg%%:*}; e=${cfg#*:}
    env $e timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${n}_b$b.json 2> $O/${n}_b$b.err
  done
done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'rs')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), 'rerank', round(d['kernel_ms_per_step']['rerank'], 4), 'scan', round(d['kernel_ms_per_step']['scan'], 3))
    except Exception as e:
        print(f, 'ERR', e)
PY
