#!/bin/bash
# The 10M-row scan at B = 1 ... 16 (one 16-row replicated tile config for all of them): scan
# kernel time per batch, with and without the selection (VX_DEBUG_TC_NOSELECT).
O=gpurun_out/${TAG:-bs}; mkdir -p $O
for b in 1 2 4 8 16; do
  timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b$b.json 2> $O/b$b.err
done
for b in 1 16; do
  VX_DEBUG_TC_NOSELECT=1 timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/nosel_b$b.json 2> $O/nosel_b$b.err
done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'bs')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()}, round(d['roofline'].get('kernel_sm_mhz', 0)))
    except Exception as e:
        print(f, 'ERR', e)
PY
