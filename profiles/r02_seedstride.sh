#!/bin/bash
# Seed sample stride A/B at the headline (10M x 768 s8 B=1024): sample-pass cost vs the full
# pass's admission work; certificate levels must stay at zero re-scans.
O=gpurun_out/${TAG:-ss}; mkdir -p $O
for r in 1 2; do for s in 64 128 96; do
  VX_DEBUG_SEED_STRIDE=$s timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/s${s}_$r.json 2> $O/s${s}_$r.err
done; done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'ss')
for f in sorted(glob.glob(f'gpurun_out/{O}/s*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()}, d.get('cert_level2'), d.get('cert_fallbacks'))
    except Exception as e:
        print(f, 'ERR', e)
PY
