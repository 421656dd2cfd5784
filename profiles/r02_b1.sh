#!/bin/bash
# B = 1 search at 10M x 768: the full pass's time with and without the sample pass's
# programmatic launch, and unseeded, alternating on one box.
O=gpurun_out/${TAG:-b1}; mkdir -p $O
for r in 1 2; do
  for cfg in "def:" "nopdl:VX_DEBUG_NO_SCAN_PDL=1" "noseed:VX_DEBUG_NO_SEED=1"; do
    n=${cfg%%:*}; e=${cfg#*:}
    env $e timeout 600 python bench.py --workload search --batch 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/${n}_$r.json 2> $O/${n}_$r.err
  done
done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'b1')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()}, d['last_step_timeline_us'])
    except Exception as e:
        print(f, 'ERR', e)
PY
