#!/bin/bash
# Small-batch re-rank staging (R = 128 chain rows, whole shared memory when B <= SMs): GPU
# suite, the search sweep, flat and AudioQuery.
O=gpurun_out/${TAG:-sr}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for b in 1 16 64 128 256; do
  timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b$b.json 2> $O/b$b.err
done
timeout 300 python bench.py --workload flat --steps 20 --warmup 5 --no-cpu-baseline > $O/flat.json 2> $O/flat.err
timeout 900 python bench.py --workload audio --steps 10 --no-cpu-baseline > $O/audio.json 2> $O/audio.err
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'sr')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 3), {k: round(v, 3) for k, v in (d.get('kernel_ms_per_step') or {}).items()})
    except Exception as e:
        print(f, 'ERR', e)
PY
