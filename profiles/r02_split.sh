#!/bin/bash
# Split small-batch re-rank (S CTAs per query): GPU suite, re-rank phases at B = 1/16/64 with
# and without the split, search sweep points, headline and flat unchanged.
O=gpurun_out/${TAG:-sp}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for b in 1 16 64; do
  for e in VX_X=0 VX_DEBUG_NO_RERANK_SPLIT=1; do
    env $e timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b${b}_$e.json 2> $O/b${b}_$e.err
  done
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/head.json 2> $O/head.err
timeout 300 python bench.py --workload flat --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/flat.json 2> $O/flat.err
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'sp')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 4), {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if v})
    except Exception as e:
        print(f, 'ERR', e)
PY
