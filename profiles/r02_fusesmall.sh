#!/bin/bash
# Small batches: standalone merge launch vs the merge fused into the re-rank (the default now
# takes the standalone merge for B <= 64; VX_DEBUG_NO_FUSE_MERGE forces it everywhere).
O=gpurun_out/${TAG:-fs}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log
cd profiles/microbench; for i in 1 2; do ./flat_timeline 16; ./flat_timeline 1; done > ../../$O/timeline.txt 2>&1; cd ../..
cat $O/timeline.txt
for r in 1 2; do
  timeout 300 python bench.py --workload flat --steps 20 --warmup 5 --no-cpu-baseline > $O/flat_$r.json 2> $O/flat_$r.err
done
timeout 900 python bench.py --workload audio --steps 10 --no-cpu-baseline > $O/audio.json 2> $O/audio.err
for b in 16 64 128; do timeout 600 python bench.py --workload search --batch $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b$b.json 2> $O/b$b.err; done
python - <<'PY'
import json, os, glob
O = os.environ.get('TAG', 'fs')
for f in sorted(glob.glob(f'gpurun_out/{O}/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'], 4), (d.get('e2e') or {}).get('value'), {k: round(v, 4) for k, v in d['kernel_ms_per_step'].items() if v})
    except Exception as e:
        print(f, 'ERR', e)
PY
