#!/bin/bash
# Query-conversion -> scan programmatic dependent launch, chunked small-batch head staging,
# 16-byte rank loads: merge microbench, flat timeline A/B, re-rank phases, GPU suite, benches.
O=gpurun_out/${TAG:-pd}; mkdir -p $O
./profiles/microbench/merge_bench > $O/merge_bench.log 2>&1
for e in "" VX_DEBUG_NO_SCAN_PDL=1; do echo "[$e]"; env $e ./profiles/microbench/flat_timeline 16; env $e ./profiles/microbench/flat_timeline 1; done > $O/flat_timeline.txt 2>&1
VX_DEBUG_RERANK_TRACE=1 timeout 600 python bench.py --graphs 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/head_trace.json 2> $O/head_trace.err
VX_DEBUG_RERANK_TRACE=1 timeout 300 python bench.py --workload flat --graphs 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/flat_trace.json 2> $O/flat_trace.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python bench.py --workload flat --steps 20 --warmup 5 --no-cpu-baseline > $O/flat.json 2> $O/flat.err
VX_DEBUG_NO_SCAN_PDL=1 timeout 300 python bench.py --workload flat --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/flat_nopdl.json 2> $O/flat_nopdl.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/head.json 2> $O/head.err
grep -A1 filter $O/merge_bench.log; cat $O/flat_timeline.txt; grep "rerank trace" $O/head_trace.err | tail -1; grep "rerank trace" $O/flat_trace.err | tail -1
tail -3 $O/pytest_gpu.log
python - <<'PY'
import json,os
O=os.environ.get('TAG','pd')
for f in ('flat','flat_nopdl','head'):
    try:
        d=json.loads(open(f'gpurun_out/{O}/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], d['ms_per_step'], d.get('kernel_ms_per_step'), d.get('e2e',{}).get('value'))
    except Exception as e: print(f, 'ERR', e)
PY
