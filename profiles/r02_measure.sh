#!/bin/bash
# Round-2 measurement set on one B200: GPU tests, smoke, the default bench line, the other
# BASELINE configs, the reference arm, the bench launch list (ncu, cold/serialised) and one
# ncu --set full capture of a named kernel.  Outputs under gpurun_out/${TAG:-m}/.
# usage: TAG=m1 KREGEX=scan_tc2 bash profiles/r02_measure.sh
set -x
O=gpurun_out/${TAG:-m}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu.txt 2>&1
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
fi
timeout 600 python bench.py > $O/bench_g1.json 2> $O/bench_g1.err
if [ -z "${SKIP_WORKLOADS:-}" ]; then
  STEPS=20 SWEEP="${SWEEP:-1 16 64 256 1024 4096}" timeout 1500 bash profiles/workloads.sh > $O/workloads.jsonl 2> $O/workloads.err
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_launch.log 2>&1
if [ -n "${KREGEX:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${KSKIP:-2} -c 1 \
    -o $O/prof_${KNAME:-kernel} -f ${KCMD:-python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e} \
    > $O/ncu_full.log 2>&1
fi
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log; tail -1 $O/bench_g1.json | cut -c1-400
cut -c1-300 $O/workloads.jsonl; tail -1 $O/bench_ref.json | cut -c1-300
