#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then the ncu launch list, then one
# `--set full` capture of the scan kernel.  Outputs under gpurun_out/.
set -u
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
$CMD > gpurun_out/prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-scan_f32} -s 2 -c 1 \
    -o gpurun_out/prof_scan -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
