#!/bin/bash
# Batch sweep of the stage (device-resident inputs), one bench line per (scan, B).
# usage: SCANS="f32 tc" BATCHES="1 4 16 64" bash profiles/sweep.sh > gpurun_out/sweep.jsonl
for s in ${SCANS:-tc}; do
  for b in ${BATCHES:-16}; do
    python bench.py --steps ${STEPS:-10} --warmup 3 --batch $b --scan $s --no-cpu-baseline --no-e2e ${EXTRA:-} 2>/dev/null | tail -1
  done
done
