#!/bin/bash
# One bench line per BASELINE.json config (configs[0..4]); outputs JSON lines on stdout.
# usage: bash profiles/workloads.sh > gpurun_out/workloads.jsonl
S=${STEPS:-20}
python bench.py --steps $S --warmup 3 2>/dev/null | tail -1                       # configs[2] headline
python bench.py --steps $S --warmup 3 --workload flat 2>/dev/null | tail -1       # configs[0]
python bench.py --steps $S --warmup 3 --workload maxsim 2>/dev/null | tail -1     # configs[1]
python bench.py --steps $S --warmup 3 --workload audio 2>/dev/null | tail -1      # configs[3]
for b in ${SWEEP:-1 16 64 256 1024 4096}; do                                      # configs[4]
  python bench.py --steps ${SWEEP_STEPS:-5} --warmup 3 --workload search --batch $b --no-cpu-baseline 2>/dev/null | tail -1
done
