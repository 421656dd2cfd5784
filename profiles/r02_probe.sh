#!/bin/bash
# Probes: random-row gather ceiling (gather_bench) and the small-batch scan vs shard length
# (tiles per CTA).  Outputs under gpurun_out/${TAG:-pr}/.
set -x
O=gpurun_out/${TAG:-pr}
mkdir -p $O
(cd profiles/microbench && timeout 300 ./gather_bench 720) > $O/gather_bench.log 2>&1
for n in 37888 75776 100000 113664 151552 227328 303104; do
  timeout 300 python bench.py --workload flat --n-docs $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $O/flat_n.jsonl
done
for b in 1 2 4 8 16 32; do
  timeout 300 python bench.py --workload flat --batch $b --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $O/flat_b.jsonl
done
cat $O/gather_bench.log
