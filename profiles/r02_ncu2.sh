#!/bin/bash
# ncu at the final code: the re-rank (ranked selection) and the flat re-rank --set full, and
# the launch lists of the headline and flat bench commands (each command ran clean first).
set -x
O=gpurun_out/${TAG:-nc2}
mkdir -p $O
timeout 300 python profiles/stage_kernels.py i8 1024 2 > $O/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rerank_kernel -s 0 -c 1 \
  -o $O/rerank -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_rerank.log 2>&1
timeout 300 python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/flat_plain.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_kernel -s 3 -c 1 \
  -o $O/rerank_flat -f python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_rerank_flat.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/head_plain.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_flat.csv python bench.py --workload flat --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_flat.log 2>&1
ls -la $O
