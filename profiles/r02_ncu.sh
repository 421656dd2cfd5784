#!/bin/bash
# Round-2 ncu captures (one kernel each, --set full) of the headline stage's kernels, plus the
# bench command's launch list.  Each after the same command ran clean without ncu.
set -x
O=gpurun_out/${TAG:-nc}
mkdir -p $O
timeout 300 python profiles/stage_kernels.py i8 1024 2 > $O/plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_tc2_kernel -s 2 -c 1 \
  -o $O/scan_tc2_i8 -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim_tc_kernel -s 0 -c 1 \
  -o $O/maxsim_tc -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_maxsim.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rerank_kernel -s 0 -c 1 \
  -o $O/rerank -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_rerank.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_tc_kernel -s 3 -c 1 \
  -o $O/scan_tc_flat -f python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_flat.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --graphs 0 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ls -la $O
