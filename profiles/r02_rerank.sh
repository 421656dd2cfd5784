#!/bin/bash
# Re-rank ring-mode sweep (rerank_kernel launch times under ncu, serialised/cold) at the headline
# stage (10M x 768 s8, B=1024, k=100), parity tests that exercise the re-rank, and the flat
# (configs[0]) launch list with graphs off.  Outputs under gpurun_out/${TAG:-rr}/.
set -x
O=gpurun_out/${TAG:-rr}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coarse.py tests/test_gpu_headline.py -m gpu -q -x > $O/pytest_rerank.log 2>&1
for cfg in "0 192 64" "3 128 64" "4 128 64" "3 192 64" "4 96 64" "3 128 32" "4 192 64"; do
  set -- $cfg
  VX_DEBUG_RERANK_STAGES=$1 VX_DEBUG_RERANK_DC=$2 VX_DEBUG_RERANK_ROWS=$3 timeout 300 \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:rerank_kernel --csv \
    --log-file $O/rr_s$1_dc$2_r$3.csv python profiles/stage_kernels.py i8 1024 3 > $O/rr_s$1_dc$2_r$3.log 2>&1
  VX_DEBUG_RERANK_STAGES=$1 VX_DEBUG_RERANK_DC=$2 VX_DEBUG_RERANK_ROWS=$3 timeout 300 \
    python profiles/stage_kernels.py i8 1024 6 > $O/stage_s$1_dc$2_r$3.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_flat.csv python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_flat.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_tc_kernel -s 3 -c 1 \
  -o $O/prof_flat_scan -f python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_flat_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_kernel -s 1 -c 1 \
  -o $O/prof_rerank -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_rerank_full.log 2>&1
tail -3 $O/pytest_rerank.log
for f in $O/stage_*.json; do echo "$f $(tail -1 $f)"; done
