#!/bin/bash
# Re-rank ring mode (warp-uniform waits) sweep at the headline stage; flat workload with the
# clean-L2 flush.  Outputs under gpurun_out/${TAG:-rr2}/.
set -x
O=gpurun_out/${TAG:-rr2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coarse.py tests/test_gpu_headline.py -m gpu -q -x > $O/pytest_rerank.log 2>&1
# CFGS: space-separated bufs:dchunk:rows triples (bufs 0 = the default)
for cfg in ${CFGS:-0:192:64 3:256:64}; do
  set -- ${cfg//:/ }
  VX_DEBUG_RERANK_BUFS=$1 VX_DEBUG_RERANK_DC=$2 VX_DEBUG_RERANK_ROWS=$3 timeout 300 \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:rerank_kernel --csv \
    --log-file $O/rr_s$1_dc$2_r$3.csv python profiles/stage_kernels.py i8 1024 3 > $O/rr_s$1_dc$2_r$3.log 2>&1
done
timeout 300 python bench.py --workload flat --steps 20 --warmup 3 > $O/bench_flat.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_flat.csv python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_flat.log 2>&1
tail -3 $O/pytest_rerank.log
tail -1 $O/bench_flat.json | cut -c1-300
