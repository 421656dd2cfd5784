#!/bin/bash
# re-rank L2-prefetch distance sweep (bufs:dchunk:rows:pf), fused merge on/off
set -x
O=gpurun_out/${TAG:-pf}
mkdir -p $O
for cfg in ${CFGS:-2:192:64:0 2:192:64:2}; do
  set -- ${cfg//:/ }
  VX_DEBUG_RERANK_BUFS=$1 VX_DEBUG_RERANK_DC=$2 VX_DEBUG_RERANK_ROWS=$3 VX_DEBUG_RERANK_PF=$4 timeout 300 \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"rerank_kernel|merge_topk" --csv \
    --log-file $O/rr_$1_$2_$3_$4.csv python profiles/stage_kernels.py i8 1024 3 > $O/rr_$1_$2_$3_$4.log 2>&1
done
