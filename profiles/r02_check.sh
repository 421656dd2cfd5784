#!/bin/bash
# Full GPU suite + smoke + headline/flat bench lines + a re-rank sweep (bufs:dchunk:rows:smemKB).
# Outputs under gpurun_out/${TAG:-ck}/.
set -x
O=gpurun_out/${TAG:-ck}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 30 > $O/bench_g1.json 2> $O/bench_g1.err
timeout 300 python bench.py --workload flat --steps 20 > $O/bench_flat.json 2> $O/bench_flat.err
for cfg in ${CFGS:-}; do
  set -- ${cfg//:/ }
  VX_DEBUG_RERANK_BUFS=$1 VX_DEBUG_RERANK_DC=$2 VX_DEBUG_RERANK_ROWS=$3 VX_DEBUG_RERANK_SMEM_KB=$4 timeout 300 \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:rerank_kernel --csv \
    --log-file $O/rr_b$1_dc$2_r$3_s$4.csv python profiles/stage_kernels.py i8 1024 3 > $O/rr_b$1_dc$2_r$3_s$4.log 2>&1
done
if [ -n "${LAUNCHES:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --graphs 0 --no-cpu-baseline --no-e2e \
  > $O/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_flat.csv python bench.py --workload flat --graphs 0 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > $O/ncu_flat.log 2>&1
fi
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
