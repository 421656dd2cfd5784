#!/bin/bash
# Strong-scaling sweep of the headline stage: one bench line per (batch, N); run on a box
# with >= max(NS) GPUs.  usage: NS="1 2 4" BATCHES="256 1024" bash profiles/scaling.sh
for b in ${BATCHES:-256 1024}; do
  for n in ${NS:-1 2 4}; do
    if [ "$n" = 1 ]; then
      timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --batch $b --no-cpu-baseline ${EXTRA:-} 2>/dev/null | tail -1
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29400 + n + b / 64)) bench.py --gpus $n --steps ${STEPS:-20} --warmup 3 --batch $b \
        --no-cpu-baseline ${EXTRA:-} 2>/dev/null | tail -1
    fi
  done
done
