#!/bin/bash
# Multi-GPU set (one box with >= 4 GPUs): multi-GPU parity tests, strong scaling 1/2/4 of the
# headline stage, the reference arm at N=4 (rank 0 only), AudioQuery with 4 replica members.
set -x
O=gpurun_out/${TAG:-mg}
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x > $O/pytest_multi.log 2>&1
NS="1 2 4" BATCHES="1024" STEPS=30 timeout 1500 bash profiles/scaling.sh > $O/scaling.jsonl 2> $O/scaling.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --workload audio --steps 20 > $O/audio_g4.json 2> $O/audio_g4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 4 --impl reference --steps 3 --warmup 3 > $O/ref_g4.json 2> $O/ref_g4.err
tail -3 $O/pytest_multi.log; cut -c1-250 $O/scaling.jsonl; tail -1 $O/audio_g4.json | cut -c1-250
