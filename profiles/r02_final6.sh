#!/bin/bash
# Final round-2 set (6) on one 4-GPU box: all GPU tests, smoke, bench N=1 (+ reference arm),
# scaling N = 1/2/4 on the same box, every BASELINE config at N=1, AudioQuery on 4 GPUs.
set -x
O=gpurun_out/${TAG:-f6}
mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > $O/bench_g1.json 2> $O/bench_g1.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
NS="1 2 4" BATCHES="1024" STEPS=30 timeout 1500 bash profiles/scaling.sh > $O/scaling.jsonl 2> $O/scaling.err
CUDA_VISIBLE_DEVICES=0 STEPS=20 SWEEP="1 16 64 256 1024 4096" timeout 1800 bash profiles/workloads.sh > $O/workloads.jsonl 2> $O/workloads.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --workload maxsim --tok-f32 --steps 20 > $O/maxsim_f32.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 \
  bench.py --gpus 4 --workload audio --steps 20 > $O/audio_g4.json 2> $O/audio_g4.err
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
