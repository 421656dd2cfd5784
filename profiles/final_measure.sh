#!/bin/bash
# End-of-round measurement set (one 4-GPU box): bench N=1, reference arm, 2/4-GPU scaling,
# the bench launch list and one ncu --set full capture of the seeded s8 pair scan.
set -x
mkdir -p gpurun_out/fm
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fm/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fm/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/fm/bench_g1.json 2>gpurun_out/fm/bench_g1.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fm/bench_ref.json 2>gpurun_out/fm/bench_ref.err
NS="2 4" BATCHES="1024" bash profiles/scaling.sh > gpurun_out/fm/scaling.jsonl 2>gpurun_out/fm/scaling.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fm/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fm/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_tc2 -s 2 -c 1 -o gpurun_out/fm/scan_i8_seeded python profiles/stage_kernels.py i8 1024 2 1 > gpurun_out/fm/ncu_scan.log 2>&1
tail -2 gpurun_out/fm/pytest_gpu.log; tail -1 gpurun_out/fm/smoke.log; tail -1 gpurun_out/fm/bench_g1.json; tail -1 gpurun_out/fm/bench_ref.json | cut -c1-300; cat gpurun_out/fm/scaling.jsonl | cut -c1-200
