O=gpurun_out/rt4; mkdir -p $O
VX_DEBUG_RERANK_TRACE=1 timeout 600 python bench.py --graphs 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/head.json 2> $O/head.err
VX_DEBUG_RERANK_TRACE=1 timeout 300 python bench.py --workload flat --graphs 0 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/flat.json 2> $O/flat.err
grep "rerank trace" $O/head.err | tail -4; grep "rerank trace" $O/flat.err | tail -2
