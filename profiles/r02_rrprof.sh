#!/bin/bash
# re-rank A/B (fused merge vs separate) and one ncu --set full capture of the re-rank
set -x
O=gpurun_out/${TAG:-rp}
mkdir -p $O
for v in 0 1; do
  if [ $v = 1 ]; then export VX_DEBUG_NO_FUSE_MERGE=1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"rerank_kernel|merge_topk" --csv \
    --log-file $O/rr_nofuse$v.csv python profiles/stage_kernels.py i8 1024 3 > $O/rr_nofuse$v.log 2>&1
done
unset VX_DEBUG_NO_FUSE_MERGE
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rerank_kernel -s 1 -c 1 \
  -o $O/prof_rerank -f python profiles/stage_kernels.py i8 1024 2 > $O/ncu_rerank_full.log 2>&1
timeout 600 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -q -x > $O/pytest.log 2>&1
tail -2 $O/pytest.log
