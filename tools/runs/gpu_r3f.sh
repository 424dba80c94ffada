#!/bin/bash
# k_gemm_2sm: last-wave K split (parity, GEMM timings A/B, config-4 breakdown, full prefill)
OUT=gpurun_out/r3f
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in 0 1; do
  PCB_GEMM_2SM_SPLIT=$v timeout 300 python tools/kbench.py > $OUT/kbench_split$v.txt 2>&1
  PCB_GEMM_2SM_SPLIT=$v timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64_split$v.txt 2>&1
done
