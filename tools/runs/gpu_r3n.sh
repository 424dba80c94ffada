#!/bin/bash
# persistent batched attention (attn_batch.cu): parity, config-4 A/B, phases
OUT=gpurun_out/r3n
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in 0 1; do PCB_ATTN_BATCH=$v timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64_batch$v.txt 2>&1; done
