#!/bin/bash
# persistent batched attention: unprofiled config-4 device time per micro-batch, A/B x3
OUT=gpurun_out/r3o
mkdir -p $OUT
for r in 1 2 3; do for v in 0 1; do
  echo "== batch=$v" >> $OUT/c4.txt
  PCB_ATTN_BATCH=$v C4_N=256 timeout 600 python tools/c4_timing.py 64 2>&1 | head -1 >> $OUT/c4.txt
done; done
