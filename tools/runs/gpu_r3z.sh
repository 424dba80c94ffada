#!/bin/bash
# config 4: micro-batch 64 vs 128 vs 256 (device time per request)
OUT=gpurun_out/r3z
mkdir -p $OUT
for mb in 64 128 256; do
  C4_N=256 timeout 600 python tools/c4_timing.py $mb 2>&1 | head -1 >> $OUT/c4.txt
done
