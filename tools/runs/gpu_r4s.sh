#!/bin/bash
# ncu source-level capture of the chain at configs[2]'s shape (2 layers): where the softmax cycles go
OUT=gpurun_out/r4s
mkdir -p $OUT
PROF_LAYERS=2 PROF_WARM=1 PROF_CACHED=16384 PROF_UNC=128 PROF_MODS=3 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:k_chain -s 1 -c 1 -o $OUT/full_k_chain_c3 python tools/prof_step.py > $OUT/full_k_chain_c3.log 2>&1
ls -la $OUT
