#!/bin/bash
# config 4: kernel-class breakdown of a 64-request micro-batch; ncu capture of one batched attention launch
OUT=gpurun_out/r3d
mkdir -p $OUT
timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_attn_tc -s 64 -c 1 -o $OUT/full_attn_batch python tools/c4_profile.py 64 > $OUT/ncu_attn.log 2>&1
