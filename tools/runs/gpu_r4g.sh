#!/bin/bash
# attention tail cycle counts (output/park loop, split merge), configs[1]
OUT=gpurun_out/r4g
mkdir -p $OUT
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c2.txt 2>&1
