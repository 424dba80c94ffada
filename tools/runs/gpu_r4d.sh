#!/bin/bash
# attention-phase tail events, configs[1] and configs[2]
OUT=gpurun_out/r4d
mkdir -p $OUT
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c2.txt 2>&1
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c3.txt 2>&1
