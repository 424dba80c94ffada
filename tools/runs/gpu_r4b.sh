#!/bin/bash
# configs[2] (16K cached + 128 uncached) chain timeline
OUT=gpurun_out/r4b
mkdir -p $OUT
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c3.txt 2>&1
