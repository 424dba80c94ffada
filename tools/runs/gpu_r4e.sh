#!/bin/bash
# K/V streaming ceiling (persistent probe) + attention cycle accounting, configs[1] / configs[2]
OUT=gpurun_out/r4e
mkdir -p $OUT
timeout 120 tools/probe/kvstream > $OUT/kvstream.txt 2>&1
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c2.txt 2>&1
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c3.txt 2>&1
