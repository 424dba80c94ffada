#!/bin/bash
# launch-boundary probes between chain launches (configs[1])
OUT=gpurun_out/r4l
mkdir -p $OUT
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c2.txt 2>&1
