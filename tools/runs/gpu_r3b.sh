#!/bin/bash
OUT=gpurun_out/r3b
mkdir -p $OUT
for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_WT=0 timeout 300 python tools/ttft_ab.py wt0 >> $OUT/ttft.txt 2>&1
done
PCB_CHAIN_WT=0 AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl_wt0.txt 2>&1
PCB_LIB_PATH=ablib/prev/libpcb200.so AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl_prev.txt 2>&1
