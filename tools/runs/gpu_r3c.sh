#!/bin/bash
OUT=gpurun_out/r3c
mkdir -p $OUT
for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_WT=0 timeout 300 python tools/ttft_ab.py wt0 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_WT=0 PCB_CHAIN_XREL=0 timeout 300 python tools/ttft_ab.py wt0_x0 >> $OUT/ttft.txt 2>&1
done
