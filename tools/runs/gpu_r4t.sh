#!/bin/bash
# chain softmax exponentials in groups of 8 with packed FFMA2 / FADD2
OUT=gpurun_out/r4t
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev_c2 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py new_c2 >> $OUT/ttft.txt 2>&1
done
PCB_CHAIN_PROBE=0 AB_CACHED=16384 AB_UNC=128 AB_MODS=3 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev_c3 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 AB_CACHED=16384 AB_UNC=128 AB_MODS=3 timeout 300 python tools/ttft_ab.py new_c3 >> $OUT/ttft.txt 2>&1
AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c2.txt 2>&1
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 AB_VARIANTS=zero-copy timeout 600 python tools/chain_ab.py 2 > $OUT/chain_tl_c3.txt 2>&1
