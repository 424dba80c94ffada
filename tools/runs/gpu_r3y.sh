#!/bin/bash
# vectorised embedding gather and argmax: parity + TTFT A/B vs previous build + launch list
OUT=gpurun_out/r3y
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py new >> $OUT/ttft.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/prof_step.py > $OUT/launches.log 2>&1
