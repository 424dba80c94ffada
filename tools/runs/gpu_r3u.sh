#!/bin/bash
# chain exchange-buffer signal: per-thread release arrivals vs one fence + relaxed arrivals
OUT=gpurun_out/r3u
mkdir -p $OUT
PCB_CHAIN_PBREL=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do
PCB_CHAIN_PROBE=0 PCB_CHAIN_PBREL=0 timeout 300 python tools/ttft_ab.py rel >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_PBREL=1 timeout 300 python tools/ttft_ab.py fence+relaxed >> $OUT/ttft.txt 2>&1
done
