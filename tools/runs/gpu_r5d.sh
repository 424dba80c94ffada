#!/bin/bash
# cooperative launch attribute on the clustered chain launch (PCB_CHAIN_COOP=1): parity tests with it on,
# then a same-box TTFT A/B (off / on, twice)
OUT=gpurun_out/r5d
mkdir -p $OUT
PCB_CHAIN_COOP=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest_coop.log 2>&1; echo rc=$? >> $OUT/pytest_coop.log
for r in 1 2; do
timeout 300 python tools/ttft_ab.py off >> $OUT/ttft.txt 2>&1
PCB_CHAIN_COOP=1 timeout 300 python tools/ttft_ab.py coop >> $OUT/ttft.txt 2>&1
done
