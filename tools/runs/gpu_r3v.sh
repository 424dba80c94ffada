#!/bin/bash
# chain softmax: next block's S loaded under the current block's math (A/B vs previous build)
OUT=gpurun_out/r3v
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_SPRE=0 timeout 300 python tools/ttft_ab.py spre0 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 PCB_CHAIN_SPRE=1 timeout 300 python tools/ttft_ab.py spre1 >> $OUT/ttft.txt 2>&1
done
