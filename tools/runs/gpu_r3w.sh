#!/bin/bash
# chain: LayerNorm-row helper out of line (fewer spills in the kernel body), A/B vs previous build
OUT=gpurun_out/r3w
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2 3; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py new >> $OUT/ttft.txt 2>&1
done
