#!/bin/bash
# chain launches spanning several layers (attention at any phase): parity, A/B, timeline
OUT=gpurun_out/r2w
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_serve.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/base/libpcb200.so timeout 300 python tools/ttft_ab.py base >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 AB_OPTS=chain_group=1 timeout 300 python tools/ttft_ab.py group1 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 AB_OPTS=chain_group=4 timeout 300 python tools/ttft_ab.py group4 >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py group9 >> $OUT/ttft.txt 2>&1
done
AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 2 > $OUT/chain_tl.txt 2>&1
