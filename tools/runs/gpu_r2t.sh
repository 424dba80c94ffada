#!/bin/bash
# chain: attention P in TMEM, 5 K/V stages (Q in the exchange buffer), O-phase residual prefetch
OUT=gpurun_out/r2t
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_serve.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
AB_VARIANTS=zero-copy timeout 300 python tools/chain_ab.py 3 > $OUT/chain_tl.txt 2>&1

for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/base/libpcb200.so timeout 300 python tools/ttft_ab.py base >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py new >> $OUT/ttft.txt 2>&1
done
