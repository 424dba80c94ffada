#!/bin/bash
OUT=gpurun_out/r3t
mkdir -p $OUT
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 --error-exitcode 9 python tools/sanitize_hd128.py > $OUT/san_synccheck.log 2>&1; echo "rc=$?" >> $OUT/san_synccheck.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do
PCB_CHAIN_PROBE=0 PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/ttft_ab.py prev >> $OUT/ttft.txt 2>&1
PCB_CHAIN_PROBE=0 timeout 300 python tools/ttft_ab.py new >> $OUT/ttft.txt 2>&1
done
