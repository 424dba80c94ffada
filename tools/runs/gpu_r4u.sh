#!/bin/bash
# paired prefill attention: 12 warps with setmaxnreg budgets (softmax warpgroups at 216 registers)
OUT=gpurun_out/r4u
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for r in 1 2; do
PCB_LIB_PATH=ablib/prev/libpcb200.so timeout 300 python tools/prefill_ab.py prev >> $OUT/prefill.txt 2>&1
timeout 300 python tools/prefill_ab.py new >> $OUT/prefill.txt 2>&1
done
PCB_LIB_PATH=ablib/prev/libpcb200.so AB_CACHED=16384 AB_UNC=128 AB_MODS=3 timeout 600 python tools/prefill_ab.py prev_c3 >> $OUT/prefill.txt 2>&1
AB_CACHED=16384 AB_UNC=128 AB_MODS=3 timeout 600 python tools/prefill_ab.py new_c3 >> $OUT/prefill.txt 2>&1
