#!/bin/bash
OUT=gpurun_out/r3m
mkdir -p $OUT
timeout 600 python tools/attn_phases_c4.py 64 > $OUT/attn_phases_c4.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py -k full_depth -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
