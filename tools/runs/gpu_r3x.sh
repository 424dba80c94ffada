#!/bin/bash
# configs[1]'s model at full depth vs the reference fixture
OUT=gpurun_out/r3x
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -rs > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
