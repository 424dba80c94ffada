#!/bin/bash
# one-warp-per-row LayerNorm: parity + config-4 breakdown A/B
OUT=gpurun_out/r3i
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for v in 0 1; do PCB_LN_WARP=$v timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64_warp$v.txt 2>&1; done
