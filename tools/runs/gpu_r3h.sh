#!/bin/bash
# vectorised LayerNorm stores: parity + config-4 breakdown
OUT=gpurun_out/r3h
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python tools/c4_profile.py 64 > $OUT/c4prof64.txt 2>&1
