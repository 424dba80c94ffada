#!/bin/bash
# prefill attention: exponential emulation A/B + correctness at the default
OUT=gpurun_out/r2s
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "paired_prefill" -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for e in 0 2 3 4; do
PCB_PREFILL_EMU=$e python - >> $OUT/attn_ab.txt 2>&1 <<'PY'
import os, sys
sys.path.insert(0, "tools")
from kbench import bench
for n in (4160, 16512):
    us = bench("attn", n, 0, 32, iters=10)
    fl = 4 * 32 * 128 * n * (n + 1) / 2
    print(f"emu={os.environ['PCB_PREFILL_EMU']} n={n}: {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s")
PY
done
