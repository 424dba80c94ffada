#!/bin/bash
# prefill attention: P store chunk 16 vs 64 keys (A/B), parity of the pair kernel
OUT=gpurun_out/r3k
mkdir -p $OUT
for ch in 16 64; do
PCB_PREFILL_CH=$ch timeout 600 python -m pytest tests/test_gpu_kernels.py -k paired -x -q -p no:cacheprovider > $OUT/pytest_ch$ch.log 2>&1; echo rc=$? >> $OUT/pytest_ch$ch.log
for r in 1 2; do
PCB_PREFILL_CH=$ch python - >> $OUT/attn_ab.txt 2>&1 <<'PY'
import os, sys
sys.path.insert(0, "tools")
from kbench import bench
for n in (4160, 16512):
    us = bench("attn", n, 0, 32, iters=10)
    fl = 4 * 32 * 128 * n * (n + 1) / 2
    print(f"ch={os.environ['PCB_PREFILL_CH']} n={n}: {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s")
PY
done
done
