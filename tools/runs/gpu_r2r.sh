#!/bin/bash
# paired-tile prefill attention: correctness, then kernel timing A/B
OUT=gpurun_out/r2r
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -k "paired_prefill or tc_path_vs_simt" tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
python - > $OUT/attn_ab.txt 2>&1 <<'PY'
import os, sys
sys.path.insert(0, "tools")
from kbench import bench
for n in (4160, 4096, 2048, 16512):
    us = bench("attn", n, 0, 32, iters=10)
    fl = 4 * 32 * 128 * n * (n + 1) / 2
    print(f"pair  n={n}: {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s")
PY
PCB_ATTN_PAIR=0 python - >> $OUT/attn_ab.txt 2>&1 <<'PY'
import os, sys
sys.path.insert(0, "tools")
from kbench import bench
for n in (4160, 4096, 2048):
    us = bench("attn", n, 0, 32, iters=10)
    fl = 4 * 32 * 128 * n * (n + 1) / 2
    print(f"single n={n}: {us:8.1f} us {fl / us / 1e6:7.1f} TFLOP/s")
PY
