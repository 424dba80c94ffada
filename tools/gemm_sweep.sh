#!/bin/bash
# splits x pipeline-depth sweep of the M=64 GEMM shapes (tuning aid)
for deep in 0 1; do for sp in 1 2 4 8; do
  echo "deep=$deep splits=$sp"
  PCB_GEMM_DEEP=$deep PCB_GEMM_SPLITS=$sp python - <<'PY'
import sys; sys.path.insert(0, "tools"); import kbench
for M, N, K, nm in [(64, 12288, 4096, "qkv"), (64, 4096, 4096, "o"), (64, 16384, 4096, "w1"), (64, 4096, 16384, "w2"), (1, 32000, 4096, "unembed")]:
    try:
        us = kbench.bench("gemm", M, N, K)
        print(f"  {nm:8s} {us:7.1f} us {(N*K*2)/us/1e3:6.0f} GB/s")
    except Exception as e:
        print("  ", nm, "ERR", e)
PY
done; done
