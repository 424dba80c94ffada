"""One GEMM shape through pcb_debug_kernel_bench (for ncu captures of the tensor-bound kernels).

  python tools/gemm_ncu.py M N K [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import bench  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 1
us = bench("gemm", M, N, K, iters=iters)
print(f"gemm M={M} N={N} K={K}: {us:.1f} us  {2 * M * N * K / us / 1e6:.1f} TFLOP/s")
