import os, sys
sys.path.insert(0, "tools"); import kbench
for M in (1, 16, 32, 64):
    us = kbench.bench("gemm", M, 12288, 4096)
    print(f"qkv M={M:3d} ctas={os.environ.get('PCB_GEMM_CTAS','all')}: {us:7.1f} us {12288*4096*2/us/1e3:6.0f} GB/s")
