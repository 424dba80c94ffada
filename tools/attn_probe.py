import os, sys
sys.path.insert(0, "tools"); import kbench
for n, P in [(64, 4096), (1, 4096), (128, 16384)]:
    us = kbench.bench("attn", n, P, 32)
    print(f"attn n={n} P={P} splits={os.environ.get('PCB_ATTN_SPLITS','auto')} hm={os.environ.get('PCB_ATTN_HM_PROBE','0')}: {us:7.1f} us  {2*(n+P)*4096*2/us/1e3:6.0f} GB/s")
