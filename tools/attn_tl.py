"""One attention launch with the CTA-0 timeline probe (PCB_ATTN_DBG): per KV block, when the
load was issued, landed, S ready, P arrived, PV issued."""
import os
import sys
os.environ["PCB_ATTN_DBG"] = "1"
sys.path.insert(0, "tools")
import kbench  # noqa: E402
for n, P in [(64, 4096), (1, 4096)]:
    print(f"== n={n} P={P}", flush=True)
    kbench.bench("attn", n, P, 32, iters=1)
