"""Per-CTA phases of the last batched attention launch of a config-4 micro-batch (PCB_ATTN_TL):
prologue, first K/V latency, streaming, softmax tail and the gaps between consecutive CTAs.
  python tools/attn_phases_c4.py [micro_batch]"""
import ctypes as C
import os
import sys

os.environ["PCB_ATTN_TL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = pcb.lib()
L.pcb_debug_attn_tl.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
buf = np.zeros((8192, 8), np.uint64)
m = pcb.Model(dict(bench.CFG_7B, n_layers=int(os.environ.get("PROF_LAYERS", "4"))), dtype=pcb.BF16)
schema_text, prompts, _ = bench.workload_c4(64, 256, mb, 8, 64)
schema = pcb.Schema.parse(schema_text)
store = pcb.ModuleStore(m)
store.encode_schema(schema)
ps = [pcb.Prompt.parse(p) for p in prompts[:mb]]
for _ in range(2):
    pcb.serve_batch(store, schema, ps, micro_batch=mb)
n = C.c_int()
assert L.pcb_debug_attn_tl(buf.ctypes.data, 8192, C.byref(n)) == 0
t = buf[: n.value].astype(np.int64)
t0 = t[:, 0].min()
names = ["entry", "prologue", "first_kv", "last_pv", "softmax_done", "merge_done"]
print(f"CTAs {n.value}, kernel span {(t[:, 5].max() - t0) / 1e3:.1f} us")
for a, b in zip(range(0, 5), range(1, 6)):
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{names[a]:>12s} -> {names[b]:<12s} median {np.median(d):7.2f}  p90 {np.percentile(d, 90):7.2f} us")
cta = (t[:, 5] - t[:, 0]) / 1e3
print(f"CTA lifetime median {np.median(cta):.2f} us; sum of lifetimes / (148 SMs x span) = "
      f"{cta.sum() / (148 * (t[:, 5].max() - t0) / 1e3):.3f}")
