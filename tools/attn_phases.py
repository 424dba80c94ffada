"""Per-CTA phases of the last attention launch of one 7B cached request (PCB_ATTN_TL):
entry skew, prologue, first K/V latency, streaming, softmax tail, cluster merge."""
import ctypes as C
import os
import statistics
import sys

os.environ["PCB_ATTN_TL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

L = pcb.lib()
L.pcb_debug_attn_tl.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int)]
buf = np.zeros((8192, 8), np.uint64)
m = pcb.Model(dict(bench.CFG_7B, n_layers=int(os.environ.get("PROF_LAYERS", "32"))), dtype=pcb.BF16)
schema_text, prompts = bench.workload(4096, 64, 1)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
for i in range(3):
    pcb.serve(st, s, prompts[i % 2], max_new_tokens=1)
n = C.c_int()
assert L.pcb_debug_attn_tl(buf.ctypes.data, 8192, C.byref(n)) == 0
t = buf[: n.value].astype(np.int64)
t0 = t[:, 0].min()
names = ["entry", "prologue", "first_kv", "last_pv", "softmax_done", "merge_done"]
print(f"CTAs {n.value}")
print("entry skew (max-min) us", (t[:, 0].max() - t0) / 1e3)
for a, b in zip(range(0, 5), range(1, 6)):
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{names[a]:>12s} -> {names[b]:<12s} median {np.median(d):7.2f}  max {d.max():7.2f} us")
print("kernel span (first entry -> last merge_done) us", (t[:, 5].max() - t0) / 1e3)
