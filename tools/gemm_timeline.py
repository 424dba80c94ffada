"""GEMM timeline of one 7B-shape cached request (PCB_GEMM_PROBE=1 is set here).

Per GEMM launch: span from the first CTA entry to the last CTA exit, the ramp (entry ->
first weight stage landed), the streaming window (first -> last stage), the tail (last
stage -> CTA done) and the gap to the next GEMM's first CTA entry; medians over CTAs.
"""
import ctypes as C
import os
import statistics
import sys

os.environ["PCB_GEMM_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import numpy as np  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

L = pcb.lib()
L.pcb_debug_gemm_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
MAXL = 1024
shapes = np.zeros((MAXL, 4), np.int64)
times = np.zeros((MAXL, 160, 4), np.uint64)


def dump():
    n = C.c_int()
    rc = L.pcb_debug_gemm_probe(shapes.ctypes.data, times.ctypes.data, MAXL, C.byref(n))
    assert rc == 0, L.pcb_last_error()
    return n.value


layers = int(os.environ.get("PROF_LAYERS", "32"))
cfg = dict(bench.CFG_7B, n_layers=layers)
schema_text, prompts = bench.workload(4096, 64, 1)
m = pcb.Model(cfg, dtype=pcb.BF16)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
for i in range(2):
    pcb.serve(st, s, prompts[0], max_new_tokens=1)
m.sync()
dump()
r = pcb.serve(st, s, prompts[1], max_new_tokens=1)
n = dump()
print(f"ttft_ms {r.timings['ttft_us'] / 1e3:.3f}  gemm launches {n}")
t0 = None
rows = []
for i in range(n):
    M, N, K, ctas = (int(x) for x in shapes[i])
    t = times[i, :ctas].astype(np.int64)
    if t0 is None:
        t0 = t[:, 0].min()
    ent, first, last, done = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
    rows.append(dict(M=M, N=N, K=K, start=(ent.min() - t0) / 1e3, end=(done.max() - t0) / 1e3,
                     span=(done.max() - ent.min()) / 1e3,
                     entry_spread=(ent.max() - ent.min()) / 1e3,
                     ramp=statistics.median((first - ent).tolist()) / 1e3,
                     stream=statistics.median((last - first).tolist()) / 1e3,
                     tail=statistics.median((done - last).tolist()) / 1e3,
                     tail_max=(done.max() - last.max()) / 1e3,
                     gbs=N * K * 2 / ((done.max() - ent.min())) if done.max() > ent.min() else 0))
tot = {}
for i, r_ in enumerate(rows):
    gap = rows[i + 1]["start"] - r_["end"] if i + 1 < len(rows) else 0.0
    r_["gap_next"] = gap
    key = (r_["N"], r_["K"])
    tot.setdefault(key, []).append(r_)
    if i < 12 or i >= n - 3:
        print(f"{i:3d} M={r_['M']:5d} N={r_['N']:5d} K={r_['K']:5d} start {r_['start']:9.1f} span {r_['span']:6.1f} "
              f"entry_spread {r_['entry_spread']:5.1f} ramp {r_['ramp']:5.1f} stream {r_['stream']:6.1f} "
              f"tail {r_['tail']:5.1f} (max {r_['tail_max']:5.1f}) gap_next {gap:6.1f} us  {r_['gbs']:6.0f} GB/s")
print("per shape (median): span / ramp / stream / tail / gap_next us, GB/s over span")
for key, rs in tot.items():
    f = lambda k: statistics.median([x[k] for x in rs])  # noqa: E731
    print(f"N={key[0]:5d} K={key[1]:5d} x{len(rs):3d}: span {f('span'):6.1f} ramp {f('ramp'):5.1f} "
          f"stream {f('stream'):6.1f} tail {f('tail'):5.1f} gap {f('gap_next'):6.1f}  {f('gbs'):6.0f} GB/s "
          f"(stream-only {key[0] * key[1] * 2 / (f('stream') * 1e3):6.0f} GB/s)")
span_all = rows[-1]["end"] - rows[0]["start"]
print(f"first GEMM entry -> last GEMM done: {span_all:.1f} us; sum of GEMM spans {sum(x['span'] for x in rows):.1f} us")
