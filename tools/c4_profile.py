"""Kernel-class breakdown of config 4 micro-batches (serve_batch): where a micro-batch's
device time goes (CUDA-event profile hooks of the library).
  python tools/c4_profile.py [micro_batch]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
m = pcb.Model(bench.CFG_7B, dtype=pcb.BF16)
schema_text, prompts, _ = bench.workload_c4(64, 256, 256, 8, 64)
schema = pcb.Schema.parse(schema_text)
store = pcb.ModuleStore(m)
store.encode_schema(schema)
ps = [pcb.Prompt.parse(p) for p in prompts[: 4 * mb]]
pcb.serve_batch(store, schema, ps[: 2 * mb], micro_batch=mb)
m.sync()
m.set_option("profile", 1)
m.profile()
m.timer_start()
pcb.serve_batch(store, schema, ps, micro_batch=mb)
dev = m.timer_stop()
prof = m.profile()
nb = len(ps) // mb
print(f"micro-batch {mb}: {dev / nb:.2f} ms per micro-batch (device, profiled)")
for k, v in prof.items():
    if v["ms"]:
        print(f"  {k:10s} {v['ms'] / nb:8.2f} ms  launches {v['launches'] / nb:6.1f}  "
              f"{v['bytes'] / (v['ms'] / 1e3) / 1e9:8.0f} GB/s  {v['flops'] / (v['ms'] / 1e3) / 1e12:7.1f} TFLOP/s")
