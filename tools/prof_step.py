"""One 7B-shape cached serve step for ncu captures (launch lists / --set full of one kernel).

Usage under gpurun:
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python tools/prof_step.py
Every kernel before the marker step is warm-up; the marker step is the last serve() call.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_04934_b200 as pcb  # noqa: E402

layers = int(os.environ.get("PROF_LAYERS", "32"))
cfg = dict(bench.CFG_7B, n_layers=layers)  # max_position 32768
schema_text, prompts = bench.workload(int(os.environ.get("PROF_CACHED", "4096")), int(os.environ.get("PROF_UNC", "64")),
                                     int(os.environ.get("PROF_MODS", "1")))  # configs[2]: 16384 128 3
m = pcb.Model(cfg, dtype=pcb.BF16)
m.set_option("zero_copy", int(os.environ.get("PROF_ZC", "1")))  # 0: requests assemble (copy) their cache
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
for i in range(int(os.environ.get("PROF_WARM", "2"))):
    pcb.serve(st, s, prompts[0], max_new_tokens=1)
m.sync()
r = pcb.serve(st, s, prompts[1], max_new_tokens=1)
print("ttft_ms", r.timings["ttft_us"] / 1e3, "launches", m.launches)
