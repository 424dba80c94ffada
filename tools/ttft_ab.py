"""Cached-TTFT A/B of library builds on one box: run once per build with PCB_LIB_PATH set
(the same box, back to back, removes box-to-box noise).

  PCB_LIB_PATH=ablib/base/libpcb200.so python tools/ttft_ab.py base
  python tools/ttft_ab.py new
Prints one line: label, median / min TTFT (ms) and device ms per request over N requests
of the configs[1] workload (7B shape, 4096 cached + 64 uncached).  AB_OPTS=k=v,... sets model
options (e.g. AB_OPTS=chain_group=1).
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

import paper_2311_04934_b200 as pcb  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "run"
n_req = int(os.environ.get("AB_N", "40"))
layers = int(os.environ.get("AB_LAYERS", "32"))
schema_text, prompts = bench.workload(int(os.environ.get("AB_CACHED", "4096")), int(os.environ.get("AB_UNC", "64")),
                                     int(os.environ.get("AB_MODS", "1")))  # configs[2]: 16384 128 3
m = pcb.Model(dict(bench.CFG_7B, n_layers=layers), dtype=pcb.BF16)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
parsed = [pcb.Prompt.parse(p) for p in prompts]
for kv in filter(None, os.environ.get("AB_OPTS", "").split(",")):  # model options, e.g. chain_group=1
    k, v = kv.split("=")
    m.set_option(k, int(v))
for i in range(5):
    pcb.serve(st, s, parsed[i % 4], max_new_tokens=1)
tt, dev = [], []
m.timer_start()
for i in range(n_req):
    r = pcb.serve(st, s, parsed[i % 4], max_new_tokens=1)
    tt.append(r.timings["ttft_us"] / 1e3)
    dev.append(r.timings["prefill_device_us"] / 1e3)
region = m.timer_stop()
print(f"{label:10s} ttft median {statistics.median(tt):.3f} min {min(tt):.3f}  device {statistics.median(dev):.3f}  "
      f"region/req {region / n_req:.3f} ms  token {r.output_tokens[0]}", flush=True)
