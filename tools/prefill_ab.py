"""Full-prefill TTFT of configs[1]'s prompt (4160 tokens, use_cache=False) in one process, for
same-box A/B of the prefill kernels (PCB_LIB_PATH selects the library).

  python tools/prefill_ab.py <label>
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2311_04934_b200 as pcb  # noqa: E402

cached, unc, mods = (int(os.environ.get(k, d)) for k, d in (("AB_CACHED", "4096"), ("AB_UNC", "64"), ("AB_MODS", "1")))
schema_text, prompts = bench.workload(cached, unc, mods)
m = pcb.Model(dict(bench.CFG_7B), dtype=pcb.BF16)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
p = pcb.Prompt.parse(prompts[0])
for _ in range(2):
    pcb.serve(st, s, p, max_new_tokens=1, use_cache=False)
t = [pcb.serve(st, s, p, max_new_tokens=1, use_cache=False).timings["ttft_us"] / 1e3 for _ in range(5)]
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'run':10s} full prefill median {statistics.median(t):.2f} min {min(t):.2f} ms")
