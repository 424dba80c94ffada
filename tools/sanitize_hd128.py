"""Small hd128 workload for compute-sanitizer: the chain attention phase (zero-copy segments and
the assembled copy), a batched micro-batch, the paired prefill attention and a 320-row prefill.

  compute-sanitizer --tool memcheck python tools/sanitize_hd128.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2311_04934_b200 as pcb  # noqa: E402

cfg = dict(n_layers=2, n_heads=2, head_dim=128, hidden=256, vocab_size=512, pos_encoding="rope",
           max_position=8192, bytes_per_element=2, seed=42)
m = pcb.Model(cfg, dtype=pcb.BF16)
schema_text, prompts = bench.workload(300, 40, 2)
s = pcb.Schema.parse(schema_text)
st = pcb.ModuleStore(m)
st.encode_schema(s)
for zc in (1, 0):
    m.set_option("zero_copy", zc)
    r = pcb.serve(st, s, prompts[0], max_new_tokens=3)
    print("serve zc", zc, r.output_tokens)
res = pcb.serve_batch(st, s, prompts[:4], micro_batch=4)
print("batch", [x.output_tokens for x in res])
m.set_option("attn_pair", 2)
t = np.arange(300) % 250
logits, _ = m.forward(t, np.arange(300))
print("prefill pair", int(np.argmax(logits[-1])))
