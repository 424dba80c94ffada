import json, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2311_04934_b200 as pcb
hg = json.load(open("/root/repo/tests/golden/host.json"))
ng = json.load(open("/root/repo/tests/golden/numeric.json"))
def inputs(name):
    if name.startswith("corpus:"):
        c = next(c for c in hg["corpus"] if c["name"] == name[7:])
        return pcb.Schema.parse(c["schema_text"]), pcb.Prompt.parse(c["prompt_text"])
    seed = int(name.split(":")[1])
    c = next(c for c in hg["random_case"] if c["seed"] == seed)
    return pcb.Schema.from_ast(c["schema"]), pcb.Prompt.from_ast(c["prompt"])
cfg = dict(n_layers=2, n_heads=2, head_dim=128, hidden=256, vocab_size=512, pos_encoding="rope",
           max_position=8192, bytes_per_element=2, seed=42)
m = pcb.Model(cfg, dtype=pcb.BF16)
skip_oracle = os.environ.get("NO_ORACLE") == "1"
for case in ng["serve"][:20]:
    schema, prompt = inputs(case["name"])
    st = pcb.ModuleStore(m)
    st.encode_schema(schema)
    res = []
    for zc in (1, 0):
        m.set_option("zero_copy", zc)
        r = pcb.serve(st, schema, prompt, 8)
        res.append((int(np.isnan(r.first_token_logits).sum()), r.timings["assemble_us"] < 1, r.cache_report["cached_token_count"], r.cache_report["uncached_token_count"]))
    m.set_option("zero_copy", 1)
    if not skip_oracle:
        pcb.oracle_serve(m, schema, prompt, 8)
    print(case["name"], res)
