"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libpcref_*.so (the reference compiled from
/root/reference/proj/core/src by oracle/Makefile) and records the reference's own
outputs on fixed inputs:

  host.json      PML ASTs / serializations / validation reports / layout plans /
                 resolved prompts for the 12-schema corpus, tests/common.hpp
                 random_case seeds 1..200 and random_ast seeds 0..299; config
                 canonical JSON + hashes; per_token_bytes KATs; synthetic_text.
  numeric.json   tiny-model (tests/common.hpp tiny_config) weight checksums, forward
                 logits of fixed token sequences (float32 bits, base64), and cached /
                 oracle / baseline serve results (tokens + first-token logits) for the
                 corpus and random_case seeds 1..40 (f32 model).
  store_ref.pcst a PCST v1 store written by the reference's ModuleStore::save.
"""
import base64
import glob
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import TINY, C1, Ref, RefError, RefModel  # noqa: E402

CORPUS = "/root/reference/proj/data/corpus"


def f32b64(a) -> str:
    return base64.b64encode(np.ascontiguousarray(a, np.float32).tobytes()).decode()


def err_or(fn):
    try:
        return fn()
    except RefError as e:
        return {"error": str(e).split(":")[0]}


def main():
    host = {"corpus": [], "random_case": [], "random_ast": [], "configs": [], "ptb": [], "synthetic": []}
    for path in sorted(glob.glob(f"{CORPUS}/*.pml")):
        if path.endswith(".prompt.pml"):
            continue
        st = open(path).read()
        pt = open(path[:-4] + ".prompt.pml").read()
        ast = Ref.parse_schema(st)
        host["corpus"].append({
            "name": os.path.basename(path), "schema_text": st, "prompt_text": pt,
            "schema_ast": ast, "schema_ast_raw": Ref.parse_schema(st, expand=False),
            "prompt_ast": Ref.parse_prompt(pt), "serialized": Ref.serialize_schema(ast),
            "prompt_serialized": Ref.serialize_prompt(Ref.parse_prompt(pt)),
            "plan": Ref.plan(st), "resolved": err_or(lambda: Ref.resolve(st, pt)),
            "validation": Ref.validate(pt, st)})
    for seed in range(1, 201):
        rc = Ref.random_case(seed)
        host["random_case"].append({
            "seed": seed, "schema": rc["schema"], "prompt": rc["prompt"], "plan": Ref.plan(rc["schema"]),
            "resolved": err_or(lambda: Ref.resolve(rc["schema"], rc["prompt"])),
            "validation": Ref.validate(rc["prompt"], rc["schema"]),
            "serialized": Ref.serialize_schema(rc["schema"]), "prompt_serialized": Ref.serialize_prompt(rc["prompt"])})
    for seed in range(300):
        a = Ref.random_ast(seed)
        text = Ref.serialize_schema(a)
        host["random_ast"].append({"seed": seed, "ast": a, "serialized": text,
                                   "reparsed": Ref.parse_schema(text, expand=False)})
    cfgs = [TINY, C1, dict(TINY, seed=43), dict(TINY, pos_encoding="alibi"), {"n_layers": 2},
            dict(n_layers=32, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
                 max_position=8192, bytes_per_element=2, seed=42)]
    for c in cfgs:
        host["configs"].append({"config": c, "canonical": Ref._str(Ref.lib().pcref_config_canonical(json.dumps(c).encode())),
                                "hash": str(Ref.config_hash(c))})
    for L, d, H, bpe in [(32, 4096, 32, 2), (40, 5120, 40, 2), (4, 256, 8, 4), (80, 8192, 64, 2)]:
        c = dict(n_layers=L, hidden=d, n_heads=H, head_dim=d // H, bytes_per_element=bpe)
        host["ptb"].append({"config": c, "bytes": Ref.per_token_bytes(c)})
    for n, seed in [(64, 1), (256, 1793), (4096, 28673)]:
        host["synthetic"].append({"n": n, "seed": seed, "text": Ref.synthetic_text(n, seed)})
    with open(os.path.join(HERE, "host.json"), "w") as f:
        json.dump(host, f, separators=(",", ":"))

    # ---- numeric (tiny f32 model) ----
    num = {"weights": {}, "forward": [], "serve": []}
    for name, cfg in (("tiny", TINY), ("c1", C1)):
        m = RefModel(cfg)
        num["weights"][name] = {t: str(m.weight_checksum(t)) for t in
                                ["embed", "unembed", "layer0.wq", "layer0.wk", "layer0.wv", "layer0.wo",
                                 "layer0.w1", "layer1.w2"]}
    m = RefModel(TINY)
    rng = np.random.default_rng(1234)
    for n, start in [(1, 0), (17, 0), (40, 100), (64, 4000)]:
        t = rng.integers(0, 259, n)
        p = np.arange(start, start + n)
        logits, kv = m.forward(t, p)
        num["forward"].append({"tokens": t.tolist(), "positions": p.tolist(), "logits": f32b64(logits[-1]),
                               "k0_row0": f32b64(kv.layer(0, 0)[0]), "v3_last": f32b64(kv.layer(3, 1)[-1])})
    cases = []
    for path in sorted(glob.glob(f"{CORPUS}/*.pml")):
        if not path.endswith(".prompt.pml"):
            cases.append(("corpus:" + os.path.basename(path), open(path).read(),
                          open(path[:-4] + ".prompt.pml").read()))
    for seed in range(1, 41):
        rc = Ref.random_case(seed)
        cases.append((f"random_case:{seed}", rc["schema"], rc["prompt"]))
    for name, s, pr in cases:
        entry = {"name": name}
        for mode in ("cached", "oracle", "baseline"):
            r = m.serve(s, pr, max_new=8, mode=mode)
            entry[mode] = {"tokens": r["output_tokens"], "logits": f32b64(r["first_token_logits"]),
                           "report": r["cache_report"]}
        num["serve"].append(entry)
    with open(os.path.join(HERE, "numeric.json"), "w") as f:
        json.dump(num, f, separators=(",", ":"))

    demo = ('<schema name="store"><module name="x">persistent text</module>'
            '<module name="y">more <param name="p" len="2"/></module></schema>')
    m.store_save(demo, os.path.join(HERE, "store_ref.pcst"), scaffold=["x", "y"])
    print("wrote", os.listdir(HERE))


if __name__ == "__main__":
    main()
