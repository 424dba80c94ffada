"""Reference outputs for the benchmarked shapes (round-2 parity fixtures).

Run here, where /root/reference exists:  python tests/golden/make_golden_parity.py
Every number comes from the UNMODIFIED reference (oracle/_ref, built by oracle/Makefile from
/root/reference/proj/core/src) on the inputs of tests/parity_cases.py:

  parity.json      c1        configs[0] as BASELINE.json states it (68-token system module +
                             512-token document + 32 uncached, fp32): cached / baseline / oracle
                             serve, 32 greedy tokens + first-token logits (engine.cpp:187-334)
                   h128      the golden serve corpus (12 corpus schemas + random_case 1..40) on a
                             head-dim-128 model: cached serve, 8 tokens + first-token logits
                   long      configs[2] shape at d 256 (3 modules, 16,384 cached + 128 uncached):
                             cached serve, 4 tokens + logits; sampled K/V rows of module doc1
  parity_w7b.npz   Llama-2-7B width (d 4096, H 32, V 32000), 2 layers: Model::forward of each
                   request's 64 suffix tokens over synthetic bf16-exact module K/V (model.cpp:
                   304-443, logits of rows 0 and 63) and a 320-row prefill without past (logits
                   of the first/last rows, K/V rows 0/160/319 of layer 1)

The 7B-width forwards take minutes on one core each; they run in parallel processes.
"""
import base64
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref, RefModel, ref_kv  # noqa: E402
from tests import parity_cases as pc  # noqa: E402


def b64(a) -> str:
    return base64.b64encode(np.ascontiguousarray(a, np.float32).tobytes()).decode()


def serve_entry(r):
    return {"tokens": r["output_tokens"], "logits": b64(r["first_token_logits"]), "report": r["cache_report"]}


def job_c1(_):
    m = RefModel(pc.C1)
    s, p = pc.c1_workload()
    return "c1", {mode: serve_entry(m.serve(s, p, max_new=32, mode=mode)) for mode in ("cached", "baseline", "oracle")}


def job_h128(alibi=0):
    with open(os.path.join(HERE, "numeric.json")) as f:
        names = [c["name"] for c in json.load(f)["serve"]]
    with open(os.path.join(HERE, "host.json")) as f:
        host = json.load(f)
    m = RefModel(pc.H128_ALIBI if alibi else pc.H128)
    out = []
    for name in names:
        if name.startswith("corpus:"):
            c = next(c for c in host["corpus"] if c["name"] == name[7:])
            s, p = c["schema_text"], c["prompt_text"]
        else:
            seed = int(name.split(":")[1])
            c = next(c for c in host["random_case"] if c["seed"] == seed)
            s, p = c["schema"], c["prompt"]
        out.append(dict(name=name, **serve_entry(m.serve(s, p, max_new=8, mode="cached"))))
    return ("h128_alibi" if alibi else "h128"), out


def job_long(_):
    m = RefModel(pc.H128_LONG)
    s, p = pc.long_workload()
    r = serve_entry(m.serve(s, p, max_new=4, mode="cached"))
    kv = m.encode_module(s, "doc1")
    rows = [0, kv.rows // 2, kv.rows - 1]
    r["doc1_rows"] = rows
    r["doc1_k1"] = b64(kv.layer(1, 0)[rows])
    r["doc1_v1"] = b64(kv.layer(1, 1)[rows])
    return "long", r


def job_w7b_request(i, alibi=False):
    m = RefModel(pc.W7B_ALIBI if alibi else pc.W7B)
    res = Ref.resolve(pc.W7B_SCHEMA, pc.W7B_PROMPTS[i])
    toks = [t for u in res["uncached"] for t in u["seg"]["tokens"]]
    pos = [q for u in res["uncached"] for q in u["seg"]["positions"]]
    mods = [pc.w7b_module_kv(int(name[3:])) for name in res["cached_imports"]]
    k = np.concatenate([x[0] for x in mods], axis=1)
    v = np.concatenate([x[1] for x in mods], axis=1)
    pp = np.concatenate([x[2] for x in mods])
    logits, _ = m.forward(toks, pos, past=ref_kv(k, v, pp))
    return f"{'alibi_' if alibi else ''}req{i}", {"tokens": np.array(toks, np.int32), "positions": np.array(pos, np.int64),
                                                   "row0": logits[0], "last": logits[-1]}


def job_w7b_full(_):
    """configs[1]'s model at full depth (32 layers): Model::forward of request 0's 64 suffix
    tokens over doc0 + doc1 (4096 synthetic cached rows).  ~30 GB of host memory and ~10 min
    of one core: run alone (`python tests/golden/make_golden_parity.py full`)."""
    m = RefModel(pc.W7B_FULL)
    res = Ref.resolve(pc.W7B_SCHEMA, pc.W7B_PROMPTS[0])
    toks = [t for u in res["uncached"] for t in u["seg"]["tokens"]]
    pos = [q for u in res["uncached"] for q in u["seg"]["positions"]]
    ks, vs, ps = [], [], []
    for name in res["cached_imports"]:
        k, v, p = pc.w7b_full_module_kv(int(name[3:]))
        ks.append(k)
        vs.append(v)
        ps.append(p)
    k = np.concatenate(ks, axis=1)
    del ks
    v = np.concatenate(vs, axis=1)
    del vs
    past = ref_kv(k, v, np.concatenate(ps))
    del k, v
    logits, _ = m.forward(toks, pos, past=past)
    return "full0", {"tokens": np.array(toks, np.int32), "positions": np.array(pos, np.int64),
                     "row0": logits[0], "last": logits[-1]}


def job_w7b_alibi(i):
    return job_w7b_request(i, alibi=True)


def job_w7b_prefill(_):
    m = RefModel(pc.W7B)
    toks = pc.w7b_prefill_tokens()
    logits, kv = m.forward(toks, list(range(len(toks))))
    rows = np.array([0, len(toks) // 2, len(toks) - 1])
    return "prefill", {"row0": logits[0], "last": logits[-1], "kv_rows": rows,
                       "k1": kv.layer(1, 0)[rows], "v1": kv.layer(1, 1)[rows]}


def run(job):
    fn, arg = job
    t = time.time()
    try:
        key, val = fn(arg)
    except Exception as e:  # noqa: BLE001  (reference errors do not pickle back to the pool)
        return f"{fn.__name__}({arg})", RuntimeError(repr(e))
    print(f"{key}: {time.time() - t:.0f}s", flush=True)
    return key, val


JOBS = {
    "prefill": [(job_w7b_prefill, 0)],
    "requests": [(job_w7b_request, i) for i in range(len(pc.W7B_PROMPTS))],
    "long": [(job_long, 0)], "h128": [(job_h128, 0)], "c1": [(job_c1, 0)],
    # ALiBi on the tensor-core paths: head-dim-128 corpus, 7B-width suffixes
    "h128_alibi": [(job_h128, 1)], "alibi_requests": [(job_w7b_alibi, i) for i in (0, 1)],
    "full": [(job_w7b_full, 0)],
}


def main(groups):
    """Regenerates the named job groups (all by default), keeping the other fixtures."""
    jobs = [j for g in groups for j in JOBS[g]]
    with mp.get_context("fork").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        results = dict(pool.map(run, jobs))
    failed = {k: v for k, v in results.items() if isinstance(v, Exception)}
    if failed:
        raise SystemExit(f"reference jobs failed: {failed}")
    jpath, npath = os.path.join(HERE, "parity.json"), os.path.join(HERE, "parity_w7b.npz")
    parity = json.load(open(jpath)) if os.path.exists(jpath) else {}
    parity.update({k: v for k, v in results.items() if k in ("c1", "h128", "long", "h128_alibi")})
    with open(jpath, "w") as f:
        json.dump(parity, f, separators=(",", ":"))
    flat = dict(np.load(npath)) if os.path.exists(npath) else {}
    for key in [k for k in results if "req" in k or k in ("prefill", "full0")]:
        for name, arr in results[key].items():
            flat[f"{key}_{name}"] = arr
    np.savez(npath, **flat)
    print("wrote", jpath, npath)


if __name__ == "__main__":
    main(sys.argv[1:] or [g for g in JOBS if g != "full"])
