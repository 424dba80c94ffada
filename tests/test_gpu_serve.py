"""Cached serving on the device vs the reference's engine (reference
proj/tests/test_engine.cpp and acceptance.cpp checks 1, 2, 4, 9-11): same schema /
prompt inputs, compare output tokens, first-token logits and cache reports."""
import base64
import os

import numpy as np
import pytest

import paper_2311_04934_b200 as pcb
from oracle.oracle import TINY, Ref, RefModel, max_rel_diff
from tests.util import BF16_REL, F32_TOL, record_sequence, rel, same_greedy_token

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

DEMO = ('<schema name="demo">You are a travel agent. <module name="city">The city is <param name="which" len="4"/>, '
        'a fine place.</module><module name="season">It is winter there.</module></schema>')


def f32(b):
    return np.frombuffer(base64.b64decode(b), np.float32)


@pytest.fixture(scope="module")
def m32():
    return pcb.Model(TINY, dtype=pcb.F32)


@pytest.fixture(scope="module")
def m16():
    return pcb.Model(TINY, dtype=pcb.BF16)


def schema_of(s):
    return pcb.Schema.parse(s) if isinstance(s, str) else pcb.Schema.from_ast(s)


def prompt_of(p):
    return pcb.Prompt.parse(p) if isinstance(p, str) else pcb.Prompt.from_ast(p)


def golden_case_inputs(host_golden, name):
    if name.startswith("corpus:"):
        c = next(c for c in host_golden["corpus"] if c["name"] == name[7:])
        return c["schema_text"], c["prompt_text"]
    seed = int(name.split(":")[1])
    c = next(c for c in host_golden["random_case"] if c["seed"] == seed)
    return c["schema"], c["prompt"]


def test_serve_matches_reference_goldens(m32, m16, host_golden, numeric_golden):
    """12 corpus schemas + random_case seeds 1..40: cached / oracle / baseline."""
    worst32, worst16, bad16 = 0.0, 0.0, 0
    for case in numeric_golden["serve"]:
        s_in, p_in = golden_case_inputs(host_golden, case["name"])
        schema, prompt = schema_of(s_in), prompt_of(p_in)
        for model, is32 in ((m32, True), (m16, False)):
            store = pcb.ModuleStore(model)
            store.encode_schema(schema)
            got = {"cached": pcb.serve(store, schema, prompt, 8),
                   "baseline": pcb.serve(store, schema, prompt, 8, use_cache=False),
                   "oracle": pcb.oracle_serve(model, schema, prompt, 8)}
            for mode, r in got.items():
                want = case[mode]
                wl = f32(want["logits"])
                assert r.cache_report["cached_token_count"] == want["report"]["cached_token_count"]
                assert r.cache_report["uncached_token_count"] == want["report"]["uncached_token_count"]
                if is32:
                    worst32 = max(worst32, float(np.max(np.abs(r.first_token_logits - wl))))
                    assert r.output_tokens == want["tokens"], (case["name"], mode)
                else:
                    worst16 = max(worst16, rel(r.first_token_logits, wl))
                    assert same_greedy_token(r.first_token_logits, wl, f"tiny bf16 {case['name']} {mode}"), \
                        (case["name"], mode)
                    bad16 += r.output_tokens != want["tokens"]
                    record_sequence(r.output_tokens, want["tokens"], f"tiny bf16 {case['name']} {mode}")
    assert worst32 <= F32_TOL, worst32
    assert worst16 <= BF16_REL, worst16
    print(f"f32 worst max-abs {worst32:.2e}; bf16 worst rel {worst16:.2e}; bf16 full-sequence mismatches {bad16}")


def test_serve_matches_live_reference_200_seeds(m32, ref):
    """acceptance check 1 style: random_case seeds 1..200, 32 greedy tokens, f32."""
    r = RefModel(TINY)
    worst = 0.0
    for seed in range(1, 201):
        rc = Ref.random_case(seed)
        schema, prompt = pcb.Schema.from_ast(rc["schema"]), pcb.Prompt.from_ast(rc["prompt"])
        store = pcb.ModuleStore(m32)
        store.encode_schema(schema)
        got = pcb.serve(store, schema, prompt, 32)
        want = r.serve(rc["schema"], rc["prompt"], max_new=32)
        assert got.output_tokens == want["output_tokens"], seed
        worst = max(worst, max_rel_diff(want["first_token_logits"], got.first_token_logits))
    assert worst <= F32_TOL


def test_cached_equals_oracle_and_single_module_equals_baseline(m32):
    schema = pcb.Schema.parse(DEMO)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    p = '<prompt schema="demo"><city><which>Rome</which></city><season/>Pack what?</prompt>'
    c = pcb.serve(store, schema, p, 8)
    o = pcb.oracle_serve(m32, schema, p, 8)
    assert c.output_tokens == o.output_tokens
    assert max_rel_diff(c.first_token_logits, o.first_token_logits) < 1e-5
    one = pcb.Schema.parse('<schema name="one"><module name="m">The quick brown fox jumps over the lazy dog.'
                           '</module></schema>')
    st = pcb.ModuleStore(m32)
    st.encode_schema(one)
    a = pcb.serve(st, one, '<prompt schema="one"><m/> and then?</prompt>', 6)
    b = pcb.serve(st, one, '<prompt schema="one"><m/> and then?</prompt>', 6, use_cache=False)
    assert a.output_tokens == b.output_tokens
    assert max_rel_diff(a.first_token_logits, b.first_token_logits) < 1e-6


def test_cache_report_miss_reencode_and_validation(m32):
    schema = pcb.Schema.parse(DEMO)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    r = pcb.serve(store, schema, '<prompt schema="demo"><city/><season/>x</prompt>', 4)
    assert r.cache_report["modules_hit"] == 3 and r.cache_report["modules_missed"] == 0
    assert r.cache_report["uncached_token_count"] == 1
    empty = pcb.ModuleStore(m32)
    miss = pcb.serve(empty, schema, '<prompt schema="demo"><city/><season/>x</prompt>', 4)
    assert miss.cache_report["modules_missed"] == 3 and len(empty) == 3
    assert miss.output_tokens == r.output_tokens
    with pytest.raises(pcb.PromptCacheError) as e:
        pcb.serve(store, schema, '<prompt schema="demo"><nope/></prompt>', 4)
    assert e.value.code == "ValidationFailed"
    with pytest.raises(pcb.PromptCacheError) as e:
        pcb.serve(store, schema, '<prompt schema="demo"><city><which>toolongbyfar</which></city></prompt>', 1)
    assert e.value.code == "ValidationFailed" and "ARG_TOO_LONG" in str(e.value)


def test_args_empty_suffix_scaffold(m32):
    schema = pcb.Schema.parse(DEMO)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    r1 = pcb.serve(store, schema, '<prompt schema="demo"><city><which>Rome</which></city>next?</prompt>', 1)
    r2 = pcb.serve(store, schema, '<prompt schema="demo"><city><which>Oslo</which></city>next?</prompt>', 1)
    assert max_rel_diff(r1.first_token_logits, r2.first_token_logits) > 1e-6
    p = pcb.Schema.parse('<schema name="p"><module name="m">some cached words</module></schema>')
    st = pcb.ModuleStore(m32)
    st.encode_schema(p)
    c = pcb.serve(st, p, '<prompt schema="p"><m/></prompt>', 4)
    o = pcb.oracle_serve(m32, p, '<prompt schema="p"><m/></prompt>', 4)
    assert len(c.output_tokens) == 4 and c.output_tokens == o.output_tokens
    store.encode_scaffold(schema, ["__anon_0", "city", "season"])
    prompt = '<prompt schema="demo"><city/><season/>go on</prompt>'
    sc = pcb.serve(store, schema, prompt, 6, use_scaffolds=True)
    assert sc.cache_report["used_scaffold"]
    base = pcb.serve(store, schema, prompt, 6, use_cache=False)
    assert sc.output_tokens == base.output_tokens
    assert max_rel_diff(sc.first_token_logits, base.first_token_logits) < 1e-6
    assert not pcb.serve(store, schema, prompt, 6).cache_report["used_scaffold"]


def test_concat_is_pure_concat_and_overlap_rejected(m32):
    schema = pcb.Schema.parse(DEMO)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    a, b = store.lookup("demo", "city"), store.lookup("demo", "season")
    ab = pcb.concat_kv(m32, [a, b])
    assert ab.rows == a.rows + b.rows
    assert np.array_equal(ab.positions(), np.concatenate([a.positions(), b.positions()]))
    assert np.array_equal(ab.k(), np.concatenate([a.k(), b.k()], axis=1))  # byte-exact
    assert np.array_equal(ab.v(), np.concatenate([a.v(), b.v()], axis=1))
    with pytest.raises(pcb.PromptCacheError) as e:
        pcb.concat_kv(m32, [a, a])
    assert e.value.code == "PositionOverlap"
    # permutation invariance of a probe token over the concatenation (acceptance check 4)
    anon = store.lookup("demo", "__anon_0")
    total = schema.plan()["total_len"]
    outs = [m32.forward([ord("?")], [total], past=pcb.concat_kv(m32, o))[0][0]
            for o in ([anon, a, b], [b, a, anon], [a, anon, b])]
    assert max_rel_diff(outs[0], outs[1]) < 1e-6 and max_rel_diff(outs[0], outs[2]) < 1e-6


def test_precompute_rows_match_reference(m32, ref):
    r = RefModel(TINY)
    schema_text = ('<schema name="demo">intro <module name="a">alpha text here</module>'
                   '<module name="b">beta <param name="p" len="3"/> tail</module></schema>')
    schema = pcb.Schema.parse(schema_text)
    store = pcb.ModuleStore(m32)
    assert store.encode_schema(schema) == 3
    for name in ("__anon_0", "a", "b"):
        got = store.lookup("demo", name)
        want = r.encode_module(schema_text, name)
        assert np.array_equal(got.positions(), want.positions())
        assert np.max(np.abs(got.k() - want.k())) <= 1e-5
        assert np.max(np.abs(got.v() - want.v())) <= 1e-5


def test_lru_capacity_and_stats(m32):
    schema = pcb.Schema.parse(DEMO)
    ptb = pcb.per_token_bytes(TINY)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    st = store.stats()
    assert st["entries"] == 3 and st["bytes_used"]["fast"] > 0
    small = pcb.ModuleStore(m32)
    small.set_capacity(pcb.FAST, 40 * ptb)
    small.encode_module(schema, "city")     # 31 tokens
    with pytest.raises(pcb.PromptCacheError) as e:
        small.set_capacity(pcb.FAST, 10 * ptb)
        small.encode_module(schema, "city")
    assert e.value.code == "CapacityExceeded"
    small.set_capacity(pcb.FAST, 60 * ptb)
    small.encode_module(schema, "season")
    small.lookup("demo", "season")
    small.encode_module(schema, "__anon_0")  # evicts the LRU entry (city) to fit
    assert small.lookup("demo", "season") is not None


def test_slow_tier_equals_fast_tier(m16):
    schema = pcb.Schema.parse(DEMO)
    fast, slow = pcb.ModuleStore(m16), pcb.ModuleStore(m16)
    fast.encode_schema(schema)
    slow.encode_schema(schema, tier=pcb.SLOW)
    assert slow.stats()["bytes_used"]["slow"] > 0
    p = '<prompt schema="demo"><city><which>Rome</which></city><season/>Pack what?</prompt>'
    a, b = pcb.serve(fast, schema, p, 6), pcb.serve(slow, schema, p, 6)
    assert a.output_tokens == b.output_tokens
    assert np.array_equal(a.first_token_logits, b.first_token_logits)
    assert b.timings["copy_us"] > 0


def test_pcst_persistence(m32, tmp_path):
    # loads a store written by the reference's ModuleStore::save, and round-trips byte-identically
    schema = pcb.Schema.parse('<schema name="store"><module name="x">persistent text</module>'
                              '<module name="y">more <param name="p" len="2"/></module></schema>')
    st = pcb.ModuleStore(m32)
    st.load(os.path.join(HERE, "golden", "store_ref.pcst"))
    assert len(st) == 3
    p1, p2 = str(tmp_path / "a.pcst"), str(tmp_path / "b.pcst")
    st.save(p1)
    assert open(p1, "rb").read() == open(os.path.join(HERE, "golden", "store_ref.pcst"), "rb").read()
    again = pcb.ModuleStore(m32)
    again.load(p1)
    again.save(p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    mine = pcb.ModuleStore(m32)
    mine.encode_schema(schema)
    r1 = pcb.serve(st, schema, '<prompt schema="store"><x/>go</prompt>', 4)
    r2 = pcb.serve(mine, schema, '<prompt schema="store"><x/>go</prompt>', 4)
    assert r1.output_tokens == r2.output_tokens
    other = pcb.Model(dict(TINY, seed=43), dtype=pcb.F32)
    with pytest.raises(pcb.PromptCacheError) as e:
        pcb.ModuleStore(other).load(p1)
    assert e.value.code == "ConfigHashMismatch"


def test_decode_cost_flat(m32):
    schema = pcb.Schema.parse(DEMO)
    store = pcb.ModuleStore(m32)
    store.encode_schema(schema)
    p = '<prompt schema="demo"><city/><season/>go</prompt>'
    b = m32.forward_tokens
    pcb.serve(store, schema, p, 1)
    one = m32.forward_tokens - b
    b = m32.forward_tokens
    pcb.serve(store, schema, p, 9)
    assert m32.forward_tokens - b - one == 8


def test_zero_copy_on_reference_corpus(host_golden, numeric_golden):
    """Every golden corpus schema / random case (unions, nested and anonymous modules,
    parameters, scaffolds-free prompts) through a bf16 model with 128-wide heads, so single
    requests take the chain attention phase and read their modules in place when eligible:
    tokens and first-token logits vs the same requests with the assembly copy, and the
    cached path vs the device oracle.  (TINY's 32-wide heads never take that path.)"""
    cfg = dict(n_layers=2, n_heads=2, head_dim=128, hidden=256, vocab_size=512, pos_encoding="rope",
               max_position=8192, bytes_per_element=2, seed=42)
    m = pcb.Model(cfg, dtype=pcb.BF16)
    worst, n_cases = 0.0, 0
    for case in numeric_golden["serve"]:
        s_in, p_in = golden_case_inputs(host_golden, case["name"])
        schema, prompt = schema_of(s_in), prompt_of(p_in)
        store = pcb.ModuleStore(m)
        store.encode_schema(schema)
        out = {}
        for zc in (1, 0):
            m.set_option("zero_copy", zc)
            out[zc] = pcb.serve(store, schema, prompt, 8)
        m.set_option("zero_copy", 1)
        o = pcb.oracle_serve(m, schema, prompt, 8)
        assert out[1].cache_report == out[0].cache_report, case["name"]
        assert same_greedy_token(out[1].first_token_logits, out[0].first_token_logits,
                                 f"zc-vs-copy {case['name']}"), case["name"]
        assert same_greedy_token(out[1].first_token_logits, o.first_token_logits,
                                 f"zc-vs-device-oracle {case['name']}"), case["name"]
        worst = max(worst, rel(out[1].first_token_logits, out[0].first_token_logits),
                    rel(out[1].first_token_logits, o.first_token_logits))
        n_cases += 1
    assert n_cases >= 40
    assert worst <= BF16_REL, worst
