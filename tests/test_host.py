"""Host layer (C++ behind the C ABI, no GPU needed): PML parsing / serialization /
validation / chat expansion and the layout + resolve integer contract, checked
bit-exactly against the reference's own outputs (tests/golden/host.json) and the
reference's known-answer tests (proj/tests/test_layout.cpp, test_pml.cpp)."""
import pytest

import paper_2311_04934_b200 as pcb


def test_corpus_parse_plan_resolve_validate(host_golden):
    assert len(host_golden["corpus"]) == 12
    for c in host_golden["corpus"]:
        s = pcb.Schema.parse(c["schema_text"])
        p = pcb.Prompt.parse(c["prompt_text"])
        assert s.ast() == c["schema_ast"], c["name"]
        assert pcb.Schema.parse(c["schema_text"], expand_chat=False).ast() == c["schema_ast_raw"], c["name"]
        assert p.ast() == c["prompt_ast"], c["name"]
        assert s.serialize() == c["serialized"], c["name"]
        assert p.serialize() == c["prompt_serialized"], c["name"]
        assert s.plan() == c["plan"], c["name"]
        assert p.resolve(s) == c["resolved"], c["name"]
        assert p.validate(s) == c["validation"], c["name"]


def test_random_cases_plan_resolve_bit_exact(host_golden):
    # tests/common.hpp random_case seeds 1..200 (in-memory ASTs replayed via JSON)
    for c in host_golden["random_case"]:
        s = pcb.Schema.from_ast(c["schema"])
        p = pcb.Prompt.from_ast(c["prompt"])
        assert s.plan() == c["plan"], c["seed"]
        if "error" in c["resolved"]:
            with pytest.raises(pcb.PromptCacheError):
                p.resolve(s)
        else:
            assert p.resolve(s) == c["resolved"], c["seed"]
        assert p.validate(s) == c["validation"], c["seed"]
        assert s.serialize() == c["serialized"], c["seed"]
        assert p.serialize() == c["prompt_serialized"], c["seed"]


def test_random_ast_serializer_round_trip(host_golden):
    # acceptance.cpp check 9: parse(serialize(ast)) == ast
    for c in host_golden["random_ast"]:
        s = pcb.Schema.from_ast(c["ast"])
        text = s.serialize()
        assert text == c["serialized"], c["seed"]
        back = pcb.Schema.parse(text, expand_chat=False)
        assert back.ast() == c["reparsed"], c["seed"]
        assert back.ast() == c["ast"], c["seed"]


def _mod(name, n, ch="x"):
    return {"k": "module", "name": name, "anon": False, "ch": [{"k": "text", "t": ch * n}]}


def test_kat_spans_50_60_110():
    # test_layout.cpp:23-37 / acceptance.cpp:212-235
    s = pcb.Schema.from_ast({"name": "s", "root": [_mod("a", 50), _mod("b", 60), _mod("c", 7)]})
    e = s.plan()["entries"]
    assert (e["a"]["start"], e["b"]["start"], e["c"]["start"]) == (0, 50, 110)
    assert s.plan()["total_len"] == 117


def test_kat_union_shared_start():
    # test_layout.cpp:39-60
    s = pcb.Schema.from_ast({"name": "s", "root": [
        _mod("pre", 10), {"k": "union", "ch": [_mod("small", 5, "a"), _mod("large", 12, "b")]}, _mod("post", 4)]})
    pl = s.plan()
    e = pl["entries"]
    assert e["small"]["start"] == e["large"]["start"] == 10
    assert e["post"]["start"] == 22
    assert pl["unions"][0]["len"] == 12
    assert e["small"]["union_group"] == e["large"]["union_group"] == 0 and e["post"]["union_group"] == -1


def test_kat_params_nested_gap_args():
    s = pcb.Schema.parse('<schema name="s"><module name="m">ab<param name="p" len="3"/>cd</module></schema>')
    m = s.plan()["entries"]["m"]
    assert m["len"] == 7 and m["params"] == [{"name": "p", "start": 2, "len": 3}]
    assert m["own_tokens"][2:5] == [256, 256, 256] and m["own_tokens"][5] == ord("c")
    s = pcb.Schema.parse('<schema name="s"><module name="outer">aa<module name="inner">bbb</module>cc</module>'
                         '</schema>')
    e = s.plan()["entries"]
    assert e["outer"]["own_positions"] == [0, 1, 5, 6] and e["inner"]["start"] == 2
    assert e["inner"]["parent"] == "outer"
    # interior free text takes the positional gap; overflow raises FREE_TEXT_OVERFLOW
    s = pcb.Schema.from_ast({"name": "s", "root": [_mod("a", 5), _mod("b", 6), _mod("c", 7)]})
    p = pcb.Prompt.from_ast({"schema": "s", "items": [
        {"k": "import", "name": "a", "args": [], "ch": []}, {"k": "text", "t": "xxxx"},
        {"k": "import", "name": "c", "args": [], "ch": []}]})
    assert p.resolve(s)["uncached"][0]["seg"]["positions"] == [5, 6, 7, 8]
    p = pcb.Prompt.from_ast({"schema": "s", "items": [
        {"k": "import", "name": "a", "args": [], "ch": []}, {"k": "text", "t": "xxxxxxx"},
        {"k": "import", "name": "c", "args": [], "ch": []}]})
    with pytest.raises(pcb.PromptCacheError) as ei:
        p.resolve(s)
    assert ei.value.code == "FreeTextOverflow"
    # trailing text after max used position; suffix_start
    p = pcb.Prompt.from_ast({"schema": "s", "items": [
        {"k": "import", "name": "c", "args": [], "ch": []}, {"k": "import", "name": "a", "args": [], "ch": []},
        {"k": "text", "t": "??"}]})
    r = p.resolve(s)
    assert r["cached_imports"] == ["a", "c"] and r["uncached"][0]["seg"]["positions"][0] == 18
    assert r["suffix_start"] == 20


def test_errors_and_codes():
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.Schema.parse("<schema><module/></schema>")
    assert ei.value.code == "SyntaxError"
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.Prompt.parse("<prompt><x/></prompt>")
    assert ei.value.code == "MissingSchemaAttr"
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.Schema.parse('<schema name="s"><module name="m"><param name="p" len="0"/></module></schema>')
    assert ei.value.code == "SyntaxError"
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.Schema.parse('<schema name="s"><bogus>x</bogus></schema>', expand_chat=True)
    assert ei.value.code == "SyntaxError"
    s = pcb.Schema.parse('<schema name="d"><module name="m">x</module></schema>')
    p = pcb.Prompt.parse('<prompt schema="d"><nope/></prompt>')
    rep = p.validate(s)
    assert not rep["ok"] and rep["issues"][0]["code"] == "UNKNOWN_MODULE"
    with pytest.raises(pcb.PromptCacheError) as ei:
        p.resolve(s)
    assert ei.value.code == "UnknownModule"


def test_config_canonical_and_hash(host_golden):
    for c in host_golden["configs"]:
        assert pcb.config_canonical(c["config"]) == c["canonical"]
        assert pcb.config_hash(c["config"]) == int(c["hash"])
    for c in host_golden["ptb"]:
        assert pcb.per_token_bytes(c["config"]) == c["bytes"]
    # Table 4 of the paper: Llama-7B 0.50 MB/token, Llama-13B 0.78 MB/token (fp16)
    assert pcb.per_token_bytes(dict(n_layers=32, hidden=4096, n_heads=32, head_dim=128, bytes_per_element=2)) == 524288
    assert pcb.per_token_bytes(dict(n_layers=40, hidden=5120, n_heads=40, head_dim=128, bytes_per_element=2)) == 819200
    with pytest.raises(pcb.PromptCacheError) as ei:
        pcb.config_hash({"n_layers": 0})
    assert ei.value.code == "InvalidConfig"


def test_c4_workload_and_partition():
    """Config-4 request generator: distinct modules in schema order, deterministic; the
    data-parallel partition covers every request exactly once."""
    import bench
    schema, prompts, picks = bench.workload_c4(64, 8, 256, 8, 4)
    assert len(prompts) == 256 and all(len(p) == 8 and p == sorted(set(p)) for p in picks)
    assert bench.workload_c4(64, 8, 256, 8, 4)[2] == picks
    assert len({tuple(p) for p in picks}) > 200  # differing module combinations
    for world in (1, 2, 3, 8):
        parts = [bench.partition(256, r, world) for r in range(world)]
        assert sorted(i for p in parts for i in p) == list(range(256))
