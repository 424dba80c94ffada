"""Differential fuzzing of the host layer against the live reference (oracle/_ref): PML
sources mutated at random -- characters dropped, duplicated or replaced by markup
fragments -- must parse to the same AST or fail with the same pc::ErrorCode, and the
same goes for serialization, validation, layout plans and resolved prompts.
Runs where the reference library is built (skipped otherwise)."""
import os
import random

import pytest

import paper_2311_04934_b200 as pcb

FRAGMENTS = ["<", ">", "/", "</module>", "<module name=\"x\">", "<union>", "</union>", "<param name=\"p\" len=\"3\"/>",
             "<param name=\"q\" len=\"0\"/>", "&amp;", "&bogus;", "&", "\"", "'", " ", "\n", "<user>", "</user>",
             "<system>", "<m/>", "<a><b>v</b></a>", "<x y=\"1\"/>", "<module>", "len=\"-2\"", "<param/>"]


def code_of(fn):
    try:
        return ("ok", fn())
    except pcb.PromptCacheError as e:
        return ("err", e.code)


def ref_code_of(ref, fn):
    from oracle.oracle import RefError
    try:
        return ("ok", fn())
    except RefError as e:
        return ("err", str(e).split(":")[0])


def mutate(rng, text):
    s = list(text)
    for _ in range(rng.randint(1, 3)):
        i = rng.randrange(len(s) + 1)
        op = rng.random()
        if op < 0.3 and i < len(s):
            del s[i]
        elif op < 0.5 and i < len(s):
            s.insert(i, s[i])
        else:
            s[i:i] = list(rng.choice(FRAGMENTS))
    return "".join(s)


def _norm_code(c):
    # the reference names the two resolve-time codes by their issue codes
    return {"FREE_TEXT_OVERFLOW": "FreeTextOverflow", "ARG_TOO_LONG": "ArgTooLong"}.get(c, c)


def test_mutated_pml_matches_reference(ref, host_golden):
    rng = random.Random(20251017)
    n_ok = n_err = 0
    for c in host_golden["corpus"]:
        for _ in range(int(os.environ.get("PCB_FUZZ_N", "60"))):
            st, pt = c["schema_text"], c["prompt_text"]
            if rng.random() < 0.5:
                st = mutate(rng, st)
            else:
                pt = mutate(rng, pt)
            for expand in (False, True):  # the expanded AST (used below) last
                ours = code_of(lambda: pcb.Schema.parse(st, expand_chat=expand).ast())
                theirs = ref_code_of(ref, lambda: ref.parse_schema(st, expand))
                assert (ours[0], _norm_code(ours[1]) if ours[0] == "err" else ours[1]) == \
                       (theirs[0], _norm_code(theirs[1]) if theirs[0] == "err" else theirs[1]), (st, expand)
            p_ours = code_of(lambda: pcb.Prompt.parse(pt).ast())
            p_theirs = ref_code_of(ref, lambda: ref.parse_prompt(pt))
            assert p_ours == p_theirs, pt
            if ours[0] == "ok" and p_ours[0] == "ok":
                s, p = pcb.Schema.parse(st), pcb.Prompt.parse(pt)
                assert s.serialize() == ref.serialize_schema(ours[1])
                assert p.serialize() == ref.serialize_prompt(p_ours[1])
                assert p.validate(s) == ref.validate(pt, st)
                assert s.plan() == ref.plan(st)
                r_ours = code_of(lambda: p.resolve(s))
                r_theirs = ref_code_of(ref, lambda: ref.resolve(st, pt))
                if r_ours[0] == "err":
                    assert r_theirs[0] == "err" and _norm_code(r_ours[1]) == _norm_code(r_theirs[1]), (st, pt)
                else:
                    assert r_ours == r_theirs, (st, pt)
                n_ok += 1
            else:
                n_err += 1
    assert n_ok > 100 and n_err > 100, (n_ok, n_err)
