"""Micro-batched cached serving (many requests with differing
module combinations from one store).  serve_batch must give what a loop of serve()
gives: bit-exact on the fp32 path (SIMT kernels are row-independent), within the bf16
tolerance with the same greedy token on the tcgen05 path (a different token count
changes the stream-K split, hence the fp32 summation order)."""
import numpy as np
import pytest

import bench
import paper_2311_04934_b200 as pcb
from oracle.oracle import C1, TINY
from tests.util import BF16_REL, F32_TOL, rel, same_greedy_token

pytestmark = pytest.mark.gpu

L7B = dict(n_layers=2, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
           max_position=32768, bytes_per_element=2, seed=42)


def small_store_case(n_modules=6, mod_len=40, n_req=7, per_req=3, n_unc=12):
    schema, prompts, picks = bench.workload_c4(n_modules, mod_len, n_req, per_req, n_unc)
    # ragged suffixes: vary the uncached length per request
    prompts = [p.replace("</prompt>", "x" * (i % 4) + "</prompt>") for i, p in enumerate(prompts)]
    return schema, prompts


def check(model, schema_text, prompts, micro_batch, is32):
    schema = pcb.Schema.parse(schema_text)
    store = pcb.ModuleStore(model)
    store.encode_schema(schema)
    single = [pcb.serve(store, schema, p, max_new_tokens=1) for p in prompts]
    batch = pcb.serve_batch(store, schema, prompts, micro_batch=micro_batch)
    assert len(batch) == len(prompts)
    for s, b in zip(single, batch):
        assert b.cache_report["cached_token_count"] == s.cache_report["cached_token_count"]
        assert b.cache_report["uncached_token_count"] == s.cache_report["uncached_token_count"]
        if is32:
            assert float(np.max(np.abs(b.first_token_logits - s.first_token_logits))) <= F32_TOL
            assert b.output_tokens == s.output_tokens
        else:
            assert rel(b.first_token_logits, s.first_token_logits) <= BF16_REL
            assert same_greedy_token(b.first_token_logits, s.first_token_logits)


@pytest.mark.parametrize("mb", [1, 3, 7])
def test_batch_equals_single_fp32(mb):
    m = pcb.Model(TINY, dtype=pcb.F32)
    check(m, *small_store_case(), micro_batch=mb, is32=True)


@pytest.mark.parametrize("mb", [2, 4])
def test_batch_equals_single_bf16(mb):
    m = pcb.Model(TINY, dtype=pcb.BF16)
    check(m, *small_store_case(), micro_batch=mb, is32=False)


@pytest.fixture(scope="module")
def m7():
    return pcb.Model(L7B, dtype=pcb.BF16)


@pytest.mark.parametrize("mb", [2, 4])
def test_batch_7b_shape(m7, mb):
    # 16-module store of 256-token modules, 8 modules + 64 uncached tokens per request:
    # micro-batch 2 -> 128 suffix rows (chain kernel), 4 -> 256 rows (stream-K tcgen05 GEMMs)
    schema, prompts, _ = bench.workload_c4(16, 256, 6, 8, 64)
    check(m7, schema, prompts, micro_batch=mb, is32=False)


@pytest.mark.parametrize("cfg,mod_len", [("c1", 40), ("7b", 100), ("7b", 256)])
def test_batch_zero_copy_equals_assembled(cfg, mod_len):
    """Micro-batches whose modules are read in place by the batched attention kernel
    (per-request segment tables over the store blocks, no assembly launch) vs the same
    micro-batches assembled into the request caches."""
    m = pcb.Model(C1 if cfg == "c1" else L7B, dtype=pcb.BF16)  # (TINY's hd 32 has no tcgen05 attention)
    schema_text, prompts = small_store_case(mod_len=mod_len, n_req=8)
    schema = pcb.Schema.parse(schema_text)
    store = pcb.ModuleStore(m)
    store.encode_schema(schema)
    out, asm = {}, {}
    m.set_option("profile", 1)
    for zc in (1, 0):
        m.set_option("zero_copy", zc)
        m.profile()
        out[zc] = pcb.serve_batch(store, schema, prompts, micro_batch=4)
        asm[zc] = m.profile()["assembly"]["launches"]
    m.set_option("profile", 0)
    m.set_option("zero_copy", 1)
    assert (asm[1], asm[0]) == (0, 2)  # the copy runs once per micro-batch (8 requests / 4) only when assembled
    for a, b in zip(out[1], out[0]):
        assert rel(a.first_token_logits, b.first_token_logits) <= BF16_REL
        assert same_greedy_token(a.first_token_logits, b.first_token_logits)
