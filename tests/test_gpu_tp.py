"""Head-sharded (tensor-parallel) serving, on ONE GPU: the T ranks
are threads of this process sharing the device through a TPGroup (the same sharded
weights, sharded module store, row-parallel partial GEMMs + all-reduce and vocab-shard
gather as the NCCL path; only the transport differs).  Every rank must produce the
same token, and it must match the unsharded model."""
import threading

import numpy as np
import pytest

import paper_2311_04934_b200 as pcb
from oracle.oracle import TINY
from tests.util import BF16_REL, F32_TOL, rel, same_greedy_token

pytestmark = pytest.mark.gpu

SCHEMA = ('<schema name="tp"><module name="sys">You are a careful reader of long documents. </module>'
          '<module name="doc">The Seine flows through Paris; the Thames through London; the Tiber '
          'through Rome. Each city grew around its river crossing.</module></schema>')
PROMPTS = ['<prompt schema="tp"><sys/><doc/>Which river runs through Rome?</prompt>',
           '<prompt schema="tp"><doc/>Name a city.</prompt>']


def run_ranks(T, fn):
    out, err = [None] * T, []

    def go(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=go, args=(r,)) for r in range(T)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    if err:
        raise err[0]
    return out


def serve_tp(cfg, dtype, T, prompts, batch=False):
    group = pcb.TPGroup(T)
    models = [pcb.Model(cfg, dtype=dtype, device=0, tp_rank=r, tp_size=T, group=group) for r in range(T)]
    schema = pcb.Schema.parse(SCHEMA)

    def rank(r):
        store = pcb.ModuleStore(models[r])
        store.encode_schema(schema)
        if batch:
            return [(x.output_tokens, x.first_token_logits) for x in pcb.serve_batch(store, schema, prompts, 2)]
        return [(x.output_tokens, x.first_token_logits) for x in
                (pcb.serve(store, schema, p, max_new_tokens=3) for p in prompts)]

    return run_ranks(T, rank)


def serve_single(cfg, dtype, prompts, max_new=3):
    m = pcb.Model(cfg, dtype=dtype)
    schema = pcb.Schema.parse(SCHEMA)
    store = pcb.ModuleStore(m)
    store.encode_schema(schema)
    return [(x.output_tokens, x.first_token_logits) for x in
            (pcb.serve(store, schema, p, max_new_tokens=max_new) for p in prompts)]


@pytest.mark.parametrize("T", [2, 4])
@pytest.mark.parametrize("dtype", [pcb.F32, pcb.BF16])
def test_tp_matches_single(T, dtype):
    ref = serve_single(TINY, dtype, PROMPTS)
    ranks = serve_tp(TINY, dtype, T, PROMPTS)
    for r in range(1, T):  # replicated results: identical on every rank
        for (ta, la), (tb, lb) in zip(ranks[0], ranks[r]):
            assert ta == tb and np.array_equal(la, lb)
    for (t, lg), (rt, rl) in zip(ranks[0], ref):
        if dtype == pcb.F32:
            assert float(np.max(np.abs(lg - rl))) <= F32_TOL
            assert t == rt
        else:
            assert rel(lg, rl) <= BF16_REL and same_greedy_token(lg, rl)


def test_tp_batch():
    ref = serve_single(TINY, pcb.BF16, PROMPTS, max_new=1)
    ranks = serve_tp(TINY, pcb.BF16, 2, PROMPTS, batch=True)
    for (t, lg), (rt, rl) in zip(ranks[0], ref):
        assert rel(lg, rl) <= BF16_REL and same_greedy_token(lg, rl)


def test_tp_7b_shape():
    # 2 layers at Llama-2-7B width, TP 2: packed tcgen05 shards (d/2 = 2048 attention
    # columns, 8192 MLP columns, 16000 vocab rows per rank)
    cfg = dict(n_layers=2, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
               max_position=8192, bytes_per_element=2, seed=42)
    ref = serve_single(cfg, pcb.BF16, PROMPTS[:1], max_new=1)
    ranks = serve_tp(cfg, pcb.BF16, 2, PROMPTS[:1])
    (t, lg), (rt, rl) = ranks[0][0], ref[0]
    assert rel(lg, rl) <= BF16_REL and same_greedy_token(lg, rl)
