"""Full-size (Llama-2-7B shape) properties of the sm_100a kernels where the CPU
reference is far too slow to run: the tcgen05 GEMM and flash attention against the
exact SIMT kernels, KV assembly byte-exactness, determinism, and cached serve ==
block-causal oracle at 7B shape with reduced depth."""
import numpy as np
import pytest

import paper_2311_04934_b200 as pcb
from tests.util import BF16_REL, rel, same_greedy_token

pytestmark = pytest.mark.gpu

L7B = dict(n_layers=2, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
           max_position=8192, bytes_per_element=2, seed=42)


@pytest.fixture(scope="module")
def m7():
    return pcb.Model(L7B, dtype=pcb.BF16)


def test_tc_path_vs_simt_7b_shape(m7):
    rng = np.random.default_rng(0)
    t = rng.integers(0, 259, 4160)
    p = np.arange(4160)
    out = {}
    for simt in (0, 1):
        m7.set_option("force_simt", simt)
        a, kv = m7.forward(t[:4096], p[:4096])          # 4096-row prefill (precompute shape)
        b, _ = m7.forward(t[4096:], p[4096:], past=kv)  # 64-token suffix over the 4096-row cache
        c, _ = m7.forward(t[:1], p[:1])
        out[simt] = (a[-1], b, c)
    m7.set_option("force_simt", 0)
    for x, y in zip(out[0], out[1]):
        assert rel(x, y) <= BF16_REL
        x2, y2 = np.atleast_2d(x), np.atleast_2d(y)
        assert all(same_greedy_token(a, b) for a, b in zip(x2, y2))


@pytest.mark.parametrize("n,P", [(129, 0), (256, 0), (300, 0), (640, 0), (1000, 0), (300, 700), (520, 64)])
def test_paired_prefill_attention(m7, n, P):
    """attn_prefill.cu (two 128-query tiles per CTA, P in TMEM, 128-key blocks) against the
    single-tile kernel and the exact SIMT attention: ragged pairs (a lone tile A), a past that is
    not a multiple of the key block, every row's logits."""
    rng = np.random.default_rng(n * 7 + P)
    t = rng.integers(0, 259, P + n)
    p = np.arange(P + n)
    out = {}
    for name, opts in (("pair", {"attn_pair": 2}), ("single", {"attn_pair": 0}), ("simt", {"force_simt_attn": 1})):
        for k, v in opts.items():
            m7.set_option(k, v)
        past = m7.forward(t[:P], p[:P])[1] if P else None
        logits, kv = m7.forward(t[P:], p[P:], past=past)
        out[name] = (logits, kv.layer(1, 0), kv.layer(1, 1))
        m7.set_option("attn_pair", 1)
        m7.set_option("force_simt_attn", 0)
    for other in ("single", "simt"):
        for x, y in zip(out["pair"], out[other]):
            assert rel(x, y) <= BF16_REL, (other, rel(x, y))
    assert all(same_greedy_token(a, b) for a, b in zip(out["pair"][0], out["simt"][0]))


@pytest.mark.parametrize("M", [1, 7, 16, 33, 64, 100, 128, 200, 256, 300])
def test_gemm_token_counts(m7, M):
    rng = np.random.default_rng(M)
    t = rng.integers(0, 259, M)
    p = np.arange(1000, 1000 + M)
    a, _ = m7.forward(t, p)
    m7.set_option("force_simt", 1)
    b, _ = m7.forward(t, p)
    m7.set_option("force_simt", 0)
    assert rel(a, b) <= BF16_REL


def test_deterministic(m7):
    rng = np.random.default_rng(5)
    t = rng.integers(0, 259, 64)
    p = np.arange(64)
    a, ka = m7.forward(t, p)
    b, kb = m7.forward(t, p)
    assert np.array_equal(a, b) and np.array_equal(ka.k(), kb.k())


def test_cached_serve_equals_oracle_7b_shape(m7):
    # 3 modules (incl. a union and a param), 4K cached rows, 64-token suffix
    doc = "".join(chr(97 + (i * 7) % 26) for i in range(2000))
    schema = pcb.Schema.parse(
        f'<schema name="big"><module name="sys">{doc[:900]}</module><union><module name="u1">{doc[900:1700]}</module>'
        f'<module name="u2">{doc[100:400]}</module></union><module name="q">Q: <param name="x" len="8"/> '
        f'{doc[:1200]}</module></schema>')
    store = pcb.ModuleStore(m7)
    store.encode_schema(schema)
    prompt = ('<prompt schema="big"><sys/><u1/><q><x>abc</x></q>' + ("What comes next in the text above" * 2)[:64]
              + '</prompt>')
    c = pcb.serve(store, schema, prompt, 4)
    o = pcb.oracle_serve(m7, schema, prompt, 4)
    assert rel(c.first_token_logits, o.first_token_logits) <= BF16_REL
    assert same_greedy_token(c.first_token_logits, o.first_token_logits)
    assert c.cache_report["cached_token_count"] > 2000


def test_assembly_bytes_at_scale(m7):
    # 3 modules x 1.3K rows at 7B width: byte-exact gather (the assembly kernel)
    rng = np.random.default_rng(7)
    kvs = []
    start = 0
    for n in (1300, 1400, 1500):
        k = rng.standard_normal((2, n, 4096)).astype(np.float32)
        v = rng.standard_normal((2, n, 4096)).astype(np.float32)
        kvs.append((m7.upload_kv(k, v, np.arange(start, start + n)), k, v))
        start += n
    cat = pcb.concat_kv(m7, [x[0] for x in kvs])
    assert np.array_equal(cat.positions(), np.arange(start))
    want_k = np.concatenate([x[0].k() for x in kvs], axis=1)
    assert np.array_equal(cat.k(), want_k)


def test_chain_and_ln_fold_full_depth():
    """32-layer Llama-2-7B shape cached request: the persistent chain with LayerNorm folded
    into its GEMMs vs the same chain with explicit LN phases vs one kernel per GEMM (the
    fold rewrites LN(h)W^T as rstd (hW^T - mean sum_k W); depth must not amplify it)."""
    cfg = dict(L7B, n_layers=32)
    m = pcb.Model(cfg, dtype=pcb.BF16)
    doc = "".join(chr(97 + (i * 11) % 26) for i in range(4096))
    schema = pcb.Schema.parse(f'<schema name="deep"><module name="doc">{doc}</module></schema>')
    store = pcb.ModuleStore(m)
    store.encode_schema(schema)
    prompt = '<prompt schema="deep"><doc/>' + ("Summarise the document above briefly " * 2)[:64] + '</prompt>'
    out = {}
    # chain_group: layers per chain launch (default 9: 4 launches for 32 layers; 1: one per layer;
    # 4: 8 launches) -- the same phases in the same order, so bit-identical logits
    for name, opts in (("fold", {"chain": 1, "ln_fold": 1}), ("ln", {"chain": 1, "ln_fold": 0}),
                       ("kernels", {"chain": 0}), ("group1", {"chain": 1, "ln_fold": 1, "chain_group": 1}),
                       ("group4", {"chain": 1, "ln_fold": 1, "chain_group": 4})):
        for k, v in opts.items():
            m.set_option(k, v)
        out[name] = pcb.serve(store, schema, prompt, 1).first_token_logits
        m.set_option("chain_group", 9)
    m.set_option("chain", 1)
    m.set_option("ln_fold", 1)
    for other in ("ln", "kernels"):
        assert rel(out["fold"], out[other]) <= BF16_REL
        assert same_greedy_token(out["fold"], out[other])
    assert np.array_equal(out["fold"], out["group1"]) and np.array_equal(out["fold"], out["group4"])


@pytest.mark.parametrize("doc_len,suffix", [(4096, 64), (700, 128), (37, 1), (0, 40), (130, 120)])
def test_chain_attention_phase(m7, doc_len, suffix):
    """The chain's attention phase (first phase of every per-layer chain: (head, key split)
    items, global-memory split merge) vs the standalone attention kernel between chains, over
    split counts 1..8 (key blocks), a lone decode-like token, an uncached prompt (P = 0) and a
    128-row suffix (the whole query tile)."""
    doc = "".join(chr(97 + (i * 7) % 26) for i in range(doc_len))
    mod = f'<module name="doc">{doc}</module>' if doc_len else ""
    schema = pcb.Schema.parse(f'<schema name="ca{doc_len}">{mod}</schema>')
    store = pcb.ModuleStore(m7)
    store.encode_schema(schema)
    tail = ("Question about the text: what letters repeat and why " * 4)[:suffix]
    prompt = f'<prompt schema="ca{doc_len}">' + ("<doc/>" if doc_len else "") + tail + "</prompt>"
    out = {}
    for v in (1, 0):
        m7.set_option("chain_attn", v)
        out[v] = pcb.serve(store, schema, prompt, 1).first_token_logits
    m7.set_option("chain_attn", 1)
    assert np.isfinite(out[1]).all()
    assert rel(out[1], out[0]) <= BF16_REL
    assert same_greedy_token(out[1], out[0])


def test_chain_attention_repeated(m7):
    """Barrier-protocol stress: many back-to-back cached requests through the chain's attention
    phase (a single P-ready mbarrier once let the softmax complete two phases before the MMA
    thread looked -- an intermittent hang, ~2 in 3 runs of tools/chain_ab.py)."""
    doc = "".join(chr(97 + (i * 5) % 26) for i in range(2000))
    schema = pcb.Schema.parse(f'<schema name="rep"><module name="doc">{doc}</module></schema>')
    store = pcb.ModuleStore(m7)
    store.encode_schema(schema)
    first = None
    for i in range(60):
        tail = ("tell me more about it please " * 3)[: 8 + (i % 5) * 14]
        r = pcb.serve(store, schema, f'<prompt schema="rep"><doc/>{tail}</prompt>', 1)
        if i % 5 == 0:
            if first is None:
                first = r.first_token_logits
            else:
                assert np.array_equal(first, r.first_token_logits)  # same prompt: bitwise repeatable


@pytest.mark.parametrize("lens", [(4096,), (100, 37, 250), (64, 128, 1, 63)])
def test_zero_copy_prefix(m7, lens):
    """Cached modules read in place by the chain's attention phase (no assembly copy) vs the
    assembled request cache: first-token logits and greedy continuation (decode steps extend
    the request's own rows behind the in-place prefix).  Module lengths off the 64-row key
    block exercise the per-segment padding masks."""
    mods = "".join(f'<module name="m{i}">' + "".join(chr(97 + (i * 3 + j * 7) % 26) for j in range(n)) + "</module>"
                   for i, n in enumerate(lens))
    schema = pcb.Schema.parse(f'<schema name="zc{len(lens)}">Intro. {mods}</schema>')
    store = pcb.ModuleStore(m7)
    store.encode_schema(schema)
    imports = "".join(f"<m{i}/>" for i in range(len(lens)))
    prompt = f'<prompt schema="zc{len(lens)}">{imports}Now answer the question in detail.</prompt>'
    out = {}
    for zc in (1, 0):
        m7.set_option("zero_copy", zc)
        r = pcb.serve(store, schema, prompt, 6)
        out[zc] = (r.first_token_logits, list(r.output_tokens), r.timings["assemble_us"])
    m7.set_option("zero_copy", 1)
    assert rel(out[1][0], out[0][0]) <= BF16_REL
    assert same_greedy_token(out[1][0], out[0][0])
    assert out[1][1][:3] == out[0][1][:3]
