"""Bring-up diagnostics on the GPU box: each section reports instead of stopping."""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2311_04934_b200 as pcb
from oracle.oracle import C1, TINY, Ref, RefModel, max_rel_diff


def section(name):
    def deco(fn):
        t = time.time()
        try:
            fn()
            print(f"[ok]   {name} ({time.time() - t:.1f}s)", flush=True)
        except Exception:
            print(f"[FAIL] {name}", flush=True)
            traceback.print_exc()
        return fn
    return deco


rng = np.random.default_rng(0)
ref = RefModel(TINY)


@section("weights checksum f32/bf16")
def _():
    for dt in (pcb.F32, pcb.BF16):
        m = pcb.Model(TINY, dtype=dt)
        for n in ["embed", "unembed", "layer0.wq", "layer3.w2"]:
            assert m.weight_checksum(n) == ref.weight_checksum(n), n


@section("f32 forward vs reference")
def _():
    m = pcb.Model(TINY, dtype=pcb.F32)
    t = rng.integers(0, 259, 40)
    p = np.arange(40)
    lr, kvr = ref.forward(t, p)
    lm, kvm = m.forward(t, p)
    print("   f32 logits max abs", np.abs(lr - lm).max(), "k", np.abs(kvr.k() - kvm.k()).max())
    l1, kv1 = m.forward(t[:30], p[:30])
    l2, _ = m.forward(t[30:], p[30:], past=kv1)
    print("   chained vs single", max_rel_diff(lm[-1], l2[-1]))


for force in (1, 0):
    @section(f"bf16 forward vs reference force_simt={force}")
    def _():
        m = pcb.Model(TINY, dtype=pcb.BF16)
        m.set_option("force_simt", force)
        t = rng.integers(0, 259, 40)
        p = np.arange(40)
        lr, _ = ref.forward(t, p)
        lm, _ = m.forward(t, p)
        rel = np.abs(lr - lm).max() / np.abs(lr).max()
        print("   bf16 rel err", rel, "argmax", lr[-1].argmax(), lm[-1].argmax())


@section("serve tiny f32 + bf16 vs reference")
def _():
    schema = ('<schema name="demo">You are a travel agent. <module name="city">The city is '
              '<param name="which" len="4"/>, a fine place.</module><module name="season">It is winter '
              'there.</module></schema>')
    prompt = '<prompt schema="demo"><city><which>Rome</which></city><season/>Pack what?</prompt>'
    rr = ref.serve(schema, prompt, max_new=8)
    for dt in (pcb.F32, pcb.BF16):
        m = pcb.Model(TINY, dtype=dt)
        s = pcb.Schema.parse(schema)
        st = pcb.ModuleStore(m)
        st.encode_schema(s)
        r = pcb.serve(st, s, prompt, max_new_tokens=8)
        d = np.abs(np.array(rr["first_token_logits"]) - r.first_token_logits).max()
        print(f"   dtype={dt} tokens ref={rr['output_tokens']} got={r.output_tokens} maxabs={d:.3e}")
        o = pcb.oracle_serve(m, s, prompt, max_new_tokens=8)
        print(f"   oracle tokens {o.output_tokens}")


@section("7B-shape GEMM tc vs simt (1 layer)")
def _():
    cfg = dict(n_layers=1, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
               max_position=8192, bytes_per_element=2, seed=42)
    m = pcb.Model(cfg, dtype=pcb.BF16)
    t = rng.integers(0, 259, 64)
    p = np.arange(4096, 4160)
    l_tc, _ = m.forward(t, p)
    m.set_option("force_simt", 1)
    l_s, _ = m.forward(t, p)
    print("   tc vs simt rel", np.abs(l_tc - l_s).max() / np.abs(l_s).max(), "argmax", l_tc[-1].argmax(),
          l_s[-1].argmax())
    for M in (1, 16, 64, 128, 300):
        t = rng.integers(0, 259, M)
        p = np.arange(M)
        m.set_option("force_simt", 0)
        a, _ = m.forward(t, p)
        m.set_option("force_simt", 1)
        b, _ = m.forward(t, p)
        print(f"   M={M} rel {np.abs(a - b).max() / np.abs(b).max():.3e}")


@section("7B-shape attention tc vs simt (1 layer)")
def _():
    cfg = dict(n_layers=1, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
               max_position=8192, bytes_per_element=2, seed=42)
    m = pcb.Model(cfg, dtype=pcb.BF16)
    t = rng.integers(0, 259, 4160)
    p = np.arange(4160)
    res = {}
    for force in (0, 1):
        m.set_option("force_simt", force)
        a, kv = m.forward(t[:4096], p[:4096])
        b, _ = m.forward(t[4096:], p[4096:], past=kv)
        c, _ = m.forward(t[4096:4097], p[4096:4097], past=kv)
        d, _ = m.forward(t[:200], p[:200])
        res[force] = (a, b, c, d)
    for i, nm in enumerate(["prefill4096", "suffix64", "suffix1", "prefill200"]):
        x, y = res[0][i], res[1][i]
        print(f"   {nm}: rel {np.abs(x - y).max() / np.abs(y).max():.3e} argmax_eq "
              f"{(x.argmax(-1) == y.argmax(-1)).mean():.3f}")
