"""Inputs of the reference-pinned parity fixtures (tests/golden/parity.json, parity_w7b.npz).

Shared by the generator (tests/golden/make_golden_parity.py, run where /root/reference
exists, against the UNMODIFIED reference compiled into oracle/_ref) and by the GPU tests
(tests/test_gpu_parity.py), so both sides see byte-identical inputs.  Everything here is
deterministic: text from the reference's synthetic_text generator (bench.cpp:22-31,
restated in bench.py), synthetic K/V from numpy's PCG64 stream rounded to bf16 so the
bf16 device store holds exactly the values the fp32 reference reads.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
from bench import question, synthetic_text, workload  # noqa: E402

# BASELINE.json configs[0]: 2 layers, d 256, 4 heads, fp32 (oracle.C1)
C1 = dict(n_layers=2, n_heads=4, head_dim=64, hidden=256, vocab_size=512, pos_encoding="rope",
          max_position=8192, bytes_per_element=4, seed=42)
# the benchmarked head width (128) on a narrow model: the chain attention phase, zero-copy
# segments, CTA-pair GEMMs and the batched attention all run at this head size
H128 = dict(n_layers=2, n_heads=2, head_dim=128, hidden=256, vocab_size=512, pos_encoding="rope",
            max_position=8192, bytes_per_element=2, seed=42)
H128_LONG = dict(H128, max_position=32768)
# Llama-2-7B width (d 4096, 32 heads of 128, vocab 32000) at 2 layers
W7B = dict(n_layers=2, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
           max_position=8192, bytes_per_element=2, seed=42)

# ALiBi variants: no RoPE, per-head linear position bias in the attention
H128_ALIBI = dict(H128, pos_encoding="alibi")
W7B_ALIBI = dict(W7B, pos_encoding="alibi")

# configs[0]: a 68-token system module + a 512-token document + 32 uncached tokens
C1_SYSTEM = "You are a careful assistant. Answer only from the document; cite it."
assert len(C1_SYSTEM) == 68


def c1_workload():
    schema = (f'<schema name="c1"><module name="sys">{C1_SYSTEM}</module>'
              f'<module name="doc">{synthetic_text(512, 7 * 512 + 1)}</module></schema>')
    prompt = f'<prompt schema="c1"><sys/><doc/>{question(32, 1000)}</prompt>'
    return schema, prompt


def long_workload():
    """configs[2] shape at narrow width: 3 modules, 16,384 cached tokens + 128 uncached."""
    schema, prompts = workload(16384, 128, 3)
    return schema, prompts[0]


# ---- 7B width: two synthetic 2048-row modules in the store, four requests ----
W7B_MOD_ROWS = 2048
W7B_SCHEMA = ('<schema name="w7b">'
              f'<module name="doc0">{synthetic_text(W7B_MOD_ROWS, 101)}</module>'
              f'<module name="doc1">{synthetic_text(W7B_MOD_ROWS, 102)}</module></schema>')
W7B_PROMPTS = [f'<prompt schema="w7b">{imp}{question(64, 11 + i)}</prompt>'
               for i, imp in enumerate(["<doc0/><doc1/>", "<doc0/>", "<doc1/>", "<doc0/><doc1/>"])]
W7B_PREFILL = 320  # rows of the no-past prefill (CTA-pair GEMM tiles + a ragged tail)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 (ties to even) -> fp32."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def w7b_module_kv(i: int):
    """Synthetic K/V [L][rows][hidden] of module doc{i} (K scaled 4x for a peaked softmax)."""
    L, d = W7B["n_layers"], W7B["hidden"]
    g = np.random.default_rng(20251017 + i)
    k = bf16_round(g.uniform(-4.0, 4.0, (L, W7B_MOD_ROWS, d)).astype(np.float32))
    v = bf16_round(g.uniform(-1.0, 1.0, (L, W7B_MOD_ROWS, d)).astype(np.float32))
    pos = np.arange(i * W7B_MOD_ROWS, (i + 1) * W7B_MOD_ROWS, dtype=np.int64)
    return k, v, pos


# the benchmarked depth: Llama-2-7B shape at all 32 layers (configs[1]'s model), one request of
# 4096 cached rows (doc0 + doc1, synthetic bf16-exact K/V) + 64 uncached tokens
W7B_FULL = dict(W7B, n_layers=32)


def w7b_full_module_kv(i: int):
    """Synthetic K/V [32][rows][hidden] of module doc{i} for the full-depth case."""
    L, d = W7B_FULL["n_layers"], W7B_FULL["hidden"]
    g = np.random.default_rng(20251117 + i)
    k = bf16_round(g.uniform(-4.0, 4.0, (L, W7B_MOD_ROWS, d)).astype(np.float32))
    v = bf16_round(g.uniform(-1.0, 1.0, (L, W7B_MOD_ROWS, d)).astype(np.float32))
    pos = np.arange(i * W7B_MOD_ROWS, (i + 1) * W7B_MOD_ROWS, dtype=np.int64)
    return k, v, pos


def w7b_prefill_tokens():
    return [ord(c) for c in synthetic_text(W7B_PREFILL, 4242)]
