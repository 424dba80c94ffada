"""Localise a tc-vs-SIMT divergence at 7B shape (2 layers): per-layer K/V rows and logits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2311_04934_b200 as pcb

L = dict(n_layers=2, n_heads=32, head_dim=128, hidden=4096, vocab_size=32000, pos_encoding="rope",
         max_position=8192, bytes_per_element=2, seed=42)
rng = np.random.default_rng(0)
t = rng.integers(0, 259, 4160)
p = np.arange(4160)


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


n = 256
m = pcb.Model(L, dtype=pcb.BF16)
m.set_option("force_simt", 1)
a0, kv0 = m.forward(t[:n], p[:n])
s0, new0 = m.forward(t[n:n + 64], p[n:n + 64], past=kv0)
m.set_option("force_simt", 0)
for opt in ("none", "force_simt_gemm", "force_simt_attn"):
    if opt != "none":
        m.set_option(opt, 1)
    s, new = m.forward(t[n:n + 64], p[n:n + 64], past=kv0)  # same (SIMT-made) past for every variant
    print(f"{opt:16s} suffix logits rel {rel(s, s0):.3e}  K0 {rel(new.layer(0, 0), new0.layer(0, 0)):.3e} "
          f"V0 {rel(new.layer(0, 1), new0.layer(0, 1)):.3e} K1 {rel(new.layer(1, 0), new0.layer(1, 0)):.3e} "
          f"V1 {rel(new.layer(1, 1), new0.layer(1, 1)):.3e}", flush=True)
    if opt != "none":
        m.set_option(opt, 0)
for sp in ("1", "2", "3"):
    os.environ["PCB_ATTN_SPLITS"] = sp
    s, _ = m.forward(t[n:n + 64], p[n:n + 64], past=kv0)
    print(f"attn splits={sp}: suffix rel {rel(s, s0):.3e}", flush=True)
