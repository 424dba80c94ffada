"""Shared numeric criteria for the parity tests."""
import sys

import numpy as np

F32_TOL = 1e-3   # north star: fp32 path max-abs <= 1e-3
BF16_REL = 2e-2  # north star: bf16 path logits rel-err <= 2e-2 (max |a-b| / max |b|)

# Every greedy-token comparison of the session: how many were identical and how many passed
# only through the tie exemption below (printed in the pytest terminal summary, conftest.py).
GREEDY = {"checked": 0, "identical": 0, "exempt": []}
# bf16 multi-token sequences that diverged from the reference after an identical first token
SEQ = {"checked": 0, "diverged": []}
# logits rel-err of the reference comparisons at the benchmarked shapes (label -> rel), printed
# in the terminal summary
RELS = {}


def rel(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def same_greedy_token(got, want, label: str = "") -> bool:
    """Identical greedy token, except where the reference's own top-2 gap is inside
    the observed bf16 error (a tie at the working precision: either token is a
    correct argmax of the true logits to within rounding).  Ties break to the lowest
    id (reference argmax_lowest, model.cpp:457-462).  Exemptions are recorded."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    g, w = int(np.argmax(got)), int(np.argmax(want))
    GREEDY["checked"] += 1
    if g == w:
        GREEDY["identical"] += 1
        return True
    err = float(np.max(np.abs(got - want)))
    ok = want[w] - want[g] <= 2 * err
    if ok:
        label = label or sys._getframe(1).f_code.co_name
        GREEDY["exempt"].append(f"{label}: token {g} vs reference {w}, reference gap {want[w] - want[g]:.2e} "
                                f"<= 2 x max-abs err {err:.2e}")
    return ok


def record_sequence(got_tokens, want_tokens, label: str = ""):
    SEQ["checked"] += 1
    if list(got_tokens) != list(want_tokens):
        k = next(i for i, (a, b) in enumerate(zip(got_tokens, want_tokens)) if a != b) \
            if any(a != b for a, b in zip(got_tokens, want_tokens)) else min(len(got_tokens), len(want_tokens))
        SEQ["diverged"].append(f"{label}: first divergence at token {k}")
