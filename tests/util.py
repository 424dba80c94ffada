"""Shared numeric criteria for the parity tests."""
import numpy as np

F32_TOL = 1e-3   # north star: fp32 path max-abs <= 1e-3
BF16_REL = 2e-2  # north star: bf16 path logits rel-err <= 2e-2 (max |a-b| / max |b|)


def rel(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def same_greedy_token(got, want) -> bool:
    """Identical greedy token, except where the reference's own top-2 gap is inside
    the observed bf16 error (a tie at the working precision: either token is a
    correct argmax of the true logits to within rounding).  Ties break to the lowest
    id (reference argmax_lowest, model.cpp:457-462)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    g, w = int(np.argmax(got)), int(np.argmax(want))
    if g == w:
        return True
    err = float(np.max(np.abs(got - want)))
    return want[w] - want[g] <= 2 * err
