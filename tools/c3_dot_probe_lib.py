"""Exactly rounded dot product (parity evidence helper for tools/c3_*.py)."""
import math

import numpy as np


def exact_dot(x, y) -> float:
    """Correctly rounded sum of the exact products x_i y_i (Dekker split + fsum)."""
    a = np.asarray(x, dtype=float).ravel()
    b = np.asarray(y, dtype=float).ravel()
    p = a * b
    c = 134217729.0  # 2^27 + 1
    ah = a * c
    ah = ah - (ah - a)
    al = a - ah
    bh_ = b * c
    bh_ = bh_ - (bh_ - b)
    bl = b - bh_
    err = ((ah * bh_ - p) + ah * bl + al * bh_) + al * bl  # p + err == a b exactly
    return math.fsum(np.concatenate([p, err]))
