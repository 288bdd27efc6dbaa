"""Shared parity bound of the GPU tests (BASELINE.json north_star, SURVEY §8(c)
"Parity contract"): iterates within a relative error of 1e-9.

`close(a, b)` holds when BOTH
  * the norm bound   ||a - b||_2   <= rtol ||b||_2 + 1e-14 sqrt(len), and
  * the entry bound  max_i |a_i - b_i| <= rtol max(||b||_inf, 1)
hold, so one entry off by more than rtol of the vector's scale fails even when the
vector is long (the norm alone would hide it: VERDICT r1 weak #2).
"""
import math

import numpy as np


def close(a, b, rtol=1e-9):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    if a.shape != b.shape:
        return False
    if b.size == 0:
        return True
    d = np.abs(a - b)
    norm_ok = np.linalg.norm(a - b) <= rtol * np.linalg.norm(b) + 1e-14 * math.sqrt(b.size)
    entry_ok = d.max() <= rtol * max(np.abs(b).max(), 1.0)
    return bool(norm_ok and entry_ok)


def worst(a, b):
    """(index, |a_i - b_i|, b_i) of the largest entry difference, for messages."""
    d = np.abs(np.asarray(a, float) - np.asarray(b, float))
    i = int(d.argmax()) if d.size else -1
    return (i, float(d[i]), float(np.asarray(b)[i])) if d.size else None
