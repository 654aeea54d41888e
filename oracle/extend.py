"""Extended interpolation set and labels (TEST-ONLY ORACLE).

PAPER.md §2.1.1 (l.140-162): for each x_i with unit normal n_i,
    x_{N+i}  = x_i + delta n_i   (outside, X_delta^+)
    x_{2N+i} = x_i - delta n_i   (inside,  X_delta^-)
and X_ext = X u X_delta^+ u X_delta^-, ordered X, X^+, X^- (l.158-162).
§2.1.2 (l.186-193): P_f = 0 on X, +1 on X^+, -1 on X^-.  BASELINE configs use
0/+delta/-delta instead (SURVEY.md §8(c) reading 2); `value` selects it.

Canonical inputs: the sums are formed in fp64 (one
multiply, one add, each correctly rounded) and rounded ONCE to fp32.
"""
from __future__ import annotations

import numpy as np


def extend(x, normals, delta: float):
    """(3N,3) float32 centres ordered [X; X + delta n; X - delta n]."""
    x = np.asarray(x, dtype=np.float64)
    n = np.asarray(normals, dtype=np.float64)
    dn = delta * n
    ext = np.concatenate([x, x + dn, x - dn], axis=0)
    return ext.astype(np.float32)


def labels(N: int, value: float):
    """(3N,) fp64 right-hand side b = [0 x N, +value x N, -value x N]."""
    return np.concatenate([np.zeros(N), np.full(N, float(value)), np.full(N, -float(value))])
