"""Density measures and sigma heuristics (TEST-ONLY ORACLE).

Eq. 7  q_X = 1/2 min_{i != j} ||x_i - x_j||
Eq. 8  (l.497-500)           h_{X,Omega} = sup_{x in Omega} min_j ||x - x_j||
                             (sup over a caller-supplied discrete sample of Omega)
l.614-619                    h_max = max_j min_{i != j} ||x_i - x_j||
Eq. 9  sigma ~ 2 q_X;  Eq. 10 sigma ~ h sqrt(2);  Eq. 11 h ~ h_max sqrt(2).
Pinned by Fig. 3 (l.505): 25 Halton points on [0,1]^2, q ~ 0.0597, h ~ 0.2667.
"""
from __future__ import annotations

import numpy as np


def _nn_dist(P, X, exclude_self: bool, chunk=1024):
    out = np.empty(P.shape[0])
    for s in range(0, P.shape[0], chunk):
        p = P[s:s + chunk]
        d2 = ((p[:, None, :] - X[None, :, :]) ** 2).sum(axis=2)
        if exclude_self:
            d2[np.arange(p.shape[0]), np.arange(s, s + p.shape[0])] = np.inf
        out[s:s + chunk] = np.sqrt(d2.min(axis=1))
    return out


def separation_distance(X):
    X = np.asarray(X, dtype=np.float64)
    return 0.5 * _nn_dist(X, X, True).min()


def h_max(X):
    X = np.asarray(X, dtype=np.float64)
    return _nn_dist(X, X, True).max()


def fill_distance(X, omega_sample):
    return _nn_dist(np.asarray(omega_sample, dtype=np.float64),
                    np.asarray(X, dtype=np.float64), False).max()


def halton(n: int, base: int, start: int = 1):
    """Radical-inverse (van der Corput) sequence in `base`, indices start..start+n-1."""
    out = np.empty(n)
    for k in range(n):
        i, f, r = start + k, 1.0, 0.0
        while i > 0:
            f /= base
            r += f * (i % base)
            i //= base
        out[k] = r
    return out


def sigma_heuristics(X, omega_sample=None):
    q = separation_distance(X)
    hm = h_max(X)
    out = dict(q=q, h_max=hm, sigma_q=2.0 * q, sigma_hmax=hm * np.sqrt(2.0) * np.sqrt(2.0))
    if omega_sample is not None:
        h = fill_distance(X, omega_sample)
        out.update(h=h, sigma_h=h * np.sqrt(2.0))
    return out
