"""Evaluation of the interpolant on a regular grid (TEST-ONLY ORACLE).

Eq. 5: P_f(xi_k) = sum_j phi(||xi_k - x_j||) c_j,
evaluated "on a dense grid of a bounding box" (§2.1.3 l.202-204).  The grid
is inclusive linspace per axis, nodes ordered x fastest (reading 10):
    xi_(i,j,k) = lo + (i,j,k) * (hi - lo)/(n - 1),  flat index i + nx (j + ny k).
Zero set: M* ~ M_ext^eps cap S_0 (l.211-221): linear interpolation along grid
edges whose endpoint values have strictly opposite signs, keeping only edges
whose both endpoints are within eps of a data point (reading 11).
"""
from __future__ import annotations

import numpy as np

from .kernel import matvec


def axes(lo, hi, n):
    return [lo[a] + np.arange(n[a], dtype=np.float64) * ((hi[a] - lo[a]) / (n[a] - 1))
            for a in range(3)]


def nodes(lo, hi, n, flat=None):
    """(M,3) node coordinates (x fastest); `flat` selects a subset of flat ids."""
    ax = axes(lo, hi, n)
    if flat is None:
        flat = np.arange(n[0] * n[1] * n[2])
    flat = np.asarray(flat, dtype=np.int64)
    i = flat % n[0]
    j = (flat // n[0]) % n[1]
    k = flat // (n[0] * n[1])
    return np.stack([ax[0][i], ax[1][j], ax[2][k]], axis=1)


def evaluate(centres, w, sigma, lo, hi, n, cutoff_sigmas=6.0, amp=None, flat=None):
    """Brute-force P_f on all (or the `flat`-selected) grid nodes."""
    return matvec(centres, w, sigma, cutoff_sigmas, amp, targets=nodes(lo, hi, n, flat))


def _min_dist(P, X, chunk=2048):
    out = np.empty(P.shape[0])
    for s in range(0, P.shape[0], chunk):
        p = P[s:s + chunk]
        d2 = ((p[:, None, :] - X[None, :, :]) ** 2).sum(axis=2)
        out[s:s + chunk] = np.sqrt(d2.min(axis=1))
    return out


def zero_crossings(F, lo, hi, n, data_points, eps):
    """Points of the masked zero set: (K,3) array."""
    F = np.asarray(F, dtype=np.float64).reshape(n[2], n[1], n[0])  # [k][j][i]
    P = nodes(lo, hi, n)
    near = (_min_dist(P, np.asarray(data_points, dtype=np.float64)) <= eps).reshape(F.shape)
    P = P.reshape(n[2], n[1], n[0], 3)
    out = []
    for axis in (2, 1, 0):  # i (x), j (y), k (z) directions in [k][j][i] layout
        sl_a = [slice(None)] * 3
        sl_b = [slice(None)] * 3
        sl_a[axis] = slice(0, -1)
        sl_b[axis] = slice(1, None)
        fa, fb = F[tuple(sl_a)], F[tuple(sl_b)]
        m = (fa * fb < 0) & near[tuple(sl_a)] & near[tuple(sl_b)]
        t = fa[m] / (fa[m] - fb[m])
        pa, pb = P[tuple(sl_a)][m], P[tuple(sl_b)][m]
        out.append(pa + t[:, None] * (pb - pa))
    return np.concatenate(out, axis=0)
