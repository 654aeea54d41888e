"""Gaussian RBF entries and the brute-force truncated matvec (TEST-ONLY ORACLE).

Eq. 6 (Table I l.299):
    A_ij = 1/(sqrt(2 pi) sigma) * exp(-||x_i - x_j||^2 / (2 sigma^2))
Truncation (l.367-369: distant interactions "can be neglected"; reading 5 of
SURVEY.md §8(c)): A_ij = 0 when ||x_i - x_j||^2 > (n_c sigma)^2, n_c = 6.
Matvec f = A w is Eq. 4 (l.257-262) computed by brute force over ALL
centres, row by row, in fp64 on the fp32 canonical centres promoted to fp64.
"""
from __future__ import annotations

import numpy as np


def amplitude(sigma: float) -> float:
    """a = 1/(sqrt(2 pi) sigma), the Eq. 6 / Table I normalisation."""
    return 1.0 / (np.sqrt(2.0 * np.pi) * sigma)


def phi(r, sigma: float, amp: float | None = None, cutoff: float | None = None):
    """phi(r) = a exp(-r^2/(2 sigma^2)), exactly 0 for r > cutoff (Eq. 6)."""
    a = amplitude(sigma) if amp is None else amp
    r = np.asarray(r, dtype=np.float64)
    v = a * np.exp(-(r * r) / (2.0 * sigma * sigma))
    if cutoff is not None:
        v = np.where(r * r <= cutoff * cutoff, v, 0.0)
    return v


def _row_values(X, xi, sigma, amp, c2, truncate):
    d2 = (X[:, 0] - xi[0]) ** 2 + (X[:, 1] - xi[1]) ** 2 + (X[:, 2] - xi[2]) ** 2
    v = amp * np.exp(-d2 / (2.0 * sigma * sigma))
    if truncate:
        v[d2 > c2] = 0.0
    return v


def matvec(centres, w, sigma: float, cutoff_sigmas: float = 6.0, amp: float | None = None,
           rows=None, truncate: bool = True, targets=None):
    """f_i = sum_j A_ij w_j (Eq. 4), brute force over all j.

    centres: (n,3) canonical coordinates (fp32 promoted to fp64 here).
    rows:    optional subset of row indices i (sampled parity at large n).
    targets: optional (m,3) evaluation points instead of centres (Eq. 5).
    """
    X = np.asarray(centres, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    a = amplitude(sigma) if amp is None else amp
    c2 = (cutoff_sigmas * sigma) ** 2
    T = X if targets is None else np.asarray(targets, dtype=np.float64)
    idx = np.arange(T.shape[0]) if rows is None else np.asarray(rows)
    out = np.empty(idx.shape[0])
    n = X.shape[0]
    blk = max(1, int(4_000_000 // max(n, 1)))
    for s in range(0, idx.shape[0], blk):
        ii = idx[s:s + blk]
        if blk == 1:
            out[s] = _row_values(X, T[ii[0]], sigma, a, c2, truncate) @ w
            continue
        d2 = ((T[ii, None, 0] - X[None, :, 0]) ** 2 + (T[ii, None, 1] - X[None, :, 1]) ** 2
              + (T[ii, None, 2] - X[None, :, 2]) ** 2)
        v = a * np.exp(-d2 / (2.0 * sigma * sigma))
        if truncate:
            v[d2 > c2] = 0.0
        out[s:s + blk] = v @ w
    return out


def dense_matrix(centres, sigma: float, cutoff_sigmas: float = 6.0, amp: float | None = None,
                 truncate: bool = True):
    """The full matrix A of Eq. 4 (small n only)."""
    X = np.asarray(centres, dtype=np.float64)
    a = amplitude(sigma) if amp is None else amp
    d2 = ((X[:, None, 0] - X[None, :, 0]) ** 2 + (X[:, None, 1] - X[None, :, 1]) ** 2
          + (X[:, None, 2] - X[None, :, 2]) ** 2)
    A = a * np.exp(-d2 / (2.0 * sigma * sigma))
    if truncate:
        A[d2 > (cutoff_sigmas * sigma) ** 2] = 0.0
    return A


def pair_count(centres, sigma: float, cutoff_sigmas: float = 6.0, targets=None, rows=None):
    """Number of ordered (target, source) pairs with r^2 <= (n_c sigma)^2
    (the 'useful pairs' of SURVEY.md §8(d)), fp64 predicate."""
    X = np.asarray(centres, dtype=np.float64)
    T = X if targets is None else np.asarray(targets, dtype=np.float64)
    idx = np.arange(T.shape[0]) if rows is None else np.asarray(rows)
    c2 = (cutoff_sigmas * sigma) ** 2
    tot = 0
    for i in idx:
        t = T[i]
        d2 = (X[:, 0] - t[0]) ** 2 + (X[:, 1] - t[1]) ** 2 + (X[:, 2] - t[2]) ** 2
        tot += int((d2 <= c2).sum())
    return tot


def _mv_worker(args):
    centres, w, sigma, cutoff_sigmas, amp, rows, targets = args
    return matvec(centres, w, sigma, cutoff_sigmas, amp, rows=rows, targets=targets)


def matvec_parallel(centres, w, sigma, cutoff_sigmas=6.0, amp=None, rows=None,
                    targets=None, procs: int = 1):
    """Same as `matvec`, rows split over `procs` worker processes (used only to
    time the oracle on the host cores for bench.py's cpu_baseline)."""
    T = centres if targets is None else targets
    idx = np.arange(np.asarray(T).shape[0]) if rows is None else np.asarray(rows)
    if procs <= 1:
        return matvec(centres, w, sigma, cutoff_sigmas, amp, rows=idx, targets=targets)
    import multiprocessing as mp
    parts = np.array_split(idx, procs)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        outs = pool.map(_mv_worker, [(centres, w, sigma, cutoff_sigmas, amp, p, targets)
                                     for p in parts])
    return np.concatenate(outs)


def matvec_local(centres, w, sigma: float, cutoff_sigmas: float = 6.0, amp: float | None = None,
                 rows=None, targets=None):
    """The same f_i = sum_j A_ij w_j as `matvec` (Eq. 4 with the truncated Eq. 6
    entries), for SAMPLED rows of large problems (c3-c5 parity at >= 1e4 rows).

    Every entry with d2 > c^2 is exactly 0 (truncation, l.367-369), so row i only
    needs the centres within c of its target.  Those are found with a library
    range search -- scipy's cKDTree ball query at radius c (1 + 1e-9), a superset
    -- and then selected by the SAME fp64 predicate d2 <= c^2 and summed with the
    same fp64 entry formula as `matvec` (in ascending j).  Pinned against `matvec`
    in tests/test_oracle_kernel.py; only the rounding order of the sum differs.
    """
    from scipy.spatial import cKDTree
    X = np.asarray(centres, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    a = amplitude(sigma) if amp is None else amp
    c = cutoff_sigmas * sigma
    c2 = c * c
    T = X if targets is None else np.asarray(targets, dtype=np.float64)
    idx = np.arange(T.shape[0]) if rows is None else np.asarray(rows)
    tree = cKDTree(X)
    nbrs = tree.query_ball_point(T[idx], c * (1.0 + 1e-9))
    out = np.empty(idx.shape[0])
    for k, i in enumerate(idx):
        j = np.sort(np.asarray(nbrs[k], dtype=np.int64))
        t = T[i]
        d2 = (X[j, 0] - t[0]) ** 2 + (X[j, 1] - t[1]) ** 2 + (X[j, 2] - t[2]) ** 2
        keep = d2 <= c2
        out[k] = (a * np.exp(-d2[keep] / (2.0 * sigma * sigma))) @ w[j[keep]]
    return out
