"""Direct and iterative solves of A c = b (TEST-ONLY ORACLE).

* lu_solve: dense LU with partial pivoting (scipy) of the truncated Eq. 4
  matrix -- the "plain definition" of the interpolation coefficients c.
* ras_blocks / ras_apply: the restricted additive Schwarz method of §3.1
  (PAPER.md l.340-359): overlapping subdomains Omega_i with non-overlapping
  cores ~Omega_i; each local system A_i x_Omega_i = b_Omega_i is solved and
  "the values x outside of the subdomain ~Omega_i are discarded" (l.358).
  The paper does not define the subdomains; the block definition below is
  DESIGN.md reading R1 (shared, as a *definition*, with the CUDA path so the
  two preconditioners can be compared; the arithmetic is written here anew):
    - non-empty cells in Morton order of their cell coordinates; cell c joins
      core floor(P(c)/core_target), P = exclusive prefix of cell counts in
      that order; empty core ids are dropped; a last core with fewer than
      core_target/2 centres is merged into the one before it;
    - core members: cells in Morton order, each cell's sorted range ascending;
    - extended set: centres j (not in the core) with
      min_{i in core} d2_32(i,j) <= float32(ov^2), ov = overlap_sigmas*sigma,
      d2_32 = ((dx*dx + dy*dy) + dz*dz) in float32 from float32 coordinates;
      candidates are the cells within Chebyshev distance ceil(ov/h)+1 of a
      core cell;
    - local ordering: [non-core members ascending by sorted index] + [core];
    - local matrix B_i = A_i + shift*a*I (reading R17: a diagonal shift keeps
      the local inverses bounded when sigma/spacing makes A_i numerically
      singular; the paper's exact local solve is shift = 0).
* gmres: restarted GMRES(m) with right preconditioning (l.359 "in
  combination with any iterative method like the Krylov subspace methods";
  l.389-391 KSPSolve), modified Gram-Schmidt Arnoldi and Givens rotations as
  in Saad, "Iterative Methods for Sparse Linear Systems", Alg. 6.9/9.5.
  Stops on the TRUE relative residual ||b - A x|| / ||b|| (reading 6).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .cells import morton3
from .kernel import amplitude, dense_matrix


def lu_solve(centres, b, sigma, cutoff_sigmas=6.0, amp=None):
    A = dense_matrix(centres, sigma, cutoff_sigmas, amp)
    lu, piv = sla.lu_factor(A)
    return sla.lu_solve((lu, piv), np.asarray(b, dtype=np.float64))


def ras_blocks(cells, sigma: float, core_target: int = 512, overlap_sigmas: float = 1.0, core_cells=None):
    """List of dicts {core, ext} with indices in SORTED (cell-list) order.

    core_cells: optional boolean mask over the cells from which the cores are
    formed (a slab of a multi-GPU partition, reading R20: every rank
    builds the blocks of its own cells; their extended sets may reach into any
    cell); default all cells."""
    S = cells["sorted"].astype(np.float32)
    dim = cells["dim"]
    h = cells["h"]
    cs, ce = cells["cell_start"].astype(np.int64), cells["cell_end"].astype(np.int64)
    counts = ce - cs
    if core_cells is not None:
        counts = np.where(core_cells, counts, 0)
    nonempty = np.nonzero(counts > 0)[0]
    cx = nonempty % dim[0]
    cy = (nonempty // dim[0]) % dim[1]
    cz = nonempty // (dim[0] * dim[1])
    order = np.argsort(morton3(cx, cy, cz), kind="stable")
    cm = nonempty[order]
    P = np.concatenate([[0], np.cumsum(counts[cm])[:-1]])
    cid = P // core_target
    _, cid = np.unique(cid, return_inverse=True)
    ncore = int(cid.max()) + 1
    if ncore > 1:
        last = counts[cm][cid == ncore - 1].sum()
        if 2 * last < core_target:
            cid[cid == ncore - 1] = ncore - 2
            ncore -= 1
    ov = overlap_sigmas * sigma
    ov2 = np.float32(ov * ov)
    R = int(np.ceil(ov / h)) + 1
    coords = np.stack([cx, cy, cz], axis=1)[order]
    blocks = []
    for k in range(ncore):
        mine = np.nonzero(cid == k)[0]
        core = np.concatenate([np.arange(cs[c], ce[c]) for c in cm[mine]])
        # candidate cells: Chebyshev dilation by R of the core cells
        cc = coords[mine]
        lo = np.maximum(cc.min(axis=0) - R, 0)
        hi = np.minimum(cc.max(axis=0) + R, dim - 1)
        cand = []
        for z in range(lo[2], hi[2] + 1):
            for y in range(lo[1], hi[1] + 1):
                for x in range(lo[0], hi[0] + 1):
                    d = np.abs(cc - np.array([x, y, z])).max(axis=1).min()
                    if d <= R:
                        lin = x + dim[0] * (y + dim[1] * z)
                        if ce[lin] > cs[lin]:
                            cand.append(np.arange(cs[lin], ce[lin]))
        cand = np.setdiff1d(np.concatenate(cand), core) if cand else np.zeros(0, np.int64)
        if cand.size:
            Sc, Sj = S[core], S[cand]
            dmin = np.full(cand.size, np.inf, dtype=np.float32)
            for i in range(core.size):
                dx = Sj[:, 0] - Sc[i, 0]
                dy = Sj[:, 1] - Sc[i, 1]
                dz = Sj[:, 2] - Sc[i, 2]
                d2 = (dx * dx + dy * dy) + dz * dz
                np.minimum(dmin, d2, out=dmin)
            extra = np.sort(cand[dmin <= ov2])
        else:
            extra = cand
        blocks.append(dict(core=core, ext=np.concatenate([extra, core])))
    return blocks


def ras_apply(blocks, sorted_centres, r, sigma, cutoff_sigmas=6.0, amp=None, factors=None,
              shift: float = 0.0):
    """z = sum_i R~_i^T B_i^{-1} R_i r (restricted additive Schwarz), sorted order,
    B_i = A_i + shift * a * I (reading R17; shift = 0 is the paper's
    exact local solve A_i^{-1}).  `factors` caches the scipy LU of each B_i (fp64)."""
    r = np.asarray(r, dtype=np.float64)
    z = np.zeros_like(r)
    a = amplitude(sigma) if amp is None or amp <= 0 else float(amp)
    for k, blk in enumerate(blocks):
        ext = blk["ext"]
        if factors is not None and k in factors:
            f = factors[k]
        else:
            B = dense_matrix(sorted_centres[ext], sigma, cutoff_sigmas, amp)
            B[np.diag_indices_from(B)] += shift * a
            f = sla.lu_factor(B)
            if factors is not None:
                factors[k] = f
        y = sla.lu_solve(f, r[ext])
        nc = blk["core"].size
        z[blk["core"]] = y[-nc:]
    return z


def gmres(apply_A, b, restart: int = 30, rtol: float = 1e-8, maxit: int = 500,
          apply_M=None, x0=None):
    """Restarted right-preconditioned GMRES(m).  Returns (x, info)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    M = (lambda v: v) if apply_M is None else apply_M
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = np.linalg.norm(b)
    hist, it, breakdown = [], 0, False
    if bnorm == 0.0:
        return x, dict(iters=0, history=hist, converged=True, rel_residual=0.0, breakdown=False)
    while True:
        r = b - apply_A(x)
        beta = np.linalg.norm(r)
        if beta / bnorm <= rtol or it >= maxit or breakdown:
            break
        m = restart
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            Z[j] = M(V[j])
            w = apply_A(Z[j])
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            hj1 = H[j + 1, j]
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if hj1 <= 1e-14 * beta:
                breakdown = True
                break
            if abs(g[j + 1]) / bnorm <= rtol or it >= maxit:
                break
            V[j + 1] = w / hj1
        y = sla.solve_triangular(H[:k, :k], g[:k])
        x = x + Z[:k].T @ y
    rel = np.linalg.norm(b - apply_A(x)) / bnorm
    return x, dict(iters=it, history=hist, converged=rel <= rtol, rel_residual=rel,
                   breakdown=breakdown)
