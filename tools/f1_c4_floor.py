"""Finding F1 at c4, from the oracle only: can the true relative
residual ||b - A w|| / ||b|| of the 6-sigma-truncated c4 system reach the north
star's 1e-6, and with which solver?

Patches of the c4 cloud (BASELINE configs[3], synth seed 0) of growing radius
around surface point 0, their +-delta extension and b = [0; +delta; -delta]
(oracle.extend) are solved in fp64 by

  * dense LU (oracle.solve.lu_solve, the plain definition):
      lu_res       ||b - A w_LU|| / ||b||
      arith_floor  u ||(|A| |w_LU|)|| / ||b||, u = 2^-53: the rounding noise of
                   evaluating the residual itself
      w_over_b     ||w_LU|| / ||b||
  * the spectrum of the truncated A (eigh): negative eigenvalues, and the share
    of ||b|| in the eigen-directions with |lambda| below 1e-12 .. 1e2 a -- a
    Krylov method reaches a residual r only after resolving every component of
    b outside the modes that hold r of it ("resolve_to_*": the |lambda| down to
    which that is);
  * fp64 right-preconditioned GMRES(50) (oracle.solve.gmres) for `F1_ITS`
    iterations with the preconditioners tried for the gate:
      bj(core, shift)       block-Jacobi of shifted local blocks (the benchmarked
                            one is core 64, shift 3e-3 a)
      ras(core, ov, shift)  restricted additive Schwarz
      2lvl-add / 2lvl-mult  bj(64, 3e-3) plus an exact coarse correction on a
                            piecewise-constant space (per block and per layer
                            0 / +delta / -delta)
  * and at radius 0.07 the same GMRES for delta = 0.1 .. 1.65 sigma (1.65 sigma
    = the paper's "1% of the bounding box" rule, at c4).

    python tools/f1_c4_floor.py > profiles/r02/f1_c4.jsonl   (~15 min on 8 cores)
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cells as OC  # noqa: E402
from oracle import extend as OE  # noqa: E402
from oracle import kernel as OK  # noqa: E402
from oracle import solve as OS  # noqa: E402
from synth import make_inputs  # noqa: E402

ITS = int(os.environ.get("F1_ITS", "300"))


def patch(d, r, delta):
    x, nrm = d["x"], d["normals"]
    sel = np.linalg.norm(x - x[0], axis=1) <= r
    X = OE.extend(x[sel], nrm[sel], delta).astype(np.float64)
    b = OE.labels(int(sel.sum()), delta).astype(np.float32).astype(np.float64)
    return X, b, int(sel.sum())


def precond_bj(X, oc, sigma, core, overlap, shift):
    blocks = OS.ras_blocks(oc, sigma, core, overlap)
    perm = oc["perm"]
    factors = {}

    def M(v):
        z = np.empty_like(v)
        z[perm] = OS.ras_apply(blocks, oc["sorted"], v[perm], sigma, factors=factors, shift=shift)
        return z
    return M, blocks


def coarse_space(blocks, perm, n, N):
    layer = np.arange(n) // N          # caller order: 0 surface, 1 +delta, 2 -delta
    cols = []
    for blk in blocks:
        idx = perm[blk["core"]]
        for L in range(3):
            m = idx[layer[idx] == L]
            if m.size:
                z = np.zeros(n)
                z[m] = 1.0
                cols.append(z)
    return np.array(cols).T


def gmres_run(A, b, M):
    t = time.time()
    w, info = OS.gmres(lambda v: A @ v, b, restart=50, rtol=1e-8, maxit=ITS, apply_M=M)
    h = info["history"]
    return dict(res=float(np.linalg.norm(b - A @ w) / np.linalg.norm(b)), its=info["iters"],
                est_at=[float(h[k - 1]) for k in (50, 100, 200, 300) if k <= len(h)], s=round(time.time() - t, 1))


def study(d, r, delta, full=True):
    sigma = d["sigma"]
    X, b, N = patch(d, r, delta)
    n = len(X)
    a = OK.amplitude(sigma)
    A = OK.dense_matrix(X, sigma)
    out = dict(radius=r, delta_over_sigma=round(delta / sigma, 3), surface_points=N, centres=n)
    w = OS.lu_solve(X, b, sigma)
    out.update(lu_res=float(np.linalg.norm(b - A @ w) / np.linalg.norm(b)),
               arith_floor=float(2.0 ** -53 * np.linalg.norm(np.abs(A) @ np.abs(w)) / np.linalg.norm(b)),
               w_over_b=float(np.linalg.norm(w) / np.linalg.norm(b)))
    oc = OC.build(X.astype(np.float32), 6 * sigma, cell_edge=6 * sigma / 3.999)
    if full:
        lam, V = np.linalg.eigh(A)
        beta = V.T @ b
        bn = np.linalg.norm(b)
        out.update(neg_eigs=int((lam < 0).sum()), lam_min_over_a=float(lam.min() / a),
                   lam_max_over_a=float(lam.max() / a), min_abs_lam_over_a=float(np.abs(lam).min() / a))
        out["b_share_below"] = {f"{t:g}a": dict(modes=int((np.abs(lam) < t * a).sum()),
                                                 share=float(np.linalg.norm(beta[np.abs(lam) < t * a]) / bn))
                                for t in (1e-12, 1e-10, 1e-8, 1e-6, 1e-4, 1e-2, 1.0)}
        order = np.argsort(np.abs(lam))
        cum = np.sqrt(np.cumsum(beta[order] ** 2)) / bn
        for tgt in (1e-4, 1e-6):
            k = min(int(np.searchsorted(cum, tgt)), n - 1)
            out[f"resolve_to_{tgt:g}"] = dict(modes_to_resolve=n - k, down_to_lam_over_a=float(abs(lam[order[k]]) / a))
    runs = {}
    cases = [("bj", 64, 0.0, 3e-3), ("bj", 64, 0.0, 1e-4), ("bj", 512, 0.0, 1e-3), ("bj", 512, 0.0, 1e-5),
             ("ras", 512, 1.0, 0.0), ("ras", 512, 1.0, 0.1)] if full else [("bj", 64, 0.0, 3e-3),
                                                                           ("bj", 512, 0.0, 1e-3)]
    for kind, core, ov, sh in cases:
        M, blocks = precond_bj(X, oc, sigma, core, ov * sigma, sh)
        runs[f"{kind}({core},{ov}sigma,{sh:g}a)"] = gmres_run(A, b, M)
    if full:
        M, blocks = precond_bj(X, oc, sigma, 64, 0.0, 3e-3)
        Z = coarse_space(blocks, oc["perm"], n, N)
        lu = sla.lu_factor(Z.T @ A @ Z)

        def Q(v):
            return Z @ sla.lu_solve(lu, Z.T @ v)

        runs[f"2lvl-add(bj64,3e-3a; coarse {Z.shape[1]})"] = gmres_run(A, b, lambda v: M(v) + Q(v))

        def Mm(v):
            q = Q(v)
            return q + M(v - A @ q)

        runs[f"2lvl-mult(bj64,3e-3a; coarse {Z.shape[1]})"] = gmres_run(A, b, Mm)
    out["gmres"] = runs
    return out


def main():
    d = make_inputs("c4")
    sigma = d["sigma"]
    for r in (0.05, 0.07, 0.09):
        print(json.dumps(study(d, r, d["delta"])), flush=True)
    for fac in (0.3, 0.5, 1.0, 1.65):
        print(json.dumps(study(d, 0.07, fac * sigma, full=False)), flush=True)


if __name__ == "__main__":
    main()
