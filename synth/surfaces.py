"""Seeded analytic surfaces: positions and exact unit normals in fp64.

Readings:
  12  Fibonacci sphere  phi_i = arccos(1 - 2(i+1/2)/N), theta_i = pi(1+sqrt5)(i+1/2)
  13  torus             theta by rejection with acceptance (R + r cos t)/(R + r),
                        phi uniform, normals from the clean point, then isotropic
                        N(0, noise^2) added to positions only
  14  blobby family     g(x) = sum_k exp(-|x-c_k|^2 / (2 s_k^2)) - 1/2, sampled
                        as a thin band |g| < 0.004 |grad g| of uniform candidates,
                        projected by 4 Newton steps; outward normal -grad g/|grad g|

These are the stand-ins for the paper's "scanned surface" point clouds
(§1, §4.1 "synthetic dataset"); the paper's own clouds (382-point
sphere, Stanford bunny) are not available and are not recreated.
"""
from __future__ import annotations

import numpy as np


def fibonacci_sphere(n: int):
    """Unit sphere, N points, outward normals == positions (reading 12)."""
    i = np.arange(n, dtype=np.float64) + 0.5
    phi = np.arccos(1.0 - 2.0 * i / n)
    theta = np.pi * (1.0 + np.sqrt(5.0)) * i
    x = np.stack([np.cos(theta) * np.sin(phi),
                  np.sin(theta) * np.sin(phi),
                  np.cos(phi)], axis=1)
    return x, x.copy()


def torus(n: int, R: float = 1.0, r: float = 0.35, noise: float = 1e-3, seed: int = 0):
    """Area-uniform torus samples with analytic normals and position noise
    (reading 13).  Draw order per chunk: (theta, u) candidates, then phi for
    the accepted ones; after all chunks, the noise for the first n points."""
    rng = np.random.default_rng(seed)
    thetas = []
    have = 0
    while have < n:
        m = max(1024, 2 * (n - have))
        t = rng.uniform(0.0, 2.0 * np.pi, m)
        u = rng.uniform(0.0, 1.0, m)
        keep = u < (R + r * np.cos(t)) / (R + r)
        thetas.append(t[keep])
        have += int(keep.sum())
    theta = np.concatenate(thetas)[:n]
    phi = rng.uniform(0.0, 2.0 * np.pi, n)
    ct, st = np.cos(theta), np.sin(theta)
    cp, sp = np.cos(phi), np.sin(phi)
    x = np.stack([(R + r * ct) * cp, (R + r * ct) * sp, r * st], axis=1)
    nrm = np.stack([ct * cp, ct * sp, st], axis=1)
    x = x + rng.normal(0.0, noise, size=x.shape)
    return x, nrm


def _blobby_params(K: int, seed: int, s0: float):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-0.6, 0.6, size=(K, 3))
    s = s0 * rng.uniform(0.7, 1.3, size=K)
    return rng, c, s


def blobby_field(x: np.ndarray, c: np.ndarray, s: np.ndarray):
    """g and grad g of the sum-of-Gaussians blob at points x (M x 3)."""
    px, py, pz = (np.ascontiguousarray(x[:, a]) for a in range(3))
    g = np.full(x.shape[0], -0.5)
    gx, gy, gz = np.zeros_like(g), np.zeros_like(g), np.zeros_like(g)
    dx, dy, dz = np.empty_like(g), np.empty_like(g), np.empty_like(g)
    e, t = np.empty_like(g), np.empty_like(g)
    for k in range(c.shape[0]):
        np.subtract(px, c[k, 0], out=dx)
        np.subtract(py, c[k, 1], out=dy)
        np.subtract(pz, c[k, 2], out=dz)
        np.multiply(dx, dx, out=e)
        np.multiply(dy, dy, out=t)
        e += t
        np.multiply(dz, dz, out=t)
        e += t
        e *= -1.0 / (2.0 * s[k] * s[k])
        np.exp(e, out=e)
        g += e
        e *= 1.0 / (s[k] * s[k])
        np.multiply(dx, e, out=t)
        gx -= t
        np.multiply(dy, e, out=t)
        gy -= t
        np.multiply(dz, e, out=t)
        gz -= t
    return g, np.stack([gx, gy, gz], axis=1)


def blobby(n: int, K: int = 16, seed: int = 0, s0: float | None = None,
           density_mod: bool = False, holes: int = 0, hole_frac: float = 0.08,
           coarse: int = 128, chunk: int = 1 << 17):
    """Points on the zero set of the blobby field (reading 14).

    density_mod: accept with p = 0.1 + 0.9 (x+1)/2 (10x density across x).
    holes: number of seeded spherical caps removed (hole_frac of the points,
    by the quantile of distance to the nearest cap centre).

    A coarse-grid prefilter keeps only candidate cells that can intersect the
    acceptance band; candidates are uniform inside the kept cells, so the
    accepted set is the same distribution as uniform candidates in [-1,1]^3.
    """
    if s0 is None:
        s0 = 0.25 if K <= 16 else 0.15
    rng, c, s = _blobby_params(K, seed, s0)
    band = 0.004
    # coarse prefilter over [-1,1]^3
    h = 2.0 / coarse
    ax = -1.0 + h * (np.arange(coarse) + 0.5)
    keep = np.zeros((coarse, coarse, coarse), dtype=bool)
    hd = 0.5 * h * np.sqrt(3.0)
    for iz in range(coarse):
        zz, yy, xx = np.meshgrid([ax[iz]], ax, ax, indexing="ij")
        p = np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)
        g, gr = blobby_field(p, c, s)
        gn = np.sqrt((gr * gr).sum(axis=1))
        keep[iz] = (np.abs(g) <= 1.5 * (band + hd) * gn + 1e-12).reshape(coarse, coarse)
    # dilate by one cell (conservative)
    dil = keep.copy()
    for a in range(3):
        dil |= np.roll(keep, 1, axis=a) | np.roll(keep, -1, axis=a)
    kz, ky, kx = np.nonzero(dil)
    cell_lo = np.stack([-1.0 + h * kx, -1.0 + h * ky, -1.0 + h * kz], axis=1)
    need = n if holes == 0 else int(np.ceil(n / (1.0 - hole_frac))) + 1
    pts, nrms = [], []
    have = 0
    while have < need:
        ci = rng.integers(0, cell_lo.shape[0], chunk)
        x = cell_lo[ci] + h * rng.random((chunk, 3))
        u = rng.random(chunk)
        g, gr = blobby_field(x, c, s)
        gn = np.sqrt((gr * gr).sum(axis=1))
        ok = np.abs(g) < band * gn
        if density_mod:
            ok &= u < 0.1 + 0.9 * (x[:, 0] + 1.0) / 2.0
        x = x[ok]
        for _ in range(4):
            g, gr = blobby_field(x, c, s)
            x = x - (g / (gr * gr).sum(axis=1))[:, None] * gr
        g, gr = blobby_field(x, c, s)
        ok = (np.abs(g) < 1e-12) & np.all(np.abs(x) <= 1.0, axis=1)
        x, gr = x[ok], gr[ok]
        pts.append(x)
        nrms.append(-gr / np.sqrt((gr * gr).sum(axis=1))[:, None])
        have += x.shape[0]
    x = np.concatenate(pts)[:need]
    nrm = np.concatenate(nrms)[:need]
    if holes:
        idx = rng.choice(need, size=holes, replace=False)
        caps = x[idx]
        d = np.full(need, np.inf)
        for cc in caps:
            d = np.minimum(d, np.sqrt(((x - cc) ** 2).sum(axis=1)))
        thr = np.quantile(d, hole_frac)
        sel = d > thr
        x, nrm = x[sel][:n], nrm[sel][:n]
    return x, nrm
