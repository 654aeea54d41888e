"""BASELINE.json configs as seeded synthetic workloads.

Each config returns the *inputs* of the paper's Alg. 1 (PAPER.md l.310-323:
"point cloud X, surface normals n_i, evaluation grid xi") plus the kernel
and solver parameters the config names.  Nothing here computes the method.

Grid placement (SURVEY.md §8(c) reading 10): c1 uses [-1.2,1.2]^3 as the
config states; the others use a cube centred on the bounding-box centre of
the surface points with side = max extent * 1.05, n^3 inclusive nodes.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .surfaces import blobby, fibonacci_sphere, torus


@dataclass(frozen=True)
class Config:
    name: str
    kind: str                 # sphere | torus | blobby
    n: int                    # surface points N (centres = 3N)
    sigma: float
    delta: float
    grid_n: int
    cutoff_sigmas: float = 6.0
    restart: int = 50
    core_target: int = 512
    overlap_sigmas: float = 1.0
    precond_kind: int = 2     # 0 none, 1 block-Jacobi, 2 RAS (include/rbf.h)
    shift: float = 0.0        # local diagonal shift in units of a (reading R17)
    local_fp32: int = 0       # fp32 on-chip local inverses (reading R17)
    cgs_passes: int = 2       # Gram-Schmidt passes per Arnoldi step (1: CGS, 2: CGS2)
    cell_div: float = 3.999   # cell edge = cutoff / cell_div (the library default)
    kw: dict = field(default_factory=dict)


CONFIGS = {
    # BASELINE.json configs[0]: unit sphere, GMRES(30), 32^3 on [-1.2,1.2]^3
    "c1": Config("c1", "sphere", 1000, 0.1, 0.01, 32, restart=30,
                 core_target=512, overlap_sigmas=3.0),
    # configs[1]: torus R=1 r=0.35, N=20k, noise 1e-3, delta 0.005, sigma 0.05, 128^3
    # (noisy data at sigma/spacing 1.9: ill-posed, finding F1; the least-bad
    # preconditioner measured is RAS(128, 1 sigma) with a shift of 1.0 a: 0.18 in 100 its)
    "c2": Config("c2", "torus", 20000, 0.05, 0.005, 128, core_target=128, overlap_sigmas=1.0, shift=1.0,
                 kw=dict(R=1.0, r=0.35, noise=1e-3)),
    # configs[2]: blobby K=16, N=200k, 10x density, sigma 0.02 (delta = 0.1 sigma, reading 4)
    # c3-c5 sit at sigma/spacing ~3-4 where exact local solves stall GMRES (DESIGN.md
    # finding F4): shifted block-Jacobi local solves, fp32 on chip (reading R17)
    "c3": Config("c3", "blobby", 200000, 0.02, 0.002, 256, core_target=64, overlap_sigmas=0.0,
                 precond_kind=1, shift=0.003, local_fp32=1, cgs_passes=1, kw=dict(K=16, density_mod=True)),
    # configs[3]: blobby K=64, N=1M, sigma 0.01, 256^3  (the metric config)
    "c4": Config("c4", "blobby", 1000000, 0.01, 0.001, 256, core_target=64, overlap_sigmas=0.0,
                 precond_kind=1, shift=0.003, local_fp32=1, cgs_passes=1, kw=dict(K=64)),
    # configs[4]: blobby K=64 with 5 caps removed, N=10M, sigma 0.004, 512^3
    "c5": Config("c5", "blobby", 10000000, 0.004, 0.0004, 512, core_target=64, overlap_sigmas=0.0,
                 precond_kind=1, shift=0.003, local_fp32=1, cgs_passes=1, kw=dict(K=64, holes=5)),
}


def grid_box(cfg: Config, x: np.ndarray):
    """(lo[3], hi[3], n[3]) of the inclusive evaluation grid."""
    n = (cfg.grid_n,) * 3
    if cfg.name == "c1" or cfg.kind == "sphere":
        return (-1.2, -1.2, -1.2), (1.2, 1.2, 1.2), n
    mn, mx = x.min(axis=0), x.max(axis=0)
    ctr = 0.5 * (mn + mx)
    side = float((mx - mn).max()) * 1.05
    lo = tuple(float(v) for v in ctr - 0.5 * side)
    hi = tuple(float(v) for v in ctr + 0.5 * side)
    return lo, hi, n


def make_inputs(name: str, seed: int = 0, n: int | None = None, **over):
    """Seeded inputs for config `name`; `n` overrides the point count
    (parity-sized variants), other keyword overrides replace Config fields."""
    cfg = CONFIGS[name]
    if n is not None:
        cfg = replace(cfg, n=n)
    if over:
        cfg = replace(cfg, **over)
    if cfg.kind == "sphere":
        x, nrm = fibonacci_sphere(cfg.n)
    elif cfg.kind == "torus":
        x, nrm = torus(cfg.n, seed=seed, **cfg.kw)
    else:
        x, nrm = blobby(cfg.n, seed=seed, **cfg.kw)
    lo, hi, gn = grid_box(cfg, x)
    return dict(cfg=cfg, seed=seed, x=np.ascontiguousarray(x), normals=np.ascontiguousarray(nrm),
                delta=cfg.delta, sigma=cfg.sigma, cutoff_sigmas=cfg.cutoff_sigmas,
                grid_lo=lo, grid_hi=hi, grid_n=gn)
