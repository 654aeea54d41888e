"""float32 replica of the cell-list build (TEST-ONLY ORACLE).

The paper's "truncation area" (Alg. 2) and its locality
argument (§3.1 l.361-369) need, for every centre, the centres within the
cutoff.  The build bins centres into cubic cells; this module fixes that
binning's arithmetic exactly so the
GPU result can be compared bit for bit:

    h      = cell_edge (default cutoff/4), fp64
    lo     = float32(float64(min_a x_a) - h/2)          per axis a
    inv_h  = float32(1/h)
    dim_a  = floor(float32(float32(max_a x_a - lo_a) * inv_h)) + 1
    c_a(x) = clip(floor(float32(float32(x_a - lo_a) * inv_h)), 0, dim_a - 1)
    key    = c_x + dim_x (c_y + dim_y c_z)              (x fastest)
    perm   = stable argsort of key                      (sorted pos -> input id)
    cell_start[k] / cell_end[k] = searchsorted(sorted keys, k, left / right)

Morton codes (bit-interleave, x in bit 0) order the non-empty cells when
forming RAS cores (see oracle.solve.ras_blocks).
"""
from __future__ import annotations

import numpy as np


def cell_params(centres, cutoff: float, cell_edge: float | None = None):
    c = np.asarray(centres, dtype=np.float32)
    h = float(cutoff) / 4.0 if not cell_edge else float(cell_edge)
    mn = c.min(axis=0)
    mx = c.max(axis=0)
    lo = (mn.astype(np.float64) - 0.5 * h).astype(np.float32)
    inv_h = np.float32(1.0 / h)
    dim = np.floor((mx - lo) * inv_h).astype(np.int64) + 1
    return lo, inv_h, dim, h


def cell_coords(centres, lo, inv_h, dim):
    c = np.asarray(centres, dtype=np.float32)
    q = np.floor((c - lo.astype(np.float32)) * np.float32(inv_h)).astype(np.int64)
    return np.clip(q, 0, dim - 1)


def build(centres, cutoff: float, cell_edge: float | None = None):
    """Returns dict(lo, inv_h, dim, h, perm, sorted, keys, cell_start, cell_end, coords)."""
    c = np.asarray(centres, dtype=np.float32)
    lo, inv_h, dim, h = cell_params(c, cutoff, cell_edge)
    q = cell_coords(c, lo, inv_h, dim)
    key = q[:, 0] + dim[0] * (q[:, 1] + dim[1] * q[:, 2])
    perm = np.argsort(key, kind="stable")
    skey = key[perm]
    ncell = int(dim[0] * dim[1] * dim[2])
    cells = np.arange(ncell)
    cell_start = np.searchsorted(skey, cells, side="left").astype(np.int32)
    cell_end = np.searchsorted(skey, cells, side="right").astype(np.int32)
    return dict(lo=lo, inv_h=inv_h, dim=dim, h=h, perm=perm.astype(np.int32),
                sorted=c[perm], keys=skey, cell_start=cell_start, cell_end=cell_end,
                coords=q[perm])


def morton3(cx, cy, cz):
    """Interleave the low 21 bits of (cx, cy, cz); x in bit 0."""
    cx, cy, cz = (np.asarray(v, dtype=np.uint64) for v in (cx, cy, cz))
    m = np.zeros(np.broadcast(cx, cy, cz).shape, dtype=np.uint64)
    for b in range(21):
        one = np.uint64(1)
        m |= ((cx >> np.uint64(b)) & one) << np.uint64(3 * b)
        m |= ((cy >> np.uint64(b)) & one) << np.uint64(3 * b + 1)
        m |= ((cz >> np.uint64(b)) & one) << np.uint64(3 * b + 2)
    return m
