"""Pins for oracle.mesh (masked marching tetrahedra, reading R24): topology
(closed, consistently oriented 2-manifolds with the Euler characteristic of
the sphere / torus), the divergence-theorem volume of a sphere, exactness on
linear fields, agreement with the independently pinned axis-edge zero
crossings, and the eps mask as a restriction of the unmasked mesh."""
from collections import Counter

import numpy as np
import pytest

from oracle import grid as G
from oracle import mesh as M


def _field(fn, lo, hi, n):
    return fn(G.nodes(lo, hi, n)).astype(np.float32)


def _topology(V, T):
    """(directed-edge multiplicities, referenced vertex count, undirected edges)."""
    de = Counter()
    for a, b, c in T:
        for e in ((a, b), (b, c), (c, a)):
            de[e] += 1
    und = {tuple(sorted(e)) for e in de}
    return de, len(np.unique(T)), len(und)


def _signed_volume(V, T):
    p0, p1, p2 = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    return np.einsum("ij,ij->i", p0, np.cross(p1, p2)).sum() / 6.0


def _closed_oriented(V, T):
    de, nv, ne = _topology(V, T)
    # every directed edge exactly once, its reverse exactly once
    assert all(m == 1 for m in de.values())
    assert all(de[(b, a)] == 1 for (a, b) in de)
    return nv - ne + len(T)


def test_sphere_closed_euler_volume():
    lo, hi, n = (-1.0,) * 3, (1.0,) * 3, (21, 21, 21)
    r = 0.73   # no node exactly on the sphere (F = 0 sides with the outside)
    F = _field(lambda P: np.linalg.norm(P, axis=1) - r, lo, hi, n)
    V, T = M.marching_tets(F, lo, hi, n, np.ones(F.size, bool))
    assert _closed_oriented(V, T) == 2                      # genus 0
    vol = _signed_volume(V, T)
    assert vol == pytest.approx(4 / 3 * np.pi * r ** 3, rel=0.03)   # outward normals
    h = 0.1
    assert np.abs(np.linalg.norm(V, axis=1) - r).max() < h * h
    # -F: inside and outside swap, normals point inward, same vertices
    V2, T2 = M.marching_tets(-F, lo, hi, n, np.ones(F.size, bool))
    np.testing.assert_array_equal(V2, V)
    assert _signed_volume(V2, T2) == pytest.approx(-vol, rel=1e-12)


def test_torus_euler_characteristic():
    lo, hi, n = (-1.5, -1.5, -0.6), (1.5, 1.5, 0.6), (31, 31, 13)
    R0, r0 = 1.0, 0.35

    def sdf(P):
        q = np.hypot(P[:, 0], P[:, 1]) - R0
        return np.hypot(q, P[:, 2]) - r0
    F = _field(sdf, lo, hi, n)
    V, T = M.marching_tets(F, lo, hi, n, np.ones(F.size, bool))
    assert _closed_oriented(V, T) == 0                      # genus 1
    assert _signed_volume(V, T) == pytest.approx(2 * np.pi ** 2 * R0 * r0 ** 2, rel=0.05)


def test_linear_field_is_exact():
    """The piecewise-linear interpolant of a linear field is the field: every
    vertex lies on the plane (to rounding) and every triangle normal points
    along +grad F; a horizontal plane's mesh area is the box's cross-section."""
    lo, hi, n = (0.0, 0.0, 0.0), (1.0, 2.0, 1.5), (6, 9, 7)
    g = np.array([0.3, -0.5, 0.8])
    F = _field(lambda P: P @ g - 0.2, lo, hi, n)
    V, T, E = M.marching_tets(F, lo, hi, n, np.ones(F.size, bool), return_edges=True)
    assert len(T) > 20
    # the vertices solve the fp32-rounded field's interpolant; against the exact
    # plane the residual is the fp32 rounding of the node values
    assert np.abs(V @ g - 0.2).max() < 1e-6
    nrm = np.cross(V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]])
    area = 0.5 * np.linalg.norm(nrm, axis=1)
    big = area > 1e-9
    assert np.all(nrm[big] @ g > 0)
    Fz = _field(lambda P: P[:, 2] - 0.55, lo, hi, n)
    Vz, Tz = M.marching_tets(Fz, lo, hi, n, np.ones(Fz.size, bool))
    nz = np.cross(Vz[Tz[:, 1]] - Vz[Tz[:, 0]], Vz[Tz[:, 2]] - Vz[Tz[:, 0]])
    assert 0.5 * np.linalg.norm(nz, axis=1).sum() == pytest.approx(1.0 * 2.0, rel=1e-6)
    assert np.all(nz[:, 2] > 0)


def test_axis_edge_vertices_equal_zero_crossings():
    lo, hi, n = (-1.5,) * 3, (1.5,) * 3, (23, 23, 23)
    F = _field(lambda P: np.linalg.norm(P, axis=1) - 1.0, lo, hi, n)
    rng = np.random.default_rng(3)
    v = rng.normal(size=(2000, 3))
    data = v / np.linalg.norm(v, axis=1, keepdims=True)
    data = data[data[:, 2] > -0.3]
    eps = 0.35
    near = M.near_mask(lo, hi, n, data, eps)
    V, T, E = M.marching_tets(F, lo, hi, n, near, return_edges=True)
    zc = G.zero_crossings(F, lo, hi, n, data, eps)
    axis_pts = np.concatenate([V[E[:, 1] == a] for a in range(3)])
    # zero_crossings orders by (axis, lower node); the mesh by (node, direction)
    # within one axis both are ascending in the lower node: equal point for point
    np.testing.assert_array_equal(axis_pts, zc)


def test_mask_restricts_unmasked_mesh():
    """The masked mesh is the unmasked one minus the cubes with a corner outside
    M_ext^eps: every masked triangle (in edge ids) is an unmasked triangle."""
    lo, hi, n = (-1.2,) * 3, (1.2,) * 3, (17, 17, 17)
    F = _field(lambda P: np.linalg.norm(P, axis=1) - 0.9, lo, hi, n)
    rng = np.random.default_rng(1)
    v = rng.normal(size=(600, 3))
    data = 0.9 * v / np.linalg.norm(v, axis=1, keepdims=True)
    data = data[data[:, 0] > 0.0]
    near = M.near_mask(lo, hi, n, data, 0.3)
    Vm, Tm, Em = M.marching_tets(F, lo, hi, n, near, return_edges=True)
    Vf, Tf, Ef = M.marching_tets(F, lo, hi, n, np.ones(F.size, bool), return_edges=True)
    key_m = [tuple(map(tuple, Em[t])) for t in Tm]
    key_f = {tuple(map(tuple, Ef[t])) for t in Tf}
    assert 0 < len(key_m) < len(key_f)
    assert all(k in key_f for k in key_m)
    # every vertex of the masked mesh lies on an edge with both ends near
    assert np.all(near[Em[:, 0]])
    # open surface: some directed edges have no reverse (the mask boundary)
    de, _, _ = _topology(Vm, Tm)
    assert any(de[(b, a)] == 0 for (a, b) in de)
    assert np.abs(np.linalg.norm(Vm, axis=1) - 0.9).max() < 0.15 ** 2
