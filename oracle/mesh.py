"""Triangle mesh of the masked zero iso-surface (TEST-ONLY ORACLE).

Alg. 1 step 4 renders the zero iso-surface of P_f from
its values on the grid xi (MATLAB ``isosurface``); §2.1.3 (l.200-221) keeps
only the part inside the eps-surrounding of the data,
M* ~ M_ext^eps cap S_0.  Reading R24 fixes the polygonisation:
marching tetrahedra on the Kuhn (Freudenthal) split of every grid cube --
the piecewise-linear interpolant of the node values on each tetrahedron has a
planar zero set, and neighbouring cubes split their shared faces along the
same diagonal, so the mesh is watertight without ambiguity tables.

Definitions (both sides follow them; this module writes them out plainly):
  * node v = (i, j, k), flat id i + nx (j + ny k) (oracle.grid layout);
    "inside" iff F[v] < 0;  near[v] iff some data point lies within eps
    (the mask of oracle.grid.zero_crossings, fp64 distances);
  * edge (v, d), d in D7 = (1,0,0) (0,1,0) (0,0,1) (1,1,0) (1,0,1) (0,1,1)
    (1,1,1) (this order), with v + d inside the grid.  It carries a vertex iff
    near[v] and near[v+d] and inside(v) != inside(v+d); the vertex is
    p_v + t (p_{v+d} - p_v) per coordinate, t = F_v / (F_v - F_{v+d}) in fp64
    of the fp32 field (the formula of oracle.grid.zero_crossings).  Vertices
    are numbered in (v, d) order;
  * cube with lower corner v (i < nx-1, j < ny-1, k < nz-1) is polygonised iff
    all 8 corners are near; its 6 tetrahedra, for the axis permutations
    pi = (x,y,z) (x,z,y) (y,x,z) (y,z,x) (z,x,y) (z,y,x) in this order, are
    q0 = v, q1 = q0 + e_pi0, q2 = q1 + e_pi1, q3 = v + (1,1,1);
  * in a tetrahedron with inside set I: |I| = 0 or 4 -> nothing; |I| = 1 or 3
    -> a = the lone corner, b < c < d the others (tet order), triangle
    (P_ab, P_ac, P_ad); |I| = 2 -> a < b inside, c < d outside, quad
    P_ac P_ad P_bd P_bc split into (P_ac, P_ad, P_bd), (P_ac, P_bd, P_bc);
  * orientation: a triangle's normal (p1-p0) x (p2-p0) points from the inside
    corners to the outside ones (towards increasing F), decided on the
    combinatorial polygon (every vertex at its edge midpoint: exact in fp64)
    as  n . (mean(outside corners) - mean(inside corners)) > 0, otherwise the
    last two vertices are swapped;
  * triangles are listed in (cube flat id, tet, triangle) order.
"""
from __future__ import annotations

import numpy as np

from .grid import _min_dist, nodes

D7 = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1)]
PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def near_mask(lo, hi, n, data_points, eps):
    """near[flat] = min_j |node - x_j| <= eps (the M_ext^eps of l.211-214)."""
    return _min_dist(nodes(lo, hi, n), np.asarray(data_points, dtype=np.float64)) <= eps


def _tet_corners(perm):
    q = [np.zeros(3, dtype=np.int64)]
    for a in perm[:2]:
        e = np.zeros(3, dtype=np.int64)
        e[a] = 1
        q.append(q[-1] + e)
    q.append(np.ones(3, dtype=np.int64))
    return q


def marching_tets(F, lo, hi, n, near, return_edges=False):
    """(V, T): V (K,3) fp64 vertices, T (M,3) int64 triangles (module docstring);
    with return_edges also E (K,2): the (lower node flat id, direction) of each
    vertex's edge."""
    nx, ny, nz = n
    F = np.asarray(F, dtype=np.float32).astype(np.float64).ravel()
    near = np.asarray(near, dtype=bool).ravel()
    P = nodes(lo, hi, n)
    inside = F < 0

    def flat(i, j, k):
        return i + nx * (j + ny * k)

    # vertices, in (node, direction) order
    vid = {}
    verts = []
    edges = []
    for v in range(nx * ny * nz):
        i, j, k = v % nx, (v // nx) % ny, v // (nx * ny)
        for d, (di, dj, dk) in enumerate(D7):
            if i + di >= nx or j + dj >= ny or k + dk >= nz:
                continue
            u = flat(i + di, j + dj, k + dk)
            if near[v] and near[u] and inside[v] != inside[u]:
                t = F[v] / (F[v] - F[u])
                pa, pb = P[v], P[u]
                vid[(v, d)] = len(verts)
                verts.append(pa + t * (pb - pa))
                edges.append((v, d))

    def edge_vertex(ca, cb):
        """vertex id on the tet edge between lattice corners ca, cb."""
        lo_c, hi_c = (ca, cb) if tuple(cb - ca) in D7 else (cb, ca)
        d = D7.index(tuple(hi_c - lo_c))
        return vid[(flat(*lo_c), d)]

    tris = []
    for k in range(nz - 1):
        for j in range(ny - 1):
            for i in range(nx - 1):
                base = np.array([i, j, k], dtype=np.int64)
                corners = [flat(*(base + np.array(c))) for c in np.ndindex(2, 2, 2)]
                if not all(near[c] for c in corners):
                    continue
                for perm in PERMS:
                    q = [base + c for c in _tet_corners(perm)]
                    ins = [bool(inside[flat(*c)]) for c in q]
                    nin = sum(ins)
                    if nin in (0, 4):
                        continue
                    if nin in (1, 3):
                        lone = [m for m in range(4) if ins[m] == (nin == 1)][0]
                        others = [m for m in range(4) if m != lone]
                        polys = [[(lone, others[0]), (lone, others[1]), (lone, others[2])]]
                    else:
                        a, b = [m for m in range(4) if ins[m]]
                        c, d = [m for m in range(4) if not ins[m]]
                        polys = [[(a, c), (a, d), (b, d)], [(a, c), (b, d), (b, c)]]
                    qin = np.mean([q[m] for m in range(4) if ins[m]], axis=0)
                    qout = np.mean([q[m] for m in range(4) if not ins[m]], axis=0)
                    for poly in polys:
                        mids = [0.5 * (q[x] + q[y]) for x, y in poly]
                        nrm = np.cross(mids[1] - mids[0], mids[2] - mids[0])
                        ids = [edge_vertex(q[x], q[y]) for x, y in poly]
                        if np.dot(nrm, qout - qin) < 0:
                            ids = [ids[0], ids[2], ids[1]]
                        tris.append(ids)
    V = np.array(verts, dtype=np.float64).reshape(-1, 3)
    T = np.array(tris, dtype=np.int64).reshape(-1, 3)
    if return_edges:
        return V, T, np.array(edges, dtype=np.int64).reshape(-1, 2)
    return V, T


def isosurface(F, lo, hi, n, data_points, eps):
    """Masked zero iso-surface mesh of a grid field (Alg. 1 step 4 restricted to
    M_ext^eps)."""
    return marching_tets(F, lo, hi, n, near_mask(lo, hi, n, data_points, eps))
