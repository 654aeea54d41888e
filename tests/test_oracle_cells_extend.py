"""Pins for oracle.extend (§2.1.1) and the float32 cell-list replica."""
import numpy as np
import pytest

from oracle import cells as C
from oracle.extend import extend, labels


def test_extend_single_point():
    # one point (0,0,1), normal (0,0,1), delta 0.1 -> (0,0,1),(0,0,1.1),(0,0,0.9)
    e = extend(np.array([[0, 0, 1.0]]), np.array([[0, 0, 1.0]]), 0.1)
    assert e.dtype == np.float32
    np.testing.assert_array_equal(e, np.float32([[0, 0, 1], [0, 0, 1.1], [0, 0, 0.9]]))
    np.testing.assert_array_equal(labels(1, 0.1), [0, 0.1, -0.1])


def test_extend_distances(c1_inputs):
    x, n, d = c1_inputs["x"], c1_inputs["normals"], c1_inputs["delta"]
    e = extend(x, n, d).astype(np.float64)
    N = len(x)
    np.testing.assert_allclose(np.linalg.norm(e[N:2 * N] - e[:N], axis=1), d, rtol=1e-4)
    np.testing.assert_allclose(np.linalg.norm(e[2 * N:] - e[:N], axis=1), d, rtol=1e-4)
    # outside points are farther from the origin on the unit sphere
    assert (np.linalg.norm(e[N:2 * N], axis=1) > 1).all()
    assert (np.linalg.norm(e[2 * N:], axis=1) < 1).all()


def _cloud(seed=0, n=4000):
    rng = np.random.default_rng(seed)
    return rng.normal(size=(n, 3)).astype(np.float32) * np.float32(0.3)


def test_cells_permutation_sorted_stable():
    X = _cloud()
    c = C.build(X, cutoff=0.2)
    perm = c["perm"]
    assert np.array_equal(np.sort(perm), np.arange(len(X)))
    k = c["keys"]
    assert (np.diff(k) >= 0).all()
    # stability: equal keys keep ascending input id
    same = np.diff(k) == 0
    assert (np.diff(perm)[same] > 0).all()
    np.testing.assert_array_equal(c["sorted"], X[perm])


def test_cells_contain_their_points_and_counts():
    X = _cloud(1)
    c = C.build(X, cutoff=0.2)
    lo, h, dim = c["lo"].astype(np.float64), c["h"], c["dim"]
    q = c["coords"]
    S = c["sorted"].astype(np.float64)
    tol = 1e-6
    assert (S >= lo + q * h - tol).all() and (S <= lo + (q + 1) * h + tol).all()
    assert (q >= 0).all() and (q < dim).all()
    # brute-force recount per cell
    lin = q[:, 0] + dim[0] * (q[:, 1] + dim[1] * q[:, 2])
    counts = np.bincount(lin, minlength=int(dim.prod()))
    np.testing.assert_array_equal(c["cell_end"] - c["cell_start"], counts)
    # each cell is one contiguous range of the sorted order
    nz = np.nonzero(counts)[0]
    for cell in nz[:200]:
        idx = np.nonzero(lin == cell)[0]
        assert idx[0] == c["cell_start"][cell] and idx[-1] == c["cell_end"][cell] - 1


def test_cells_range_query_equals_bruteforce():
    """SPEC-derived invariant: a stencil query over the cells returns
    exactly the brute-force range query."""
    X = _cloud(2, 3000)
    r = 0.2
    c = C.build(X, cutoff=r)
    S = c["sorted"].astype(np.float64)
    dim, q = c["dim"], c["coords"]
    R = int(np.ceil(r / c["h"])) + 1
    rng = np.random.default_rng(3)
    for i in rng.choice(len(S), 40, replace=False):
        got = []
        for dz in range(-R, R + 1):
            for dy in range(-R, R + 1):
                for dx in range(-R, R + 1):
                    cc = q[i] + np.array([dx, dy, dz])
                    if (cc < 0).any() or (cc >= dim).any():
                        continue
                    lin = cc[0] + dim[0] * (cc[1] + dim[1] * cc[2])
                    for j in range(c["cell_start"][lin], c["cell_end"][lin]):
                        if ((S[j] - S[i]) ** 2).sum() <= r * r:
                            got.append(j)
        brute = np.nonzero(((S - S[i]) ** 2).sum(axis=1) <= r * r)[0]
        assert sorted(got) == list(brute)


def test_morton_interleave():
    assert int(C.morton3(1, 0, 0)) == 1
    assert int(C.morton3(0, 1, 0)) == 2
    assert int(C.morton3(0, 0, 1)) == 4
    assert int(C.morton3(3, 0, 0)) == 0b1001
    assert int(C.morton3(5, 6, 7)) == int("111110101", 2)
