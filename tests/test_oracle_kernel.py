"""Pins for oracle.kernel (Eq. 6 entries, Eq. 4 brute-force matvec).

Independent anchors: tabulated constants (1/sqrt(2 pi), e^{-1/2}, e^{-18}),
the Poisson-summation closed form of a Gaussian lattice sum, special cases
(single site, far sites), linearity and symmetry.
"""
import numpy as np
import pytest

from oracle import kernel as K

INV_SQRT_2PI = 0.398942280401432685715673861243  # 1/sqrt(2 pi)


def test_phi_closed_forms():
    # Table I / Eq. 6 normalisation at r = 0, sigma = 1
    assert K.phi(0.0, 1.0) == pytest.approx(INV_SQRT_2PI, rel=1e-15)
    # sigma = 0.157 (Fig. 5 caption), r = sigma:
    # 1/(sqrt(2 pi) 0.157) * e^{-1/2}; decimal evaluation = 1.541214805854416
    assert K.phi(0.157, 0.157) == pytest.approx(1.54121480585441627, rel=1e-14)
    # 6 sigma cutoff tail, inclusive: a e^{-18} with e^{-18} = 1.522997974471263e-8
    assert K.phi(6.0, 1.0, cutoff=6.0) == pytest.approx(INV_SQRT_2PI * 1.52299797447126284e-8,
                                                         rel=1e-13)
    assert K.phi(6.0 * (1 + 1e-9), 1.0, cutoff=6.0) == 0.0


def _lattice(h, half):
    g = np.arange(-half, half + 1) * h
    X = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    centre = int(np.nonzero((X == 0).all(axis=1))[0][0])
    return X, centre


def test_matvec_poisson_summation():
    """sum over Z^3 of a exp(-|kh|^2/(2 sigma^2)) = 2 pi sigma^2 / h^3 up to
    exp(-2 pi^2 sigma^2/h^2) (Poisson summation); with sigma/h = 1.37 that term
    is 1e-16.  Pins the normalisation, the 2 sigma^2, and all three axes."""
    h, sigma = 0.01, 0.0137
    X, c = _lattice(h, 20)  # half-width 20h = 14.6 sigma: untruncated tail < 1e-40
    exact = 2.0 * np.pi * sigma ** 2 / h ** 3
    f = K.matvec(X, np.ones(len(X)), sigma, rows=[c], truncate=False)[0]
    assert f == pytest.approx(exact, rel=1e-12)
    ft = K.matvec(X, np.ones(len(X)), sigma, 6.0, rows=[c])[0]
    # truncation removes the 3-D Gaussian mass beyond 6 sigma (~7.3e-8)
    assert 1e-8 < (exact - ft) / exact < 2e-7


def test_matvec_special_cases():
    sigma = 0.1
    a = 1.0 / (np.sqrt(2 * np.pi) * sigma)
    f = K.matvec(np.zeros((1, 3)), np.array([2.5]), sigma)
    assert f[0] == pytest.approx(2.5 * a, rel=1e-15)
    X = np.array([[0, 0, 0], [0.61, 0, 0]], dtype=np.float64)  # beyond 6 sigma
    f = K.matvec(X, np.array([1.0, -3.0]), sigma)
    np.testing.assert_allclose(f, [a, -3 * a], rtol=1e-15)


def test_matvec_linear_symmetric_and_matches_dense():
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, (300, 3)).astype(np.float32)
    sigma = 0.15
    w1, w2 = rng.normal(size=300), rng.normal(size=300)
    f1, f2 = K.matvec(X, w1, sigma), K.matvec(X, w2, sigma)
    np.testing.assert_allclose(K.matvec(X, w1 + 2 * w2, sigma), f1 + 2 * f2, rtol=1e-12, atol=1e-12)
    A = K.dense_matrix(X, sigma)
    assert np.array_equal(A, A.T)
    np.testing.assert_allclose(A @ w1, f1, rtol=1e-12, atol=1e-12)
    # row-block path (n small => blocked branch) equals row-by-row
    np.testing.assert_allclose(K.matvec(X, w1, sigma, rows=np.arange(5)), f1[:5], rtol=1e-14)


def test_untruncated_matrix_positive_definite():
    """the Gaussian gives positive definite matrices
    (distinct points, untruncated)."""
    rng = np.random.default_rng(2)
    X = rng.uniform(0, 1, (150, 3))
    A = K.dense_matrix(X, 0.1, truncate=False)
    np.linalg.cholesky(A)
    assert np.linalg.eigvalsh(A).min() > 0


def test_pair_count_bruteforce():
    X = np.array([[0, 0, 0], [0.5, 0, 0], [0, 0.7, 0]], dtype=np.float64)
    # sigma = 0.1, cutoff 0.6: pairs (0,0),(1,1),(2,2),(0,1),(1,0)
    assert K.pair_count(X, 0.1) == 5


def test_matvec_parallel_equals_matvec_in_row_order():
    """The multi-process row split (bench cpu_baseline, c3/c4 parity sampling)
    returns the rows of `matvec` in the order asked for (row blocks of the split
    re-concatenated), with the same per-row arithmetic."""
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, (1500, 3)).astype(np.float32)
    w = rng.normal(size=1500)
    sigma = 0.08
    rows = rng.choice(1500, 101, replace=False)     # unsorted, odd count: uneven parts
    ref = K.matvec(X, w, sigma, rows=rows)
    g = K.matvec(X, np.abs(w), sigma, rows=rows)
    for procs in (1, 2, 3):
        f = K.matvec_parallel(X, w, sigma, rows=rows, procs=procs)
        assert f.shape == ref.shape
        assert (np.abs(f - ref) <= 1e-14 * g).all(), procs
    T = rng.uniform(-1, 1, (37, 3))
    np.testing.assert_allclose(K.matvec_parallel(X, w, sigma, targets=T, procs=2),
                               K.matvec(X, w, sigma, targets=T), rtol=0,
                               atol=1e-14 * np.abs(K.matvec(X, np.abs(w), sigma, targets=T)).max())


def test_matvec_local_equals_bruteforce_including_cutoff_boundary():
    """matvec_local (range search + the same fp64 predicate) against brute force:
    random clouds, rows, grid-like targets, and pairs placed EXACTLY on the
    cutoff sphere in fp64 (d2 == c^2 is included) or one ulp beyond it."""
    rng = np.random.default_rng(6)
    sigma = 0.05
    X = rng.uniform(-0.4, 0.4, (4000, 3)).astype(np.float32).astype(np.float64)
    w = rng.normal(size=len(X))
    rows = rng.choice(len(X), 300, replace=False)
    ref = K.matvec(X, w, sigma, rows=rows)
    g = K.matvec(X, np.abs(w), sigma, rows=rows)
    assert (np.abs(K.matvec_local(X, w, sigma, rows=rows) - ref) <= 1e-13 * g).all()
    T = rng.uniform(-0.5, 0.5, (200, 3))
    ref = K.matvec(X, w, sigma, targets=T)
    g = K.matvec(X, np.abs(w), sigma, targets=T)
    assert (np.abs(K.matvec_local(X, w, sigma, targets=T) - ref) <= 1e-13 * g + 1e-300).all()
    # boundary: c = 0.3 = 6 sigma; x-offsets 0.25 exactly on the sphere? use a
    # representable case: sigma = 0.125, c = 0.75, offsets (0.75, 0, 0) and
    # (0.45, 0.6, 0) have d2 == 0.5625 exactly; nextafter(0.75) lies beyond
    s2 = 0.125
    Xb = np.array([[0, 0, 0], [0.75, 0, 0], [0.45, 0.6, 0], [np.nextafter(0.75, 1), 0, 0]])
    wb = np.array([1.0, 1.0, 1.0, 1.0])
    fl = K.matvec_local(Xb, wb, s2, rows=[0])
    fb = K.matvec(Xb, wb, s2, rows=[0])
    a = K.amplitude(s2)
    np.testing.assert_allclose(fb, [a * (1 + 2 * np.exp(-18.0))], rtol=1e-15)
    np.testing.assert_allclose(fl, fb, rtol=1e-15)
