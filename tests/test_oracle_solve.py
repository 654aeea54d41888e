"""Pins for oracle.solve: dense LU, RAS blocks/apply, GMRES(m)+RAS, and the
c1 pipeline end to end (sphere zero set within 5e-3 of radius 1)."""
import numpy as np
import pytest

from oracle import cells as C
from oracle import grid as G
from oracle import kernel as K
from oracle import solve as S
from oracle.extend import extend, labels


def test_lu_single_site_closed_form():
    # 1x1 system a c = b  =>  c = b sqrt(2 pi) sigma   (SPEC S:393 idea)
    sigma = 0.2
    c = S.lu_solve(np.zeros((1, 3)), np.array([0.7]), sigma)
    assert c[0] == pytest.approx(0.7 * np.sqrt(2 * np.pi) * sigma, rel=1e-14)


def test_lu_recovers_constructed_solution():
    """b = A 1 via the row-wise brute-force matvec; the dense LU of the
    separately assembled matrix must return the all-ones vector."""
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (400, 3)).astype(np.float32)
    b = K.matvec(X, np.ones(400), 0.1)
    c = S.lu_solve(X, b, 0.1)
    np.testing.assert_allclose(c, 1.0, atol=1e-8)


def _small_problem(seed=0, n=300, sigma=0.12):
    rng = np.random.default_rng(seed)
    X = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    b = rng.normal(size=n)
    return X, b, sigma


def test_gmres_unpreconditioned_matches_lu():
    X, b, sigma = _small_problem()
    A = K.dense_matrix(X, sigma)
    x, info = S.gmres(lambda v: A @ v, b, restart=40, rtol=1e-12, maxit=2000)
    assert info["converged"]
    np.testing.assert_allclose(x, S.lu_solve(X, b, sigma), rtol=1e-8, atol=1e-9)


def test_gmres_residual_history_monotone_within_cycle():
    X, b, sigma = _small_problem(1)
    A = K.dense_matrix(X, sigma)
    m = 10
    _, info = S.gmres(lambda v: A @ v, b, restart=m, rtol=1e-10, maxit=200)
    h = np.array(info["history"])
    for s in range(0, len(h), m):
        cyc = h[s:s + m]
        assert (np.diff(cyc) <= 1e-15).all()


def test_ras_single_block_is_exact():
    """RAS with one subdomain is the exact inverse: GMRES
    converges in one iteration."""
    X, b, sigma = _small_problem(2, n=200)
    cells = C.build(X, 6 * sigma)
    blocks = S.ras_blocks(cells, sigma, core_target=10_000, overlap_sigmas=1.0)
    assert len(blocks) == 1
    Ss = cells["sorted"]
    A = K.dense_matrix(Ss, sigma)
    bs = b[cells["perm"]]
    x, info = S.gmres(lambda v: A @ v, bs, restart=5, rtol=1e-10,
                      apply_M=lambda r: S.ras_apply(blocks, Ss, r, sigma))
    assert info["iters"] == 1 and info["converged"]


def test_ras_shift_single_block_solves_shifted_system():
    """Reading R17: with one subdomain and shift mu the RAS apply is
    (A + mu a I)^{-1} r with a = 1/(sqrt(2 pi) sigma).  Checked by multiplying
    back with the brute-force row matvec (an independent code path) plus the
    mu a r term; a dropped a, a wrong sign or an off-diagonal shift fails."""
    X, _, sigma = _small_problem(4, n=200)
    cells = C.build(X, 6 * sigma)
    blocks = S.ras_blocks(cells, sigma, core_target=10_000, overlap_sigmas=0.0)
    Ss = cells["sorted"].astype(np.float64)
    r = np.random.default_rng(5).normal(size=200)
    a = 1.0 / (np.sqrt(2 * np.pi) * sigma)
    for mu in (0.0, 0.01, 0.3):
        z = S.ras_apply(blocks, Ss, r, sigma, shift=mu)
        back = K.matvec(Ss, z, sigma) + mu * a * z
        np.testing.assert_allclose(back, r, rtol=0, atol=1e-9 * np.abs(r).max())


def test_ras_shift_large_limit_and_monotone_norm():
    """mu -> infinity: B^{-1} r -> r / (mu a) (Neumann series, error O(||A||/(mu a)));
    ||z|| decreases with mu for the SPD single-site-dominated blocks used here."""
    X, _, sigma = _small_problem(6, n=150, sigma=0.05)
    cells = C.build(X, 6 * sigma)
    blocks = S.ras_blocks(cells, sigma, core_target=40, overlap_sigmas=0.0)
    Ss = cells["sorted"].astype(np.float64)
    r = np.random.default_rng(7).normal(size=150)
    a = 1.0 / (np.sqrt(2 * np.pi) * sigma)
    mu = 1e6
    z = S.ras_apply(blocks, Ss, r, sigma, shift=mu)
    np.testing.assert_allclose(z * mu * a, r, rtol=1e-4)
    norms = [np.linalg.norm(S.ras_apply(blocks, Ss, r, sigma, shift=m)) for m in (0.01, 0.1, 1.0, 10.0)]
    assert all(x > y for x, y in zip(norms, norms[1:]))


def test_shifted_block_jacobi_beats_exact_ras_at_flat_ratio():
    """DESIGN.md finding F4 in miniature: at sigma/spacing ~3 with +-delta
    triplets (delta = 0.1 sigma) the exact local solves make GMRES stall,
    while shifted block-Jacobi local solves (mu = 0.01) make progress."""
    from synth.surfaces import fibonacci_sphere
    xs, nrm = fibonacci_sphere(1500)
    sel = xs[:, 2] > 0.55                           # a cap: ~340 surface points
    xs, nrm = xs[sel], nrm[sel]
    spacing = np.sqrt(4 * np.pi / 1500)
    sigma = 3.0 * spacing
    delta = 0.1 * sigma
    X = extend(xs, nrm, delta).astype(np.float32)
    b = labels(len(xs), delta)
    cells = C.build(X, 6 * sigma)
    Ss = cells["sorted"].astype(np.float64)
    bs = b[cells["perm"]]
    A = K.dense_matrix(Ss, sigma)
    res = {}
    for name, ov, mu in (("exact-ras", 1.0, 0.0), ("shifted-bj", 0.0, 0.01)):
        blocks = S.ras_blocks(cells, sigma, core_target=128, overlap_sigmas=ov)
        facs = {}
        _, info = S.gmres(lambda v: A @ v, bs, restart=30, rtol=1e-12, maxit=30,
                          apply_M=lambda r: S.ras_apply(blocks, Ss, r, sigma, factors=facs, shift=mu))
        res[name] = info["rel_residual"]
    assert res["shifted-bj"] < 1e-2 and res["shifted-bj"] < 0.1 * res["exact-ras"], res


def test_ras_blocks_partition_and_overlap(c1_inputs):
    d = c1_inputs
    X = extend(d["x"], d["normals"], d["delta"])
    sigma = d["sigma"]
    cells = C.build(X, 6 * sigma)
    ov = 3 * sigma
    blocks = S.ras_blocks(cells, sigma, core_target=512, overlap_sigmas=3.0)
    cores = np.concatenate([b["core"] for b in blocks])
    assert np.array_equal(np.sort(cores), np.arange(len(X)))     # cores partition
    Ss = cells["sorted"].astype(np.float64)
    for b in blocks:
        core, ext = b["core"], b["ext"]
        assert np.array_equal(ext[-core.size:], core)             # core last
        extra = ext[:-core.size]
        assert (np.diff(extra) > 0).all() and not np.isin(extra, core).any()
        # brute force: every centre within ov(1-1e-5) of the core is in ext,
        # none farther than ov(1+1e-5)
        d2 = ((Ss[:, None, :] - Ss[None, core, :]) ** 2).sum(axis=2).min(axis=1)
        must = np.nonzero(d2 <= (ov * (1 - 1e-5)) ** 2)[0]
        assert np.isin(must, ext).all()
        assert (d2[ext] <= (ov * (1 + 1e-5)) ** 2).all()
    sizes = [b["core"].size for b in blocks]
    assert min(sizes) >= 256


@pytest.fixture(scope="module")
def c1_solution(c1_inputs):
    d = c1_inputs
    X = extend(d["x"], d["normals"], d["delta"])
    N = len(d["x"])
    b = labels(N, d["delta"])
    sigma = d["sigma"]
    cells = C.build(X, 6 * sigma)
    Ss = cells["sorted"]
    perm = cells["perm"]
    A = K.dense_matrix(Ss, sigma)
    blocks = S.ras_blocks(cells, sigma, 512, 3.0)
    fac = {}
    xs, info = S.gmres(lambda v: A @ v, b[perm], restart=30, rtol=1e-8, maxit=500,
                       apply_M=lambda r: S.ras_apply(blocks, Ss, r, sigma, factors=fac))
    w = np.empty_like(xs)
    w[perm] = xs
    return dict(X=X, b=b, w=w, info=info, sigma=sigma, d=d)


def test_c1_gmres_ras_vs_lu(c1_solution):
    s = c1_solution
    info = s["info"]
    assert info["converged"] and info["rel_residual"] <= 1e-8
    assert info["iters"] < 60        # survey [M3]: 15 iterations
    w_lu = S.lu_solve(s["X"], s["b"], s["sigma"])
    # interpolation conditions through the independent row-wise matvec
    f = K.matvec(s["X"], s["w"], s["sigma"])
    assert np.linalg.norm(f - s["b"]) / np.linalg.norm(s["b"]) <= 1e-8
    f_lu = K.matvec(s["X"], w_lu, s["sigma"])
    assert np.linalg.norm(f_lu - s["b"]) / np.linalg.norm(s["b"]) <= 1e-10
    # kappa ~ 2e7 (survey [M1]) bounds weight differences by ~kappa * 1e-8
    assert np.linalg.norm(s["w"] - w_lu) / np.linalg.norm(w_lu) < 1e-2


def test_c1_sphere_zero_set(c1_solution):
    """§2.1.3: the masked zero set M_ext^eps cap S_0 reconstructs the unit
    sphere; reading 11 gate: max | |p| - 1 | <= 5e-3 on 32^3, eps = 2 sigma."""
    s = c1_solution
    d = s["d"]
    F = G.evaluate(s["X"], s["w"], s["sigma"], d["grid_lo"], d["grid_hi"], d["grid_n"])
    pts = G.zero_crossings(F, d["grid_lo"], d["grid_hi"], d["grid_n"], d["x"], 2 * s["sigma"])
    assert len(pts) > 1000
    err = np.abs(np.linalg.norm(pts, axis=1) - 1.0)
    assert err.max() <= 5e-3
    # exact zeros: nodes with no centre within the cutoff
    far = G._min_dist(G.nodes(d["grid_lo"], d["grid_hi"], d["grid_n"]),
                      s["X"].astype(np.float64)) > 6 * s["sigma"]
    assert (F[far] == 0).all() and (F[~far] != 0).all()


def test_truncated_operator_indefinite_at_high_ratio():
    """DESIGN.md finding F1 (pins the reading that c2-c5 are ill-posed at the 1e-6 gate):
    the Eq.6 matrix truncated at 6 sigma is positive definite on c1's sphere
    (sigma/spacing 0.89; lambda_min 2.69e-6) but, on a torus at sigma/spacing
    1.9 (c2's ratio), truncation error (1.5e-8 a per dropped entry) exceeds the Gaussian
    matrix's smallest eigenvalues and many eigenvalues turn negative -- while the
    UNtruncated matrix stays positive semi-definite (Bochner: the Gaussian is PD)."""
    from synth.surfaces import torus, fibonacci_sphere
    x, nrm = fibonacci_sphere(1000)
    X = extend(x, nrm, 0.01)
    ev = np.linalg.eigvalsh(K.dense_matrix(X, 0.1))
    assert ev[0] > 0 and ev[0] == pytest.approx(2.69e-6, rel=0.05)
    n = 1000
    x, nrm = torus(n, noise=0.0, seed=0)
    sigma = 1.9 * np.sqrt(4 * np.pi ** 2 * 0.35 / n)
    X = extend(x, nrm, 0.1 * sigma)
    ev_t = np.linalg.eigvalsh(K.dense_matrix(X, sigma))
    ev_u = np.linalg.eigvalsh(K.dense_matrix(X, sigma, truncate=False))
    a = K.amplitude(sigma)
    assert (ev_t < 0).sum() > 100
    assert ev_t[0] < -1e-9 * a
    assert ev_u[0] > -1e-12 * ev_u[-1]          # rounding-level only
