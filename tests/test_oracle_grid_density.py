"""Pins for oracle.grid (node layout, Eq. 5 on a Gaussian bump, zero set of
an analytic field) and oracle.density (Fig. 3 values printed in the paper)."""
import numpy as np
import pytest

from oracle import density as D
from oracle import grid as G


def test_grid_nodes_layout():
    P = G.nodes((0, 0, 0), (1, 2, 3), (2, 3, 4))
    assert P.shape == (24, 3)
    np.testing.assert_allclose(P[0], [0, 0, 0])
    np.testing.assert_allclose(P[1], [1, 0, 0])      # x fastest
    np.testing.assert_allclose(P[2], [0, 1, 0])
    np.testing.assert_allclose(P[6], [0, 0, 1])
    np.testing.assert_allclose(P[-1], [1, 2, 3])     # inclusive endpoints


def test_grid_single_centre_gaussian():
    """One centre with weight 1: P_f(xi) = a exp(-|xi|^2/(2 sigma^2)) on the
    grid, zero beyond the cutoff; the Riemann sum over the grid of P_f equals
    a (sqrt(2 pi) sigma)^3 / h^3 up to truncation (Gaussian integral)."""
    sigma = 0.1
    lo, hi, n = (-1, -1, -1), (1, 1, 1), (81, 81, 81)
    F = G.evaluate(np.zeros((1, 3)), np.ones(1), sigma, lo, hi, n)
    h = 2.0 / 80
    a = 1 / (np.sqrt(2 * np.pi) * sigma)
    total = F.sum() * h ** 3
    assert total == pytest.approx(a * (np.sqrt(2 * np.pi) * sigma) ** 3, rel=1e-6)
    centre = 40 + 81 * (40 + 81 * 40)
    assert F[centre] == pytest.approx(a, rel=1e-15)
    assert F[0] == 0.0


def test_zero_crossings_of_sphere_field():
    """f = |p| - 1 sampled on a grid: crossings lie on the unit sphere to
    within the linear-interpolation error O(h^2)."""
    lo, hi, n = (-1.5,) * 3, (1.5,) * 3, (40, 40, 40)
    P = G.nodes(lo, hi, n)
    F = np.linalg.norm(P, axis=1) - 1.0
    rng = np.random.default_rng(0)
    v = rng.normal(size=(4000, 3))
    data = v / np.linalg.norm(v, axis=1, keepdims=True)
    pts = G.zero_crossings(F, lo, hi, n, data, 0.3)
    h = 3.0 / 39
    assert len(pts) > 500
    assert np.abs(np.linalg.norm(pts, axis=1) - 1).max() < h * h


def test_halton_fig3_pins():
    """Fig. 3 caption: 25 Halton points on [0,1]^2 have
    q_X ~ 0.0597 and h_{X,Omega} ~ 0.2667 (fill distance over a 401^2 grid)."""
    import os
    gold = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "fig3_halton.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                gold[k] = [float(x) for x in v]
    n = int(gold["n_points"][0])
    P = np.stack([D.halton(n, int(gold["bases"][0])), D.halton(n, int(gold["bases"][1]))], axis=1)
    g = np.linspace(0, 1, 401)
    Om = np.stack(np.meshgrid(g, g), -1).reshape(-1, 2)
    assert D.separation_distance(P) == pytest.approx(gold["q_X"][0], abs=5e-5)
    assert D.fill_distance(P, Om) == pytest.approx(gold["h_X_Omega"][0], abs=5e-5)
    assert D.halton(4, 2).tolist() == [0.5, 0.25, 0.75, 0.125]


def test_density_small_cases():
    X = np.array([[0, 0, 0], [1.0, 0, 0], [3.0, 0, 0]])
    assert D.separation_distance(X) == 0.5
    assert D.h_max(X) == 2.0
    s = D.sigma_heuristics(X)
    assert s["sigma_q"] == 1.0 and s["sigma_hmax"] == pytest.approx(4.0)
