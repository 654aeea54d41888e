"""GPU density measures (Eq.7-11) against the
oracle (oracle/density.py, pinned by the Fig. 3 values) -- every distance is
computed with the oracle's fp64 rounding, so the comparisons are exact."""
import os

import numpy as np
import pytest
import torch

from oracle import density as D
from synth import make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


@pytest.fixture(scope="module")
def ctx(R):
    return R.Context(0)


def _dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _gold():
    gold = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "fig3_halton.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                gold[k] = [float(x) for x in v]
    return gold


def test_fig3_halton_values(R, ctx):
    """Fig. 3 caption: 25 Halton points on [0,1]^2: q ~ 0.0597, h ~ 0.2667."""
    gold = _gold()
    n = int(gold["n_points"][0])
    P2 = np.stack([D.halton(n, int(gold["bases"][0])), D.halton(n, int(gold["bases"][1]))], axis=1)
    P = np.concatenate([P2, np.zeros((n, 1))], axis=1)
    g = np.linspace(0, 1, 401)
    Om2 = np.stack(np.meshgrid(g, g), -1).reshape(-1, 2)
    Om = np.concatenate([Om2, np.zeros((len(Om2), 1))], axis=1)
    out = R.density(ctx, _dev(P), _dev(Om))
    assert out["q"] == pytest.approx(gold["q_X"][0], abs=5e-5)
    assert out["h"] == pytest.approx(gold["h_X_Omega"][0], abs=5e-5)
    assert out["q"] == D.separation_distance(P2)            # bit-identical
    assert out["h"] == D.fill_distance(P2, Om2)
    assert out["sigma_q"] == 2 * out["q"]                   # Eq. 9


@pytest.mark.parametrize("name,n", [("c1", None), ("c3", 4000), ("c2", 3000)])
def test_nn_distances_equal_oracle(R, ctx, name, n):
    d = make_inputs(name, n=n)
    X = d["x"]
    nn = R.nn_distance(ctx, _dev(X)).cpu().numpy()
    ref = D._nn_dist(X, X, True)
    np.testing.assert_array_equal(nn, ref)
    out = R.density(ctx, _dev(X))
    assert out["q"] == D.separation_distance(X) and out["h_max"] == D.h_max(X)
    assert np.isnan(R.density(ctx, _dev(X)).get("h", np.nan))


def test_queries_outside_duplicates_and_degenerate(R, ctx):
    rng = np.random.default_rng(4)
    X = rng.uniform(-1, 1, (3000, 3))
    X[10] = X[20]                                            # a duplicate: separation 0
    Q = np.concatenate([rng.uniform(-5, 5, (500, 3)), [[40.0, -30.0, 7.0]], X[:5]])
    got = R.nn_distance(ctx, _dev(X), _dev(Q)).cpu().numpy()
    np.testing.assert_array_equal(got, D._nn_dist(Q, X, False))
    assert R.density(ctx, _dev(X))["q"] == 0.0
    # all points on a line (two degenerate extents)
    L = np.stack([np.linspace(0, 1, 500) ** 2, np.zeros(500), np.zeros(500)], axis=1)
    np.testing.assert_array_equal(R.nn_distance(ctx, _dev(L)).cpu().numpy(), D._nn_dist(L, L, True))
    with pytest.raises(R.RbfError):
        R.density(ctx, _dev(X[:1]))
