"""Neighbour-list form of the solver's symmetric fp32 operator
(rbf_ctx_neighbour_lists, summation.cu ensure_nl / nl_build_kernel): the tile
source lists are the traversal's culled rows written out once per cell
structure (Alg.2 "truncation area"); the products must equal the
traversal form's up to the atomics' summation order and the oracle's
brute-force truncated sum (Eq.4 / Eq.6) per row."""
import numpy as np
import pytest
import torch

from oracle import extend as OE
from oracle import kernel as OK
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


def dev(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def torus(R, ctx):
    d = make_inputs("c2")          # 60k centres, noisy torus (near-duplicate centres)
    X = OE.extend(d["x"], d["normals"], d["delta"])
    return d, X


def _products(R, ctx, cells, kern, w, nl):
    ctx.neighbour_lists(nl)
    try:
        return host(R.matvec_op(ctx, cells, kern, dev(w, torch.float32), op=R.OP_SYM_WIDE))
    finally:
        ctx.neighbour_lists(True)


def test_nl_equals_traversal_and_oracle(R, ctx, torus):
    d, X = torus
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    cells = R.Cells(ctx, dev(X, torch.float32), kern)
    rng = np.random.default_rng(7)
    w = rng.normal(size=len(X))
    w32 = w.astype(np.float32).astype(np.float64)
    f_nl = _products(R, ctx, cells, kern, w, True)
    f_nl2 = _products(R, ctx, cells, kern, w, True)      # the cached list
    f_tr = _products(R, ctx, cells, kern, w, False)
    rows = np.sort(rng.choice(len(X), 3000, replace=False))
    ref = OK.matvec(X, w32, sigma, rows=rows)
    g = OK.matvec(X, np.abs(w32), sigma, rows=rows)
    for f in (f_nl, f_nl2, f_tr):
        assert (np.abs(f[rows] - ref) <= 5e-5 * g).all()
        assert np.linalg.norm(f[rows] - ref) <= 1e-4 * np.linalg.norm(ref)
    # the two forms evaluate the same pairs except those the list drops because
    # they lie beyond the cutoff of every target of a 32-target group (each such
    # term <= 2^-26 of its weight's peak entry, reading R18), and sum in another
    # order: a few ulp of the row's absolute sum g
    assert (np.abs(f_nl[rows] - f_tr[rows]) <= 5e-6 * g).all()
    # the cached list gives the same pairs; only the atomics' order differs
    assert (np.abs(f_nl[rows] - f_nl2[rows]) <= 2e-6 * g).all()


def test_nl_rebuilt_when_the_cutoff_changes(R, ctx, torus):
    """The list is keyed by the culling radius: a product with a narrower kernel
    on the same cells rebuilds it (a stale list would miss or add pairs)."""
    d, X = torus
    k1, k2 = R.Kernel(d["sigma"]), R.Kernel(0.6 * d["sigma"])
    cells = R.Cells(ctx, dev(X, torch.float32), k1)
    rng = np.random.default_rng(8)
    w = rng.normal(size=len(X))
    w32 = w.astype(np.float32).astype(np.float64)
    rows = np.sort(rng.choice(len(X), 2000, replace=False))
    for sig, kern in ((d["sigma"], k1), (0.6 * d["sigma"], k2), (d["sigma"], k1)):
        f = _products(R, ctx, cells, kern, w, True)
        ref = OK.matvec(X, w32, sig, rows=rows)
        g = OK.matvec(X, np.abs(w32), sig, rows=rows)
        assert (np.abs(f[rows] - ref) <= 5e-5 * g).all(), sig


def test_nl_solve_matches_traversal_solve(R, ctx, torus):
    """The benchmarked solver configuration (shifted block-Jacobi, OP_SYM_WIDE)
    with and without neighbour lists: same iteration counts within a few, both
    true residuals certified by the oracle's fp64 matvec."""
    d, X = torus
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    cells = R.Cells(ctx, dev(X, torch.float32), kern)
    b = OE.labels(len(d["x"]), d["delta"])
    out = {}
    for nl in (True, False):
        ctx.neighbour_lists(nl)
        try:
            w, rep = R.gmres_solve(ctx, cells, kern, dev(b, torch.float32), restart=50, rtol=1e-6, kind=1,
                                   core_target=64, overlap_sigmas=0.0, shift=0.003, local_fp32=1, max_iters=60,
                                   op=R.OP_SYM_WIDE)
        finally:
            ctx.neighbour_lists(True)
        res = np.linalg.norm(b - OK.matvec(X, host(w), sigma)) / np.linalg.norm(b)
        out[nl] = (res, rep)
        assert res <= 1.5 * rep["rel_residual_true"] + 1e-12, (nl, res, rep["rel_residual_true"])
    assert abs(out[True][1]["iters_phase1"] - out[False][1]["iters_phase1"]) <= 5, out
    assert out[True][0] <= 2 * out[False][0] + 1e-7 and out[False][0] <= 2 * out[True][0] + 1e-7, out
