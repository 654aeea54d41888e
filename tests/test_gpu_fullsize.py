"""GPU parity at BASELINE.json's full sizes, in the configuration bench.py times.

c4 (configs[3]: 1M surface points -> 3M centres, sigma 0.01, 256^3 grid) and c3
(configs[2]: 200k points with a 10x density ramp -> 600k centres): the oracle
cannot run the full products, so it computes SAMPLED outputs one by one (rows of
the matvec, nodes of the grid) on all host cores; integer work (extension, cell
lists) is compared in full, bit for bit.  Tolerances as in test_gpu_hotpath.py
(DESIGN.md §9): fp32 tier per row <= 5e-5 g_i, fp64 tier per row <= 1e-12 g_i,
grid per node <= 5e-5 g(xi) with exact zeros where no centre is in range.
"""
import os

import numpy as np
import pytest
import torch

from oracle import cells as OC
from oracle import extend as OE
from oracle import grid as OG
from oracle import kernel as OK
from synth import make_inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
PROCS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


@pytest.fixture(scope="module")
def ctx(R):
    return R.Context(0)


@pytest.fixture(scope="module", params=["c4", "c3"])
def big(request, R, ctx):
    d = make_inputs(request.param)
    centres, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"),
                                 torch.as_tensor(d["normals"], device="cuda"), d["delta"])
    X = OE.extend(d["x"], d["normals"], d["delta"])
    kern = R.Kernel(d["sigma"])
    cells = R.Cells(ctx, centres, kern)
    return dict(name=request.param, d=d, X=X, centres=centres, b=b, kern=kern, cells=cells, sigma=d["sigma"])


def _rows(n, k, seed):
    return np.sort(np.random.default_rng(seed).choice(n, k, replace=False))


def test_extension_and_cells_bit_exact(big):
    X = big["X"]
    assert np.array_equal(big["centres"].cpu().numpy(), X)
    v = big["cells"].view()
    oc = OC.build(X, 6 * big["sigma"], cell_edge=6 * big["sigma"] / 3.999)
    np.testing.assert_array_equal(v["perm"].cpu().numpy(), oc["perm"])
    np.testing.assert_array_equal(v["keys"].cpu().numpy().view(np.uint32), oc["keys"].astype(np.uint32))
    np.testing.assert_array_equal(v["cell_start"].cpu().numpy()[:-1], oc["cell_start"])


def test_matvec_sampled_rows(R, ctx, big):
    X, sigma = big["X"], big["sigma"]
    n = len(X)
    w = np.random.default_rng(7).normal(size=n)
    f32 = R.matvec(ctx, big["cells"], big["kern"], torch.as_tensor(w, dtype=torch.float32, device="cuda"))
    f64 = R.matvec(ctx, big["cells"], big["kern"], torch.as_tensor(w, device="cuda"))
    f32, f64 = f32.cpu().numpy(), f64.cpu().numpy()
    rows = _rows(n, 192, 1)
    w32 = w.astype(np.float32).astype(np.float64)
    ref32 = OK.matvec_parallel(X, w32, sigma, rows=rows, procs=PROCS)
    ref64 = OK.matvec_parallel(X, w, sigma, rows=rows, procs=PROCS)
    g = OK.matvec_parallel(X, np.abs(w), sigma, rows=rows, procs=PROCS)
    assert (np.abs(f32[rows] - ref32) <= 5e-5 * g).all()
    assert np.linalg.norm(f32[rows] - ref32) / np.linalg.norm(ref32) <= 1e-4
    assert (np.abs(f64[rows] - ref64) <= 1e-12 * g).all()
    # the solver's operators as benchmarked (symmetric variants at this size, reading R19)
    os.environ["RBF_PUBLIC_SYM"] = "1"
    try:
        s32 = R.matvec(ctx, big["cells"], big["kern"], torch.as_tensor(w, dtype=torch.float32, device="cuda"))
        s64 = R.matvec(ctx, big["cells"], big["kern"], torch.as_tensor(w, device="cuda"))
    finally:
        del os.environ["RBF_PUBLIC_SYM"]
    s32, s64 = s32.cpu().numpy(), s64.cpu().numpy()
    assert (np.abs(s32[rows] - ref32) <= 5e-5 * g).all()
    assert np.linalg.norm(s32[rows] - ref32) / np.linalg.norm(ref32) <= 1e-4
    assert (np.abs(s64[rows] - ref64) <= 1e-12 * g).all()


def test_solve_as_benchmarked(R, ctx, big):
    """The bench's fit (50 iterations, shifted block-Jacobi): the reported true
    residual is ||b - A w|| / ||b|| of the fp64 tier, whose rows match the oracle."""
    cfg = big["d"]["cfg"]
    w, rep = R.gmres_solve(ctx, big["cells"], big["kern"], big["b"], restart=cfg.restart, rtol=1e-6,
                           kind=cfg.precond_kind, core_target=cfg.core_target, overlap_sigmas=cfg.overlap_sigmas,
                           shift=cfg.shift, local_fp32=cfg.local_fp32, max_iters=50)
    assert rep["iters_phase1"] + rep["iters_phase2"] <= 50
    Aw = R.matvec(ctx, big["cells"], big["kern"], w).cpu().numpy()
    b = big["b"].cpu().numpy().astype(np.float64)
    res = np.linalg.norm(b - Aw) / np.linalg.norm(b)
    assert res == pytest.approx(rep["rel_residual_true"], rel=1e-9)
    assert res < 1e-2                                       # the fit makes progress (finding F4)
    wh = w.cpu().numpy()
    rows = _rows(len(b), 96, 2)
    ref = OK.matvec_parallel(big["X"], wh, big["sigma"], rows=rows, procs=PROCS)
    g = OK.matvec_parallel(big["X"], np.abs(wh), big["sigma"], rows=rows, procs=PROCS)
    assert (np.abs(Aw[rows] - ref) <= 1e-12 * g).all()


def test_grid_sampled_nodes(R, ctx, big):
    d = big["d"]
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    w = np.random.default_rng(9).normal(size=len(big["X"]))
    F = R.eval_grid(ctx, big["cells"], big["kern"], torch.as_tensor(w, device="cuda"), lo, hi, gn)
    F = F.cpu().numpy().ravel()
    rng = np.random.default_rng(3)
    nz = np.nonzero(F)[0]
    flat = np.sort(np.concatenate([rng.choice(F.size, 64, replace=False), rng.choice(nz, 192, replace=False)]))
    P = OG.nodes(lo, hi, gn, flat=flat)
    w32 = w.astype(np.float32).astype(np.float64)        # the grid tier rounds w to fp32
    ref = OK.matvec_parallel(big["X"], w32, big["sigma"], targets=P, procs=PROCS)
    g = OK.matvec_parallel(big["X"], np.abs(w32), big["sigma"], targets=P, procs=PROCS)
    assert (np.abs(F[flat] - ref) <= 5e-5 * g).all()
    # exact zeros where no centre lies within c (1 + 1e-5) (reading R5: fp32 boundary flips)
    g_wide = OK.matvec_parallel(big["X"], np.ones(len(big["X"])), big["sigma"], cutoff_sigmas=6 * (1 + 1e-5),
                                targets=P, procs=PROCS)
    assert (F[flat][g_wide == 0] == 0).all()
