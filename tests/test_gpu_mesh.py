"""GPU parity of Alg.1 steps 3-4 on the eps-surrounding:
rbf_eval_grid_masked (P_f on M_ext^eps only, §2.1.3) and the
marching-tetrahedra mesh of the zero iso-surface (reading R24)
against oracle/mesh.py on the same field -- vertices (fp64 arithmetic on both
sides) and triangles bit for bit, in the same order."""
import numpy as np
import pytest
import torch

from oracle import extend as OE
from oracle import grid as OG
from oracle import kernel as OK
from oracle import mesh as OM
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


def _closed_euler(T):
    from collections import Counter
    de = Counter()
    for a, b, c in T:
        for e in ((a, b), (b, c), (c, a)):
            de[e] += 1
    assert all(m == 1 for m in de.values()) and all(de[(b, a)] == 1 for (a, b) in de)
    return len(np.unique(T)) - len(de) // 2 + len(T)


@pytest.fixture(scope="module")
def c1_fit(R, ctx):
    d = make_inputs("c1")
    X = OE.extend(d["x"], d["normals"], d["delta"])
    kern = R.Kernel(d["sigma"])
    c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                           d["delta"])
    cells = R.Cells(ctx, c, kern)
    w, rep = R.gmres_solve(ctx, cells, kern, b, restart=30, rtol=1e-8, overlap_sigmas=3.0)
    return dict(d=d, X=X, kern=kern, cells=cells, w=w)


def test_c1_masked_field_and_mesh(R, ctx, c1_fit):
    d, w = c1_fit["d"], c1_fit["w"]
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    data = torch.as_tensor(d["x"], device="cuda")
    eps = 2 * d["sigma"]
    full = R.eval_grid(ctx, c1_fit["cells"], c1_fit["kern"], w, lo, hi, gn).cpu().numpy().ravel()
    masked = R.eval_grid_masked(ctx, c1_fit["cells"], c1_fit["kern"], w, lo, hi, gn, data, eps).cpu().numpy().ravel()
    near = OM.near_mask(lo, hi, gn, d["x"], eps)
    assert 0 < near.sum() < near.size
    # on M_ext^eps the masked field is the full field bit for bit; NaN elsewhere
    assert np.array_equal(masked[near].view(np.uint32), full[near].view(np.uint32))
    assert np.isnan(masked[~near]).all()
    Fm = torch.empty(full.size, dtype=torch.float32, device="cuda")
    V, T = R.isosurface(ctx, c1_fit["cells"], c1_fit["kern"], w, lo, hi, gn, data, eps, field=Fm)
    assert np.array_equal(Fm.cpu().numpy().view(np.uint32), masked.view(np.uint32))
    Vo, To, Eo = OM.marching_tets(masked, lo, hi, gn, near, return_edges=True)
    V, T = V.cpu().numpy(), T.cpu().numpy()
    assert len(To) > 1000
    np.testing.assert_array_equal(V, Vo)
    np.testing.assert_array_equal(T, To)
    # the zero set of the sphere fit: the axis-edge vertices (the zero crossings of
    # reading R11) within 5e-3 of radius 1; the diagonal edges are up to sqrt(3)
    # longer, so their linear interpolation error is up to 3x larger
    rad = np.abs(np.linalg.norm(V, axis=1) - 1.0)
    assert rad[Eo[:, 1] < 3].max() <= 5e-3
    assert rad.max() <= 3 * 5e-3
    # with eps = 2 sigma the whole sphere is inside the mask: a closed genus-0 surface
    assert _closed_euler(T) == 2
    # outward orientation (labels +delta outside): positive enclosed volume ~ 4/3 pi
    vol = np.einsum("ij,ij->i", V[T[:, 0]], np.cross(V[T[:, 1]], V[T[:, 2]])).sum() / 6
    assert vol == pytest.approx(4 / 3 * np.pi, rel=0.02)


def test_mesh_from_field_matches_oracle(R, ctx):
    """Analytic fields (torus, tilted plane, a random field for every tet case),
    mask from a few data points with a partial cover."""
    rng = np.random.default_rng(5)
    lo, hi, gn = (-1.5, -1.45, -0.7), (1.5, 1.45, 0.8), (29, 25, 17)
    P = OG.nodes(lo, hi, gn)
    fields = {
        "torus": np.hypot(np.hypot(P[:, 0], P[:, 1]) - 1.0, P[:, 2]) - 0.35,
        "plane": P @ np.array([0.3, -0.5, 0.8]) - 0.1,
        "random": rng.normal(size=len(P)),
    }
    for name, F in fields.items():
        F = F.astype(np.float32)
        for data, eps in ((np.zeros((1, 3)), 10.0), (rng.uniform(-1.5, 1.5, size=(40, 3)), 0.6)):
            near = OM.near_mask(lo, hi, gn, data, eps)
            V, T = R.mesh_from_field(ctx, torch.as_tensor(F, device="cuda"), lo, hi, gn,
                                     torch.as_tensor(data, device="cuda"), eps)
            Vo, To = OM.marching_tets(F, lo, hi, gn, near)
            np.testing.assert_array_equal(V.cpu().numpy(), Vo, err_msg=name)
            np.testing.assert_array_equal(T.cpu().numpy(), To, err_msg=name)
            if name == "torus" and eps == 10.0:
                assert _closed_euler(To) == 0


def test_mesh_degenerate_inputs(R, ctx):
    lo, hi, gn = (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), (5, 6, 7)
    n = 5 * 6 * 7
    data = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    # no sign change: empty mesh
    V, T = R.mesh_from_field(ctx, torch.ones(n, device="cuda"), lo, hi, gn, data, 5.0)
    assert V.shape == (0, 3) and T.shape == (0, 3)
    # no data: empty mask, empty mesh
    V, T = R.mesh_from_field(ctx, torch.randn(n, device="cuda"), lo, hi, gn, data[:0], 5.0)
    assert V.shape == (0, 3) and T.shape == (0, 3)
    # minimal grid: one cube
    F = np.array([-1, 1, 1, 1, 1, 1, 1, 2], dtype=np.float32)
    V, T = R.mesh_from_field(ctx, torch.as_tensor(F, device="cuda"), lo, hi, (2, 2, 2), data, 5.0)
    Vo, To = OM.marching_tets(F, lo, hi, (2, 2, 2), np.ones(8, bool))
    np.testing.assert_array_equal(V.cpu().numpy(), Vo)
    np.testing.assert_array_equal(T.cpu().numpy(), To)
    assert len(To) == 6                        # corner 0 is in all 6 tetrahedra
    with pytest.raises(R.RbfError):
        R.mesh_from_field(ctx, torch.ones(n, device="cuda"), lo, hi, gn, data, 0.0)
