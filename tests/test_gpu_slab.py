"""GPU checks of the slab partition's kernels.

Only one GPU is available to the tests, so each rank r of a W-way partition is
emulated in turn (RBF_SLAB_EMULATE="r/W": the cells get rank r's slab; the
window is read from the full vector instead of arriving by NCCL).  This checks
everything rank-local -- the slab plan on device data, tile ranges, source
windows, pointer shifts, node-layer ownership, slab-local blocks -- against:
  * the host plan (rbf_slab_plan) on the ORACLE's cell replica (bit-exact ranges);
  * the single-GPU result (itself parity-tested against the oracle): every
    owned matvec entry and owned grid layer is bit-identical to it, because a
    tile's arithmetic does not depend on which rank runs it;
  * the oracle's block definition restricted to the slab's cells.
The NCCL exchange itself is covered on CPU by tests/test_dist_cpu.py (gloo).
"""
import os

import numpy as np
import pytest
import torch

from oracle import cells as OC
from oracle import extend as OE
from oracle import solve as OS
from synth import make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


@pytest.fixture(scope="module")
def setup(R):
    ctx = R.Context(0)
    d = make_inputs("c3", n=4000)          # 10x density ramp along x: unequal planes
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    Xd = torch.as_tensor(X, device="cuda")
    full = R.Cells(ctx, Xd, kern)
    w = torch.as_tensor(np.random.default_rng(3).normal(size=len(X)), device="cuda")
    f32 = R.matvec(ctx, full, kern, w.float()).cpu().numpy()
    f64 = R.matvec(ctx, full, kern, w).cpu().numpy()
    lo, hi, gn = d["grid_lo"], d["grid_hi"], (40, 40, 40)
    F = R.eval_grid(ctx, full, kern, w, lo, hi, gn).cpu().numpy()
    return dict(ctx=ctx, d=d, X=X, Xd=Xd, kern=kern, sigma=sigma, full=full, w=w, f32=f32, f64=f64,
                grid=(lo, hi, gn), F=F, info=full.info(), perm=full.view()["perm"].cpu().numpy())


def _emulated(R, s, rank, world):
    os.environ["RBF_SLAB_EMULATE"] = f"{rank}/{world}"
    try:
        return R.Cells(s["ctx"], s["Xd"], s["kern"])
    finally:
        del os.environ["RBF_SLAB_EMULATE"]


def _host_plan(R, s, world):
    oc = OC.build(s["X"], 6 * s["sigma"], cell_edge=6 * s["sigma"] / 3.999)
    dim = oc["dim"]
    per_plane = int(dim[0] * dim[1])
    cs, ce = oc["cell_start"].astype(np.int64), oc["cell_end"].astype(np.int64)
    ps = np.concatenate([cs[::per_plane][: dim[2]], [len(s["X"])]])
    weight = ((ce - cs).astype(np.float64) ** 2).reshape(dim[2], per_plane).sum(axis=1)
    return oc, R.slab_plan(ps, weight, s["info"]["reach"] + 1, world)


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_slabs_match_single_gpu(R, setup, world):
    s = setup
    oc, plan = _host_plan(R, s, world)
    perm = s["perm"]
    lo, hi, gn = s["grid"]
    covered_rows = np.zeros(len(s["X"]), dtype=int)
    layers = np.zeros(gn[2], dtype=int)
    for r in range(world):
        c = _emulated(R, s, r, world)
        sl = c.slab()
        o0, o1 = sl["own"]
        assert (o0, o1) == (plan["own_lo"][r], plan["own_hi"][r])
        assert sl["window"] == (plan["win_lo"][r], plan["win_hi"][r]) or o0 == o1
        assert sl["planes"] == (plan["plane_lo"][r], plan["plane_lo"][r + 1])
        covered_rows[o0:o1] += 1
        mine = perm[o0:o1]                                   # caller indices of the owned targets
        g32 = R.matvec(s["ctx"], c, s["kern"], s["w"].float()).cpu().numpy()
        g64 = R.matvec(s["ctx"], c, s["kern"], s["w"]).cpu().numpy()
        np.testing.assert_array_equal(g32[mine], s["f32"][mine])
        np.testing.assert_array_equal(g64[mine], s["f64"][mine])
        G = R.eval_grid(s["ctx"], c, s["kern"], s["w"], lo, hi, gn).cpu().numpy()
        own_layers = [k for k in range(gn[2]) if np.any(G[k] != 0)]
        for k in own_layers:
            np.testing.assert_array_equal(G[k], s["F"][k])
        layers[own_layers] += 1
        # slab-local block-Jacobi blocks = the oracle's definition on the slab's cells
        P = R.Precond(s["ctx"], c, s["kern"], kind=1, core_target=64, shift=0.003, local_fp32=1)
        cores, exts, _ = P.blocks()
        sub = dict(oc)
        dim = oc["dim"]
        pz = np.arange(len(oc["cell_start"])) // (dim[0] * dim[1])
        keep = (pz >= sl["planes"][0]) & (pz < sl["planes"][1])
        sub["cell_end"] = np.where(keep, oc["cell_end"], oc["cell_start"])
        ref = OS.ras_blocks(sub, s["sigma"], 64, 0.0) if o1 > o0 else []
        assert len(cores) == len(ref)
        for k, blk in enumerate(ref):
            np.testing.assert_array_equal(cores[k] + o0, blk["core"])
            np.testing.assert_array_equal(exts[k] + o0, blk["ext"])
    assert (covered_rows == 1).all()                        # slabs partition the targets
    nonzero_layers = [k for k in range(gn[2]) if np.any(s["F"][k] != 0)]
    assert (layers[nonzero_layers] == 1).all()              # every layer owned once


def test_emulated_cells_refuse_the_solver(R, setup):
    s = setup
    c = _emulated(R, s, 0, 2)
    b = torch.zeros(len(s["X"]), dtype=torch.float32, device="cuda")
    with pytest.raises(R.RbfError):
        R.gmres_solve(s["ctx"], c, s["kern"], b)


@pytest.mark.parametrize("op", ["OP_SYM", "OP_SYM_WIDE"])
def test_emulated_slabs_symmetric_solver_operator(R, setup, op):
    """The solver's symmetric fp32/fp64 operators (reading R19) on emulated slabs:
    each rank's owned rows equal the single-GPU symmetric product to the tiers'
    accuracy (the atomics reorder the last bits), and the single-GPU symmetric
    product equals the one-sided one likewise."""
    s = setup
    perm = s["perm"]
    opv = getattr(R, op)
    full32 = R.matvec_op(s["ctx"], s["full"], s["kern"], s["w"].float(), op=opv).cpu().numpy()
    full64 = R.matvec_op(s["ctx"], s["full"], s["kern"], s["w"], op=opv).cpu().numpy()
    g = np.abs(s["f64"]).max()
    np.testing.assert_allclose(full32, s["f32"], rtol=0, atol=1e-5 * g)
    np.testing.assert_allclose(full64, s["f64"], rtol=0, atol=1e-12 * g)
    for r in range(2):
        c = _emulated(R, s, r, 2)
        o0, o1 = c.slab()["own"]
        mine = perm[o0:o1]
        g32 = R.matvec_op(s["ctx"], c, s["kern"], s["w"].float(), op=opv).cpu().numpy()
        g64 = R.matvec_op(s["ctx"], c, s["kern"], s["w"], op=opv).cpu().numpy()
        np.testing.assert_allclose(g32[mine], s["f32"][mine], rtol=0, atol=1e-5 * g)
        np.testing.assert_allclose(g64[mine], s["f64"][mine], rtol=0, atol=1e-12 * g)
