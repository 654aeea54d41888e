"""The multi-rank slab partition executed on ONE GPU.

W contexts of this process join an in-process loopback group
(rbf_loopback_group_create / rbf_create_loopback): each rank runs in its own
host thread on its own stream and the library's multi-rank code path runs
unchanged -- slab plan, halo exchange of the source window, the symmetric
operators' reverse halo reduction, Krylov all-reduces, the gathers of the
solution and of the grid layers -- with device copies between the ranks'
buffers in place of NCCL (transport.h).  Checked against:
  * the host plan (rbf_slab_plan) on the ORACLE's cell replica (bit-exact ranges);
  * the single-GPU result: one-sided matvec rows and grid layers are
    BIT-identical (a tile's arithmetic does not depend on which rank runs it);
  * the ORACLE's products for the symmetric operators (pairs across slabs are
    evaluated once, by the lower rank, and sent back) and the oracle's fp64
    residual for the distributed GMRES solve;
  * the oracle's block definition restricted to each slab's cells.
"""
import threading

import numpy as np
import pytest
import torch

from oracle import cells as OC
from oracle import extend as OE
from oracle import kernel as OK
from oracle import solve as OS
from synth import make_inputs

pytestmark = pytest.mark.gpu
TIMEOUT = 600


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


def run_ranks(R, world, fn):
    """fn(ctx, rank) on `world` threads, one loopback context (own stream) each.
    Returns the per-rank results; re-raises the first exception."""
    group = R.LoopbackGroup(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ctx = R.Context(0, stream=st, loopback=(group, r))
                try:
                    out[r] = fn(ctx, r)
                    st.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:   # noqa: BLE001 -- reported below
            err[r] = e

    torch.cuda.synchronize()
    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(TIMEOUT)
    assert not any(t.is_alive() for t in th), "loopback ranks did not finish (deadlock?)"
    for e in err:
        if e is not None:
            raise e
    group.close()
    return out


@pytest.fixture(scope="module")
def setup(R):
    ctx = R.Context(0)
    d = make_inputs("c3", n=4000)          # 10x density ramp along x: unequal planes
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    Xd = torch.as_tensor(X, device="cuda")
    full = R.Cells(ctx, Xd, kern)
    w = np.random.default_rng(3).normal(size=len(X))
    wt = torch.as_tensor(w, device="cuda")
    f32 = R.matvec(ctx, full, kern, wt.float()).cpu().numpy()
    f64 = R.matvec(ctx, full, kern, wt).cpu().numpy()
    lo, hi, gn = d["grid_lo"], d["grid_hi"], (40, 40, 40)
    F = R.eval_grid(ctx, full, kern, wt, lo, hi, gn).cpu().numpy()
    useful, _ = R.matvec_pairs(ctx, full, kern)
    Xo = X.astype(np.float64)
    return dict(d=d, X=X, kern=kern, sigma=sigma, w=w, f32=f32, f64=f64, grid=(lo, hi, gn), F=F,
                info=full.info(), perm=full.view()["perm"].cpu().numpy(), useful=useful,
                ref32=OK.matvec(Xo, w.astype(np.float32).astype(np.float64), sigma),
                ref64=OK.matvec(Xo, w, sigma), g=OK.matvec(Xo, np.abs(w), sigma))


def _host_plan(R, s, world):
    oc = OC.build(s["X"], 6 * s["sigma"], cell_edge=6 * s["sigma"] / 3.999)
    dim = oc["dim"]
    per_plane = int(dim[0] * dim[1])
    cs, ce = oc["cell_start"].astype(np.int64), oc["cell_end"].astype(np.int64)
    ps = np.concatenate([cs[::per_plane][: dim[2]], [len(s["X"])]])
    weight = ((ce - cs).astype(np.float64) ** 2).reshape(dim[2], per_plane).sum(axis=1)
    return oc, R.slab_plan(ps, weight, s["info"]["reach"] + 1, world)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_partition_products_and_grid(R, setup, world):
    s = setup
    oc, plan = _host_plan(R, s, world)
    lo, hi, gn = s["grid"]

    def rank(ctx, r):
        Xd = torch.as_tensor(s["X"], device="cuda")
        wt = torch.as_tensor(s["w"], device="cuda")
        c = R.Cells(ctx, Xd, s["kern"])
        res = dict(slab=c.slab())
        res["f32"] = R.matvec(ctx, c, s["kern"], wt.float()).cpu().numpy()
        res["f64"] = R.matvec(ctx, c, s["kern"], wt).cpu().numpy()
        for op in ("OP_SYM", "OP_SYM_WIDE", "OP_SYM_ROT", "OP_ONESIDED"):
            res[op] = (R.matvec_op(ctx, c, s["kern"], wt.float(), op=getattr(R, op)).cpu().numpy(),
                       R.matvec_op(ctx, c, s["kern"], wt, op=getattr(R, op)).cpu().numpy())
        # the wide operator's two distributed forms: peer memory (default on this
        # transport: one kernel reads and updates the other ranks' buffers) and
        # the copy-based halo exchange + reverse reduction (NCCL's form)
        ctx.peer_memory(False)
        res["OP_SYM_WIDE_copy"] = (R.matvec_op(ctx, c, s["kern"], wt.float(), op=R.OP_SYM_WIDE).cpu().numpy(),
                                   R.matvec_op(ctx, c, s["kern"], wt, op=R.OP_SYM_WIDE).cpu().numpy())
        ctx.peer_memory(True)
        res["F"] = R.eval_grid(ctx, c, s["kern"], wt, lo, hi, gn).cpu().numpy()
        part = torch.full((gn[2], gn[1], gn[0]), -1.0, device="cuda")
        res["layers"] = R.eval_grid_slab(ctx, c, s["kern"], wt, lo, hi, gn, part)
        res["part"] = part.cpu().numpy()
        res["useful"] = R.matvec_pairs(ctx, c, s["kern"])[0]
        P = R.Precond(ctx, c, s["kern"], kind=1, core_target=64, shift=0.003, local_fp32=1)
        res["blocks"] = P.blocks()
        P.close()
        # the paper's distributed RASM: cores from the slab, ext sets across slabs
        P = R.Precond(ctx, c, s["kern"], kind=2, core_target=128, overlap_sigmas=1.0)
        res["ras_blocks"] = P.blocks()
        P.close()
        return res

    out = run_ranks(R, world, rank)
    covered = np.zeros(len(s["X"]), dtype=int)
    layers = np.zeros(gn[2], dtype=int)
    for r, res in enumerate(out):
        sl = res["slab"]
        o0, o1 = sl["own"]
        assert (o0, o1) == (plan["own_lo"][r], plan["own_hi"][r])
        assert sl["window"] == (plan["win_lo"][r], plan["win_hi"][r]) or o0 == o1
        assert sl["planes"] == (plan["plane_lo"][r], plan["plane_lo"][r + 1])
        covered[o0:o1] += 1
        # replicated out: every rank returns the full vectors / field
        np.testing.assert_array_equal(res["f32"], s["f32"])
        np.testing.assert_array_equal(res["f64"], s["f64"])
        np.testing.assert_array_equal(res["F"], s["F"])
        k0, k1 = res["layers"]
        np.testing.assert_array_equal(res["part"][k0:k1], s["F"][k0:k1])
        assert (res["part"][:k0] == -1).all() and (res["part"][k1:] == -1).all()
        layers[k0:k1] += 1
        # solver operators across slabs against the oracle (tier tolerances)
        for op in ("OP_SYM", "OP_SYM_WIDE", "OP_SYM_ROT", "OP_ONESIDED", "OP_SYM_WIDE_copy"):
            a32, a64 = res[op]
            assert (np.abs(a32 - s["ref32"]) <= 5e-5 * s["g"]).all(), (op, r)
            assert (np.abs(a64 - s["ref64"]) <= 1e-12 * s["g"]).all(), (op, r)
        # slab-local block-Jacobi blocks = the oracle's definition on the slab's cells
        cores, exts, _ = res["blocks"]
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
        # RAS blocks: cores from the slab's cells, extended sets from every cell
        cores, exts, _ = res["ras_blocks"]
        ref = OS.ras_blocks(oc, s["sigma"], 128, 1.0, core_cells=keep) if o1 > o0 else []
        assert len(cores) == len(ref)
        for k, blk in enumerate(ref):
            np.testing.assert_array_equal(cores[k] + o0, blk["core"])
            np.testing.assert_array_equal(exts[k] + o0, blk["ext"])
    assert (covered == 1).all()                     # slabs partition the targets
    assert (layers == 1).all()                      # every node layer owned once
    # the wide plan's interior tiles (run while the halo is exchanged on the aux
    # stream) are a prefix of each rank's wide tiles; at W = 2 and 3 the slabs
    # are thick enough for the overlapped path to run (checked above by the
    # OP_SYM_WIDE / OP_SYM_ROT rows against the oracle)
    interior = [res["slab"]["wide_interior"] for res in out]
    for res in out:
        t0, t1 = res["slab"]["wide_tiles"]
        assert 0 <= res["slab"]["wide_interior"] <= t1 - t0
    if world < 8:
        assert sum(interior) > 0
    # per-rank useful pairs of the slab plan (balanced by sum n_c^2) add up to the whole
    per_rank = np.array([res["useful"] for res in out])
    assert per_rank.sum() == s["useful"]
    if world == 8:
        print(f"\nW=8 useful pairs per rank / (W=1 / 8): {np.round(per_rank / (s['useful'] / 8), 3).tolist()}")


@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_distributed_ras_apply(R, world):
    """The paper's distributed RASM applied across W slabs: z = sum_i
    R~_i^T A_i^-1 R_i r over every rank's blocks (cores from the slab, extended
    sets through the halo) against the ORACLE's RAS apply of the same blocks
    (fp64 scipy LU), gathered on every rank."""
    d = make_inputs("c2", n=3000)
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    r = np.random.default_rng(5).normal(size=len(X)).astype(np.float32)
    oc = OC.build(X, 6 * sigma, cell_edge=6 * sigma / 3.999)
    dim = oc["dim"]
    pz = np.arange(len(oc["cell_start"])) // (dim[0] * dim[1])

    def rank(ctx, k):
        c = R.Cells(ctx, torch.as_tensor(X, device="cuda"), kern)
        P = R.Precond(ctx, c, kern, kind=2, core_target=512, overlap_sigmas=1.3)
        z = P.apply(torch.as_tensor(r, device="cuda")).cpu().numpy()
        blocks = P.blocks()
        P.close()
        return z, blocks, c.slab()

    out = run_ranks(R, world, rank)
    blocks = []
    for z, (cores, exts, _), sl in out:
        o0 = sl["own"][0]
        keep = (pz >= sl["planes"][0]) & (pz < sl["planes"][1])
        ref = OS.ras_blocks(oc, sigma, 512, 1.3, core_cells=keep) if sl["own"][1] > o0 else []
        assert len(ref) == len(cores)
        for k, blk in enumerate(ref):
            np.testing.assert_array_equal(cores[k] + o0, blk["core"])
            np.testing.assert_array_equal(exts[k] + o0, blk["ext"])
        blocks += ref
    np.testing.assert_array_equal(out[0][0], out[-1][0])
    perm = oc["perm"]
    zs = OS.ras_apply(blocks, oc["sorted"], r.astype(np.float64)[perm], sigma)
    zref = np.empty_like(zs)
    zref[perm] = zs
    err = np.linalg.norm(out[0][0] - zref) / np.linalg.norm(zref)
    assert err <= 1e-3, err


@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_distributed_solve(R, world):
    """rbf_gmres_solve over W ranks (the distributed RASM: cores in the slab,
    extended sets through the halo; fp32 -> fp64 phases; symmetric operators
    with reverse halo reduction; all-reduced Krylov dots): reaches the 1e-6 gate
    on c1's Fibonacci sphere at 8000 points (24k centres, sigma 0.035 so that
    sigma/spacing stays c1's 0.89, delta = 0.1 sigma; ~40 cell planes, >= 5 per
    slab at W = 8), certified by the ORACLE's fp64 matvec, and every rank returns
    the same weights.  The deterministic one-sided variant (OP_ONESIDED) too.
    (Slabs of one cell plane -- an 8-way split of the flat c2 torus -- turn the
    cores into thin sheets and exact RAS stalls.)"""
    d = make_inputs("c1", n=8000, sigma=0.035, delta=0.0035)
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    ctx1 = R.Context(0)
    cells1 = R.Cells(ctx1, torch.as_tensor(X, device="cuda"), kern)
    # the paper's distributed RASM: cores in the slab, extended sets reaching
    # 1.3 sigma into the neighbouring slabs through the halo
    kw = dict(restart=30, rtol=1e-6, kind=2, core_target=512, overlap_sigmas=3.0, max_iters=400)
    w1, rep1 = R.gmres_solve(ctx1, cells1, kern, torch.as_tensor(b, device="cuda"), **kw)
    res1 = np.linalg.norm(b - OK.matvec(X.astype(np.float64), w1.cpu().numpy(), sigma)) / np.linalg.norm(b)
    assert res1 <= 1.5e-6, (res1, rep1)
    for op, peer in ((R.OP_AUTO, True), (R.OP_SYM_WIDE, True), (R.OP_SYM_WIDE, False), (R.OP_ONESIDED, True)):
        def rank(ctx, r):
            ctx.peer_memory(peer)
            c = R.Cells(ctx, torch.as_tensor(X, device="cuda"), kern)
            w, rep = R.gmres_solve(ctx, c, kern, torch.as_tensor(b, device="cuda"), op=op, **kw)
            return w.cpu().numpy(), rep

        out = run_ranks(R, world, rank)
        w0 = out[0][0]
        for w, rep in out:
            np.testing.assert_array_equal(w, w0)    # replicated out, identical on every rank
        res = np.linalg.norm(b - OK.matvec(X.astype(np.float64), w0, sigma)) / np.linalg.norm(b)
        rep = out[0][1]
        assert rep["converged"] == 1 and res <= 1.5e-6, (op, res, rep, res1, rep1)
        assert res == pytest.approx(rep["rel_residual_true"], rel=1e-3)
        its, its1 = rep["iters_phase1"] + rep["iters_phase2"], rep1["iters_phase1"] + rep1["iters_phase2"]
        assert its <= 2 * its1 + 10, (op, its, its1)


def test_loopback_reconstruct_host(R):
    """rbf_reconstruct_host (host buffers in, weights + field out) over 2 ranks:
    both ranks return the same weights and field; the field matches the
    single-GPU one from the same weights to the grid tier's accuracy."""
    d = make_inputs("c1")
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]

    def rank(ctx, r):
        w, F, rep = R.reconstruct_host(ctx, X, b, kern, lo, hi, gn, kind=2, core_target=512, overlap_sigmas=3.0,
                                       restart=30, rtol=1e-6, max_iters=400)
        return w.numpy().copy(), F.numpy().copy(), rep

    out = run_ranks(R, 2, rank)
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    w = out[0][0]
    res = np.linalg.norm(b - OK.matvec(X.astype(np.float64), w, sigma)) / np.linalg.norm(b)
    assert res <= 1.5e-6, (res, out[0][2])
    ctx1 = R.Context(0)
    cells1 = R.Cells(ctx1, torch.as_tensor(X, device="cuda"), kern)
    F1 = R.eval_grid(ctx1, cells1, kern, torch.as_tensor(w, device="cuda"), lo, hi, gn).cpu().numpy()
    np.testing.assert_array_equal(out[0][1], F1)


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_isosurface(R, setup, world):
    """rbf_isosurface over slab ranks: each rank evaluates the masked node blocks
    of its own layers, the layers are gathered (NaN outside M_ext^eps travels as
    data), and every rank's mesh equals the single-GPU mesh bit for bit."""
    s = setup
    lo, hi, gn = s["grid"]
    data = np.ascontiguousarray(s["d"]["x"], dtype=np.float64)
    eps = 2 * s["sigma"]
    ctx = R.Context(0)
    c1 = R.Cells(ctx, torch.as_tensor(s["X"], device="cuda"), s["kern"])
    wt = torch.as_tensor(s["w"], device="cuda")
    F1 = torch.empty(gn[0] * gn[1] * gn[2], dtype=torch.float32, device="cuda")
    V1, T1 = R.isosurface(ctx, c1, s["kern"], wt, lo, hi, gn, torch.as_tensor(data, device="cuda"), eps, field=F1)
    V1, T1, F1 = V1.cpu().numpy(), T1.cpu().numpy(), F1.cpu().numpy()
    assert len(T1) > 100

    def rank(ctx, r):
        c = R.Cells(ctx, torch.as_tensor(s["X"], device="cuda"), s["kern"])
        F = torch.empty(gn[0] * gn[1] * gn[2], dtype=torch.float32, device="cuda")
        V, T = R.isosurface(ctx, c, s["kern"], torch.as_tensor(s["w"], device="cuda"), lo, hi, gn,
                            torch.as_tensor(data, device="cuda"), eps, field=F)
        return V.cpu().numpy(), T.cpu().numpy(), F.cpu().numpy()

    for V, T, F in run_ranks(R, world, rank):
        assert np.array_equal(F.view(np.uint32), F1.view(np.uint32))
        np.testing.assert_array_equal(V, V1)
        np.testing.assert_array_equal(T, T1)


@pytest.mark.parametrize("world", [2, 3])
def test_loopback_sharded_inputs(R, world):
    """SURVEY §8(b)'s sharded interface: rank r passes only its shard of the
    caller-order centres and right-hand side (global ids [id0, id0 + n_r); the
    ranges are assigned to ranks in a shuffled order to exercise the tiling
    check) and receives its shard of the weights -- equal bit for bit to the
    replicated call's cells and weights."""
    d = make_inputs("c1")
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32)
    kern = R.Kernel(d["sigma"])
    kw = dict(restart=30, rtol=1e-6, kind=2, core_target=512, overlap_sigmas=3.0, max_iters=400)
    n = len(X)
    cuts = np.linspace(0, n, world + 1).astype(int)
    order = np.random.default_rng(world).permutation(world)       # rank r holds range order[r]

    def rank(ctx, r):
        k = order[r]
        lo, hi = int(cuts[k]), int(cuts[k + 1])
        c = R.Cells(ctx, torch.as_tensor(X[lo:hi], device="cuda"), kern, id0=lo)
        full = R.Cells(ctx, torch.as_tensor(X, device="cuda"), kern)
        vs, vf = c.view(), full.view()
        same = all(torch.equal(vs[key], vf[key]) for key in ("perm", "keys", "cell_start"))
        ws, rep = R.gmres_solve_shard(ctx, c, kern, torch.as_tensor(b[lo:hi], device="cuda"), lo, **kw)
        wf, _ = R.gmres_solve(ctx, full, kern, torch.as_tensor(b, device="cuda"), **kw)
        return same, ws.cpu().numpy(), wf.cpu().numpy()[lo:hi], c.n

    for same, ws, wf, nc in run_ranks(R, world, rank):
        assert same and nc == n
        np.testing.assert_array_equal(ws, wf)
    # shards that do not tile [0, n) are rejected on every rank
    def bad(ctx, r):
        with pytest.raises(R.RbfError):
            R.Cells(ctx, torch.as_tensor(X[:10], device="cuda"), kern, id0=5 * r + 1)
        return True
    assert all(run_ranks(R, world, bad))
