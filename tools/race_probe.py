"""Race / synchronisation probe (run as a subprocess per library build).

    python tools/race_probe.py LIB OUT.npz

Runs every kernel family of librbf on small seeded inputs -- cell build, the
public fp32 / fp64 products, the symmetric solver operators, the grid (full and
eps-masked), zero set, marching tetrahedra, density, the preconditioners
(fp64 batched LU with DSMEM cluster panels, on-chip fp32 Gauss-Jordan with and
without pivoting over all size bins, the packed block-Jacobi apply), a GMRES
solve with the deterministic operator and a 2-rank loopback product -- and
saves every result.  tests/test_gpu_race_probe.py compares the CHECKED build
(csrc/checks.h: device bounds checks, lane/warp jitter at every shared-memory
hand-over) with the product build: deterministic results must be bit-identical
(a missing __syncwarp / __syncthreads / mbarrier wait would let jittered lanes
read stale shared memory), the atomics-ordered symmetric products equal to
fp32 rounding.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from oracle import extend as OE  # noqa: E402  (inputs only: the +/-delta set)
from synth import make_inputs  # noqa: E402

lib, out_path = sys.argv[1], sys.argv[2]
R.load_library(lib)
ctx = R.Context(0)
res = {}


def keep(name, t):
    torch.cuda.synchronize()
    res[name] = t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


d = make_inputs("c2", n=3000)
X = torch.as_tensor(OE.extend(d["x"], d["normals"], d["delta"]), device="cuda")
b = torch.as_tensor(OE.labels(len(d["x"]), d["delta"]).astype(np.float32), device="cuda")
kern = R.Kernel(d["sigma"])
cells = R.Cells(ctx, X, kern)
v = cells.view()
keep("perm", v["perm"])
keep("cell_start", v["cell_start"])
w = torch.as_tensor(np.random.default_rng(0).normal(size=X.shape[0]), device="cuda")
keep("mv32", R.matvec(ctx, cells, kern, w.float()))
keep("mv64", R.matvec(ctx, cells, kern, w))
for name, op in (("sym", R.OP_SYM), ("symw", R.OP_SYM_WIDE), ("symr", R.OP_SYM_ROT)):
    keep(f"atomic_{name}32", R.matvec_op(ctx, cells, kern, w.float(), op=op))
    keep(f"atomic_{name}64", R.matvec_op(ctx, cells, kern, w, op=op))
lo, hi, gn = d["grid_lo"], d["grid_hi"], (40, 40, 40)
F = R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
keep("grid", F)
keep("grid_coarse", R.eval_grid(ctx, cells, kern, w, lo, hi, (8, 8, 8)))
xd = torch.as_tensor(d["x"], device="cuda")
keep("grid_masked", R.eval_grid_masked(ctx, cells, kern, w, lo, hi, gn, xd, 2 * d["sigma"]))
keep("zero_set", R.zero_set(ctx, F.reshape(-1), lo, hi, gn, xd, 2 * d["sigma"]))
V, T = R.mesh_from_field(ctx, F.reshape(-1), lo, hi, gn, xd, 2 * d["sigma"])
keep("mesh_v", V)
keep("mesh_t", T)
keep("density", np.array(list(R.density(ctx, xd).values()), dtype=np.float64))
r = torch.as_tensor(np.random.default_rng(1).normal(size=X.shape[0]).astype(np.float32), device="cuda")
for name, kw in (("ras_lu64", dict(kind=2, core_target=256, overlap_sigmas=1.3)),
                 ("bj_gj48", dict(kind=1, core_target=48, shift=0.003, local_fp32=1)),
                 ("bj_gj128", dict(kind=1, core_target=128, shift=0.003, local_fp32=1)),
                 ("bj_gj200", dict(kind=1, core_target=200, shift=0.003, local_fp32=1)),
                 ("bj_gj_piv", dict(kind=1, core_target=128, shift=0.003, local_fp32=1, pivot=1)),
                 ("ras_gj_full", dict(kind=1, core_target=96, shift=0.003, local_fp32=1, w_layout=1))):
    P = R.Precond(ctx, cells, kern, **kw)
    keep("pc_" + name, P.apply(r))
    P.close()
wsol, rep = R.gmres_solve(ctx, cells, kern, b, restart=20, kind=1, core_target=64, shift=0.003, local_fp32=1,
                          max_iters=25, op=R.OP_ONESIDED)
keep("gmres_w", wsol)
# 2-rank loopback: deterministic one-sided product gathered on every rank
import threading  # noqa: E402
group = R.LoopbackGroup(2)
lb = [None, None]


def rank(q):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        c2 = R.Context(0, stream=st, loopback=(group, q))
        cl = R.Cells(c2, X, kern)
        lb[q] = R.matvec(c2, cl, kern, w).cpu().numpy()
        st.synchronize()
        c2.close()


th = [threading.Thread(target=rank, args=(q,)) for q in range(2)]
[t.start() for t in th]
[t.join() for t in th]
res["loopback_mv64_r0"], res["loopback_mv64_r1"] = lb
np.savez(out_path, **res)
print("race_probe ok", len(res), "results")
