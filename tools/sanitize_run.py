"""Small end-to-end workload for compute-sanitizer (racecheck / synccheck /
memcheck): every kernel family of librbf on c1/c2-sized inputs -- cell build,
public and solver fp32/fp64 products (one-sided, symmetric 64-target, wide,
rotation), grid, zero set, density, RAS with the fp64 batched LU (DSMEM cluster
panels), block-Jacobi with on-chip fp32 Gauss-Jordan + packed apply, the GMRES
solve, the assembled CSR operator and a 2-rank loopback solve.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from oracle import extend as OE  # noqa: E402  (inputs only)
from synth import make_inputs  # noqa: E402

small = "--small" in sys.argv
ctx = R.Context(0)
d = make_inputs("c2", n=1000 if small else 3000)
X = torch.as_tensor(OE.extend(d["x"], d["normals"], d["delta"]), device="cuda")
b = torch.as_tensor(OE.labels(len(d["x"]), d["delta"]).astype(np.float32), device="cuda")
kern = R.Kernel(d["sigma"])
cells = R.Cells(ctx, X, kern)
w = torch.randn(X.shape[0], device="cuda", dtype=torch.float64)
R.matvec(ctx, cells, kern, w.float())
R.matvec(ctx, cells, kern, w)
for op in (R.OP_SYM, R.OP_SYM_WIDE, R.OP_SYM_ROT):
    R.matvec_op(ctx, cells, kern, w.float(), op=op)
    R.matvec_op(ctx, cells, kern, w, op=op)
R.matvec_pairs(ctx, cells, kern)
lo, hi, gn = d["grid_lo"], d["grid_hi"], (24, 24, 24)
F = R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
R.eval_grid(ctx, cells, kern, w, lo, hi, (8, 8, 8))     # difference-form blocks
R.eval_grid_pairs(ctx, cells, kern, lo, hi, gn)
R.zero_set(ctx, F.reshape(-1), lo, hi, gn, torch.as_tensor(d["x"], device="cuda"), 2 * d["sigma"])
R.density(ctx, torch.as_tensor(d["x"], device="cuda"))
P = R.Precond(ctx, cells, kern, kind=2, core_target=512, overlap_sigmas=1.3)   # fp64 batched LU
P.apply(b)
P = R.Precond(ctx, cells, kern, kind=1, core_target=64, shift=0.003, local_fp32=1)   # on-chip GJ, packed apply
P.apply(b)
P = R.Precond(ctx, cells, kern, kind=1, core_target=64, shift=0.0, local_fp32=1, pivot=1)
P.apply(b)
R.gmres_solve(ctx, cells, kern, b, restart=20, rtol=1e-6, kind=2, core_target=512, overlap_sigmas=1.3, max_iters=30)
R.gmres_solve(ctx, cells, kern, b, restart=20, kind=1, core_target=64, shift=0.003, local_fp32=1, max_iters=20,
              op=R.OP_SYM_WIDE)
A = R.AssembledOperator(ctx, cells, kern)
A.spmv(w.float())
torch.cuda.synchronize()
if "--no-loopback" not in sys.argv:
    import threading
    group = R.LoopbackGroup(2)
    errs = []

    def rank(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                c2 = R.Context(0, stream=st, loopback=(group, r))
                cl = R.Cells(c2, X, kern)
                R.gmres_solve(c2, cl, kern, b, restart=20, kind=2, core_target=512, overlap_sigmas=1.3, max_iters=20,
                              op=R.OP_SYM_WIDE)
                R.eval_grid(c2, cl, kern, w, lo, hi, gn)
                st.synchronize()
                c2.close()
        except Exception as e:   # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs
print("sanitize_run ok")
