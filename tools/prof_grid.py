"""Small driver for ncu of the grid path: cell build, a short solve, the full
grid (sum_f32_kernel<1> + mark_node_blocks) and rbf_isosurface (eps mask,
masked grid, marching tetrahedra) of a config (argv[1], default c4).

    ncu --set full -k regex:"sum_f32_kernel|mark_node_blocks|near_kernel|mt_" -o out python tools/prof_grid.py c4
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

d = make_inputs(sys.argv[1] if len(sys.argv) > 1 else "c4")
cfg = d["cfg"]
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
x = torch.as_tensor(d["x"], device="cuda")
c, b = R.extend_points(ctx, x, torch.as_tensor(d["normals"], device="cuda"), d["delta"])
cells = R.Cells(ctx, c, kern)
w, _ = R.gmres_solve(ctx, cells, kern, b, restart=50, kind=cfg.precond_kind, core_target=cfg.core_target,
                     overlap_sigmas=cfg.overlap_sigmas, shift=cfg.shift, local_fp32=cfg.local_fp32, max_iters=3)
lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
V, T = R.isosurface(ctx, cells, kern, w, lo, hi, gn, x, 2 * d["sigma"])
torch.cuda.synchronize()
print("mesh", V.shape[0], T.shape[0])
