"""Small driver for ncu: cell build, a few solver iterations (operator variant
argv[2], default OP_AUTO; argv[3] iterations, default 3) and one grid evaluation of a config (argv[1], c4).

    ncu --set full -k regex:sum_f32_symb -s 1 -c 1 -o out python tools/prof_step.py c4
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

d = make_inputs(sys.argv[1] if len(sys.argv) > 1 else "c4")
op = int(sys.argv[2]) if len(sys.argv) > 2 else R.OP_AUTO
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = d["cfg"]
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
cells = R.Cells(ctx, c, kern)
w, _ = R.gmres_solve(ctx, cells, kern, b, restart=50, kind=cfg.precond_kind, core_target=cfg.core_target,
                     overlap_sigmas=cfg.overlap_sigmas, shift=cfg.shift, local_fp32=cfg.local_fp32, max_iters=iters,
                     op=op)
R.eval_grid(ctx, cells, kern, w, d["grid_lo"], d["grid_hi"], d["grid_n"])
torch.cuda.synchronize()
