"""Run a few solver iterations with the wide symmetric fp32 tier (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

os.environ.setdefault("RBF_SUM_SYM", "2")
d = make_inputs(sys.argv[1] if len(sys.argv) > 1 else "c4")
cfg = d["cfg"]
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
cells = R.Cells(ctx, c, kern)
R.gmres_solve(ctx, cells, kern, b, restart=50, kind=cfg.precond_kind, core_target=cfg.core_target,
              overlap_sigmas=cfg.overlap_sigmas, shift=cfg.shift, local_fp32=cfg.local_fp32, max_iters=3)
torch.cuda.synchronize()
