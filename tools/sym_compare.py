"""Compare the fp32-tier matvec variants of the solver on one config (reading R19):
one-sided (RBF_SUM_SYM=0), symmetric on the 64-target plan (1), symmetric on the
wide 128-target plan (2).  Prints per variant: ms per matvec (library CUDA
events), the 50-iteration fit's true residual, the agreement with the one-sided
product."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    if len(sys.argv) > 2:
        R.load_library(sys.argv[2])      # an experimental build of librbf.so
    d = make_inputs(name)
    cfg = d["cfg"]
    ctx = R.Context(0)
    kern = R.Kernel(d["sigma"])
    c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                           d["delta"])
    div = float(os.environ.get("CELL_DIV", "3.999"))
    cells = R.Cells(ctx, c, kern, cell_edge=6 * d["sigma"] / div)
    kw = dict(restart=50, kind=cfg.precond_kind, core_target=cfg.core_target, overlap_sigmas=cfg.overlap_sigmas,
              shift=cfg.shift, local_fp32=cfg.local_fp32, max_iters=50)
    ref_w = None
    modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2"]
    for mode in modes:
        os.environ["RBF_SUM_SYM"] = mode
        R.gmres_solve(ctx, cells, kern, b, **kw)          # warm
        torch.cuda.synchronize()
        ctx.profile(True)
        ctx.profile_query()
        w, rep = R.gmres_solve(ctx, cells, kern, b, **kw)
        prof = ctx.profile_query()
        ctx.profile(False)
        t, nl = prof["matvec_f32"]
        if ref_w is None:
            ref_w = w.clone()
        print(json.dumps(dict(config=name, sym=mode, ms_per_matvec=t / max(nl, 1), res=rep["rel_residual_true"],
                              w_rel_diff=float((w - ref_w).norm() / ref_w.norm()))), flush=True)
    del os.environ["RBF_SUM_SYM"]


if __name__ == "__main__":
    main()
