"""The c4 solve far past the benchmark's 50 iterations (F1): GMRES(50)
+ shifted block-Jacobi (the bench's preconditioner) with the two-phase
fp32 -> fp64 operator, up to `--iters` iterations toward rtol 1e-6, with the
library's residual history.  Prints one JSON line.

    python tools/c4_long_solve.py [--config c4] [--iters 1000] [--op 0]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--iters", type=int, default=1000)
ap.add_argument("--op", type=int, default=0)
ap.add_argument("--shift", type=float, default=None)
ap.add_argument("--core", type=int, default=None)
ap.add_argument("--restart", type=int, default=None)
args = ap.parse_args()
d = make_inputs(args.config)
cfg = d["cfg"]
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
cells = R.Cells(ctx, c, kern)
torch.cuda.synchronize()
t = time.perf_counter()
kw = dict(restart=args.restart or cfg.restart, rtol=1e-6, kind=cfg.precond_kind,
          core_target=args.core or cfg.core_target, overlap_sigmas=cfg.overlap_sigmas,
          shift=cfg.shift if args.shift is None else args.shift, local_fp32=cfg.local_fp32,
          cgs_passes=cfg.cgs_passes, max_iters=args.iters, op=args.op, history_cap=args.iters + 64)
w, rep = R.gmres_solve(ctx, cells, kern, b, **kw)
torch.cuda.synchronize()
wall = time.perf_counter() - t
h = rep.pop("history")
ht = rep.pop("history_true")
print(json.dumps(dict(config=args.config, solver=kw | {"history_cap": None}, wall_s=wall, report=rep,
                      est_every_50=h[49::50], true_per_restart=ht)))
