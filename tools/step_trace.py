"""Where the bench step's time goes beyond the profiled stages: CUDA events
between the public calls of one step (extend, cells, solve, grid), host clock
per call, the solver's own host timers, and the profiled stages.

    python tools/step_trace.py [config] [steps]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402


def main(name="c4", steps=4):
    steps = int(steps)
    d = make_inputs(name)
    cfg = d["cfg"]
    ctx = R.Context(0)
    kern = R.Kernel(d["sigma"], d["cutoff_sigmas"])
    x = torch.as_tensor(d["x"], device="cuda")
    nrm = torch.as_tensor(d["normals"], device="cuda")
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    kw = dict(restart=cfg.restart, rtol=1e-6, phase1_rtol=1e-4, kind=cfg.precond_kind, core_target=cfg.core_target,
              overlap_sigmas=cfg.overlap_sigmas, shift=cfg.shift, local_fp32=cfg.local_fp32,
              cgs_passes=cfg.cgs_passes, max_iters=50)
    for it in range(steps + 2):
        ctx.profile(True)
        ctx.profile_query()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        hs = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record()
        centres, b = R.extend_points(ctx, x, nrm, d["delta"])
        ev[1].record(); hs.append(time.perf_counter())
        cells = R.Cells(ctx, centres, kern)
        ev[2].record(); hs.append(time.perf_counter())
        w, rep = R.gmres_solve(ctx, cells, kern, b, **kw)
        ev[3].record(); hs.append(time.perf_counter())
        field = R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
        ev[4].record(); hs.append(time.perf_counter())
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        prof = ctx.profile_query()
        dev = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        host = [1e3 * (hs[0] - t0)] + [1e3 * (hs[i + 1] - hs[i]) for i in range(3)]
        print(json.dumps(dict(step=it, wall_ms=round(1e3 * (t1 - t0), 1),
                              dev_ms=dict(zip(["extend", "cells", "solve", "grid"], [round(v, 2) for v in dev])),
                              host_ms=dict(zip(["extend", "cells", "solve", "grid"], [round(v, 2) for v in host])),
                              solver=dict(t_setup=round(1e3 * rep["t_setup"], 2), t_phase1=round(1e3 * rep["t_phase1"], 2),
                                          t_phase2=round(1e3 * rep["t_phase2"], 2)),
                              prof={k: round(v[0], 2) for k, v in prof.items()})),
              flush=True)
        del cells, w, field


if __name__ == "__main__":
    main(*sys.argv[1:])
