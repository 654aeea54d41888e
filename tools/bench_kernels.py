"""Kernel-level timing of the summation tiers and the cell build (CUDA events).

    python tools/bench_kernels.py --config c4 [--n N] [--iters 20]

Prints one JSON line per kernel: useful/visited pairs, ms per launch, pairs/s.
Used for tuning; bench.py is the contract benchmark.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402


def timed(fn, iters, warm=3):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    torch.cuda.synchronize()
    for a, b in evs:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    return t[len(t) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--f64", action="store_true")
    ap.add_argument("--precond", action="store_true", help="time the config's preconditioner setup + apply")
    ap.add_argument("--lib", default=None, help="alternative librbf .so (tools/build_variant.sh)")
    ap.add_argument("--ops", default="AUTO,SYM_WIDE,SYM_ROT,SYM")
    ap.add_argument("--no-grid", action="store_true")
    args = ap.parse_args()
    if args.lib:
        R.load_library(args.lib)
    t0 = time.time()
    d = make_inputs(args.config, n=args.n)
    tgen = time.time() - t0
    ctx = R.Context(0)
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    centres, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"),
                                 torch.as_tensor(d["normals"], device="cuda"), d["delta"])
    n = centres.shape[0]
    cells = R.Cells(ctx, centres, kern)
    tb = timed(lambda: R.Cells(ctx, centres, kern), 5, warm=1)
    info = cells.info()
    useful, visited = R.matvec_pairs(ctx, cells, kern)
    w = torch.randn(n, device="cuda", dtype=torch.float32)
    f = torch.empty_like(w)
    t32 = timed(lambda: R.matvec(ctx, cells, kern, w, out=f), args.iters)
    out = dict(config=args.config, centres=n, gen_s=round(tgen, 1), cells=info, build_ms=tb,
               useful=useful, visited=visited, useful_frac=useful / visited,
               matvec_f32_ms=t32, useful_pairs_per_s=useful / (t32 * 1e-3),
               visited_pairs_per_s=visited / (t32 * 1e-3))
    # the solver's operator (OP_AUTO: the symmetric wide-plan kernel at >= 2^18
    # centres), kernel-only time from the library's CUDA-event profiler, and
    # its agreement with the one-sided fp64 product
    wd64 = w.double()
    ref = R.matvec(ctx, cells, kern, wd64)
    g = R.matvec(ctx, cells, kern, wd64.abs())
    for name in args.ops.split(","):
        op = getattr(R, "OP_" + name)
        for _ in range(2):
            fo = R.matvec_op(ctx, cells, kern, w, op=op)
        ctx.profile(True)
        ctx.profile_query()
        for _ in range(args.iters):
            fo = R.matvec_op(ctx, cells, kern, w, op=op)
        pr = ctx.profile_query()
        ctx.profile(False)
        tm, nl = pr["matvec_f32"]
        err = ((fo.double() - ref).abs() / g.clamp_min(1e-300)).max().item()
        out[f"op_{name}"] = dict(kernel_ms=tm / max(nl, 1), frac_mufu=useful / (tm / max(nl, 1) * 1e-3) / 4.65312e12,
                                 max_err_over_g=err)
    if args.f64:
        w64 = w.double()
        f64 = torch.empty_like(w64)
        t64 = timed(lambda: R.matvec(ctx, cells, kern, w64, out=f64), max(3, args.iters // 4), warm=1)
        out.update(matvec_f64_ms=t64, f64_useful_pairs_per_s=useful / (t64 * 1e-3))
    if args.precond:
        cfg = d["cfg"]
        kw = dict(kind=cfg.precond_kind, core_target=cfg.core_target, overlap_sigmas=cfg.overlap_sigmas,
                  shift=cfg.shift, local_fp32=cfg.local_fp32)
        P = R.Precond(ctx, cells, kern, **kw)
        tp = timed(lambda: R.Precond(ctx, cells, kern, **kw), 3, warm=1)
        z = P.apply(w)
        ta = timed(lambda: P.apply(w, out=z), args.iters)
        out.update(precond_setup_ms=tp, precond_apply_ms=ta)
    if args.no_grid:
        print(json.dumps(out))
        return
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    wd = w.double()
    field = R.eval_grid(ctx, cells, kern, wd, lo, hi, gn)
    tg = timed(lambda: R.eval_grid(ctx, cells, kern, wd, lo, hi, gn, out=field), max(3, args.iters // 2))
    out.update(grid=gn, grid_ms=tg, grid_nonzero=int((field != 0).sum().item()))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
