"""Sweep tile-plan settings for the fp32 summation on one config (CUDA events)."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R
from synth import make_inputs
from tools.bench_kernels import timed

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
d = make_inputs(cfg)
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"), d["delta"])
w = torch.randn(c.shape[0], device="cuda")
f = torch.empty_like(w)
for mode, span, cap in [(1, 2, 64), (0, 2, 64), (0, 3, 64), (0, 4, 64), (0, 2, 32), (1, 1, 32)]:
    cells = R.Cells(ctx, c, kern, tile_cap=cap, tile_span=span, tile_mode=mode)
    u, v = R.matvec_pairs(ctx, cells, kern)
    t = timed(lambda: R.matvec(ctx, cells, kern, w, out=f), 10)
    print(json.dumps(dict(cfg=cfg, mode=mode, span=span, cap=cap, ntiles=cells.info()["ntiles"], useful=u, visited=v,
                          frac=round(u / v, 3), ms=round(t, 3), useful_Tps=round(u / t / 1e9, 3),
                          frac_of_peak=round(u / t / 1e9 / 4.653, 3))), flush=True)
