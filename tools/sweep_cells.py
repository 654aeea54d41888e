"""Sweep the cell edge / tile span of the fp32 summation on one config (CUDA events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402
from tools.bench_kernels import timed  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
d = make_inputs(cfg)
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
w = torch.randn(c.shape[0], device="cuda")
f = torch.empty_like(w)
cut = 6 * d["sigma"]
for div, span in [(3.999, 2), (3.5, 2), (4.5, 2), (4.5, 3), (5.0, 3), (6.0, 3), (6.0, 4), (8.0, 4)]:
    cells = R.Cells(ctx, c, kern, cell_edge=cut / div, tile_span=span)
    u, v = R.matvec_pairs(ctx, cells, kern)
    t = timed(lambda: R.matvec(ctx, cells, kern, w, out=f), 10)
    print(json.dumps(dict(cfg=cfg, div=div, span=span, ntiles=cells.info()["ntiles"], frac=round(u / v, 3),
                          ms=round(t, 3), frac_of_peak=round(u / t / 1e9 / 4.653, 3))), flush=True)
