"""Sweep the wide (symmetric) tile plan: RBF_WIDE_SPAN / RBF_WIDE_CAP and the
cell edge, timing the solver's symmetric fp32 operator (RBF_PUBLIC_SYM=1)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402
from tools.bench_kernels import timed  # noqa: E402

os.environ["RBF_PUBLIC_SYM"] = "1"
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
d = make_inputs(cfg)
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
w = torch.randn(c.shape[0], device="cuda", dtype=torch.float32)
f = torch.empty_like(w)
cut = 6 * d["sigma"]
for div, span, cap in [(3.999, 4, 128), (3.999, 3, 128), (3.999, 2, 128), (3.999, 4, 96), (4.999, 4, 128),
                       (4.999, 5, 128), (4.999, 3, 128), (5.999, 6, 128), (5.999, 4, 128), (2.999, 3, 128),
                       (2.999, 2, 128)]:
    os.environ["RBF_WIDE_SPAN"], os.environ["RBF_WIDE_CAP"] = str(span), str(cap)
    cells = R.Cells(ctx, c, kern, cell_edge=cut / div)
    t = timed(lambda: R.matvec(ctx, cells, kern, w, out=f), 10)
    print(json.dumps(dict(cfg=cfg, div=div, span=span, cap=cap, ms=round(t, 4))), flush=True)
    del cells
