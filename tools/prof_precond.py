"""Build the RAS preconditioner of a config once (for launch-list profiling)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R
from synth import make_inputs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
d = make_inputs(cfg, n=n)
ctx = R.Context(0)
kern = R.Kernel(d["sigma"])
c, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"), d["delta"])
cells = R.Cells(ctx, c, kern)
torch.cuda.synchronize()
t = time.time()
P = R.Precond(ctx, cells, kern, core_target=d["cfg"].core_target, overlap_sigmas=d["cfg"].overlap_sigmas)
torch.cuda.synchronize()
print("precond build s", time.time() - t, "blocks", P.blocks()[2] if False else "")
