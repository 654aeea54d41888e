"""Debug driver: distributed solve on W loopback ranks for the c2 n=3000 torus."""
import sys, os, threading
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R
from oracle import extend as OE, kernel as OK
from synth import make_inputs
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_loopback import run_ranks
d = make_inputs("c2", n=3000)
X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32)
sigma = d["sigma"]; kern = R.Kernel(sigma)
for world, kw in [(8, dict(kind=2, core_target=512, overlap_sigmas=1.3)), (8, dict(kind=1, core_target=128)),
                  (4, dict(kind=2, core_target=512, overlap_sigmas=1.3)), (6, dict(kind=2, core_target=512, overlap_sigmas=1.3)),
                  (8, dict(kind=0)), (1, dict(kind=0))]:
    def rank(ctx, r):
        c = R.Cells(ctx, torch.as_tensor(X, device="cuda"), kern)
        w, rep = R.gmres_solve(ctx, c, kern, torch.as_tensor(b, device="cuda"), restart=50, rtol=1e-6, max_iters=150,
                               history_cap=200, **kw)
        return w.cpu().numpy(), rep, c.slab()
    out = run_ranks(R, world, rank)
    w, rep, _ = out[0]
    res = np.linalg.norm(b - OK.matvec(X.astype(np.float64), w, sigma)) / np.linalg.norm(b)
    print(world, kw, "res %.3e" % res, "true", ["%.2e" % v for v in rep["history_true"]], "est10", ["%.2e" % v for v in rep["history"][::10]])
    print("   slabs", [o[2]["own"] for o in out])
