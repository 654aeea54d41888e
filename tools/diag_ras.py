"""Diagnostic: per-block accuracy of the GPU RAS apply vs the oracle (fp64 LU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from oracle import cells as OC, extend as OE, solve as OS, kernel as OK  # noqa: E402
from synth import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
core = int(sys.argv[3]) if len(sys.argv) > 3 else 512
ov = float(sys.argv[4]) if len(sys.argv) > 4 else 1.3
d = make_inputs(name, n=n)
X = OE.extend(d["x"], d["normals"], d["delta"])
sigma = d["sigma"]
h = 6 * sigma / 3.999
ctx = R.Context(0)
kern = R.Kernel(sigma)
cells = R.Cells(ctx, torch.as_tensor(X, device="cuda"), kern, cell_edge=h)
P = R.Precond(ctx, cells, kern, core_target=core, overlap_sigmas=ov)
cores, exts, nbytes = P.blocks()
ms = np.array([len(e) for e in exts])
print("blocks", len(cores), "m min/mean/max", ms.min(), ms.mean(), ms.max(), "bytes", nbytes, flush=True)
oc = OC.build(X, 6 * sigma, cell_edge=h)
perm = oc["perm"]
rng = np.random.default_rng(0)
r = rng.normal(size=len(X)).astype(np.float32)
z = P.apply(torch.as_tensor(r, device="cuda")).cpu().numpy()
zs_gpu = z[perm]
blocks = OS.ras_blocks(oc, sigma, core, ov)
rs = r.astype(np.float64)[perm]
import scipy.linalg as sla  # noqa: E402
worst = []
for k, blk in enumerate(blocks[: min(len(blocks), 40)]):
    A = OK.dense_matrix(oc["sorted"][blk["ext"]], sigma)
    y = sla.solve(A, rs[blk["ext"]])
    nc = blk["core"].size
    zr = y[-nc:]
    zg = zs_gpu[blk["core"]]
    e = np.linalg.norm(zg - zr) / np.linalg.norm(zr)
    cond = np.linalg.cond(A)
    worst.append((e, k, len(blk["ext"]), cond))
worst.sort(reverse=True)
for e, k, m, cond in worst[:10]:
    print(f"block {k} m {m} rel err {e:.3e} cond {cond:.3e}")
