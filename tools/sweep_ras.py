"""Sweep RAS / GMRES settings on the GPU (diagnostic; prints one line per case)."""
import itertools
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth.surfaces import torus, fibonacci_sphere, blobby  # noqa: E402

ctx = R.Context(0)


def run(kind, n, noise, sigma, delta, ov, core, p1=1e-4, restart=50, maxit=300):
    if kind == "torus":
        x, nrm = torus(n, noise=noise, seed=0)
    elif kind == "sphere":
        x, nrm = fibonacci_sphere(n)
    else:
        x, nrm = blobby(n, K=64, seed=0)
    xs = torch.as_tensor(x, device="cuda")
    ns = torch.as_tensor(nrm, device="cuda")
    c, b = R.extend_points(ctx, xs, ns, delta)
    kern = R.Kernel(sigma)
    cells = R.Cells(ctx, c, kern)
    t = time.time()
    try:
        w, rep = R.gmres_solve(ctx, cells, kern, b, restart=restart, rtol=1e-6, phase1_rtol=p1,
                               core_target=core, overlap_sigmas=ov, max_iters=maxit)
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"{kind} n={n} noise={noise} sig={sigma} del={delta} ov={ov} core={core} p1={p1}: "
              f"it {rep['iters_phase1']}+{rep['iters_phase2']} res {rep['rel_residual_true']:.2e} "
              f"conv {rep['converged']} blocks {rep['nblocks']} MB {rep['precond_bytes']/1e6:.0f} "
              f"setup {rep['t_setup']:.2f}s total {dt:.2f}s", flush=True)
    except R.RbfError as e:
        print(kind, n, noise, sigma, delta, ov, core, "ERR", e, flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "torus"
    if which == "torus":
        for noise, delta, ov in itertools.product([0.0, 1e-3], [0.005, 0.02], [1.3, 3.0]):
            run("torus", 20000, noise, 0.05, delta, ov, 512, p1=1.0)
        run("torus", 3000, 1e-3, 0.05, 0.005, 1.3, 512, p1=1.0)
        run("torus", 8000, 1e-3, 0.05, 0.005, 1.3, 512, p1=1.0)
        run("torus", 20000, 1e-3, 0.05, 0.005, 1.3, 512, p1=1e-4)
    elif which == "sphere":
        for ov in [1.0, 2.0, 3.0]:
            run("sphere", 1000, 0, 0.1, 0.01, ov, 512, p1=1.0)
            run("sphere", 1000, 0, 0.1, 0.01, ov, 512, p1=1e-4)
