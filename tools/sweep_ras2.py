import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R
from synth.surfaces import torus
ctx = R.Context(0)
def setup(n, sigma, delta=0.005, noise=1e-3):
    x, nrm = torus(n, noise=noise, seed=0)
    c, b = R.extend_points(ctx, torch.as_tensor(x, device="cuda"), torch.as_tensor(nrm, device="cuda"), delta)
    kern = R.Kernel(sigma)
    return c, b, kern, R.Cells(ctx, c, kern)
for n, sigma in [(20000, 0.05), (20000, 0.035), (20000, 0.025), (8000, 0.05), (5000, 0.05)]:
    c, b, kern, cells = setup(n, sigma)
    sp = np.sqrt(4*np.pi**2*0.35/n)
    for kind, ov in [(0, 0), (1, 0), (2, 1.3), (2, 3.0)]:
        P = R.Precond(ctx, cells, kern, kind=kind, core_target=512, overlap_sigmas=ov)
        z = P.apply(b)
        Az = R.matvec(ctx, cells, kern, z.double())
        amp = (Az.norm() / b.double().norm()).item()
        w, rep = R.gmres_solve(ctx, cells, kern, b, precond=P, restart=50, rtol=1e-6, phase1_rtol=1.0, max_iters=200)
        print(f"n={n} sigma={sigma} ratio={sigma/sp:.2f} kind={kind} ov={ov}: |AMb|/|b|={amp:.3e} it={rep['iters_phase2']} res={rep['rel_residual_true']:.2e}", flush=True)
