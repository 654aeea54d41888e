"""Preconditioner sweep at a BASELINE config on the GPU (diagnostic).

    python tools/sweep_precond.py c4 [iters]

One line per (kind, core, overlap, shift, fp32) case: true residual after a
fixed GMRES budget (the paper's Table II protocol), setup seconds, solve
seconds, W bytes.  Used to choose the benchmark's preconditioner (F4).
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

CASES = [
    # kind, core, overlap, shift, fp32
    (0, 0, 0.0, 0.0, 0),
    (1, 128, 0.0, 0.01, 1),
    (1, 96, 0.0, 0.01, 1),
    (1, 64, 0.0, 0.01, 1),
    (1, 64, 0.0, 0.003, 1),
    (1, 48, 0.0, 0.01, 1),
    (1, 32, 0.0, 0.01, 1),
    (1, 192, 0.0, 0.01, 1),
    (1, 512, 0.0, 0.01, 0),
    (2, 128, 1.0, 1.0, 0),
    (2, 512, 1.0, 0.0, 0),
]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    d = make_inputs(name)
    ctx = R.Context(0)
    kern = R.Kernel(d["sigma"])
    x = torch.as_tensor(d["x"], device="cuda")
    nrm = torch.as_tensor(d["normals"], device="cuda")
    centres, b = R.extend_points(ctx, x, nrm, d["delta"])
    cells = R.Cells(ctx, centres, kern)
    for kind, core, ov, mu, f32 in CASES:
        torch.cuda.synchronize()
        t = time.time()
        try:
            w, rep = R.gmres_solve(ctx, cells, kern, b, kind=kind, core_target=core or 512, overlap_sigmas=ov,
                                   shift=mu, local_fp32=f32, restart=50, rtol=1e-6, phase1_rtol=1e-4,
                                   max_iters=iters)
        except R.RbfError as e:
            print(f"kind={kind} core={core} ov={ov} mu={mu} fp32={f32}: ERR {e}", flush=True)
            continue
        torch.cuda.synchronize()
        dt = time.time() - t
        print(f"kind={kind} core={core} ov={ov} mu={mu} fp32={f32}: it {rep['iters_phase1']}+{rep['iters_phase2']} "
              f"res {rep['rel_residual_true']:.3e} blocks {rep['nblocks']} W {rep['precond_bytes'] / 1e9:.2f} GB "
              f"setup {rep['t_setup']:.3f}s ph1 {rep['t_phase1']:.3f}s total {dt:.3f}s", flush=True)
        del w


if __name__ == "__main__":
    main()
