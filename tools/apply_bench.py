"""Block-Jacobi apply at c4: full fp32 inverses (RBF_APPLY_FULL=1) vs packed
symmetric triangles, CUDA-event timed (median of 5 x 20 applies, public call:
gather + apply + scatter).

    python tools/apply_bench.py [config]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402


def timed(fn, n=20, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / n)
    return sorted(ts)[len(ts) // 2]


def main(name="c4"):
    R.load_library()
    ctx = R.Context(0)
    d = make_inputs(name)
    centres, b = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"),
                                 torch.as_tensor(d["normals"], device="cuda"), d["delta"])
    kern = R.Kernel(d["sigma"])
    cells = R.Cells(ctx, centres, kern)
    cfg = d["cfg"]
    kw = dict(kind=cfg.precond_kind, core_target=cfg.core_target, overlap_sigmas=cfg.overlap_sigmas,
              shift=cfg.shift, local_fp32=cfg.local_fp32)
    w = torch.randn(cells.n, device="cuda", dtype=torch.float32)
    out = {"config": name, "cap_env": os.environ.get("RBF_APPLY_CAP")}
    for label, full in (("full", True), ("packed", False)):
        if full:
            os.environ["RBF_APPLY_FULL"] = "1"
        P = R.Precond(ctx, cells, kern, **kw)
        os.environ.pop("RBF_APPLY_FULL", None)
        z = P.apply(w)
        out[label + "_ms"] = timed(lambda: P.apply(w, out=z))
        out[label + "_z"] = z.double().norm().item()
        del P
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:])
