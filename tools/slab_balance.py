"""Slab partition of a config over W ranks, as the library plans it (rbf_slab_plan
on the real cell structure), evaluated on one GPU through the loopback transport:
per-rank owned centres, source-window (halo) sizes and useful pairs per matvec
(rbf_matvec_pairs on each rank's tiles), the imbalance max/mean and the
compute-bound speedup bound W1_pairs / max_rank_pairs.  Plan evidence for the
multi-GPU scaling target (no timing: W ranks time-share one GPU here).

    python tools/slab_balance.py c4 8
"""
import json
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
d = make_inputs(name)
kern = R.Kernel(d["sigma"])
ctx = R.Context(0)
X, _ = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"), torch.as_tensor(d["normals"], device="cuda"),
                       d["delta"])
cells = R.Cells(ctx, X, kern)
useful1, _ = R.matvec_pairs(ctx, cells, kern)
out = {"config": name, "centres": int(X.shape[0]), "useful_pairs_w1": int(useful1), "worlds": {}}
del cells
for W in worlds:
    group = R.LoopbackGroup(W)
    res = [None] * W

    def rank(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c2 = R.Context(0, stream=st, loopback=(group, r))
            cl = R.Cells(c2, X, kern)
            sl = cl.slab()
            u, v = R.matvec_pairs(c2, cl, kern)
            res[r] = dict(own=sl["own"][1] - sl["own"][0], window=sl["window"][1] - sl["window"][0],
                          useful=int(u), wide_tiles=sl["wide_tiles"][1] - sl["wide_tiles"][0],
                          wide_interior=sl["wide_interior"])
            st.synchronize()
            del cl
            c2.close()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(W)]
    [t.start() for t in th]
    [t.join() for t in th]
    group.close()
    u = np.array([r["useful"] for r in res], dtype=np.float64)
    own = np.array([r["own"] for r in res], dtype=np.float64)
    halo = np.array([r["window"] - r["own"] for r in res], dtype=np.float64)
    out["worlds"][W] = {"per_rank": res, "useful_sum": int(u.sum()), "imbalance_max_over_mean": float(u.max() / u.mean()),
                        "speedup_bound_compute": float(useful1 / u.max()),
                        "halo_over_own_mean": float((halo / np.maximum(own, 1)).mean())}
    print(f"W={W}: useful max/mean {u.max() / u.mean():.3f}, compute-bound speedup {useful1 / u.max():.2f}, "
          f"halo/own {float((halo / np.maximum(own, 1)).mean()):.2f}", flush=True)
print(json.dumps(out))
