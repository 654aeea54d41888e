"""Offline model of the symmetric fp32 matvec's work on a tile plan (CPU, numpy):
for every target tile of a plan (the library's run-chunk plan, cells.cu
plan_row mode 0), the exponentials the symmetric kernel evaluates = 32 T x
(own tile padded to 4 + box-culled sources after the tile padded to 4), and the
useful share.  Used to compare plans (cap, span) before touching the kernel.

    python tools/plan_sim.py [config] [cap] [span] [sample_tiles]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cells as OC  # noqa: E402
from oracle import extend as OE  # noqa: E402
from synth import make_inputs  # noqa: E402


def plan(cs, ce, dim, cap, span):
    tiles = []
    for row in range(dim[1] * dim[2]):
        base = row * dim[0]
        cur_s = cur_n = cur_x0 = 0
        last_x = -2
        for x in range(dim[0]):
            s, m = cs[base + x], ce[base + x] - cs[base + x]
            if m == 0:
                continue
            if cur_n > 0 and (x != last_x + 1 or x - cur_x0 >= span):
                tiles.append((cur_s, cur_n)); cur_n = 0
            off = 0
            while off < m:
                if cur_n == 0:
                    cur_s, cur_x0 = s + off, x
                take = min(cap - cur_n, m - off)
                cur_n += take; off += take
                if cur_n == cap:
                    tiles.append((cur_s, cur_n)); cur_n = 0
            last_x = x
        if cur_n > 0:
            tiles.append((cur_s, cur_n))
    return np.array(tiles, dtype=np.int64)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    span = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    nsample = int(sys.argv[4]) if len(sys.argv) > 4 else 3000
    d = make_inputs(name)
    X = OE.extend(d["x"], d["normals"], d["delta"])
    sigma = d["sigma"]
    c = 6 * sigma
    oc = OC.build(X, c, cell_edge=c / 3.999)
    S = oc["sorted"].astype(np.float64)
    dim = oc["dim"]
    T = plan(oc["cell_start"], oc["cell_end"], dim, cap, span)
    cnt = T[:, 1]
    slots = 32 * ((cnt + 31) // 32)
    print(f"{name} cap {cap} span {span}: tiles {len(T)}, mean targets {cnt.mean():.1f}, "
          f"slot fill {cnt.sum() / slots.sum():.3f}")
    rng = np.random.default_rng(0)
    pick = rng.choice(len(T), min(nsample, len(T)), replace=False)
    from scipy.spatial import cKDTree
    tree = cKDTree(S)
    ex = useful = 0.0
    cc = c * (1 + 1e-5)
    for i in pick:
        s0, n = T[i]
        P = S[s0:s0 + n]
        lo, hi = P.min(0), P.max(0)
        ctr = 0.5 * (lo + hi)
        half = 0.5 * (hi - lo)
        cand = np.array(tree.query_ball_point(ctr, np.linalg.norm(half) + cc), dtype=np.int64)
        cand = cand[cand >= s0 + n]
        g = np.maximum(0, np.maximum(lo - S[cand], S[cand] - hi))
        kept = cand[(g * g).sum(1) <= cc * cc]
        tslots = 32 * ((n + 31) // 32)
        ex += tslots * (((n + 3) // 4) * 4 + ((len(kept) + 3) // 4) * 4)
        # useful ordered pairs of these targets (self included), as the metric counts them
        nb = tree.query_ball_point(P, c, return_length=True)
        useful += nb.sum()
    print(f"  exponentials per useful ordered pair: {ex / useful:.3f}  (sample of {len(pick)} tiles)")


if __name__ == "__main__" and not (len(sys.argv) > 5 and sys.argv[5] == "groups"):
    main()


def group_mask_model(name="c4", cap=128, span=4, nsample=1500):
    """Exponentials if each staged source skipped the 32-target groups whose box it
    cannot reach (per source, and OR-ed over the 4 consecutive sources the kernel
    processes together)."""
    d = make_inputs(name)
    X = OE.extend(d["x"], d["normals"], d["delta"])
    sigma = d["sigma"]
    c = 6 * sigma
    oc = OC.build(X, c, cell_edge=c / 3.999)
    S = oc["sorted"].astype(np.float64)
    T = plan(oc["cell_start"], oc["cell_end"], oc["dim"], cap, span)
    from scipy.spatial import cKDTree
    tree = cKDTree(S)
    rng = np.random.default_rng(0)
    cc = c * (1 + 1e-5)
    base = per_src = or4 = 0
    for i in rng.choice(len(T), min(nsample, len(T)), replace=False):
        s0, n = T[i]
        P = S[s0:s0 + n]
        lo, hi = P.min(0), P.max(0)
        cand = np.array(tree.query_ball_point(0.5 * (lo + hi), np.linalg.norm(0.5 * (hi - lo)) + cc), dtype=np.int64)
        cand = np.sort(cand[cand >= s0 + n])
        g = np.maximum(0, np.maximum(lo - S[cand], S[cand] - hi))
        kept = cand[(g * g).sum(1) <= cc * cc]
        ng = (n + 31) // 32
        m = np.zeros((len(kept), ng), dtype=bool)
        for t in range(ng):
            Q = P[32 * t:32 * t + 32]
            ql, qh = Q.min(0), Q.max(0)
            gg = np.maximum(0, np.maximum(ql - S[kept], S[kept] - qh))
            m[:, t] = (gg * gg).sum(1) <= cc * cc
        base += len(kept) * ng
        per_src += m.sum()
        k4 = (len(kept) + 3) // 4 * 4
        mm = np.zeros((k4, ng), dtype=bool)
        mm[:len(kept)] = m
        or4 += mm.reshape(-1, 4, ng).any(axis=1).sum() * 4
    print(f"sym-ring source x group evaluations: box {base:.3e}, per-source group cull {per_src / base:.3f}, "
          f"OR over 4 consecutive {or4 / base:.3f}")


if __name__ == "__main__" and len(sys.argv) > 5 and sys.argv[5] == "groups":
    group_mask_model(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
