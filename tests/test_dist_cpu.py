"""World-size-2/3 gloo tests of the multi-rank path (CPU only): the benchmark
max-over-ranks time and summed-work reduction (paper_1305_5179_b200.dist)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1305_5179_b200.dist import reduce_max_sum, throughput
    ms, work, rate = throughput(100.0 + 50.0 * rank, 1e9 * (rank + 1))
    mx, sm = reduce_max_sum([rank, -rank], [1.0, rank])
    out[rank] = (ms, work, rate, mx, sm)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_reduction_gloo():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        ms, work, rate, mx, sm = out[r]
        assert ms == 150.0                      # max over ranks
        assert work == 3e9                      # sum over ranks
        assert rate == pytest.approx(3e9 / 0.150)
        assert mx == [1.0, 0.0] and sm == [2.0, 1.0]


def test_single_process_identity():
    from paper_1305_5179_b200.dist import throughput
    ms, work, rate = throughput(20.0, 4e9)
    assert (ms, work) == (20.0, 4e9) and rate == pytest.approx(2e11)


# ---- slab partition ------------------
# The library's world > 1 path partitions the sorted order into slabs of whole z
# cell planes (rbf_slab_plan, host code) and, per matvec, assembles each rank's
# source window from its own slice plus the owners' slices (grouped
# send/recv).  The tests below run that protocol on CPU ranks (gloo) with the
# oracle's fp64 products standing in for the kernels: the distributed product,
# its dot products and the gathered result must equal the undistributed ones.

def _plane_data(X, sigma):
    import numpy as np
    from oracle import cells as OC
    cut = 6 * sigma
    oc = OC.build(X, cut, cell_edge=cut / 3.999)
    dim = oc["dim"]
    per_plane = int(dim[0] * dim[1])
    cs = oc["cell_start"].astype(np.int64)
    ce = oc["cell_end"].astype(np.int64)
    ps = np.concatenate([cs[::per_plane][: dim[2]], [len(X)]])
    counts = (ce - cs).reshape(dim[2], per_plane)
    weight = (counts.astype(np.float64) ** 2).sum(axis=1)
    reach = int(np.ceil(cut / oc["h"])) + 1
    return oc, ps, weight, reach


def _slab_worker(rank, world, port, out):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1305_5179_b200 as R
    from oracle import kernel as OK
    from oracle import extend as OE
    from synth import make_inputs

    d = make_inputs("c2", n=1500)
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    sigma = d["sigma"]
    oc, ps, weight, reach = _plane_data(X, sigma)
    S = oc["sorted"].astype(np.float64)
    P = R.slab_plan(ps, weight, reach, world)
    o0, o1 = int(P["own_lo"][rank]), int(P["own_hi"][rank])
    h0, h1 = int(P["win_lo"][rank]), int(P["win_hi"][rank])
    w = np.random.default_rng(5).normal(size=len(X))        # replicated input (sorted order)
    w_loc = torch.tensor(w[o0:o1])
    # halo exchange exactly as dist.cu::halo_exchange: send my slice inside q's
    # window, receive q's slice inside mine
    win = torch.zeros(h1 - h0, dtype=torch.float64)
    win[o0 - h0:o1 - h0] = w_loc
    reqs = []
    for q in range(world):
        if q == rank:
            continue
        slo, shi = max(o0, int(P["win_lo"][q])), min(o1, int(P["win_hi"][q]))
        if shi > slo:
            reqs.append(dist.isend(w_loc[slo - o0:shi - o0].clone(), q))
        rlo, rhi = max(int(P["own_lo"][q]), h0), min(int(P["own_hi"][q]), h1)
        if rhi > rlo:
            buf = torch.empty(rhi - rlo, dtype=torch.float64)
            reqs.append((dist.irecv(buf, q), buf, rlo))
    for r_ in reqs:
        if isinstance(r_, tuple):
            r_[0].wait()
            win[r_[2] - h0:r_[2] - h0 + r_[1].numel()] = r_[1]
        else:
            r_.wait()
    # local rows of the product from the window only (oracle arithmetic)
    f_loc = OK.matvec(S[h0:h1], win.numpy(), sigma, targets=S[o0:o1]) if o1 > o0 else np.zeros(0)
    # distributed dot: local partial + all-reduce
    dot = torch.tensor([float(f_loc @ w[o0:o1])], dtype=torch.float64)
    dist.all_reduce(dot)
    # gather (the library broadcasts every owner's slice)
    full = torch.zeros(len(X), dtype=torch.float64)
    full[o0:o1] = torch.tensor(f_loc)
    dist.all_reduce(full)
    out[rank] = (full.numpy(), float(dot.item()), (o0, o1, h0, h1), P["plane_lo"].tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_partition_matvec_gloo(world):
    import numpy as np
    from oracle import kernel as OK
    from oracle import extend as OE
    from synth import make_inputs

    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_slab_worker, args=(world, port, out), nprocs=world, join=True)
    d = make_inputs("c2", n=1500)
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32)
    oc, ps, weight, reach = _plane_data(X, d["sigma"])
    S = oc["sorted"].astype(np.float64)
    w = np.random.default_rng(5).normal(size=len(X))
    ref = OK.matvec(S, w, d["sigma"])
    ranges = [out[r][2] for r in range(world)]
    # slabs tile the sorted order, windows contain the slab
    assert ranges[0][0] == 0 and ranges[-1][1] == len(X)
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]
    for o0, o1, h0, h1 in ranges:
        assert h0 <= o0 <= o1 <= h1 or o0 == o1
    for r in range(world):
        full, dot, _, plane_lo = out[r]
        np.testing.assert_allclose(full, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        assert dot == pytest.approx(float(ref @ w), rel=1e-12)
        assert plane_lo == out[0][3]                         # every rank computed the same plan


def test_slab_plan_balances_pair_weight():
    """rbf_slab_plan on the c3-like 10x density ramp: slab weights within one
    plane's weight of the ideal share, contiguous cover, windows = slab +- reach."""
    import numpy as np
    import paper_1305_5179_b200 as R
    rng = np.random.default_rng(0)
    dimz = 200
    counts = rng.integers(0, 50, dimz) * np.linspace(1, 10, dimz).astype(np.int64)
    ps = np.concatenate([[0], np.cumsum(counts)])
    weight = counts.astype(np.float64) ** 2
    for world in (1, 2, 4, 8):
        P = R.slab_plan(ps, weight, 5, world)
        lo = P["plane_lo"]
        assert lo[0] == 0 and lo[-1] == dimz and (np.diff(lo) >= 0).all()
        share = weight.sum() / world
        for r in range(world):
            wr = weight[lo[r]:lo[r + 1]].sum()
            assert abs(wr - share) <= weight.max()
            assert P["own_lo"][r] == ps[lo[r]] and P["own_hi"][r] == ps[lo[r + 1]]
            if lo[r + 1] > lo[r]:
                assert P["win_lo"][r] == ps[max(0, lo[r] - 5)]
                assert P["win_hi"][r] == ps[min(dimz, lo[r + 1] + 5)]
    with pytest.raises(R.RbfError):
        R.slab_plan(ps, -weight, 5, 2)
