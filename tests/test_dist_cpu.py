"""World-size-2 gloo test of the multi-rank path (CPU only): the benchmark's
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
