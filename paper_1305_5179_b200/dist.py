"""Multi-rank plumbing for the benchmark and multi-GPU runs (torch.distributed).

The data plane of a multi-GPU solve (halo exchange, Krylov allreduce, gathers)
runs inside librbf over NCCL; the Python side only needs the
bench's timing reductions below -- the max of the per-rank device times and the
sum of the per-rank work -- which work on any backend (NCCL on GPUs, gloo on
CPU for the tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def reduce_max_sum(values_max, values_sum, device=None):
    """All-reduce two lists of floats: element-wise MAX of the first and SUM of
    the second over all ranks.  Returns (list, list).  Identity without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(v) for v in values_max], [float(v) for v in values_sum]
    dev = device if device is not None else torch.device("cpu")
    tm = torch.tensor([float(v) for v in values_max], dtype=torch.float64, device=dev)
    ts = torch.tensor([float(v) for v in values_sum], dtype=torch.float64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    dist.all_reduce(ts, op=dist.ReduceOp.SUM)
    return tm.tolist(), ts.tolist()


def throughput(ms_rank: float, work_rank: float, device=None):
    """(max-over-ranks milliseconds, summed work, summed work / max seconds)."""
    (ms,), (work,) = reduce_max_sum([ms_rank], [work_rank], device)
    return ms, work, work / (ms * 1e-3) if ms > 0 else float("nan")
