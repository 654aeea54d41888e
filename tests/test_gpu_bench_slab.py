"""The bench's N > 1 slab mode end to end on a one-GPU box: `torchrun
--nproc-per-node 2 bench.py --gpus 2` with every rank on cuda:0 (test hook
RBF_BENCH_SHARED_GPU=1: gloo process group) over the CUDA-IPC transport.  It
checks the plumbing -- launch, the distributed-vs-single-GPU self-check, the
timed loop, max-over-ranks timing, one JSON line from rank 0 -- not performance
(two ranks time-share one GPU: the numbers are not a measurement)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_slab_two_ranks_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, RBF_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "c3", "--steps", "1", "--warmup", "1", "--no-e2e"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert "ipc transport" in out["config"]["parallelism"]
    assert out["value"] > 0 and out["detail"]["rel_residual_true"] < 1e-2
