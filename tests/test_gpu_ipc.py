"""The multi-rank slab partition over the CUDA-IPC peer-memory transport
(rbf_create_ipc: one process per rank, exchange arenas mapped into each other,
interprocess events + a shared-memory host barrier) executed by real separate
processes -- all on the one GPU of the test box (CUDA IPC maps memory between
processes on the same device as it does across NVLink peers).  Each rank
(tools/ipc_worker.py) compares the distributed results with its own single-GPU
results of the same calls: one-sided products and grid bit-identical, the
symmetric operators to fp32/fp64 rounding of the atomics order; the distributed
GMRES solve (RASM across slabs, symmetric operator) reaches the 1e-6 gate,
certified here by the ORACLE's fp64 matvec, with identical weights on every rank."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import extend as OE
from oracle import kernel as OK
from synth import make_inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_transport_multiprocess(tmp_path, world):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tools", "ipc_worker.py"), str(tmp_path)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=420)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-4000:]
    res = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    own = sorted(tuple(r["slab"]) for r in res)
    assert own[0][0] == 0 and all(own[k][1] == own[k + 1][0] for k in range(world - 1))   # slabs tile the range
    for r in res:
        for k in ("mv32", "mv64", "grid"):
            assert np.array_equal(r[f"{k}_d"].view(np.uint8), r[f"{k}_s"].view(np.uint8)), k
        for k, tol in (("symw32", 1e-5), ("symw64", 1e-12)):
            scale = np.abs(r[f"{k}_s"]).max()
            assert np.abs(r[f"{k}_d"] - r[f"{k}_s"]).max() <= tol * scale, k        # peer-memory form
            assert np.abs(r[f"{k}_copy"] - r[f"{k}_s"]).max() <= tol * scale, k     # copy-based halo form
        np.testing.assert_array_equal(r["w_solve"], res[0]["w_solve"])
    d = make_inputs("c1", n=8000, sigma=0.035, delta=0.0035)
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32).astype(np.float64)
    b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32).astype(np.float64)
    resid = np.linalg.norm(b - OK.matvec(X, res[0]["w_solve"], d["sigma"])) / np.linalg.norm(b)
    rel_true, converged = res[0]["rep_solve"][:2]
    assert converged == 1 and resid <= 1.5e-6, (resid, res[0]["rep_solve"])
    assert resid == pytest.approx(rel_true, rel=1e-3)
