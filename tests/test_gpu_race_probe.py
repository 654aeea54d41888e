"""Race / synchronisation evidence without compute-sanitizer (closed on the GPU
pool: profiles/r02/race_probe.md).  tools/race_probe.py runs every kernel
family twice under the product build and once under the CHECKED build
(csrc/checks.h: device bounds checks that trap, lane/warp jitter at every
shared-memory hand-over: ring stores, flushes, block barriers, cluster
barriers, mbarrier waits).  Deterministic results are bit-identical run to run
and between the builds -- a missing __syncwarp / __syncthreads / wait would let
a jittered lane read stale shared memory; the symmetric products (atomic
accumulation order) agree to fp32 rounding."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib, out):
    cmd = [sys.executable, os.path.join(ROOT, "tools", "race_probe.py"), lib, out]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return dict(np.load(out))


def test_checked_build_matches_product(tmp_path):
    from paper_1305_5179_b200 import build as B
    prod = B.build()
    checked = B.build(checked=True)
    a = _run(prod, str(tmp_path / "a.npz"))
    a2 = _run(prod, str(tmp_path / "a2.npz"))
    c = _run(checked, str(tmp_path / "c.npz"))
    assert set(a) == set(c) == set(a2)
    for k in sorted(a):
        if k.startswith("atomic_"):
            scale = np.abs(a[k]).max()
            assert np.abs(a[k] - c[k]).max() <= 1e-5 * scale, k
            assert np.abs(a[k] - a2[k]).max() <= 1e-5 * scale, k
        else:
            assert a[k].shape == c[k].shape, k
            assert np.array_equal(a[k].view(np.uint8), a2[k].view(np.uint8)), f"{k}: not deterministic"
            assert np.array_equal(a[k].view(np.uint8), c[k].view(np.uint8)), f"{k}: checked build differs"
    np.testing.assert_array_equal(a["loopback_mv64_r0"], a["mv64"])
