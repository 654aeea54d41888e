"""the assembled (CSR) operator -- the paper's own GPU
solve path (Alg.2) -- against the matrix-free fp32 tier and the oracle."""
import numpy as np
import pytest
import torch

from oracle import extend as OE
from oracle import kernel as OK
from synth import make_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


@pytest.mark.parametrize("name,n", [("c2", None), ("c1", None)])
def test_csr_spmv_matches_matrix_free_and_oracle(R, name, n):
    ctx = R.Context(0)
    d = make_inputs(name, n=n)
    X = OE.extend(d["x"], d["normals"], d["delta"])
    sigma = d["sigma"]
    kern = R.Kernel(sigma)
    cells = R.Cells(ctx, torch.as_tensor(X, dtype=torch.float32, device="cuda"), kern)
    A = R.AssembledOperator(ctx, cells, kern)
    info = A.info()
    useful, _ = R.matvec_pairs(ctx, cells, kern)
    assert abs(info["nnz"] - useful) <= 1e-5 * useful + 2      # fp32 boundary flips only
    assert info["bytes"] >= 8 * info["nnz"]
    w = np.random.default_rng(8).normal(size=len(X))
    wt = torch.as_tensor(w, dtype=torch.float32, device="cuda")
    f_csr = A.spmv(wt).cpu().numpy()
    f_mf = R.matvec(ctx, cells, kern, wt).cpu().numpy()
    assert np.linalg.norm(f_csr - f_mf) / np.linalg.norm(f_mf) <= 1e-5
    rows = np.sort(np.random.default_rng(1).choice(len(X), 500, replace=False))
    w32 = w.astype(np.float32).astype(np.float64)
    ref = OK.matvec(X, w32, sigma, rows=rows)
    g = OK.matvec(X, np.abs(w32), sigma, rows=rows)
    assert (np.abs(f_csr[rows] - ref) <= 5e-5 * g).all()
