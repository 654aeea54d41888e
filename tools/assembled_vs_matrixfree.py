"""time the assembled CSR operator (the paper's GPU path)
against the matrix-free fp32 summation on one config (CUDA events).

    python tools/assembled_vs_matrixfree.py [c4] [iters]

Prints one JSON line: nnz, CSR bytes, assembly seconds, ms per SpMV and per
matrix-free matvec, achieved HBM bandwidth of the SpMV, agreement of the two.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from synth import make_inputs  # noqa: E402
from tools.bench_kernels import timed  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    d = make_inputs(name)
    ctx = R.Context(0)
    kern = R.Kernel(d["sigma"])
    centres, _ = R.extend_points(ctx, torch.as_tensor(d["x"], device="cuda"),
                                 torch.as_tensor(d["normals"], device="cuda"), d["delta"])
    cells = R.Cells(ctx, centres, kern)
    useful, _ = R.matvec_pairs(ctx, cells, kern)
    w = torch.randn(centres.shape[0], device="cuda")
    f1, f2 = torch.empty_like(w), torch.empty_like(w)
    t_mf = timed(lambda: R.matvec(ctx, cells, kern, w, out=f1), iters)
    A = R.AssembledOperator(ctx, cells, kern)
    info = A.info()
    t_csr = timed(lambda: A.spmv(w, out=f2), iters)
    rel = float((f1 - f2).norm() / f1.norm())
    print(json.dumps(dict(config=name, centres=centres.shape[0], useful_pairs=useful, nnz=info["nnz"],
                          csr_gb=info["bytes"] / 1e9, assemble_s=info["t_assemble"], spmv_ms=t_csr,
                          matrix_free_ms=t_mf, spmv_hbm_tbs=8 * info["nnz"] / (t_csr * 1e-3) / 1e12,
                          matrix_free_speedup=t_csr / t_mf, rel_l2_difference=rel)))


if __name__ == "__main__":
    main()
