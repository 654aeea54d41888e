"""One rank of the multi-process test of the CUDA-IPC peer-memory transport
(tests/test_gpu_ipc.py): WORLD processes, all on cuda:0 (several processes may
share one device through CUDA IPC), torch.distributed over gloo for the group
key.  Each rank runs the distributed one-sided and symmetric products, the
grid, and a distributed GMRES solve on the same replicated input, and its own
single-GPU reference of the same calls; it saves everything to OUT_DIR/rank{r}.npz.

    RANK=r WORLD_SIZE=W MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tools/ipc_worker.py OUT_DIR
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_5179_b200 as R  # noqa: E402
from oracle import extend as OE  # noqa: E402  (inputs only: the +/-delta set)
from synth import make_inputs  # noqa: E402

out_dir = sys.argv[1]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
ctx = R.Context(0, distributed=True, transport="ipc")
solo = R.Context(0)
assert ctx.world == world and ctx.rank == rank
res = {}
# products and grid on c3's density ramp (unequal planes)
d = make_inputs("c3", n=4000)
X = torch.as_tensor(OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32), device="cuda")
kern = R.Kernel(d["sigma"])
w = torch.as_tensor(np.random.default_rng(3).normal(size=X.shape[0]), device="cuda")
cd, cs = R.Cells(ctx, X, kern), R.Cells(solo, X, kern)
res["slab"] = np.array(cd.slab()["own"])
ctx.peer_memory(False)   # the copy-based halo form of the wide operator, then the peer-memory form (default)
res["symw32_copy"] = R.matvec_op(ctx, cd, kern, w.float(), op=R.OP_SYM_WIDE).cpu().numpy()
res["symw64_copy"] = R.matvec_op(ctx, cd, kern, w, op=R.OP_SYM_WIDE).cpu().numpy()
ctx.peer_memory(True)
for name, ctx_, c in (("d", ctx, cd), ("s", solo, cs)):
    res[f"mv32_{name}"] = R.matvec(ctx_, c, kern, w.float()).cpu().numpy()
    res[f"mv64_{name}"] = R.matvec(ctx_, c, kern, w).cpu().numpy()
    res[f"symw32_{name}"] = R.matvec_op(ctx_, c, kern, w.float(), op=R.OP_SYM_WIDE).cpu().numpy()
    res[f"symw64_{name}"] = R.matvec_op(ctx_, c, kern, w, op=R.OP_SYM_WIDE).cpu().numpy()
    lo, hi = d["grid_lo"], d["grid_hi"]
    res[f"grid_{name}"] = R.eval_grid(ctx_, c, kern, w, lo, hi, (40, 40, 40)).cpu().numpy()
# distributed GMRES with the paper's RASM on the 24k-centre sphere (tests/test_gpu_loopback.py)
d = make_inputs("c1", n=8000, sigma=0.035, delta=0.0035)
X = torch.as_tensor(OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float32), device="cuda")
b = torch.as_tensor(OE.labels(len(d["x"]), d["delta"]).astype(np.float32), device="cuda")
kern = R.Kernel(d["sigma"])
cd = R.Cells(ctx, X, kern)
wd, rep = R.gmres_solve(ctx, cd, kern, b, restart=30, rtol=1e-6, kind=2, core_target=512, overlap_sigmas=3.0,
                        max_iters=400, op=R.OP_SYM_WIDE)
res["w_solve"] = wd.cpu().numpy()
res["rep_solve"] = np.array([rep["rel_residual_true"], rep["converged"], rep["iters_phase1"], rep["iters_phase2"]])
torch.cuda.synchronize()
np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
del cd, cs
ctx.close()
solo.close()
dist.destroy_process_group()
print(f"rank {rank} ok")
