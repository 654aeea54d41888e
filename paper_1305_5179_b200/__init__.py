"""B200-native Gaussian-RBF implicit-surface hot path (arXiv 1305.5179).

The product path is librbf.so (C-ABI, include/rbf.h: hand-written sm_100a
CUDA) and the thin ctypes binding in `rbf`.  This package never imports the
CPU oracle (oracle/, test infrastructure only) and has no CPU fallback.
"""
from .rbf import (OP_AUTO, OP_ONESIDED, OP_SYM, OP_SYM_WIDE, OP_SYM_ROT, AssembledOperator, Cells, Context, Kernel, Precond,
                  LoopbackGroup, RbfError, SolveReport, density, eval_grid, eval_grid_masked, eval_grid_pairs, eval_grid_slab, isosurface, extend_points, gmres_solve, gmres_solve_shard, launch_count,
                  load_library, matvec, matvec_op, matvec_pairs, mesh_from_field, nccl_unique_id, nn_distance, reconstruct_host,
                  sigma_auto, slab_plan, zero_set)

__all__ = ["OP_AUTO", "OP_ONESIDED", "OP_SYM", "OP_SYM_WIDE", "OP_SYM_ROT", "AssembledOperator", "Cells", "Context", "Kernel",
           "Precond", "LoopbackGroup", "RbfError", "SolveReport", "density", "eval_grid", "eval_grid_masked", "eval_grid_pairs", "isosurface", "mesh_from_field", "eval_grid_slab", "extend_points",
           "gmres_solve", "gmres_solve_shard", "launch_count", "load_library", "matvec", "matvec_op", "matvec_pairs", "nccl_unique_id",
           "nn_distance", "reconstruct_host", "sigma_auto", "slab_plan", "zero_set"]
