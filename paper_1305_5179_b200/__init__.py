"""B200-native Gaussian-RBF implicit-surface hot path (arXiv 1305.5179).

The product path is librbf.so (C-ABI, include/rbf.h: hand-written sm_100a
CUDA) and the thin ctypes binding in `rbf`.  This package never imports the
CPU oracle (oracle/, test infrastructure only) and has no CPU fallback.
"""
from .rbf import (AssembledOperator, Context, Cells, Kernel, Precond, RbfError, SolveReport, density, eval_grid, eval_grid_pairs, extend_points,
                  gmres_solve, launch_count, load_library, matvec, matvec_pairs, nccl_unique_id, nn_distance, reconstruct_host,
                  slab_plan, zero_set)

__all__ = ["AssembledOperator", "Context", "Cells", "Kernel", "Precond", "RbfError", "SolveReport", "density", "eval_grid", "eval_grid_pairs",
           "extend_points", "gmres_solve", "launch_count", "load_library", "matvec", "matvec_pairs", "nccl_unique_id", "nn_distance",
           "reconstruct_host", "slab_plan", "zero_set"]
